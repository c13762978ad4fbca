// Red-black SOR on a colour-split layout (reference: sor.py:162-203, the
// press halo les.py:341-355): the streaming solver for grids whose working
// set does not fit the SMs' shared memory (the resident solver's domain).
//
// Layout.  Cell (i, j, k) has colour c = (ig + j + k + 1) & 1 (ig = global
// i), the colour red-black pass nrd = c updates (sor.py:174-178:
// ((i-1)+(j-1)+(k-1)+nrd) even).  Each colour has its own array of
// (im+2) x (jm+2) rows of KHP slots; cell (i, j, k) lives in array c, row
// (i, j), slot k >> 1.  KHP = ceil((km+2)/2) rounded up to a multiple of 4,
// so every row starts 16-byte aligned.  In row (i, j) the colour-c cells
// have k = 2t + s with s = (c + ig + j + 1) & 1, and every neighbour of a
// colour-c cell is in the other array:
//   E/W/N/S: rows (i+-1, j) / (i, j+-1), the same slot t;
//   T/B:     the same row, slots t + s and t + s - 1.
// A colour pass therefore reads the other array, its own cells and the
// colour's rhs, and writes its own cells, all unit-stride: a thread takes
// four consecutive slots (one 16-byte access per array and neighbour row,
// plus one scalar for the T/B shift), a warp 512 contiguous bytes.  The
// natural layout's pass strides over both colours (every 32-byte sector it
// touches is half the other colour), which is what kept the unfused pass at
// ~20 B/cell/iteration of DRAM traffic instead of 16.
//
// p and rhs are split once per solve (k_split_pack) and p is merged back
// once at the end (k_split_unpack), which also applies the final halo_fn of
// the press policy in closed form and the press stage's non-finite check.
// Arithmetic: sor_point's expression and order (A8), bitwise equal to the
// other solvers; the residual is summed per thread in slot order, per block
// by a fixed shuffle tree, and per iteration by launch_reduce_res.
#include "lesb_common.cuh"
#include "lesb_kernels.h"

namespace lesb {

SplitGeo split_geo(const Geo& g) {
  SplitGeo s;
  const int kh = (g.km + 2 + 1) / 2;
  s.khp = (kh + 3) & ~3;
  s.kh4 = s.khp / 4;
  s.spi = (long long)(g.jm + 2) * s.khp;
  s.n = (long long)(g.im + 2) * s.spi;
  return s;
}

bool split_supported(const Geo& g, const SorC& cf) {
  // scalar weights and cn1 (build_uniform_coeffs), 32-bit indices
  return cf.uni && !cf.cn1 && 4 * split_geo(g).n < (1LL << 31);
}

namespace {

constexpr int RBS_NT = 256;  // threads per pass block (x: float4 groups of a row, y: rows)
constexpr int RBS_R = 2;     // rows per thread (j, j + blockDim.y)

inline void rbs_shape(const SplitGeo& s, int* bx, int* by) {
  *bx = s.kh4 < 32 ? s.kh4 : 32;
  *by = RBS_NT / *bx;
  if (*by < 1) *by = 1;
}

// Split p and rhs: a warp per natural row (i, j), lanes over k.
__global__ void __launch_bounds__(256) k_split_pack(Geo g, SplitGeo sg, const float* __restrict__ p,
                                                    const float* __restrict__ rhs, float* __restrict__ ps,
                                                    float* __restrict__ rs) {
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= nrow) return;
  const int lane = threadIdx.x & 31;
  const int i = (int)(row / (g.jm + 2)), j = (int)(row - (long long)i * (g.jm + 2));
  const int par = (i + g.ioff + j + 1) & 1;
  const float* src_p = p + row * (g.km + 2);
  const float* src_r = rhs + row * (g.km + 2);
  const long long rb = row * sg.khp;
  for (int k = lane; k < g.km + 2; k += 32) {
    const int c = (par + k) & 1;
    const long long d = c * sg.n + rb + (k >> 1);
    ps[d] = src_p[k];
    rs[d] = src_r[k];
  }
}

// One colour pass (colour c) in place on the split arrays.  POL 0: stored
// halo; POL 1: press remaps (the W/B sources are the updated cell itself,
// read before it is written; the S/N sources have the other colour for even
// jm, and for odd jm the y halo rows hold a pre-pass snapshot, y_stored).
template <int POL>
__global__ void __launch_bounds__(RBS_NT) k_sor_rbs(Geo g, SplitGeo sg, float* __restrict__ ps,
                                                    const float* __restrict__ rs, SorC cf, float om, int c,
                                                    int y_stored, double* __restrict__ partials) {
  __shared__ double red[RBS_NT / 32];
  const int q = blockIdx.x * blockDim.x + threadIdx.x;  // float4 group of the row
  const int i = blockIdx.z + 1;
  const int ig = i + g.ioff;
  float* own = ps + (long long)c * sg.n;
  const float* oth = ps + (long long)(c ^ 1) * sg.n;
  const float* rc = rs + (long long)c * sg.n;
  const int spi = (int)sg.spi, khp = sg.khp;
  const bool wfix = POL == 1 && i == 1 && g.west_bc;   // W -> the cell itself
  const bool efix = POL == 1 && i == g.im && g.east_bc;  // E -> 0
  double acc = 0.0;
  float4 cv[RBS_R], rel4[RBS_R];
  int base[RBS_R];
  bool act[RBS_R];
  // all rows' loads are issued before the first store (a colour pass writes
  // only its own colour and reads the other one: nothing aliases)
#pragma unroll
  for (int r = 0; r < RBS_R; ++r) {
    const int j = (blockIdx.y * RBS_R + r) * blockDim.y + threadIdx.y + 1;
    act[r] = j <= g.jm && q < sg.kh4;
    base[r] = 0;
    rel4[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    cv[r] = rel4[r];
    if (!act[r]) continue;
    const int s = (c + ig + j + 1) & 1;
    const int t0 = 4 * q;
    const int b = i * spi + j * khp + t0;
    base[r] = b;
    const float4 pc = *reinterpret_cast<const float4*>(own + b);
    const float4 rh = *reinterpret_cast<const float4*>(rc + b);
    const float4 mid = *reinterpret_cast<const float4*>(oth + b);
    const float4 pe = efix ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(oth + b + spi);
    const float4 pw = wfix ? pc : *reinterpret_cast<const float4*>(oth + b - spi);
    const int jn = (POL == 1 && j == g.jm && !y_stored) ? 1 : j + 1;
    const int js = (POL == 1 && j == 1 && !y_stored) ? g.jm : j - 1;
    const float4 pn = *reinterpret_cast<const float4*>(oth + b + (jn - j) * khp);
    const float4 pso = *reinterpret_cast<const float4*>(oth + b + (js - j) * khp);
    // T/B: s = 0 -> T = mid[m], B = mid[m-1] (m = 0: slot t0-1);
    //      s = 1 -> T = mid[m+1] (m = 3: slot t0+4), B = mid[m]
    const int kf = 2 * t0 + s;  // k of the group's first cell
    float extra = 0.0f;
    if (s == 0 && t0 > 0) extra = oth[b - 1];
    if (s == 1 && kf + 6 <= g.km) extra = oth[b + 4];
    const float pcv[4] = {pc.x, pc.y, pc.z, pc.w};
    const float md[4] = {mid.x, mid.y, mid.z, mid.w};
    const float ev[4] = {pe.x, pe.y, pe.z, pe.w};
    const float wv[4] = {pw.x, pw.y, pw.z, pw.w};
    const float nv[4] = {pn.x, pn.y, pn.z, pn.w};
    const float sv[4] = {pso.x, pso.y, pso.z, pso.w};
    const float rv[4] = {rh.x, rh.y, rh.z, rh.w};
    float out[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int k = kf + 2 * m;
      out[m] = 0.0f;
      if (k < 1 || k > g.km) continue;
      float pT = s == 0 ? md[m] : (m < 3 ? md[m + 1] : extra);
      float pB = s == 0 ? (m > 0 ? md[m - 1] : extra) : md[m];
      if (POL == 1) {
        if (k == g.km) pT = 0.0f;
        if (k == 1) pB = pcv[m];
      }
      // sor.py:164-171: E, W, N, S, T, B summed left to right; sor.py:197
      float nb = cf.w2l * ev[m];
      nb = nb + cf.w2s * wv[m];
      nb = nb + cf.w3l * nv[m];
      nb = nb + cf.w3s * sv[m];
      nb = nb + cf.w4l * pT;
      nb = nb + cf.w4s * pB;
      out[m] = om * (cf.cn1s * (nb - rv[m]) - pcv[m]);
    }
    cv[r] = pc;
    rel4[r] = make_float4(out[0], out[1], out[2], out[3]);
  }
#pragma unroll
  for (int r = 0; r < RBS_R; ++r) {
    if (!act[r]) continue;
    // non-interior slots (k halo, row padding) get rel = 0: p + 0 == p for
    // every value, including -0.0 + 0.0?  No (-0 + 0 = +0): store them as read
    const int j = (blockIdx.y * RBS_R + r) * blockDim.y + threadIdx.y + 1;
    const int s = (c + ig + j + 1) & 1;
    const int kf = 8 * q + s;
    const float pcv[4] = {cv[r].x, cv[r].y, cv[r].z, cv[r].w};
    const float rl[4] = {rel4[r].x, rel4[r].y, rel4[r].z, rel4[r].w};
    float nv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int k = kf + 2 * m;
      const bool in = k >= 1 && k <= g.km;
      nv[m] = in ? pcv[m] + rl[m] : pcv[m];
      if (in) acc += (double)rl[m] * (double)rl[m];
    }
    *reinterpret_cast<float4*>(own + base[r]) = make_float4(nv[0], nv[1], nv[2], nv[3]);
  }
  // fixed-order block reduction
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  const int ltid = threadIdx.x + threadIdx.y * blockDim.x;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  if ((ltid & 31) == 0) red[ltid >> 5] = acc;
  __syncthreads();
  if (ltid == 0) {
    double sum = 0.0;
    for (int w = 0; w < nw; ++w) sum += red[w];
    partials[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = sum;
  }
}

// Pre-pass snapshot of the y halo rows (press policy, odd jm): the colour-c
// pass reads p[i, 0, k] = p[i, jm, k] and p[i, jm+1, k] = p[i, 1, k] in the
// other array, whose sources (rows jm and 1) are colour-c cells.
__global__ void k_split_refresh_y(Geo g, SplitGeo sg, float* __restrict__ ps, int c) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y + 1;
  if (t >= sg.khp) return;
  const float* own = ps + (long long)c * sg.n + i * sg.spi;
  float* oth = ps + (long long)(c ^ 1) * sg.n + i * sg.spi;
  oth[t] = own[(long long)g.jm * sg.khp + t];
  oth[(long long)(g.jm + 1) * sg.khp + t] = own[sg.khp + t];
}

// Merge the split p back into the natural layout: a warp per natural row,
// lanes over k.  PRESS: halo cells (not on a neighbour slab's plane) take
// the closed-form halo_fn source (k: 0 -> 1, km+1 -> 0; then j periodic;
// then i: 0 -> 1, im+1 -> 0), which reproduces the reference's final
// _pressure_halo call; STORED: every cell as stored.  flags: the press
// stage's non-finite check over the whole result.
template <int POL>
__global__ void __launch_bounds__(256) k_split_unpack(Geo g, SplitGeo sg, const float* __restrict__ ps,
                                                      float* __restrict__ p, unsigned* flags) {
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  unsigned bits = 0;
  if (row < nrow) {
    const int i = (int)(row / (g.jm + 2)), j = (int)(row - (long long)i * (g.jm + 2));
    const bool rowhalo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1;
    const bool foreign = (i == 0 && !g.west_bc) || (i == g.im + 1 && !g.east_bc);
    const bool remap = POL == 1 && !foreign;
    const bool zero_row = remap && i == g.im + 1;
    const int ii = (remap && i == 0) ? 1 : i;
    const int jj = (remap && rowhalo) ? (j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j)) : j;
    const int par = (ii + g.ioff + jj + 1) & 1;
    const float* src = ps + ((long long)ii * (g.jm + 2) + jj) * sg.khp;
    float* dst = p + row * (g.km + 2);
    for (int k = lane; k < g.km + 2; k += 32) {
      float val;
      if (zero_row || (remap && k == g.km + 1)) {
        val = 0.0f;
      } else {
        const int kk = (remap && k == 0) ? 1 : k;
        val = src[((par + kk) & 1) * sg.n + (kk >> 1)];
      }
      dst[k] = val;
      if (flags && !finite32(val)) bits = F_PRESS;
    }
  }
  if (flags) flag_or(flags, bits);
}

}  // namespace

void launch_split_pack(const Geo& g, const float* p, const float* rhs, float* split, cudaStream_t st) {
  const SplitGeo sg = split_geo(g);
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  k_split_pack<<<(unsigned)((nrow + 7) / 8), 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n);
}

int sor_blocks_split(const Geo& g) {
  const SplitGeo sg = split_geo(g);
  int bx, by;
  rbs_shape(sg, &bx, &by);
  return ((sg.kh4 + bx - 1) / bx) * ((g.jm + by * RBS_R - 1) / (by * RBS_R)) * g.im;
}

void launch_rbs_pass(const Geo& g, float* split, const SorC& cf, float om, int c, int policy, double* partials,
                     cudaStream_t st) {
  const SplitGeo sg = split_geo(g);
  int bx, by;
  rbs_shape(sg, &bx, &by);
  const int y_stored = (policy == 1 && (g.jm & 1)) ? 1 : 0;
  if (y_stored) k_split_refresh_y<<<dim3((sg.khp + 127) / 128, g.im), 128, 0, st>>>(g, sg, split, c);
  dim3 grid((sg.kh4 + bx - 1) / bx, (g.jm + by * RBS_R - 1) / (by * RBS_R), g.im);
  if (policy == 1)
    k_sor_rbs<1><<<grid, dim3(bx, by), 0, st>>>(g, sg, split, split + 2 * sg.n, cf, om, c, y_stored, partials);
  else
    k_sor_rbs<0><<<grid, dim3(bx, by), 0, st>>>(g, sg, split, split + 2 * sg.n, cf, om, c, 0, partials);
}

void launch_split_unpack(const Geo& g, const float* split, float* p, int policy, unsigned* flags, cudaStream_t st) {
  const SplitGeo sg = split_geo(g);
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  const unsigned nb = (unsigned)((nrow + 7) / 8);
  if (policy == 1) k_split_unpack<1><<<nb, 256, 0, st>>>(g, sg, split, p, flags);
  else k_split_unpack<0><<<nb, 256, 0, st>>>(g, sg, split, p, flags);
}

}  // namespace lesb
