// SOR pressure solver kernels (reference: gmcf_mini/sor.py:162-309 and the
// press halo les.py:341-355).
//
// Halo policies (solve_pressure's halo_fn):
//   STORED (halo_fn=None): the halo keeps whatever p0 held; read it directly.
//   PRESS  (les._pressure_halo): boundary values are read through the
//          closed-form face remap of SURVEY Appendix B instead of being
//          materialised before every colour pass:
//            W  p[0,j,k]    -> p[1,j,k]  (the point itself)
//            E  p[im+1,j,k] -> 0
//            S  p[i,0,k]    -> p[i,jm,k]
//            N  p[i,jm+1,k] -> p[i,1,k]
//            B  p[i,j,0]    -> p[i,j,1]  (the point itself)
//            T  p[i,j,km+1] -> 0
//          A colour pass reads the pre-pass value of every remapped source:
//          the W/B sources are the updated point itself (read before it is
//          written) and, for even jm, the S/N sources have the other colour.
//          For odd jm they share the colour, so the y halo planes are
//          snapshotted before each pass instead (k_refresh_y) and read stored.
//          One materialisation (k_press_halo) after the last pass reproduces
//          the reference's final halo_fn call, including edges and corners.
#include <cstdlib>

#include "lesb_common.cuh"
#include "lesb_kernels.h"

namespace lesb {

constexpr int RB_NT = 320;  // threads per colour-pass block: x = colour cells of a column, y = j (45 x 7 at km = 90: 98% of 10 warps)
constexpr int RB_NW = RB_NT / 32;
constexpr int RB_R = 4;     // rows per thread (j, j + by, ...)

// Block shape of a colour pass: x spans the colour's cells of a column (so a
// warp runs on into the next j row instead of idling), y the rows.
static inline void rb_shape(const Geo& g, int* bx, int* by) {
  const int kh = (g.km + 1) / 2;
  *bx = kh < RB_NT ? kh : RB_NT;
  *by = RB_NT / *bx;
}

template <int POL, bool UNI = false, typename IDX = long long>
__device__ __forceinline__ float sor_point(const Geo& g, const float* __restrict__ p, const float* __restrict__ rhs,
                                           const SorC& cf, float om, IDX c, int i, int j, int k, int y_stored,
                                           float& pc_out) {
  const IDX si = (IDX)g.si, sj = (IDX)g.sj;
  const float pc = p[c];
  float pE, pW, pN, pS, pT, pB;
  if (POL == 3) {  // press, cell away from the x and y faces: only the k remaps
    pE = p[c + si];
    pW = p[c - si];
    pN = p[c + sj];
    pS = p[c - sj];
    pT = (k == g.km) ? 0.0f : p[c + 1];
    pB = (k == 1) ? pc : p[c - 1];
  } else if (POL == 1) {
    pE = (i == g.im && g.east_bc) ? 0.0f : p[c + si];
    pW = (i == 1 && g.west_bc) ? pc : p[c - si];
    pN = (j == g.jm && !y_stored) ? p[c - (IDX)(g.jm - 1) * sj] : p[c + sj];
    pS = (j == 1 && !y_stored) ? p[c + (IDX)(g.jm - 1) * sj] : p[c - sj];
    pT = (k == g.km) ? 0.0f : p[c + 1];
    pB = (k == 1) ? pc : p[c - 1];
  } else {
    pE = p[c + si];
    pW = p[c - si];
    pN = p[c + sj];
    pS = p[c - sj];
    pT = p[c + 1];
    pB = p[c - 1];
  }
  // sor.py:164-171: E, W, N, S, T, B summed left to right
  float nb, cn1;
  if (UNI) {  // every entry of each weight vector equal (build_uniform_coeffs), cn1 a scalar
    nb = cf.w2l * pE;
    nb = nb + cf.w2s * pW;
    nb = nb + cf.w3l * pN;
    nb = nb + cf.w3s * pS;
    nb = nb + cf.w4l * pT;
    nb = nb + cf.w4s * pB;
    cn1 = cf.cn1s;
  } else {
    nb = cf.cn2l[i - 1] * pE;
    nb = nb + cf.cn2s[i - 1] * pW;
    nb = nb + cf.cn3l[j - 1] * pN;
    nb = nb + cf.cn3s[j - 1] * pS;
    nb = nb + cf.cn4l[k - 1] * pT;
    nb = nb + cf.cn4s[k - 1] * pB;
    cn1 = cf.cn1 ? cf.cn1[((long long)(i - 1) * g.jm + (j - 1)) * g.km + (k - 1)] : cf.cn1s;
  }
  pc_out = pc;
  // sor.py:197: reltmp = omega * (cn1 * (nb - rhs) - p)
  return om * (cn1 * (nb - rhs[c]) - pc);
}

// One red-black colour pass, in place (sor.py:194-200).  Thread x enumerates
// the colour's cells along k: k = 1 + ((i0 + j0 + nrd) & 1) + 2 t.  UNI uses
// the scalar weights and 32-bit indices (grids below 2^31 cells).
template <int POL, bool UNI>
__global__ void __launch_bounds__(RB_NT) k_sor_rb(Geo g, float* __restrict__ p, const float* __restrict__ rhs,
                                                         SorC cf, float om, int nrd, int y_stored,
                                                         double* __restrict__ partials) {
  __shared__ double red[RB_NW];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.z + 1;
  const int ig0 = i + g.ioff - 1;
  // RB_R rows per thread (j0, j0 + by, ...): every row's loads are issued
  // before the first store -- a colour pass writes only its own colour and
  // reads only the other one plus the centre, so nothing aliases -- which
  // keeps RB_R times more bytes in flight per thread
  float pc[RB_R], rel[RB_R];
  long long cc[RB_R];
  bool ok[RB_R];
#pragma unroll
  for (int q = 0; q < RB_R; ++q) {
    const int j = (blockIdx.y * RB_R + q) * blockDim.y + threadIdx.y + 1;
    const int k = 1 + ((ig0 + (j - 1) + nrd) & 1) + 2 * t;
    ok[q] = j <= g.jm && k <= g.km;
    cc[q] = 0;
    rel[q] = 0.0f;
    pc[q] = 0.0f;
    if (!ok[q]) continue;
    if (UNI) {
      const int c = i * (int)g.si + j * g.sj + k;
      cc[q] = c;
      // press: rows away from the x and y faces need only the k remaps
      // (block-uniform in i, row-uniform in j)
      if (POL == 1 && i > 1 && i < g.im && j > 1 && j < g.jm)
        rel[q] = sor_point<3, true, int>(g, p, rhs, cf, om, c, i, j, k, y_stored, pc[q]);
      else
        rel[q] = sor_point<POL, true, int>(g, p, rhs, cf, om, c, i, j, k, y_stored, pc[q]);
    } else {
      const long long c = cidx(g, i, j, k);
      cc[q] = c;
      rel[q] = sor_point<POL>(g, p, rhs, cf, om, c, i, j, k, y_stored, pc[q]);
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < RB_R; ++q) {
    if (!ok[q]) continue;
    p[cc[q]] = pc[q] + rel[q];
    acc += (double)rel[q] * (double)rel[q];
  }
  // fixed-order block reduction over the block's (possibly partial) warps
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

// One twinned (Jacobi) sweep: read src everywhere, write the interior of dst
// (sor.py:206-246).
constexpr int TW_BX = 32, TW_BY = 8, TW_NW = TW_BX * TW_BY / 32;

// TW_R rows per thread (j, j + TW_BY, ...): src and dst never alias, so all
// rows' loads go out together; UNI: scalar weights and 32-bit indexing.
constexpr int TW_R = 4;
template <int POL, bool UNI>
__global__ void __launch_bounds__(TW_BX* TW_BY) k_sor_tw(Geo g, const float* __restrict__ src,
                                                         float* __restrict__ dst, const float* __restrict__ rhs,
                                                         SorC cf, float om, double* __restrict__ partials) {
  __shared__ double red[TW_NW];
  const int k = blockIdx.x * TW_BX + threadIdx.x + 1;
  const int i = blockIdx.z + 1;
  float pc[TW_R], rel[TW_R];
  long long cc[TW_R];
  bool ok[TW_R];
#pragma unroll
  for (int q = 0; q < TW_R; ++q) {
    const int j = (blockIdx.y * TW_R + q) * TW_BY + threadIdx.y + 1;
    ok[q] = j <= g.jm && k <= g.km;
    cc[q] = 0;
    pc[q] = rel[q] = 0.0f;
    if (!ok[q]) continue;
    if (UNI) {
      const int c = i * (int)g.si + j * g.sj + k;
      cc[q] = c;
      if (POL == 1 && i > 1 && i < g.im && j > 1 && j < g.jm)  // press away from the x / y faces
        rel[q] = sor_point<3, true, int>(g, src, rhs, cf, om, c, i, j, k, 0, pc[q]);
      else
        rel[q] = sor_point<POL, true, int>(g, src, rhs, cf, om, c, i, j, k, 0, pc[q]);
    } else {
      const long long c = cidx(g, i, j, k);
      cc[q] = c;
      rel[q] = sor_point<POL>(g, src, rhs, cf, om, c, i, j, k, 0, pc[q]);
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < TW_R; ++q) {
    if (!ok[q]) continue;
    dst[cc[q]] = pc[q] + rel[q];
    acc += (double)rel[q] * (double)rel[q];
  }
  const double s = block_sum<TW_NW>(acc, red);
  if (threadIdx.x == 0 && threadIdx.y == 0)
    partials[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
}

// Snapshot of the y halo planes used by the stencils (odd jm, PRESS policy).
__global__ void k_refresh_y(Geo g, float* __restrict__ p) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int i = blockIdx.y + 1;
  if (k > g.km) return;
  p[cidx(g, i, 0, k)] = p[cidx(g, i, g.jm, k)];
  p[cidx(g, i, g.jm + 1, k)] = p[cidx(g, i, 1, k)];
}

// Final halo_fn(p) of the press policy in closed form: resolve k (0 -> 1,
// km+1 -> 0), then j (periodic), then i (0 -> 1, im+1 -> 0).  Reads src and
// writes the whole array to dst (src == dst: in place; halo sources are
// interior cells, which are not written).  Optionally checks every cell of
// the result for finiteness (press stage, les.py:413-415).
__global__ void k_press_halo(Geo g, const float* src, float* dst, unsigned* flags) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int i = blockIdx.z;
  unsigned bits = 0;
  if (k <= g.km + 1 && j <= g.jm + 1) {
    const long long c = cidx(g, i, j, k);
    const bool halo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1 || k == 0 || k == g.km + 1;
    const bool foreign = (i == 0 && !g.west_bc) || (i == g.im + 1 && !g.east_bc);
    float val;
    if (halo && !foreign) {
      if (k == g.km + 1 || i == g.im + 1) {
        val = 0.0f;
      } else {
        const int kk = k == 0 ? 1 : k;
        const int jj = j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j);
        const int ii = i == 0 ? 1 : i;
        val = src[cidx(g, ii, jj, kk)];
      }
      dst[c] = val;
    } else {
      val = src[c];
      if (src != dst) dst[c] = val;
    }
    if (flags && !finite32(val)) bits = F_PRESS;
  }
  if (flags) flag_or(flags, bits);
}

// The same by rows: a warp takes PH_R consecutive (i, j) rows, lanes over k
// (one row decode per warp instead of a div/mod per element, all PH_R rows'
// loads in flight at once).  The 3-D launch above is latency bound (one
// dependent load per thread: ~470 us on 600x600x90, ~300 GB/s); this is
// bound by HBM.
constexpr int PH_R = 4, PH_WARPS = 8;
template <int NK>
__global__ void __launch_bounds__(PH_WARPS * 32) k_press_halo_rows(Geo g, const float* src, float* dst,
                                                                    unsigned* flags) {
  const int lane = threadIdx.x & 31;
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  const long long r0 = ((long long)blockIdx.x * PH_WARPS + (threadIdx.x >> 5)) * PH_R;
  float val[PH_R][NK];
  unsigned bits = 0;
#pragma unroll
  for (int q = 0; q < PH_R; ++q) {
    const long long row = r0 + q;
    const int i = (int)(row / (g.jm + 2)), j = (int)(row - (long long)i * (g.jm + 2));
    const bool rowhalo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1;
    const bool foreign = (i == 0 && !g.west_bc) || (i == g.im + 1 && !g.east_bc);
    // the row whose values this row takes: itself, or (press) its closed-form source
    const bool zero_row = rowhalo && !foreign && i == g.im + 1;
    const int ii = (rowhalo && !foreign && i == 0) ? 1 : i;
    const int jj = (rowhalo && !foreign) ? (j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j)) : j;
    const float* s = src + cidx(g, ii, jj, 0);
#pragma unroll
    for (int u = 0; u < NK; ++u) {
      const int k = lane + 32 * u;
      val[q][u] = 0.0f;
      if (row >= nrow || k > g.km + 1 || zero_row) continue;
      const int kk = (foreign || k > 0) ? k : 1;   // bottom: p[.,.,0] -> p[.,.,1]
      val[q][u] = (!foreign && k == g.km + 1) ? 0.0f : s[kk];
    }
  }
#pragma unroll
  for (int q = 0; q < PH_R; ++q) {
    const long long row = r0 + q;
    if (row >= nrow) continue;
    const int i = (int)(row / (g.jm + 2)), j = (int)(row - (long long)i * (g.jm + 2));
    const bool rowhalo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1;
    const bool foreign = (i == 0 && !g.west_bc) || (i == g.im + 1 && !g.east_bc);
    float* d = dst + cidx(g, i, j, 0);
#pragma unroll
    for (int u = 0; u < NK; ++u) {
      const int k = lane + 32 * u;
      if (k > g.km + 1) continue;
      const bool halo = !foreign && (rowhalo || k == 0 || k == g.km + 1);
      if (halo || src != dst) d[k] = val[q][u];
      if (flags && !finite32(val[q][u])) bits = F_PRESS;
    }
  }
  if (flags) flag_or(flags, bits);
}

// residuals[it] = (sum of pass-0 partials) + (sum of pass-1 partials), each
// summed by one fixed-order tree (deterministic; numpy's pairwise order is
// matched only to rtol ~1e-15).
// res[it]: both passes' partials of iteration it ([2][nblk], contiguous) in
// one fixed-order block reduction (1024 threads: the rows are short, so the
// reduction is load-latency bound and wants every load in flight at once)
constexpr int RES_RED_THREADS = 1024;
__global__ void __launch_bounds__(RES_RED_THREADS) k_reduce_res(const double* __restrict__ partials, int nblk,
                                                                 double* __restrict__ out) {
  __shared__ double red[RES_RED_THREADS / 32];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (programmatic launch: the partials are upstream output)
  const int it = blockIdx.x;
  const double* q = partials + (long long)it * 2 * nblk;
  double a = 0.0;
#pragma unroll 4
  for (int b = threadIdx.x; b < 2 * nblk; b += RES_RED_THREADS) a += q[b];
  a = block_sum<RES_RED_THREADS / 32>(a, red);
  if (threadIdx.x == 0) out[it] = a;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int sor_blocks_rb(const Geo& g) {
  const int kh = (g.km + 1) / 2;
  int bx, by;
  rb_shape(g, &bx, &by);
  return ((kh + bx - 1) / bx) * ((g.jm + by * RB_R - 1) / (by * RB_R)) * g.im;
}
int sor_blocks_tw(const Geo& g) {
  return ((g.km + TW_BX - 1) / TW_BX) * ((g.jm + TW_BY * TW_R - 1) / (TW_BY * TW_R)) * g.im;
}

void launch_rb_pass(const Geo& g, float* p, const float* rhs, const SorC& cf, float om, int nrd, int policy,
                    double* partials, cudaStream_t st) {
  const int kh = (g.km + 1) / 2;
  int bx, by;
  rb_shape(g, &bx, &by);
  dim3 grid((kh + bx - 1) / bx, (g.jm + by * RB_R - 1) / (by * RB_R), g.im);
  dim3 block(bx, by);
  const int y_stored = (policy == 1 && (g.jm & 1)) ? 1 : 0;
  if (y_stored) {
    dim3 gy((g.km + 127) / 128, g.im);
    k_refresh_y<<<gy, 128, 0, st>>>(g, p);
  }
  const bool uni = cf.uni && !cf.cn1 && (long long)(g.im + 3) * g.si < (1LL << 31);
  if (policy == 1) {
    if (uni) k_sor_rb<1, true><<<grid, block, 0, st>>>(g, p, rhs, cf, om, nrd, y_stored, partials);
    else k_sor_rb<1, false><<<grid, block, 0, st>>>(g, p, rhs, cf, om, nrd, y_stored, partials);
  } else {
    if (uni) k_sor_rb<0, true><<<grid, block, 0, st>>>(g, p, rhs, cf, om, nrd, 0, partials);
    else k_sor_rb<0, false><<<grid, block, 0, st>>>(g, p, rhs, cf, om, nrd, 0, partials);
  }
}

void launch_tw_sweep(const Geo& g, const float* src, float* dst, const float* rhs, const SorC& cf, float om,
                     int policy, double* partials, cudaStream_t st) {
  dim3 grid((g.km + TW_BX - 1) / TW_BX, (g.jm + TW_BY * TW_R - 1) / (TW_BY * TW_R), g.im);
  dim3 block(TW_BX, TW_BY);
  const bool uni = cf.uni && !cf.cn1 && (long long)(g.im + 3) * g.si < (1LL << 31);
  if (policy == 1) {
    if (uni) k_sor_tw<1, true><<<grid, block, 0, st>>>(g, src, dst, rhs, cf, om, partials);
    else k_sor_tw<1, false><<<grid, block, 0, st>>>(g, src, dst, rhs, cf, om, partials);
  } else {
    if (uni) k_sor_tw<0, true><<<grid, block, 0, st>>>(g, src, dst, rhs, cf, om, partials);
    else k_sor_tw<0, false><<<grid, block, 0, st>>>(g, src, dst, rhs, cf, om, partials);
  }
}

void launch_press_halo(const Geo& g, float* p, unsigned* flags, cudaStream_t st) {
  launch_press_halo_copy(g, p, p, flags, st);
}

void launch_press_halo_copy(const Geo& g, const float* src, float* dst, unsigned* flags, cudaStream_t st) {
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  const unsigned nblk = (unsigned)((nrow + PH_R * PH_WARPS - 1) / (PH_R * PH_WARPS));
  const int nk = (g.km + 2 + 31) / 32;
  if (nk <= 4) {  // km + 2 <= 128: rows (otherwise the 3-D launch)
    switch (nk) {
      case 1: k_press_halo_rows<1><<<nblk, PH_WARPS * 32, 0, st>>>(g, src, dst, flags); return;
      case 2: k_press_halo_rows<2><<<nblk, PH_WARPS * 32, 0, st>>>(g, src, dst, flags); return;
      case 3: k_press_halo_rows<3><<<nblk, PH_WARPS * 32, 0, st>>>(g, src, dst, flags); return;
      default: k_press_halo_rows<4><<<nblk, PH_WARPS * 32, 0, st>>>(g, src, dst, flags); return;
    }
  }
  int bx = ((g.km + 2 + 31) / 32) * 32;
  if (bx > 128) bx = 128;
  int by = 256 / bx;
  dim3 grid((g.km + 2 + bx - 1) / bx, (g.jm + 2 + by - 1) / by, g.im + 2);
  k_press_halo<<<grid, dim3(bx, by), 0, st>>>(g, src, dst, flags);
}

// Stage 1 of the residual reduction for long partial rows: block (c, r) sums
// chunk c (RED_CHUNK consecutive partials) of row r = 2 it + pass, in a fixed
// order, so the two-stage sum is deterministic.
constexpr int RED_CHUNK = 4096;
__global__ void k_reduce_chunks(const double* __restrict__ partials, int nblk, int nch, double* __restrict__ out) {
  __shared__ double red[8];
  const int c = blockIdx.x, r = blockIdx.y;
  const double* q = partials + (long long)r * nblk + (long long)c * RED_CHUNK;
  const int n = min(RED_CHUNK, nblk - c * RED_CHUNK);
  double a = 0.0;
  for (int b = threadIdx.x; b < n; b += blockDim.x) a += q[b];
  a = block_sum<8>(a, red);
  if (threadIdx.x == 0) out[(long long)r * nch + c] = a;
}

int reduce_scratch(int nblk, int n_iter) {
  const int nch = (nblk + RED_CHUNK - 1) / RED_CHUNK;
  return nch > 1 ? 2 * n_iter * nch : 0;
}

// res[it] = sum over both passes of iteration it of the per-block partials
// ([n_iter][2][nblk]).  Rows longer than one chunk are first cut into chunk
// sums (written after the partials: the caller sizes the buffer with
// reduce_scratch), so a 600x600x90 solve reduces in microseconds instead of
// one 256-thread block per iteration walking ~150k partials.
void launch_reduce_res(const double* partials, int nblk, int n_iter, double* out, cudaStream_t st) {
  const int nch = (nblk + RED_CHUNK - 1) / RED_CHUNK;
  if (nch <= 1) {
    static const bool pdl = !(std::getenv("LESB_PDL") && std::atoi(std::getenv("LESB_PDL")) == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_iter);
    cfg.blockDim = dim3(RES_RED_THREADS);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_reduce_res, partials, nblk, out);
    return;
  }
  double* scratch = const_cast<double*>(partials) + (long long)2 * n_iter * nblk;
  k_reduce_chunks<<<dim3(nch, 2 * n_iter), 256, 0, st>>>(partials, nblk, nch, scratch);
  k_reduce_res<<<n_iter, RES_RED_THREADS, 0, st>>>(scratch, nch, out);
}

int sor_kernels_per_solve(const Geo& g, const SorC& cf, int n_iter, int scheme, int policy, bool resident,
                          bool natural) {
  if (resident && scheme == 0) return 1;
  const bool oddy = policy == 1 && (g.jm & 1);
  const int red = (int)(reduce_scratch(scheme == 0 ? sor_blocks_rb(g) : sor_blocks_tw(g), n_iter) > 0) + 1;
  if (scheme == 0 && !natural && split_supported(g, cf))  // pack, passes (+ y snapshots), unpack, reduction
    return 1 + (oddy ? 4 : 2) * n_iter + 1 + ((int)(reduce_scratch(sor_blocks_split(g), n_iter) > 0) + 1);
  if (scheme == 1 && !natural && tws_supported(g, cf))  // pack, 2 sweeps per iteration, unpack, reduction
    return 1 + 2 * n_iter + 1 + ((int)(reduce_scratch(sor_blocks_tws(g), n_iter) > 0) + 1);
  int per_iter = 2;
  if (scheme == 0 && oddy) per_iter = 4;
  return per_iter * n_iter + (policy == 1 ? 1 : 0) + red;
}

// Enqueue a full solve on p (in place).  TWINNED needs pb initialised to a
// copy of p by the caller (make_twinned, sor.py:145-150).
cudaError_t enqueue_sor(const Geo& g, float* p, float* pb, const float* rhs, const SorC& cf, float om, int n_iter,
                        int scheme, int policy, double* partials, double* res_dev, unsigned* flags, cudaStream_t st,
                        const ExchangeHook* hook, const SorMarks* marks, const ResidentBufs* res) {
  const bool hooked = hook && hook->fn;
  if (scheme == 0 && res && res->use && !hooked && resident_supported(g, cf, res->device)) {
    // one launch: passes, press halo + its non-finite check, residuals
    ResidentCall call{&g,      res->device, p,          rhs,      &cf,      om,      n_iter,
                      policy,  res->xbuf,   res->epoch, partials, res_dev,  flags,   res->err,
                      res->peer_w, res->peer_e};
    const bool book = res->book && !res->peer_w && !res->peer_e;
    if (book) call.book = res->book;
    cudaError_t e = launch_sor_resident(call, st);
    if (e != cudaSuccess) return e;
    if (book && res->book_used) *res->book_used = true;
    if (marks && marks->after_passes) cudaEventRecordWithFlags(marks->after_passes, st, cudaEventRecordExternal);
    return cudaGetLastError();
  }
  if (scheme == 0 && res && res->split && !res->natural && split_supported(g, cf)) {
    // colour-split streaming passes: split p and rhs, 2 n_iter unit-stride
    // passes (each followed by the slab's plane exchange of the colour it
    // wrote), merge back with the final halo_fn and the press check
    // x-slabs with mapped neighbours: the edge-plane exchange is fused into
    // the pass kernel (PassGhost); otherwise the hook exchanges the colour's
    // planes after every pass
    const SplitGeo sg = split_geo(g);
    const int nblk = sor_blocks_split(g);
    const bool gho = res->ghost.on() && ghost_supported(g, n_iter);
    launch_split_pack(g, p, rhs, res->split, policy, st);
    if (gho) launch_ghost_prologue(g, res->split, res->ghost, st);
    for (int it = 0; it < n_iter; ++it) {
      for (int c = 0; c < 2; ++c) {
        PassGhost gp = res->ghost;
        gp.pass = 2 * it + c;
        launch_rbs_pass(g, res->split, cf, om, c, policy, partials + ((long long)it * 2 + c) * nblk, st,
                        gho ? &gp : nullptr);
        if (hooked && !gho) hook->fn(hook->ctx, res->split + c * sg.n, sg.spi);
      }
    }
    if (marks && marks->after_passes) cudaEventRecordWithFlags(marks->after_passes, st, cudaEventRecordExternal);
    launch_split_unpack(g, res->split, p, policy, policy == 1 ? flags : nullptr, st);
    if (hooked && (policy == 1 || gho)) hook->fn(hook->ctx, p, g.si);  // the inner x halo planes: final values
    launch_reduce_res(partials, nblk, n_iter, res_dev, st);
    return cudaGetLastError();
  }
  if (scheme == 1 && res && res->split && !res->natural && !hooked && tws_supported(g, cf)) {
    // twinned sweeps on the colour-split layout: pack p into both buffers
    // (the stored / closed-form halos live in both), sweep A -> B -> A, the
    // newest iterate ends in A (component 0, sor.py:308-309)
    const SplitGeo sg = split_geo(g);
    float* A = res->split;
    float* B = res->split + 4 * sg.n;
    const float* R = res->split + 2 * sg.n;
    const int nblk = sor_blocks_tws(g);
    launch_split_pack(g, p, rhs, res->split, policy, st, B);
    for (int it = 0; it < n_iter; ++it) {
      launch_tws_sweep(g, A, B, R, cf, om, policy, partials + ((long long)it * 2 + 0) * nblk, st);
      launch_tws_sweep(g, B, A, R, cf, om, policy, partials + ((long long)it * 2 + 1) * nblk, st);
    }
    if (marks && marks->after_passes) cudaEventRecordWithFlags(marks->after_passes, st, cudaEventRecordExternal);
    launch_split_unpack(g, A, p, policy, policy == 1 ? flags : nullptr, st);
    launch_reduce_res(partials, nblk, n_iter, res_dev, st);
    return cudaGetLastError();
  }
  const int nblk = scheme == 0 ? sor_blocks_rb(g) : sor_blocks_tw(g);
  for (int it = 0; it < n_iter; ++it) {
    for (int nrd = 0; nrd < 2; ++nrd) {
      double* part = partials + ((long long)it * 2 + nrd) * nblk;
      if (scheme == 0) {
        launch_rb_pass(g, p, rhs, cf, om, nrd, policy, part, st);
        if (hooked) hook->fn(hook->ctx, p, g.si);
      } else {
        const float* s = nrd == 0 ? p : pb;
        float* d = nrd == 0 ? pb : p;
        launch_tw_sweep(g, s, d, rhs, cf, om, policy, part, st);
        if (hooked) hook->fn(hook->ctx, d, g.si);
      }
    }
  }
  if (marks && marks->after_passes) cudaEventRecordWithFlags(marks->after_passes, st, cudaEventRecordExternal);
  if (policy == 1) {
    launch_press_halo(g, p, flags, st);
    if (hooked) hook->fn(hook->ctx, p, g.si);
  }
  launch_reduce_res(partials, nblk, n_iter, res_dev, st);
  return cudaGetLastError();
}

}  // namespace lesb
