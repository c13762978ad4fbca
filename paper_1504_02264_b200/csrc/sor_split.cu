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
// colour's rhs, and writes its own cells, all unit-stride.  The natural
// layout's pass strides over both colours (every sector it touches is half
// the other colour), which kept it at ~20 B/cell/iteration of DRAM traffic
// instead of 16.
//
// Pass kernel.  A thread owns four consecutive slots (16-byte accesses) of
// RBS_R consecutive rows j of one plane i and issues all their loads before
// computing: its own cells, rhs, the other colour's rows (i+-1, j) and one
// scalar for the T/B shift per row, and the other colour's rows j0-1 ..
// j0+RBS_R of plane i once (row j's N is row j+1's centre row) -- for two
// rows, twelve 16-byte loads and two 4-byte loads for eight cells, all in
// flight together.  RBS_R is even, so the parity s of a thread's first row
// is uniform per block (it depends on c and the plane) and the T/B
// selection is compiled per parity.
//
// Halo policy.  STORED (halo_fn=None): the halos are p0's, read as stored.
// PRESS (les._pressure_halo before every pass): the pack writes the
// closed-form halo, and the pass keeps every halo cell a
// stencil reads equal to its current source by mirror writes, so the pass
// itself reads every neighbour plainly:
//   W  p[0,j,k]    = p[1,j,k]   the cell itself: stored with it (other array, plane 0)
//   B  p[i,j,0]    = p[i,j,1]   the cell itself: stored with it (other array, slot 0)
//   E  p[im+1,j,k] = 0, T p[i,j,km+1] = 0: written by the pack, never changed
//   S/N (even jm)  p[i,0,k] = p[i,jm,k], p[i,jm+1,k] = p[i,1,k]: rows jm / 1
//                  are the same colour as rows 0 / jm+1 and are mirrored
//                  into them when written; their readers run in the next pass
//   S/N (odd jm)   the halo rows and their sources share the pass: a
//                  pre-pass snapshot (k_split_refresh_y), as the reference's
//                  halo_fn before the pass
// Each mirrored slot is read in the pass only by the thread that writes it,
// before it writes it.  k_split_unpack merges p back with the final halo_fn
// in closed form and the press stage's non-finite check.
//
// Arithmetic: A8 in the reference's order, bitwise equal to the other
// solvers; the residual of a cell is fma((f64)rel, (f64)rel, acc) -- the
// f64 product of two f32 values is exact, so this is the reference's
// sum += rel*rel term -- summed per thread in row/slot order, per block by a
// fixed shuffle tree, per iteration by launch_reduce_res.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

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

// build-time switches (scripts/build_variant.sh -D...): rows per thread,
// minimum resident blocks
#ifndef RBS_ROWS
#define RBS_ROWS 2
#endif
#ifndef RBS_MINB
#define RBS_MINB 1
#endif
constexpr int RBS_NT = 256;        // threads per pass block (x: float4 groups of a row, y: row runs)
constexpr int RBS_R = RBS_ROWS;    // consecutive rows per thread (even: uniform first-row parity)

inline void rbs_shape(const SplitGeo& s, int* bx, int* by) {
  *bx = s.kh4 < RBS_NT ? s.kh4 : RBS_NT;
  *by = RBS_NT / *bx;
  if (*by < 1) *by = 1;
}

// Split p and rhs: a warp per natural row (i, j), lanes over k.  PRESS:
// halo cells (not on a neighbour slab's plane) take the closed-form
// halo_fn value (k: 0 -> 1, km+1 -> 0; then j periodic; then i: 0 -> 1,
// im+1 -> 0) -- the state the reference's halo_fn leaves before pass 0.
template <int POL, bool COPY>
__global__ void __launch_bounds__(256) k_split_pack(Geo g, SplitGeo sg, const float* __restrict__ p,
                                                    const float* __restrict__ rhs, float* __restrict__ ps,
                                                    float* __restrict__ rs, float* __restrict__ ps2) {
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= nrow) return;
  const int lane = threadIdx.x & 31;
  const int i = (int)(row / (g.jm + 2)), j = (int)(row - (long long)i * (g.jm + 2));
  const int par = (i + g.ioff + j + 1) & 1;
  const bool rowhalo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1;
  const bool foreign = (i == 0 && !g.west_bc) || (i == g.im + 1 && !g.east_bc);
  const bool remap = POL == 1 && !foreign;
  const bool zero_row = remap && i == g.im + 1;
  const int ii = (remap && i == 0) ? 1 : i;
  const int jj = (remap && rowhalo) ? (j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j)) : j;
  const float* src_p = p + ((long long)ii * (g.jm + 2) + jj) * (g.km + 2);
  const float* src_r = rhs + row * (g.km + 2);
  const long long rb = row * sg.khp;
  for (int k = lane; k < g.km + 2; k += 32) {
    float val;
    if (zero_row || (remap && k == g.km + 1)) val = 0.0f;
    else val = src_p[(remap && k == 0) ? 1 : k];
    const int c = (par + k) & 1;
    const long long d = c * sg.n + rb + (k >> 1);
    ps[d] = val;
    rs[d] = src_r[k];
    if (COPY) ps2[d] = val;
  }
}

// k_split_pack with four cells of a row per thread (16-byte loads, 8-byte
// stores into each colour array): rows of km + 2 = 4q words start 16-byte
// aligned and a group's four cells are two consecutive slots of each colour.
// Same per-cell rules as k_split_pack.
template <int POL, bool COPY>
__global__ void __launch_bounds__(256) k_split_pack4(Geo g, SplitGeo sg, const float* __restrict__ p,
                                                     const float* __restrict__ rhs, float* __restrict__ ps,
                                                     float* __restrict__ rs, float* __restrict__ ps2) {
  const int G = (g.km + 2) >> 2;  // groups per row
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  if (t >= nrow * G) return;
  const long long row = t / G;
  const int k0 = 4 * (int)(t - row * G);
  const int i = (int)(row / (g.jm + 2)), j = (int)(row - (long long)i * (g.jm + 2));
  const int par = (i + g.ioff + j + 1) & 1;
  const bool rowhalo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1;
  const bool foreign = (i == 0 && !g.west_bc) || (i == g.im + 1 && !g.east_bc);
  const bool remap = POL == 1 && !foreign;
  const bool zero_row = remap && i == g.im + 1;
  const int ii = (remap && i == 0) ? 1 : i;
  const int jj = (remap && rowhalo) ? (j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j)) : j;
  const float4 P = *reinterpret_cast<const float4*>(p + ((long long)ii * (g.jm + 2) + jj) * (g.km + 2) + k0);
  const float4 R = *reinterpret_cast<const float4*>(rhs + row * (g.km + 2) + k0);
  float v[4] = {P.x, P.y, P.z, P.w};
  if (remap && k0 == 0) v[0] = P.y;  // p[0] -> p[1]
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (zero_row || (remap && k0 + e == g.km + 1)) v[e] = 0.0f;
  const int c0 = (par + k0) & 1;
  const long long d0 = (long long)c0 * sg.n + row * sg.khp + (k0 >> 1);
  const long long d1 = (long long)(1 - c0) * sg.n + row * sg.khp + (k0 >> 1);
  *reinterpret_cast<float2*>(ps + d0) = make_float2(v[0], v[2]);
  *reinterpret_cast<float2*>(ps + d1) = make_float2(v[1], v[3]);
  *reinterpret_cast<float2*>(rs + d0) = make_float2(R.x, R.z);
  *reinterpret_cast<float2*>(rs + d1) = make_float2(R.y, R.w);
  if (COPY) {
    *reinterpret_cast<float2*>(ps2 + d0) = make_float2(v[0], v[2]);
    *reinterpret_cast<float2*>(ps2 + d1) = make_float2(v[1], v[3]);
  }
}

// Pass loads go through the read-only (non-coherent) path: within a pass the
// only locations written besides the thread's own cells are the PRESS
// mirror slots, each read earlier in the pass by the thread that writes it.
__device__ __forceinline__ float4 ld4(const float* a) { return __ldg(reinterpret_cast<const float4*>(a)); }
__device__ __forceinline__ float ld1(const float* a) { return __ldg(a); }
__device__ __forceinline__ void st4(float* a, float x, float y, float z, float w) {
  *reinterpret_cast<float4*>(a) = make_float4(x, y, z, w);
}

// One row of four cells: S is the row parity (compile time).  nb/rel in
// the reference's order (sor.py:164-171, 197).
template <int S>
__device__ __forceinline__ void rbs_row(const SorC& cf, float om, const float4& C, const float4& RH, const float4& E,
                                        const float4& W, const float4& N, const float4& So, const float4& M,
                                        float extra, const bool (&in)[4], float (&val)[4], double& acc) {
  const float cv[4] = {C.x, C.y, C.z, C.w};
  const float rv[4] = {RH.x, RH.y, RH.z, RH.w};
  const float ev[4] = {E.x, E.y, E.z, E.w};
  const float wv[4] = {W.x, W.y, W.z, W.w};
  const float nv[4] = {N.x, N.y, N.z, N.w};
  const float sv[4] = {So.x, So.y, So.z, So.w};
  // T/B: S = 0 -> T = m[t], B = m[t-1] (t0-1: extra); S = 1 -> T = m[t+1] (t0+4: extra), B = m[t]
  const float mv[6] = {S == 0 ? extra : M.x, M.x, M.y, M.z, M.w, S == 1 ? extra : M.w};
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float pT = S == 0 ? mv[m + 1] : mv[m + 2];
    const float pB = S == 0 ? mv[m] : mv[m + 1];
    float nb = cf.w2l * ev[m];
    nb = nb + cf.w2s * wv[m];
    nb = nb + cf.w3l * nv[m];
    nb = nb + cf.w3s * sv[m];
    nb = nb + cf.w4l * pT;
    nb = nb + cf.w4s * pB;
    const float rel = om * (cf.cn1s * (nb - rv[m]) - cv[m]);
    // non-interior slots (k halo, row padding) keep their stored value
    val[m] = in[m] ? cv[m] + rel : cv[m];
    const double d = in[m] ? (double)rel : 0.0;
    acc = __fma_rn(d, d, acc);
  }
}

// The rows of one thread: RBS_R consecutive rows from j0 (S0 = parity of
// row j0), four slots each, marching along j with the other colour's rows
// j-1, j, j+1 in registers.
template <int POL, int S0>
__device__ __forceinline__ void rbs_march(const Geo& g, const SplitGeo& sg, float* own, float* oth, const float* rh,
                                          const SorC& cf, float om, int q, int i, int j0, double& acc) {
  const int spi = (int)sg.spi, khp = sg.khp;
  // cells m of a parity-s row are interior iff 1 <= 8q + s + 2m <= km
  bool in0[4], in1[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int k0 = 8 * q + 2 * m;
    in0[m] = k0 >= 1 && k0 <= g.km;
    in1[m] = k0 + 1 <= g.km;
  }
  const bool wmir = POL != 0 && i == 1 && g.west_bc;
  const int nr = min(RBS_R, g.jm - j0 + 1);  // rows of this thread
  // every load of the thread's rows first (a colour pass writes only its own
  // colour and the mirror slots, which no load of the pass reads): the
  // other colour's rows j0-1 .. j0+R (row j's N is row j+1's centre row, its
  // S row j-1's), and per row its own cells, rhs, the rows (i+-1, j) and the
  // T/B shift scalar -- slot t0-1 (parity 0; for q = 0 the previous row's
  // last slot, in bounds) or t0+4 (parity 1; the next row's first slot for
  // the last group)
  float4 O[RBS_R + 2], C[RBS_R], RH[RBS_R], E[RBS_R], W[RBS_R];
  float X[RBS_R];
  O[0] = ld4(oth - khp);
#pragma unroll
  for (int r = 0; r < RBS_R; ++r) {
    if (r < nr) {
      const int ro = r * khp;
      O[r + 1] = ld4(oth + ro);
      C[r] = ld4(own + ro);
      RH[r] = ld4(rh + ro);
      E[r] = ld4(oth + ro + spi);
      W[r] = ld4(oth + ro - spi);
      X[r] = ld1(oth + ro + (((S0 + r) & 1) == 0 ? -1 : 4));
      if (r == nr - 1) O[r + 2] = ld4(oth + ro + khp);  // the last row's N
    }
  }
#pragma unroll
  for (int r = 0; r < RBS_R; ++r) {
    if (r >= nr) break;
    const int j = j0 + r;
    const int ro = r * khp;
    float val[4];
    if (((S0 + r) & 1) == 0) {
      rbs_row<0>(cf, om, C[r], RH[r], E[r], W[r], O[r + 2], O[r], O[r + 1], X[r], in0, val, acc);
    } else {
      rbs_row<1>(cf, om, C[r], RH[r], E[r], W[r], O[r + 2], O[r], O[r + 1], X[r], in1, val, acc);
      if (POL != 0 && q == 0) oth[ro] = val[0];  // B mirror: p[i,j,0] = p[i,j,1]
    }
    st4(own + ro, val[0], val[1], val[2], val[3]);
    if (wmir) st4(oth + ro - spi, val[0], val[1], val[2], val[3]);  // W mirror: p[0,j,k] = p[1,j,k]
    if (POL == 1) {  // even jm: p[i,jm+1,k] = p[i,1,k], p[i,0,k] = p[i,jm,k] (same colour)
      if (j == 1) st4(own + ro + g.jm * khp, val[0], val[1], val[2], val[3]);
      if (j == g.jm) st4(own + ro - g.jm * khp, val[0], val[1], val[2], val[3]);
    }
  }
}

// One colour pass (colour c) in place on the split arrays.
// POL 0: stored halo; 1: press, even jm (y mirrors); 2: press, odd jm
// (y halo rows refreshed before the pass).  Every thread's first row is
// odd (1 + a multiple of RBS_R), so its parity (c + ig) & 1 is uniform per
// block: one block-uniform branch picks the compiled parity.  The residual
// is reduced per warp (one partial per warp, no block barrier: warps that
// finish early leave).
template <int POL>
__global__ void __launch_bounds__(RBS_NT, RBS_MINB) k_sor_rbs(Geo g, SplitGeo sg, float* __restrict__ ps,
                                                    const float* __restrict__ rs, SorC cf, float om, int c,
                                                    double* __restrict__ partials) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;  // float4 group of the rows
  const int i = blockIdx.z + 1;
  const int j0 = 1 + (blockIdx.y * blockDim.y + threadIdx.y) * RBS_R;
  double acc = 0.0;
  if (q < sg.kh4 && j0 <= g.jm) {
    const int off = i * (int)sg.spi + j0 * sg.khp + 4 * q;
    float* own = ps + (long long)c * sg.n + off;
    float* oth = ps + (long long)(c ^ 1) * sg.n + off;  // read; PRESS mirrors write W/B halo slots
    const float* rh = rs + (long long)c * sg.n + off;
    if (((c + i + g.ioff) & 1) == 0) rbs_march<POL, 0>(g, sg, own, oth, rh, cf, om, q, i, j0, acc);
    else rbs_march<POL, 1>(g, sg, own, oth, rh, cf, om, q, i, j0, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  const int ltid = threadIdx.x + threadIdx.y * blockDim.x;
  if ((ltid & 31) == 0) {
    const int wpb = (blockDim.x * blockDim.y + 31) >> 5;
    const long long blk = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    partials[blk * wpb + (ltid >> 5)] = acc;
  }
}

// ---------------------------------------------------------------------------
// The same pass with the tiles staged in shared memory by TMA bulk copies
// (cp.async.bulk, 1-D: every tile input is one contiguous run of the split
// layout), so the bytes in flight do not live in registers.  A tile is
// TR consecutive rows of one plane: its own cells and rhs (TR rows each),
// the other colour's rows (i+-1, j0 .. j0+TR-1) and (i, j0-1 .. j0+TR) --
// five copies, one mbarrier.  Persistent CTAs walk the tiles (plane-major,
// so the CTAs in flight share their E/W planes through L2) with an NS-stage
// ring: the copies of the next NS-1 tiles are in flight while a tile is
// computed from shared memory.  A thread computes four slots of two
// consecutive rows of a tile (TR even: the first row's parity is uniform
// per tile), stores straight to global memory, and the CTA's residual is
// reduced per warp at the end (fixed tile order: deterministic).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ float4 lds4(const float* a) { return *reinterpret_cast<const float4*>(a); }

// ---- fused plane exchange of x-slabs (PassGhost) ----
// tag of pass p (-1: the state before the first pass) in solve `epoch`
__device__ __forceinline__ unsigned ghost_tag(unsigned epoch, int p) {
  return (epoch << 12) | (unsigned)((p + 1) & 0xfff);
}
__device__ __forceinline__ void gld2(const unsigned long long* a, bool sys, unsigned long long& x,
                                     unsigned long long& y) {
  if (sys) asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(a));
  else asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(a));
}
__device__ __forceinline__ void gst2(unsigned long long* a, bool sys, unsigned long long x, unsigned long long y) {
  if (sys) asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(a), "l"(x), "l"(y) : "memory");
  else asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(a), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ unsigned long long gword(float v, unsigned tag) {
  return ((unsigned long long)tag << 32) | __float_as_uint(v);
}
// four ghost words of the neighbour's pass: spin until every tag is the
// expected one (each word is written with one single-copy-atomic 64-bit
// store, so a matching tag carries its value); a wait longer than ~2 s
// sets *err and returns what it has (the host reports the timeout)
__device__ __forceinline__ float4 ghost_ld4(const unsigned long long* a, unsigned tag, bool sys, unsigned* err) {
  unsigned long long w0, w1, w2, w3;
  gld2(a, sys, w0, w1);
  gld2(a + 2, sys, w2, w3);
  if ((unsigned)(w0 >> 32) != tag || (unsigned)(w1 >> 32) != tag || (unsigned)(w2 >> 32) != tag ||
      (unsigned)(w3 >> 32) != tag) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while ((unsigned)(w0 >> 32) != tag || (unsigned)(w1 >> 32) != tag || (unsigned)(w2 >> 32) != tag ||
           (unsigned)(w3 >> 32) != tag) {
      __nanosleep(64);
      gld2(a, sys, w0, w1);
      gld2(a + 2, sys, w2, w3);
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 2000000000ull) {
        atomicExch(err, 1u);
        break;
      }
    }
  }
  return make_float4(__uint_as_float((unsigned)w0), __uint_as_float((unsigned)w1), __uint_as_float((unsigned)w2),
                     __uint_as_float((unsigned)w3));
}
__device__ __forceinline__ void ghost_st4(unsigned long long* a, const float (&v)[4], unsigned tag, bool sys) {
  gst2(a, sys, gword(v[0], tag), gword(v[1], tag));
  gst2(a + 2, sys, gword(v[2], tag), gword(v[3], tag));
}

// the per-tile ghost pointers of a thread: its first row's words in this
// pass's slots (nullptr where the tile has no such exchange)
struct TileGhost {
  const unsigned long long* rw;  // read W: my_w, slot of pass p-1
  const unsigned long long* re;  // read E: my_e, slot of pass p-1
  unsigned long long* pw;        // publish to the west neighbour (its my_e), slot of pass p
  unsigned long long* pe;        // publish to the east neighbour (its my_w), slot of pass p
  unsigned rtag, wtag;
  bool sys;
  unsigned* err;
};

struct RbtPlan {
  int rpt;     // rows per thread per tile (even)
  int tr;      // rows per tile
  int ns;      // pipeline stages
  int ntj;     // tiles per plane
  int ntiles;  // tiles per pass
  int grid;    // persistent CTAs
  int threads; // block size (1-D): kh4 * tr / rpt compute threads, padded to whole warps
  size_t smem; // dynamic shared memory bytes
};

// stage layout (floats): own[tr*khp] rhs[tr*khp] E[tr*khp] W[tr*khp] mid[(tr+2)*khp]

// Rows r0 .. r0+RPT-1 of a tile staged at st (RPT even: the first row's
// parity S0 is the tile's).  o = float offset of the thread's first cell in
// the colour arrays (32-bit: split_supported bounds the arrays).
// MODE 0: red-black pass; 1: red-black pass of an x-slab with the fused
// ghost-plane exchange; 2: twinned sweep (both colours, src -> dst).  The
// modes are separate instantiations: the ghost and twinned code paths cost
// registers and scheduling freedom even when not taken (31 -> 42 us per
// pass at 512^2x90 when they were runtime branches).
template <int POL, int S0, int RPT, int MODE>
__device__ __forceinline__ void rbt_rows(const Geo& g, const float* st, int plane, int khp, int spi, float* own_g,
                                         float* oth_g, const SorC& cf, float om, const bool (&in0)[4],
                                         const bool (&in1)[4], bool lead, int i, int j, int o, int sro, int nr,
                                         double& acc, const TileGhost& tg) {
  const float* s_own = st + sro;
  const float* s_rhs = s_own + plane;
  const float* s_e = s_own + 2 * plane;
  const float* s_w = s_own + 3 * plane;
  const float* s_mid = s_own + 4 * plane + khp;  // the tile's mid rows start one row in (row -1 is staged)
  const bool wmir = POL != 0 && i == 1 && g.west_bc;
#pragma unroll
  for (int h = 0; h < RPT; ++h) {
    if (h >= nr) break;
    const int ro = h * khp;
    const float4 C = lds4(s_own + ro), RH = lds4(s_rhs + ro);
    // x neighbours: staged, or (slab edge planes) the neighbour's words of its previous pass
    const float4 E = (MODE == 1 && tg.re) ? ghost_ld4(tg.re + ro, tg.rtag, tg.sys, tg.err) : lds4(s_e + ro);
    const float4 W = (MODE == 1 && tg.rw) ? ghost_ld4(tg.rw + ro, tg.rtag, tg.sys, tg.err) : lds4(s_w + ro);
    const float4 So = lds4(s_mid + ro - khp), M = lds4(s_mid + ro), N = lds4(s_mid + ro + khp);
    float val[4];
    const int go = o + ro;
    if (((S0 + h) & 1) == 0) {
      rbs_row<0>(cf, om, C, RH, E, W, N, So, M, s_mid[ro - 1], in0, val, acc);
    } else {
      rbs_row<1>(cf, om, C, RH, E, W, N, So, M, s_mid[ro + 4], in1, val, acc);
      if (POL != 0 && lead) oth_g[go] = val[0];  // B mirror: p[i,j,0] = p[i,j,1]
    }
    if (POL != 0 && lead && ((S0 + h) & 1) == 0) {
      // slot 0 of this row is the k = 0 halo cell, set by the other colour's
      // B mirror (twinned: in this launch; red-black: in the previous pass,
      // possibly after this tile's early load): leave it
      own_g[go + 1] = val[1];
      own_g[go + 2] = val[2];
      own_g[go + 3] = val[3];
    } else {
      st4(own_g + go, val[0], val[1], val[2], val[3]);
    }
    if (MODE == 1 && tg.pw) ghost_st4(tg.pw + ro, val, tg.wtag, tg.sys);  // straight into the neighbours' ghost planes
    if (MODE == 1 && tg.pe) ghost_st4(tg.pe + ro, val, tg.wtag, tg.sys);
    if (wmir) st4(oth_g + go - spi, val[0], val[1], val[2], val[3]);  // W mirror: p[0,j,k] = p[1,j,k]
    if (POL == 1 || POL == 3) {  // p[i,jm+1,k] = p[i,1,k], p[i,0,k] = p[i,jm,k]
      // even jm: the same colour (own array); odd jm (twinned only, POL 3:
      // the sweep never reads what it writes): the other colour's array
      float* yt = POL == 1 ? own_g : oth_g;
      if (j + h == 1) st4(yt + go + g.jm * khp, val[0], val[1], val[2], val[3]);
      if (j + h == g.jm) st4(yt + go - g.jm * khp, val[0], val[1], val[2], val[3]);
    }
  }
}

// One colour pass (c >= 0: red-black, in place: src == dst) or one twinned
// (Jacobi) sweep over both colours (c < 0: src -> dst, both colours' tiles
// interleaved per plane row chunk so they share their loads in L2).
// POL 0: stored halo; 1: press, even jm (y mirrors into the same colour);
// 2: press, odd jm, red-black (y halo rows refreshed before the pass);
// 3: press, odd jm, twinned (y mirrors into the other colour of dst).
// (dst is declared __restrict__ although it equals src in the red-black
// pass: src is read only by the TMA engine, never through a generic load)
template <int POL, int RPT, int MODE>
__global__ void __launch_bounds__(512) k_sor_rbt(Geo g, SplitGeo sg, const float* src, float* __restrict__ dst,
                                                 const float* __restrict__ rs, SorC cf, float om, int c_fixed,
                                                 RbtPlan pl, double* __restrict__ partials, PassGhost gh) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem_raw);
  float* stages = reinterpret_cast<float*>(smem_raw + 128);
  const int khp = sg.khp;
  const int spi = (int)sg.spi;
  const int plane = pl.tr * khp;
  const int sfl = (5 * pl.tr + 2) * khp;
  const int ncol = MODE == 2 ? 2 : 1;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int ncomp = sg.kh4 * (pl.tr / RPT);  // compute threads
  const int ncw = (ncomp + 31) >> 5;         // compute warps
  (void)ncw;
  if (tid == 0) {
    for (int s = 0; s < pl.ns; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tile t (plane-major): plane position t / ntj, rows from 1 + (t % ntj) * tr;
  // the CTA walks t = blockIdx.x + k * gridDim.x with incremental (pos, jt).
  // With the fused slab exchange the edge planes go first (position 0: plane
  // 1, position 1: plane im), so their words reach the neighbours early.
  const bool ghosts = MODE == 1 && (gh.my_w || gh.my_e);
  auto plane_of = [&](int pos) {
    if (!ghosts) return 1 + pos;
    return pos == 0 ? 1 : (pos == 1 ? g.im : pos);
  };
  // tile t -> (plane position, row chunk, colour)
  // (division by ntj through a float reciprocal and one correction each way:
  // an integer division per tile and thread cost ~7% of the pass)
  const float rntj = 1.0f / (float)pl.ntj;
  auto decode = [&](int t, int& pos, int& jt, int& c) {
    const int r = ncol == 2 ? (t >> 1) : t;
    c = ncol == 2 ? (t & 1) : c_fixed;
    pos = __float2int_rz(((float)r + 0.5f) * rntj);
    jt = r - pos * pl.ntj;
    if (jt < 0) {
      --pos;
      jt += pl.ntj;
    } else if (jt >= pl.ntj) {
      ++pos;
      jt -= pl.ntj;
    }
  };
  // part: 1 = own cells + rhs (+ the stage's whole expect_tx), 2 = the other
  // colour's rows, 3 = both.  In a red-black pass (MODE 0) part 1 depends
  // on no earlier launch (the own colour was last written two passes ago;
  // the slot the previous pass's B mirror writes is never stored back from a
  // load), so it is issued before griddepcontrol.wait.
  auto issue = [&](int t, int s, int part = 3) {
    int pos, jt, c;
    decode(t, pos, jt, c);
    const int i = plane_of(pos);
    const int j0 = 1 + jt * pl.tr;
    const int nrow = min(pl.tr, g.jm - j0 + 1);
    const unsigned rb = (unsigned)(nrow * khp * 4);
    float* st = stages + s * sfl;
    const int go = i * spi + j0 * khp;
    const float* own_s = src + (long long)c * sg.n;
    const float* oth_s = src + (long long)(c ^ 1) * sg.n;
    const float* rhs_g = rs + (long long)c * sg.n;
    const bool skip_e = MODE == 1 && gh.my_e && i == g.im, skip_w = MODE == 1 && gh.my_w && i == 1;  // ghost planes
    if (part & 1) {
      mbar_expect_tx(&bar[s], (skip_e ? 0u : rb) + (skip_w ? 0u : rb) + 2 * rb + rb + 2u * khp * 4);
      bulk_g2s(st, own_s + go, rb, &bar[s]);
      bulk_g2s(st + plane, rhs_g + go, rb, &bar[s]);
    }
    if (part & 2) {
      if (!skip_e) bulk_g2s(st + 2 * plane, oth_s + go + spi, rb, &bar[s]);
      if (!skip_w) bulk_g2s(st + 3 * plane, oth_s + go - spi, rb, &bar[s]);
      bulk_g2s(st + 4 * plane, oth_s + go - khp, rb + 2u * khp * 4, &bar[s]);
    }
  };
  // programmatic dependent launch: this grid may have started while the
  // previous launch drains; the own cells and rhs of the first tiles depend
  // on no launch later than the one before the previous (whose completion
  // the previous launch waited for before it let this grid start)
  const int my0 = (pl.ntiles * ncol - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (MODE == 0 && tid == 0)
    for (int k = 0; k < pl.ns && k < my0; ++k) issue((int)blockIdx.x + k * (int)gridDim.x, k, 1);
  // everything below may read what the previous launch wrote; only then may
  // the next launch start (so its early loads see this grid's predecessor)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned rtag = 0, wtag = 0;
  if (ghosts) {
    const unsigned ep = *(volatile const unsigned*)gh.epoch;
    rtag = ghost_tag(ep, gh.pass - 1);
    wtag = ghost_tag(ep, gh.pass);
  }
  const int my = (pl.ntiles * ncol - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // tiles of this CTA
  double acc = 0.0;
  if (tid == 0)
    for (int k = 0; k < pl.ns && k < my; ++k) issue((int)blockIdx.x + k * (int)gridDim.x, k, MODE == 0 ? 2 : 3);
  // per-thread invariants: its slot group q, its rows r0 .. r0+RPT-1 of a tile
  const bool active = tid < ncomp;
  const int q = active ? tid % sg.kh4 : 0, r0 = active ? RPT * (tid / sg.kh4) : pl.tr;
  bool in0[4], in1[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int k0 = 8 * q + 2 * m;
    in0[m] = k0 >= 1 && k0 <= g.km;
    in1[m] = k0 + 1 <= g.km;
  }
  const bool lead = q == 0;
  const int sro = r0 * khp + 4 * q;  // the thread's offset inside a staged array
  // the compute cursor: one colour (MODE 0, 1) walks (position, rows)
  // incrementally by gridDim tiles; the twinned sweep decodes each tile
  int cur_pos, cur_jt, cur_c;
  decode((int)blockIdx.x, cur_pos, cur_jt, cur_c);
  const int dpos = (int)gridDim.x / pl.ntj, djt = (int)gridDim.x % pl.ntj;
  float* own_g = dst + (long long)cur_c * sg.n;
  float* oth_g = dst + (long long)(cur_c ^ 1) * sg.n;
  for (int k = 0; k < my; ++k) {
    const int s = k % pl.ns;
    int ii, jt, c;
    if (MODE == 2) {
      decode((int)blockIdx.x + k * (int)gridDim.x, ii, jt, c);
      own_g = dst + (long long)c * sg.n;
      oth_g = dst + (long long)(c ^ 1) * sg.n;
    } else {
      ii = cur_pos;
      jt = cur_jt;
      c = c_fixed;
      cur_pos += dpos;
      cur_jt += djt;
      if (cur_jt >= pl.ntj) {
        cur_jt -= pl.ntj;
        ++cur_pos;
      }
    }
    mbar_wait(&bar[s], (unsigned)((k / pl.ns) & 1));
    const int j = 1 + jt * pl.tr + r0;
    const int nr = g.jm - j + 1;  // rows left in the plane from the thread's first row
    if (active && nr > 0) {
      const int pi = plane_of(ii);
      const int o = pi * spi + j * khp + 4 * q;
      const float* st = stages + s * sfl;
      TileGhost tg{nullptr, nullptr, nullptr, nullptr, rtag, wtag, gh.sys != 0, gh.err};
      if (ghosts) {
        const int go = j * khp + 4 * q;  // the thread's word offset inside a ghost plane slot
        const int rs_ = ((gh.pass - 1) & 3) * spi + go, ws_ = (gh.pass & 3) * spi + go;
        if (pi == 1 && gh.my_w) tg.rw = gh.my_w + rs_;
        if (pi == g.im && gh.my_e) tg.re = gh.my_e + rs_;
        if (pi == 1 && gh.to_w) tg.pw = gh.to_w + ws_;
        if (pi == g.im && gh.to_e) tg.pe = gh.to_e + ws_;
      }
      // only an x-slab's edge-plane tiles take the ghost path; the others run
      // the plain pass code (the ghost branches slow every tile otherwise)
      constexpr int M0 = MODE == 1 ? 0 : MODE;
      const bool gtile = MODE == 1 && (tg.rw || tg.re || tg.pw || tg.pe);
      if (((c + pi + g.ioff) & 1) == 0) {
        if (gtile)
          rbt_rows<POL, 0, RPT, 1>(g, st, plane, khp, spi, own_g, oth_g, cf, om, in0, in1, lead, pi, j, o, sro, nr, acc,
                                   tg);
        else
          rbt_rows<POL, 0, RPT, M0>(g, st, plane, khp, spi, own_g, oth_g, cf, om, in0, in1, lead, pi, j, o, sro, nr,
                                    acc, tg);
      } else {
        if (gtile)
          rbt_rows<POL, 1, RPT, 1>(g, st, plane, khp, spi, own_g, oth_g, cf, om, in0, in1, lead, pi, j, o, sro, nr, acc,
                                   tg);
        else
          rbt_rows<POL, 1, RPT, M0>(g, st, plane, khp, spi, own_g, oth_g, cf, om, in0, in1, lead, pi, j, o, sro, nr,
                                    acc, tg);
      }
    }
    __syncthreads();  // every thread is done with stage s
    if (tid == 0 && k + pl.ns < my) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async overwrite
      issue((int)blockIdx.x + (k + pl.ns) * (int)gridDim.x, s);
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) partials[(long long)blockIdx.x * ((blockDim.x + 31) >> 5) + (tid >> 5)] = acc;
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
// the closed-form halo_fn source, which reproduces the reference's final
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

// k_split_unpack with four cells of a row per thread (see k_split_pack4)
template <int POL>
__global__ void __launch_bounds__(256) k_split_unpack4(Geo g, SplitGeo sg, const float* __restrict__ ps,
                                                       float* __restrict__ p, unsigned* flags) {
  // programmatic dependent launch after the last pass
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int G = (g.km + 2) >> 2;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  unsigned bits = 0;
  if (t < nrow * G) {
    const long long row = t / G;
    const int k0 = 4 * (int)(t - row * G);
    const int i = (int)(row / (g.jm + 2)), j = (int)(row - (long long)i * (g.jm + 2));
    const bool rowhalo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1;
    const bool foreign = (i == 0 && !g.west_bc) || (i == g.im + 1 && !g.east_bc);
    const bool remap = POL == 1 && !foreign;
    const bool zero_row = remap && i == g.im + 1;
    const int ii = (remap && i == 0) ? 1 : i;
    const int jj = (remap && rowhalo) ? (j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j)) : j;
    const int par = (ii + g.ioff + jj + 1) & 1;
    const long long sb = ((long long)ii * (g.jm + 2) + jj) * sg.khp + (k0 >> 1);
    const int c0 = (par + k0) & 1;
    const float2 A = *reinterpret_cast<const float2*>(ps + (long long)c0 * sg.n + sb);        // k0, k0 + 2
    const float2 B = *reinterpret_cast<const float2*>(ps + (long long)(1 - c0) * sg.n + sb);  // k0 + 1, k0 + 3
    float v[4] = {A.x, B.x, A.y, B.y};
    if (remap && k0 == 0) v[0] = B.x;  // p[0] -> p[1]
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (zero_row || (remap && k0 + e == g.km + 1)) v[e] = 0.0f;
      if (flags && !finite32(v[e])) bits = F_PRESS;
    }
    *reinterpret_cast<float4*>(p + row * (g.km + 2) + k0) = make_float4(v[0], v[1], v[2], v[3]);
  }
  if (flags) flag_or(flags, bits);
}

}  // namespace

void launch_split_pack(const Geo& g, const float* p, const float* rhs, float* split, int policy, cudaStream_t st,
                       float* p_copy) {
  const SplitGeo sg = split_geo(g);
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  if (((g.km + 2) & 3) == 0) {  // 16-byte row groups
    const unsigned nb4 = (unsigned)((nrow * ((g.km + 2) >> 2) + 255) / 256);
    if (p_copy) {
      if (policy == 1) k_split_pack4<1, true><<<nb4, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, p_copy);
      else k_split_pack4<0, true><<<nb4, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, p_copy);
    } else {
      if (policy == 1) k_split_pack4<1, false><<<nb4, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, nullptr);
      else k_split_pack4<0, false><<<nb4, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, nullptr);
    }
    return;
  }
  const unsigned nb = (unsigned)((nrow + 7) / 8);
  if (p_copy) {
    if (policy == 1) k_split_pack<1, true><<<nb, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, p_copy);
    else k_split_pack<0, true><<<nb, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, p_copy);
  } else {
    if (policy == 1) k_split_pack<1, false><<<nb, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, nullptr);
    else k_split_pack<0, false><<<nb, 256, 0, st>>>(g, sg, p, rhs, split, split + 2 * sg.n, nullptr);
  }
}

static dim3 rbs_grid(const Geo& g, const SplitGeo& sg, int* bx, int* by) {
  rbs_shape(sg, bx, by);
  return dim3((sg.kh4 + *bx - 1) / *bx, (g.jm + *by * RBS_R - 1) / (*by * RBS_R), g.im);
}

// LESB_SPLIT_REG=1: the register-staged pass kernel (k_sor_rbs) instead of
// the TMA-staged one (A/B experiments)
static bool use_reg_kernel() {
  static const int v = [] {
    const char* e = std::getenv("LESB_SPLIT_REG");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

// Tile plan of the TMA pass: ~256 threads (two rows each) per tile, two
// stages, as many CTAs per SM as fit (occupancy query: two at km = 90),
// persistent.  Measured at 512x512x90 (stored / press, us per iteration):
// 42 rows x 2 stages 74.5 / 80.9; 20 x 3: 77.7 / 86.8; 30 x 3: 78.5 / 87.1;
// 42 x 3 (one CTA per SM): 93.8 / 105.8; 10 x 4: 94.0 / 103.0.
static RbtPlan rbt_plan(const Geo& g, const SplitGeo& sg) {
  RbtPlan pl{};
  static const int env_tr = std::getenv("LESB_RBT_TR") ? std::atoi(std::getenv("LESB_RBT_TR")) : 0;
  static const int env_ns = std::getenv("LESB_RBT_NS") ? std::atoi(std::getenv("LESB_RBT_NS")) : 0;
  static const int env_rpt = std::getenv("LESB_RBT_RPT") ? std::atoi(std::getenv("LESB_RBT_RPT")) : 0;
  const int rpt = 2;  // (4 rows per thread measured slower; RBT_RPT kept as a template parameter)
  (void)env_rpt;
  // ~144 threads per tile (24 rows at km = 90): measured across 150^2-600^2 x 90,
  // both halo policies, against 16-60 rows (the old 42-row default was 6-15%
  // slower at 300^2: its 2400 tiles leave a ninth round for 32 of 296 CTAs)
  int tr = env_tr > 0 ? env_tr : rpt * std::max(1, 288 / (2 * sg.kh4));
  tr = std::max(rpt, tr - tr % rpt);
  while (tr > rpt && sg.kh4 * (tr / rpt) > 512) tr -= rpt;
  const size_t stage = (size_t)(5 * tr + 2) * sg.khp * sizeof(float);
  int ns = env_ns > 0 ? env_ns : 2;
  while (ns > 2 && 128 + ns * stage > 200 * 1024) --ns;
  pl.rpt = rpt;
  pl.tr = tr;
  pl.ns = std::min(ns, 8);
  // whole warps (the residual is shuffle-reduced per warp): padding threads compute nothing
  pl.threads = ((sg.kh4 * (tr / rpt) + 31) / 32) * 32;
  pl.smem = 128 + ns * stage;
  pl.ntj = (g.jm + tr - 1) / tr;
  pl.ntiles = pl.ntj * g.im;
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static bool attr = false;
  if (!attr) {
#define RBT_ATTR(P, M) cudaFuncSetAttribute(k_sor_rbt<P, 2, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
    RBT_ATTR(0, 0); RBT_ATTR(1, 0); RBT_ATTR(2, 0);
    RBT_ATTR(0, 1); RBT_ATTR(1, 1); RBT_ATTR(2, 1);
    RBT_ATTR(0, 2); RBT_ATTR(1, 2); RBT_ATTR(3, 2);
#undef RBT_ATTR
    attr = true;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sor_rbt<1, 2, 1>, pl.threads, pl.smem);
  if (per < 1) per = 1;
  pl.grid = std::min(pl.ntiles, sms * per);
  static const bool verbose = std::getenv("LESB_RBT_VERBOSE") != nullptr;
  if (verbose)
    std::fprintf(stderr, "rbt_plan im=%d jm=%d km=%d: tr=%d threads=%d smem=%zu per=%d grid=%d ntiles=%d\n", g.im, g.jm,
                 g.km, pl.tr, pl.threads, pl.smem, per, pl.grid, pl.ntiles);
  return pl;
}

static bool rbt_ok(const SplitGeo& sg) { return sg.kh4 <= 512 && !use_reg_kernel(); }

bool ghost_supported(const Geo& g, int n_iter) { return rbt_ok(split_geo(g)) && 2 * n_iter <= 4094; }

// bump the solve epoch, then publish the slab's initial colour-1 edge-plane
// values (tag of pass -1, slot 3) into the neighbours' ghost planes
__global__ void k_ghost_epoch(unsigned* epoch) {
  if (threadIdx.x == 0) *epoch += 1;
}
__global__ void k_ghost_publish0(Geo g, SplitGeo sg, const float* __restrict__ ps, PassGhost gh) {
  const unsigned tag = ghost_tag(*(volatile const unsigned*)gh.epoch, -1);
  const float* c1 = ps + sg.n;  // colour 1
  const int spi = (int)sg.spi;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < spi; w += gridDim.x * blockDim.x) {
    const unsigned long long slot = 3ull * spi + w;
    if (gh.to_w) {
      const unsigned long long v = gword(c1[spi + w], tag);  // plane 1
      if (gh.sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(gh.to_w + slot), "l"(v) : "memory");
      else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(gh.to_w + slot), "l"(v) : "memory");
    }
    if (gh.to_e) {
      const unsigned long long v = gword(c1[(long long)g.im * spi + w], tag);  // plane im
      if (gh.sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(gh.to_e + slot), "l"(v) : "memory");
      else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(gh.to_e + slot), "l"(v) : "memory");
    }
  }
}

void launch_ghost_prologue(const Geo& g, const float* split, const PassGhost& gh, cudaStream_t st) {
  k_ghost_epoch<<<1, 32, 0, st>>>(gh.epoch);
  const SplitGeo sg = split_geo(g);
  k_ghost_publish0<<<(unsigned)std::min<long long>(148, (sg.spi + 255) / 256), 256, 0, st>>>(g, sg, split, gh);
}

int sor_blocks_split(const Geo& g) {  // residual partials per pass: one per warp
  const SplitGeo sg = split_geo(g);
  if (rbt_ok(sg)) {
    const RbtPlan pl = rbt_plan(g, sg);
    return pl.grid * ((pl.threads + 31) / 32);
  }
  int bx, by;
  const dim3 gr = rbs_grid(g, sg, &bx, &by);
  return gr.x * gr.y * gr.z * ((bx * by + 31) / 32);
}

void launch_rbs_pass(const Geo& g, float* split, const SorC& cf, float om, int c, int policy, double* partials,
                     cudaStream_t st, const PassGhost* ghp) {
  const PassGhost gh = ghp ? *ghp : PassGhost{};
  float* ps = split;
  const SplitGeo sg = split_geo(g);
  float* rs = split + 2 * sg.n;
  const int pol = policy == 1 ? ((g.jm & 1) ? 2 : 1) : 0;
  if (pol == 2)  // odd jm: the y halo rows are a pre-pass snapshot
    k_split_refresh_y<<<dim3((sg.khp + 127) / 128, g.im), 128, 0, st>>>(g, sg, split, c);
  if (rbt_ok(sg)) {
    const RbtPlan pl = rbt_plan(g, sg);
    const dim3 block(pl.threads);
    const bool gho = gh.my_w || gh.my_e;
    // programmatic stream serialisation: the pass may start while the
    // previous launch drains (its griddepcontrol.wait orders the dependent
    // accesses); LESB_PDL=0 launches it plainly
    static const bool pdl = !(std::getenv("LESB_PDL") && std::atoi(std::getenv("LESB_PDL")) == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.grid);
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    const float* cps = ps;
#define RBT_GO(P, M) cudaLaunchKernelEx(&cfg, k_sor_rbt<P, 2, M>, g, sg, cps, ps, (const float*)rs, cf, om, c, pl, partials, gh)
    if (gho) {
      // (no early start for the slab passes: in one process the slabs' grids
      // share the SMs, and early CTAs parked at griddepcontrol.wait hold slots
      // another slab's pass needs -- 2 slabs of 600x300x90: +24% vs +8%)
      cfg.numAttrs = 0;
      if (pol == 2) RBT_GO(2, 1);
      else if (pol == 1) RBT_GO(1, 1);
      else RBT_GO(0, 1);
    } else {
      if (pol == 2) RBT_GO(2, 0);
      else if (pol == 1) RBT_GO(1, 0);
      else RBT_GO(0, 0);
    }
#undef RBT_GO
    return;
  }
  int bx, by;
  const dim3 grid = rbs_grid(g, sg, &bx, &by);
  const dim3 block(bx, by);
  if (pol == 2) k_sor_rbs<2><<<grid, block, 0, st>>>(g, sg, split, rs, cf, om, c, partials);
  else if (pol == 1) k_sor_rbs<1><<<grid, block, 0, st>>>(g, sg, split, rs, cf, om, c, partials);
  else k_sor_rbs<0><<<grid, block, 0, st>>>(g, sg, split, rs, cf, om, c, partials);
}

bool tws_supported(const Geo& g, const SorC& cf) { return split_supported(g, cf) && rbt_ok(split_geo(g)); }

int sor_blocks_tws(const Geo& g) {  // residual partials per sweep: one per warp of the persistent grid
  const SplitGeo sg = split_geo(g);
  const RbtPlan pl = rbt_plan(g, sg);
  return pl.grid * ((pl.threads + 31) / 32);
}

// One twinned (Jacobi) sweep (sor.py:206-246) on the colour-split layout:
// src (both colours) -> dst (both colours), the halo of the press policy
// kept in dst by the same mirror writes as the red-black pass (the
// reference applies halo_fn to the new component after every sweep,
// sor.py:292-307).
void launch_tws_sweep(const Geo& g, const float* src, float* dst, const float* rhs_split, const SorC& cf, float om,
                      int policy, double* partials, cudaStream_t st) {
  const SplitGeo sg = split_geo(g);
  const RbtPlan pl = rbt_plan(g, sg);
  const dim3 block(pl.threads);
  const PassGhost gh{};
  const int pol = policy == 1 ? ((g.jm & 1) ? 3 : 1) : 0;
  static const bool pdl = !(std::getenv("LESB_PDL") && std::atoi(std::getenv("LESB_PDL")) == 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;  // (a sweep waits for the previous one before any access)
#define RBT_TW(P) cudaLaunchKernelEx(&cfg, k_sor_rbt<P, 2, 2>, g, sg, src, dst, rhs_split, cf, om, -1, pl, partials, gh)
  if (pol == 3) RBT_TW(3);
  else if (pol == 1) RBT_TW(1);
  else RBT_TW(0);
#undef RBT_TW
}

void launch_split_unpack(const Geo& g, const float* split, float* p, int policy, unsigned* flags, cudaStream_t st) {
  const SplitGeo sg = split_geo(g);
  const long long nrow = (long long)(g.im + 2) * (g.jm + 2);
  if (((g.km + 2) & 3) == 0) {  // 16-byte row groups, launched programmatically after the last pass
    static const bool pdl = !(std::getenv("LESB_PDL") && std::atoi(std::getenv("LESB_PDL")) == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((nrow * ((g.km + 2) >> 2) + 255) / 256));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    if (policy == 1) cudaLaunchKernelEx(&cfg, k_split_unpack4<1>, g, sg, split, p, flags);
    else cudaLaunchKernelEx(&cfg, k_split_unpack4<0>, g, sg, split, p, flags);
    return;
  }
  const unsigned nb = (unsigned)((nrow + 7) / 8);
  if (policy == 1) k_split_unpack<1><<<nb, 256, 0, st>>>(g, sg, split, p, flags);
  else k_split_unpack<0><<<nb, 256, 0, st>>>(g, sg, split, p, flags);
}

}  // namespace lesb
