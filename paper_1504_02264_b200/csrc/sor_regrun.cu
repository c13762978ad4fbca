// Register-run variant of the persistent red-black SOR (reference semantics:
// gmcf_mini/sor.py:181-203, the halo policies of sor.cu, the final halo_fn
// call of the press policy les.py:341-355, residuals sor.py:199-203).
//
// Same tiling and LL face exchange as sor_resident.cu, different work
// mapping.  Every thread owns one RUN: up to RK consecutive cells (both
// colours) of one column, held in registers.  A colour pass updates the run's
// cells of that colour:
//   * centre, top and bottom come from the registers (only the two cells just
//     outside the run are re-read from shared memory);
//   * east / west / north / south and rhs come from shared memory (plain
//     [column][k] layout, odd column stride).  The lanes of a warp own runs in
//     consecutive columns at the same k, so these loads are bank-conflict free;
//   * the new value goes to registers and to shared memory and, for
//     tile-boundary columns, to the face buffer.
// That is 5 shared loads + 1 store per cell update (the generic kernel needs
// 8 + 1, with conflicts) and no per-cell index arithmetic: a run is fully
// unrolled, every access is a base register plus an immediate, and cells past
// the end of a partial run are predicated off.
//
// Boundary columns get short runs (RK_B) in their own warps, so their cells,
// and with them the faces the neighbours wait for, are published early in a
// pass while the longer interior runs (RK_I) are still being updated.
//
// Arithmetic per point is sor_point's (same op order, -fmad=false): results
// are bitwise identical to the other solvers and the reference.
#include <cooperative_groups.h>

#include <cstdlib>

#include "lesb_common.cuh"
#include "lesb_kernels.h"

namespace cg = cooperative_groups;

namespace lesb {

constexpr int RR_THREADS = 1024;
constexpr int RR_WARPS = RR_THREADS / 32;
constexpr int RK_B = 10;  // cells per boundary-column run
constexpr int RK_I = 20;  // cells per interior-column run
constexpr int RCV_BATCH = 2;  // face values each thread has in flight while receiving

struct RRPlan {
  int ni, nj;       // tile grid
  int ti_max, tj_max;
  int nseg_b, nseg_i;  // runs per boundary / interior column
  size_t smem;
  long long xbuf;   // 64-bit words of the face exchange buffer
  bool ok;
};

struct RRArgs {
  Geo g;
  RRPlan pl;
  float* p;
  const float* rhs;
  float om, cn1;
  float w2l, w2s, w3l, w3s, w4l, w4s;
  int n_iter;
  unsigned long long* xbuf;  // [4][ntiles][4 faces][fmax][km+2] (value, tag) words
  unsigned* epoch;
  double* partials;          // [2 n_iter][ntiles][RR_WARPS]
  double* res;               // [n_iter]
  unsigned* pflags;
  unsigned* err;
};

__device__ __forceinline__ void rr_st_ll(unsigned long long* a, float v, unsigned tag) {
  const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long rr_ld_ll(const unsigned long long* a) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(a) : "memory");
  return w;
}

__device__ __forceinline__ int rr_tile_lo(int t, int n, int nt) { return 1 + (int)(((long long)t * n) / nt); }

extern __shared__ float rr_smem[];

// A run in shared-memory index space: p of cell k0 - 1 + m is rr_smem[c + m];
// its east / west / north / south neighbours are at +sI / -sI / +cw / -cw and
// its rhs at +rh (the offsets are per-tile constants).
struct RunCtx {
  int c, sI, cw, rh;
  int ncell;
  bool wphys, bot;
  int4 pub;            // face offsets (+ k) of a boundary column, -1 if none
  int k0;
};

// Update the run's cells at positions m = Q, Q+2, ... (m = k - k0 + 1).
template <bool PRESS, int RK, int Q, bool PUB>
__device__ __forceinline__ double rr_pass(const RRArgs& a, float (&P)[RK + 2], const RunCtx& r,
                                          unsigned long long* X, unsigned tag) {
  double acc = 0.0;
#pragma unroll
  for (int m = (Q ? 1 : 2); m <= RK; m += 2) {
    const bool live = m <= r.ncell;
    const int x = r.c + m;
    const float pc = P[m];
    const float pE = rr_smem[x + r.sI];
    float pW = rr_smem[x - r.sI];
    const float pN = rr_smem[x + r.cw];
    const float pS = rr_smem[x - r.cw];
    const float pT = P[m + 1];
    float pB = P[m - 1];
    const float rh = rr_smem[x + r.rh];
    if (PRESS) {
      pW = r.wphys ? pc : pW;            // physical west: p[0] -> p[1]
      if (m == 1) pB = r.bot ? pc : pB;  // bottom: p[.,.,0] -> p[.,.,1]
    }
    // sor.py:164-171: E, W, N, S, T, B summed left to right
    float nb = a.w2l * pE;
    nb = nb + a.w2s * pW;
    nb = nb + a.w3l * pN;
    nb = nb + a.w3s * pS;
    nb = nb + a.w4l * pT;
    nb = nb + a.w4s * pB;
    // sor.py:197: reltmp = omega * (cn1 * (nb - rhs) - p)
    const float rel = a.om * (a.cn1 * (nb - rh) - pc);
    const float np = pc + rel;
    P[m] = live ? np : pc;
    if (live) rr_smem[x] = np;
    if (PUB && live) {
      const int k = r.k0 - 1 + m;
      if (r.pub.x >= 0) rr_st_ll(X + r.pub.x + k, np, tag);
      if (r.pub.y >= 0) rr_st_ll(X + r.pub.y + k, np, tag);
      if (r.pub.z >= 0) rr_st_ll(X + r.pub.z + k, np, tag);
      if (r.pub.w >= 0) rr_st_ll(X + r.pub.w + k, np, tag);
    }
    const double r2 = (double)rel * (double)rel;
    acc += live ? r2 : 0.0;
  }
  return acc;
}

// One run's registers: P[m] holds p of cell k0 - 1 + m (RK_I + 2 slots; a
// boundary run uses the first RK_B + 2).
template <int RK, bool PUB>
__device__ __forceinline__ void rr_init_run(const RRArgs& a, float (&P)[RK_I + 2], const RunCtx& r, int par,
                                            long long bstride, long long tile_off, unsigned tag0, bool active) {
#pragma unroll
  for (int m = 0; m < RK + 2; ++m) P[m] = (active && m <= r.ncell + 1) ? rr_smem[r.c + m] : 0.0f;
  // initial publish: colour-0 cells as pass -2, colour-1 cells as pass -1
  if (PUB && active) {
#pragma unroll
    for (int m = 1; m <= RK; ++m) {
      if (m <= r.ncell) {
        const int colr = (par + m) & 1;  // colour of cell k0 - 1 + m
        unsigned long long* X = a.xbuf + (2 + colr) * bstride + tile_off;
        const int k = r.k0 - 1 + m;
        const unsigned tag = tag0 + (unsigned)colr;
        if (r.pub.x >= 0) rr_st_ll(X + r.pub.x + k, P[m], tag);
        if (r.pub.y >= 0) rr_st_ll(X + r.pub.y + k, P[m], tag);
        if (r.pub.z >= 0) rr_st_ll(X + r.pub.z + k, P[m], tag);
        if (r.pub.w >= 0) rr_st_ll(X + r.pub.w + k, P[m], tag);
      }
    }
  }
}

// One colour pass of one run.
template <bool PRESS, int RK, bool PUB>
__device__ __forceinline__ double rr_run_pass(const RRArgs& a, float (&P)[RK_I + 2], const RunCtx& r, int Q,
                                              int km, unsigned long long* X, unsigned tag) {
  // the two cells just outside the run, when an updated cell needs them
  if (Q == 1 && r.k0 > 1) P[0] = rr_smem[r.c];
  if (Q == (RK & 1) && r.k0 + RK <= km) P[RK + 1] = rr_smem[r.c + RK + 1];
  float (&PP)[RK + 2] = *reinterpret_cast<float (*)[RK + 2]>(&P);
  return Q ? rr_pass<PRESS, RK, 1, PUB>(a, PP, r, X, tag) : rr_pass<PRESS, RK, 0, PUB>(a, PP, r, X, tag);
}

template <bool PRESS>
__global__ void __launch_bounds__(RR_THREADS, 1) k_sor_regrun(RRArgs a) {
  float* smem = rr_smem;
  __shared__ double red[RR_WARPS];
  const Geo& g = a.g;
  const RRPlan& pl = a.pl;
  const int tid = threadIdx.x, nth = RR_THREADS;
  const int lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int ntiles = pl.ni * pl.nj;
  const int ti = tile / pl.nj, tj = tile % pl.nj;
  const int I0 = rr_tile_lo(ti, g.im, pl.ni), I1 = rr_tile_lo(ti + 1, g.im, pl.ni);
  const int J0 = rr_tile_lo(tj, g.jm, pl.nj), J1 = rr_tile_lo(tj + 1, g.jm, pl.nj);
  const int TI = I1 - I0, TJ = J1 - J0;
  const int km = g.km, KC = km + 2, KT = (km + 1) >> 1;
  const int CW = KC | 1;  // odd column stride: lanes in different columns hit different banks
  const int sI = (TJ + 2) * CW;
  const long long ncol_h_max = (long long)(pl.ti_max + 2) * (pl.tj_max + 2);
  const long long arr = (ncol_h_max * CW + 3) & ~3LL;
  float* S = smem;          // p   [TI+2][TJ+2][CW]
  float* RH = smem + arr;   // rhs [TI+2][TJ+2][CW], interior columns
  int4* rcvtab = reinterpret_cast<int4*>(smem + 2 * arr);
  const int fmax = pl.ti_max > pl.tj_max ? pl.ti_max : pl.tj_max;
  const long long fstride = (long long)fmax * KC;
  const long long tstride = 4 * fstride;
  const long long bstride = tstride * ntiles;

  auto colbase = [&](int li, int lj) { return (li * (TJ + 2) + lj) * CW; };

  int nbr[4];
  nbr[0] = ti > 0 ? tile - pl.nj : -1;
  nbr[1] = ti < pl.ni - 1 ? tile + pl.nj : -1;
  nbr[2] = tj > 0 ? tile - 1 : (PRESS ? ti * pl.nj + pl.nj - 1 : -1);
  nbr[3] = tj < pl.nj - 1 ? tile + 1 : (PRESS ? ti * pl.nj : -1);
  const int wrap_flip = g.jm & 1;

  const int nfc = 2 * TJ + 2 * TI;
  for (int q = tid; q < nfc; q += nth) {
    int f, m;
    if (q < 2 * TJ) { f = q / TJ; m = q - f * TJ; }
    else { f = 2 + (q - 2 * TJ) / TI; m = (q - 2 * TJ) - (f - 2) * TI; }
    const int rli = f == 0 ? 0 : (f == 1 ? TI + 1 : 1 + m);
    const int rlj = f == 2 ? 0 : (f == 3 ? TJ + 1 : 1 + m);
    const bool wrap = (f == 2 && tj == 0) || (f == 3 && tj == pl.nj - 1);
    const int si_ = I0 - 1 + rli, sj0 = J0 - 1 + rlj;
    const int sj_ = sj0 == 0 ? g.jm : (sj0 == g.jm + 1 ? 1 : sj0);
    rcvtab[q] = make_int4(colbase(rli, rlj), nbr[f] < 0 ? -1 : (int)(nbr[f] * tstride + (f ^ 1) * fstride + m * KC),
                          wrap ? wrap_flip : 0, (si_ + sj_) & 1);
  }

  // ---- load the tile, its rhs and its halo columns: warp per column, all of
  // a column's loads in flight before the stores ----
  const int ncol_h = (TI + 2) * (TJ + 2);
  for (int col = warp; col < ncol_h; col += RR_WARPS) {
    const int li = col / (TJ + 2), lj = col - li * (TJ + 2);
    const bool ih = li == 0 || li == TI + 1, jh = lj == 0 || lj == TJ + 1;
    if (ih && jh) continue;
    const int i = I0 - 1 + li, j = J0 - 1 + lj;
    const int jj = j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j);
    const bool xphys = ih && (i == 0 || i == g.im + 1);
    const bool inner = !ih && !jh;
    const float* src = a.p + cidx(g, i, PRESS ? jj : j, 0);
    const float* rsrc = a.rhs + cidx(g, i, j, 0);
    float* dst = S + colbase(li, lj);
    float* rdst = RH + colbase(li, lj);
    for (int k0 = 0; k0 <= km + 1; k0 += 128) {
      float v[4], rv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + lane + 32 * u;
        const bool kh = k == 0 || k == km + 1;
        v[u] = 0.0f;
        rv[u] = 0.0f;
        if (k <= km + 1) {
          if (!PRESS || !(kh || xphys)) v[u] = src[k];  // press: top / east 0, bottom / west remapped
          if (inner && !kh) rv[u] = rsrc[k];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + lane + 32 * u;
        if (k <= km + 1) {
          dst[k] = v[u];
          if (inner) rdst[k] = rv[u];
        }
      }
    }
  }
  __syncthreads();

  // ---- my run: boundary columns' runs first (short), then interior runs;
  // within a class lanes take consecutive columns at the same k ----
  const int ncol = TI * TJ;
  const int nbnd = (TI <= 2 || TJ <= 2) ? ncol : 2 * TJ + 2 * (TI - 2);
  const int nint = ncol - nbnd;
  const int nrun_b = pl.nseg_b * nbnd;
  const bool bnd = tid < nrun_b;
  const bool active = tid < nrun_b + pl.nseg_i * nint;
  int gseg = 0, li = 1, lj = 1;
  if (active) {
    int cc;
    if (bnd) {
      gseg = tid / nbnd;
      cc = tid - gseg * nbnd;
    } else {
      const int r = tid - nrun_b;
      gseg = r / nint;
      cc = r - gseg * nint;
    }
    if (nbnd == ncol) {
      li = 1 + cc / TJ;
      lj = 1 + cc % TJ;
    } else if (!bnd) {
      li = 2 + cc / (TJ - 2);
      lj = 2 + cc % (TJ - 2);
    } else if (cc < TJ) {
      li = 1; lj = 1 + cc;
    } else if (cc < 2 * TJ) {
      li = TI; lj = 1 + (cc - TJ);
    } else {
      const int r = cc - 2 * TJ;
      li = 2 + (r >> 1);
      lj = (r & 1) ? TJ : 1;
    }
  }
  const int i = I0 - 1 + li, j = J0 - 1 + lj;
  const int RK = bnd ? RK_B : RK_I;
  const int k0 = 1 + gseg * RK;
  RunCtx r;
  r.k0 = k0;
  r.ncell = active ? min(RK, km - k0 + 1) : 0;
  const int cC = colbase(li, lj);
  r.c = cC + k0 - 1;
  r.sI = sI;
  r.cw = CW;
  r.rh = (int)arr;
  r.wphys = PRESS && g.west_bc && i == 1;
  r.bot = PRESS && k0 == 1;
  r.pub = make_int4(li == 1 ? (int)(0 * fstride + (lj - 1) * KC) : -1,
                    li == TI ? (int)(1 * fstride + (lj - 1) * KC) : -1,
                    lj == 1 ? (int)(2 * fstride + (li - 1) * KC) : -1,
                    lj == TJ ? (int)(3 * fstride + (li - 1) * KC) : -1);
  const int par = (i + j + k0) & 1;  // cell k0-1+m has colour (par + m) & 1

  const unsigned tag0 = 1u + *a.epoch;
  const long long tile_off = (long long)tile * tstride;
  float P[RK_I + 2];
  if (bnd) rr_init_run<RK_B, true>(a, P, r, par, bstride, tile_off, tag0, active);
  else rr_init_run<RK_I, false>(a, P, r, par, bstride, tile_off, tag0, active);

  // receive walk over (face column q, cell index t)
  const int nrcv = nfc * KT;
  const int rq0 = tid / KT, rt0 = tid - rq0 * KT;
  const int rdq = nth / KT, rdr = nth - rdq * KT;
  bool timed_out = false;
  for (int n = 0; n < 2 * a.n_iter; ++n) {
    const int nrd = n & 1;
    // receive the neighbours' faces into the halo columns: pass n-1's publish,
    // or pass n-2's across an odd-jm periodic wrap (those halo cells were last
    // read in pass n-2, before the previous barrier)
    {
      const int ob1 = ((n + 3) & 3) * (int)bstride, ob2 = ((n + 2) & 3) * (int)bstride;
      const unsigned t1 = tag0 + (unsigned)(n + 1);
      int q = rq0, t = rt0;
      for (int w0 = 0; w0 < nrcv; w0 += RCV_BATCH * RR_THREADS) {
        int off[RCV_BATCH], dst[RCV_BATCH];  // dst: smem index | flip << 30, or -1
        unsigned long long v[RCV_BATCH];
#pragma unroll
        for (int u = 0; u < RCV_BATCH; ++u) {
          dst[u] = -1;
          if (q < nfc) {
            const int4 e = rcvtab[q];
            const int kps = (((1 - nrd) ^ e.z) + e.w + 1) & 1;
            const int k = 2 * t + 2 - kps;
            if (e.y >= 0 && k <= km) {
              off[u] = (e.z ? ob2 : ob1) + e.y + k;
              dst[u] = (e.x + k) | (e.z << 30);
              v[u] = rr_ld_ll(a.xbuf + off[u]);
            }
          }
          t += rdr;
          q += rdq;
          if (t >= KT) {
            t -= KT;
            ++q;
          }
        }
#pragma unroll
        for (int u = 0; u < RCV_BATCH; ++u) {
          if (dst[u] < 0) continue;
          const unsigned want = t1 - (unsigned)(dst[u] >> 30);
          unsigned spins = 0;
          while ((unsigned)(v[u] >> 32) != want && !timed_out) {
            if (++spins > (1u << 22)) {  // ~seconds: never hang the GPU
              atomicOr(a.err, 1u);
              timed_out = true;
            }
            v[u] = rr_ld_ll(a.xbuf + off[u]);
          }
          S[dst[u] & 0x3FFFFFFF] = __uint_as_float((unsigned)v[u]);
        }
      }
    }
    __syncthreads();
    double acc = 0.0;
    if (active) {
      const int Q = (nrd + par) & 1;  // updated positions m have parity Q
      unsigned long long* X = a.xbuf + (n & 3) * bstride + tile_off;
      const unsigned tag = tag0 + (unsigned)(n + 2);
      if (bnd) acc = rr_run_pass<PRESS, RK_B, true>(a, P, r, Q, km, X, tag);
      else acc = rr_run_pass<PRESS, RK_I, false>(a, P, r, Q, km, X, tag);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) a.partials[((long long)n * ntiles + tile) * RR_WARPS + warp] = acc;
    if (timed_out) break;
  }
  __syncthreads();

  // ---- write the tile back (warp per column); press: closed-form halo ----
  unsigned bad = 0;
  for (int cc = warp; cc < ncol; cc += RR_WARPS) {
    const int wli = 1 + cc / TJ, wlj = 1 + (cc - (cc / TJ) * TJ);
    const int wi = I0 - 1 + wli, wj = J0 - 1 + wlj;
    const int cb = colbase(wli, wlj);
    int ti_[2] = {wi, (PRESS && wi == 1) ? 0 : -1};
    int tj_[3] = {wj, (PRESS && wj == 1) ? g.jm + 1 : -1, (PRESS && wj == g.jm) ? 0 : -1};
    for (int k = lane; k <= km + 1; k += 32) {
      const int kr = k == 0 ? 1 : (k > km ? km : k);
      const float v = S[cb + kr];
      const bool own = k >= 1 && k <= km;
      if (own && !finite32(v)) bad = F_PRESS;
      const float hv = (k == km + 1) ? 0.0f : v;
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (ti_[x] < 0) continue;
#pragma unroll
        for (int y = 0; y < 3; ++y) {
          if (tj_[y] < 0) continue;
          const bool self = x == 0 && y == 0;
          if (self && !own && !PRESS) continue;
          a.p[cidx(g, ti_[x], tj_[y], k)] = self && own ? v : hv;
        }
      }
      if (PRESS && wi == g.im) {
#pragma unroll
        for (int y = 0; y < 3; ++y)
          if (tj_[y] >= 0) a.p[cidx(g, g.im + 1, tj_[y], k)] = 0.0f;
      }
    }
  }
  if (a.pflags) flag_or(a.pflags, bad);

  cg::this_grid().sync();
  if (tid == 0 && tile == 0) *a.epoch += (unsigned)(2 * a.n_iter + 2);
  const int per_pass = ntiles * RR_WARPS;
  for (int it = tile; it < a.n_iter; it += ntiles) {
    double tot = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      const double* q = a.partials + (long long)(2 * it + pass) * per_pass;
      double v = 0.0;
      for (int b = tid; b < per_pass; b += nth) v += q[b];
      v = block_sum<RR_WARPS>(v, red);
      __syncthreads();
      tot += v;
    }
    if (tid == 0) a.res[it] = tot;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int rr_num_sms = -1, rr_max_smem = -1;

static size_t rr_smem_bytes(int tim, int tjm, int km) {
  const size_t cw = (size_t)((km + 2) | 1);
  const size_t arr = (((size_t)(tim + 2) * (tjm + 2) * cw) + 3) & ~(size_t)3;
  // p and rhs arrays, receive table, and RK_I floats of slack: a partial run's
  // discarded positions may read past the last column
  return 4 * (2 * arr) + 16ull * 2 * (tim + tjm) + 4 * RK_I;
}

static int rr_runs(int tim, int tjm, int km) {
  const int ncol = tim * tjm;
  const int nbnd = (tim <= 2 || tjm <= 2) ? ncol : 2 * tjm + 2 * (tim - 2);
  return nbnd * ((km + RK_B - 1) / RK_B) + (ncol - nbnd) * ((km + RK_I - 1) / RK_I);
}

RRPlan plan_regrun(const Geo& g, int device) {
  RRPlan pl{};
  pl.ok = false;
  if (rr_num_sms < 0) {
    cudaDeviceGetAttribute(&rr_num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&rr_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  }
  if (rr_num_sms <= 0 || !g.west_bc || !g.east_bc || g.ioff != 0) return pl;
  pl.nseg_b = (g.km + RK_B - 1) / RK_B;
  pl.nseg_i = (g.km + RK_I - 1) / RK_I;
  size_t best = (size_t)-1;
  for (int ni = 1; ni <= g.im && ni <= rr_num_sms; ++ni) {
    for (int nj = 1; nj <= g.jm && ni * nj <= rr_num_sms; ++nj) {
      const int tim = (g.im + ni - 1) / ni, tjm = (g.jm + nj - 1) / nj;
      if (rr_runs(tim, tjm, g.km) > RR_THREADS) continue;
      const size_t smem = rr_smem_bytes(tim, tjm, g.km);
      if (smem > (size_t)rr_max_smem - 2048) continue;
      const size_t cost = (size_t)tim * tjm * 4 + 2 * (size_t)(tim + tjm);
      if (cost < best) {
        best = cost;
        pl.ni = ni;
        pl.nj = nj;
        pl.ti_max = tim;
        pl.tj_max = tjm;
        pl.smem = smem;
      }
    }
  }
  if (best == (size_t)-1) return pl;
  const int fmax = pl.ti_max > pl.tj_max ? pl.ti_max : pl.tj_max;
  pl.xbuf = 4LL * pl.ni * pl.nj * 4 * fmax * (g.km + 2);
  pl.ok = true;
  return pl;
}

RRPlanView regrun_view(const Geo& g, int device) {
  RRPlan pl = plan_regrun(g, device);
  return RRPlanView{pl.ok ? pl.ni * pl.nj : 0, pl.ok ? pl.xbuf : 0, pl.ok ? pl.ni * pl.nj * RR_WARPS : 0, pl.ok};
}

template <bool PRESS>
static cudaError_t rr_set_smem_attr(size_t smem) {
  static size_t attr_set = 0;
  if (attr_set >= smem) return cudaSuccess;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, k_sor_regrun<PRESS>);
  if (e != cudaSuccess) return e;
  const int dyn_max = rr_max_smem - (int)fa.sharedSizeBytes;
  e = cudaFuncSetAttribute(k_sor_regrun<PRESS>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
  if (e != cudaSuccess) return e;
  attr_set = (size_t)dyn_max;
  return cudaSuccess;
}

cudaError_t launch_sor_regrun(const Geo& g, int device, float* p, const float* rhs, const SorC& cf, float om,
                              int n_iter, int policy, void* xbuf, unsigned* epoch, double* partials, double* res,
                              unsigned* pflags, unsigned* err, cudaStream_t st) {
  RRPlan pl = plan_regrun(g, device);
  if (!pl.ok || !cf.uni || cf.cn1) return cudaErrorInvalidValue;
  cudaError_t e = policy == 1 ? rr_set_smem_attr<true>(pl.smem) : rr_set_smem_attr<false>(pl.smem);
  if (e != cudaSuccess) return e;
  RRArgs a{g,      pl,     p,      rhs, om,       cf.cn1s, cf.w2l, cf.w2s, cf.w3l, cf.w3s, cf.w4l,
           cf.w4s, n_iter, (unsigned long long*)xbuf, epoch, partials, res, pflags, err};
  void* args[] = {&a};
  const void* fn = policy == 1 ? (const void*)k_sor_regrun<true> : (const void*)k_sor_regrun<false>;
  return cudaLaunchCooperativeKernel(fn, dim3(pl.ni * pl.nj), dim3(RR_THREADS), args, pl.smem, st);
}

}  // namespace lesb
