// Colour-fused, out-of-place red-black SOR iteration (reference semantics:
// gmcf_mini/sor.py:181-203 -- halo_fn, colour-0 pass, halo_fn, colour-1
// pass, halo_fn -- with the halo policies of sor.cu).
//
// One launch performs one whole iteration, reading the field as it stood at
// the start of the iteration (pa) and writing the field after both colour
// passes (pb):
//   red  (nrd = 0) cells:  r' = f(old black neighbours, old red centre)
//   black(nrd = 1) cells:  b' = f(neighbour values as they stand before the
//                                black pass: r' for red cells, old for black)
// A CTA owns a TI x TJ tile of columns (full k).  It stages pa for the tile
// plus a two-column apron in shared memory (colour-split: cell (i,j,k) of
// colour c = (i+j+k+1)&1 at slot k>>1 of colour array c), computes r' in
// place for the tile plus a one-column apron (identical arithmetic to the
// neighbouring tile's, so the redundant values are bitwise equal), computes
// b' in place for the tile, and writes the tile to pb.  Per iteration p moves
// once in and once out and rhs once in (apron re-reads hit L2): 12 B per cell
// and iteration from HBM, against 16 B for two unfused colour passes.
//
// Boundary values follow the reference's halo_fn before every pass:
//   STORED: halo cells keep their stored values (pa's halo, copied into pb
//           once per solve).
//   PRESS:  the closed-form remap is applied while
//           staging: west/bottom halo cells take the value of the cell they
//           mirror (p[0]=p[1], p[.,.,0]=p[.,.,1]), east/top halo cells are 0,
//           and the periodic y halo is staged as the cells it wraps to.  With
//           even jm the wrapped cells have the same colours as their halo
//           positions and are updated like real neighbours; with odd jm they
//           have the other colour and keep their pre-pass values, which is
//           the reference's snapshot semantics.
// Arithmetic per point is sor_point's (same op order, -fmad=false).
//
// Staging moves 16-byte chunks (four consecutive k) when km + 2 is a multiple
// of 4 (VEC), splitting each chunk into the two colour arrays in registers;
// otherwise element by element.  Work items are walked with an incremental
// (column, t) decode over a shared column table: no integer division per item.
#include "lesb_common.cuh"
#include "lesb_kernels.h"

namespace lesb {

constexpr int FZ_THREADS = 512;
constexpr int FZ_WARPS = FZ_THREADS / 32;

struct FzArgs {
  Geo g;
  const float* pa;
  float* pb;
  const float* rhs;
  float om, cn1;
  float w2l, w2s, w3l, w3s, w4l, w4s;
  int ti, tj;     // tile extents (max)
  int ntj;        // tiles along j
  int kk;         // slots per colour column (even)
  double* partials;  // [2][nblocks]: red sums, then black sums
};

// red-pass column table entry .x: staged column base (floats) |
// parity(i+j) << 28 | red-updated << 29 | in-tile << 30;  .y: global offset
// of the column's rhs (k = 0) or -1
constexpr unsigned FZ_BASE = 0x0FFFFFFFu;

// Walk items (c, t), c in [0, n), t in [0, KT), item = c * KT + t; thread
// tid takes items tid, tid + FZ_THREADS, ...
struct Walk {
  int c, t, dq, dr, KT;
  __device__ __forceinline__ explicit Walk(int KT_) : KT(KT_) {
    const int w = threadIdx.x;
    c = w / KT_;
    t = w - c * KT_;
    dq = FZ_THREADS / KT_;
    dr = FZ_THREADS - dq * KT_;
  }
  __device__ __forceinline__ void next() {
    t += dr;
    c += dq;
    if (t >= KT) {
      t -= KT;
      ++c;
    }
  }
};

// split four consecutive k (k0 even, colour c0 at k0) into the colour arrays
__device__ __forceinline__ void put4(float* base, int KK, int c0, int k0, float4 x) {
  *reinterpret_cast<float2*>(base + c0 * KK + (k0 >> 1)) = make_float2(x.x, x.z);
  *reinterpret_cast<float2*>(base + (c0 ^ 1) * KK + (k0 >> 1)) = make_float2(x.y, x.w);
}

template <bool PRESS, bool VEC>
__global__ void __launch_bounds__(FZ_THREADS) k_sor_rbfused(FzArgs a) {
  extern __shared__ __align__(16) float sm[];
  __shared__ double red[FZ_WARPS];
  const Geo& g = a.g;
  const int tid = threadIdx.x;
  const int bt = blockIdx.x;
  const int ti = bt / a.ntj, tj = bt - ti * a.ntj;
  const int I0 = 1 + ti * a.ti, J0 = 1 + tj * a.tj;
  const int TI = min(a.ti, g.im - I0 + 1), TJ = min(a.tj, g.jm - J0 + 1);
  const int km = g.km, KK = a.kk, KT = (km + 1) >> 1;
  const int CWS = 2 * KK;                    // floats per staged column (two colours)
  const int NJ = TJ + 4;                     // staged columns along j (2-column apron)
  const int NJr = TJ + 2;
  const int ncs = (TI + 4) * NJ;             // staged p columns
  const int nrc = (TI + 2) * NJr;            // staged rhs columns (= red-pass columns)
  float* S = sm;                                            // p  [(TI+4)][(TJ+4)][2][KK]
  float* R = sm + (size_t)(a.ti + 4) * (a.tj + 4) * CWS;    // rhs [(TI+2)][(TJ+2)][2][KK]
  int2* tab = reinterpret_cast<int2*>(R + (size_t)(a.ti + 2) * (a.tj + 2) * CWS);   // [nrc]
  int2* stab = tab + (((a.ti + 2) * (a.tj + 2) + 1) & ~1);                          // [ncs]
  auto sbase = [&](int li, int lj) { return (li * NJ + lj) * CWS; };

  // ---- tables ----
  // staging: .x global offset of the source column (k = 0) or -1 (zero
  // column), .y colour of k = 0 at the staged position
  for (int col = tid; col < ncs; col += FZ_THREADS) {
    const int li = col / NJ, lj = col - li * NJ;
    const int gi = I0 - 2 + li, gj = J0 - 2 + lj;
    int si = gi, sj = gj;
    bool zero_col = gi < 0 || gi > g.im + 1 || ((gj < 0 || gj > g.jm + 1) && !PRESS);
    if (PRESS) {
      if (gi > g.im) zero_col = true;                // east halo: 0
      if (gi == 0) si = 1;                           // west halo mirrors i = 1
      if (gj < 1 || gj > g.jm) sj = ((gj - 1) % g.jm + g.jm) % g.jm + 1;  // periodic y
    }
    stab[col] = make_int2(zero_col ? -1 : (int)cidx(g, si, sj, 0), (gi + gj + 1) & 1);
    if (li >= 1 && li <= TI + 2 && lj >= 1 && lj <= TJ + 2) {
      const bool real = gi >= 1 && gi <= g.im && gj >= 1 && gj <= g.jm;
      const bool image = PRESS && !(g.jm & 1) && gi >= 1 && gi <= g.im && !real;
      const bool intile = li >= 2 && li <= TI + 1 && lj >= 2 && lj <= TJ + 1;
      tab[(li - 1) * NJr + (lj - 1)] =
          make_int2((int)((unsigned)sbase(li, lj) | ((unsigned)((gi + gj) & 1) << 28) |
                          ((real || image) ? (1u << 29) : 0u) | (intile ? (1u << 30) : 0u)),
                    (real || image) ? (int)cidx(g, gi, PRESS ? sj : gj, 0) : -1);
    }
  }
  __syncthreads();

  // ---- stage pa (tile + 2 apron columns) and rhs (tile + 1 apron) ----
  if (VEC) {
    const int NCH = (km + 2) >> 2;  // 16-byte chunks per column
    Walk w(NCH);
    while (w.c < ncs) {
      float4 v[4];
      int col[4], k0[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        col[u] = w.c;
        k0[u] = 4 * w.t;
        if (w.c < ncs) {
          const int src = stab[w.c].x;
          v[u] = src >= 0 ? *reinterpret_cast<const float4*>(a.pa + src + k0[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        w.next();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (col[u] >= ncs) continue;
        float4 x = v[u];
        if (PRESS) {
          if (k0[u] == 0) x.x = x.y;  // bottom mirrors k = 1
          const int top = km + 1 - k0[u];
          if (top == 0) x.x = 0.f;
          else if (top == 1) x.y = 0.f;
          else if (top == 2) x.z = 0.f;
          else if (top == 3) x.w = 0.f;
        }
        const int li = col[u] / NJ, lj = col[u] - li * NJ;
        put4(S + sbase(li, lj), KK, stab[col[u]].y, k0[u], x);
      }
    }
    Walk wr(NCH);
    while (wr.c < nrc) {
      float4 v[4];
      int col[4], k0[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        col[u] = -1;
        if (wr.c < nrc) {
          const int src = tab[wr.c].y;
          if (src >= 0) {
            col[u] = wr.c;
            k0[u] = 4 * wr.t;
            v[u] = *reinterpret_cast<const float4*>(a.rhs + src + k0[u]);
          }
        }
        wr.next();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (col[u] < 0) continue;
        const int c0 = (int)((((unsigned)tab[col[u]].x >> 28) & 1u) ^ 1u);  // colour of k = 0
        put4(R + col[u] * CWS, KK, c0, k0[u], v[u]);
      }
    }
  } else {
    Walk w(km + 2);
    for (; w.c < ncs; w.next()) {
      const int2 e = stab[w.c];
      const int k = w.t;
      int sk = k;
      bool z = e.x < 0;
      if (PRESS) {
        if (k == 0) sk = 1;           // bottom mirrors k = 1
        if (k == km + 1) z = true;    // top: 0
      }
      const float v = z ? 0.0f : a.pa[e.x + sk];
      const int li = w.c / NJ, lj = w.c - li * NJ;
      S[sbase(li, lj) + ((e.y ^ (k & 1)) * KK) + (k >> 1)] = v;
    }
    Walk wr(km + 2);
    for (; wr.c < nrc; wr.next()) {
      const int2 e = tab[wr.c];
      const int k = wr.t;
      if (e.y < 0 || k < 1 || k > km) continue;
      const int c0 = (int)((((unsigned)e.x >> 28) & 1u) ^ 1u);
      R[wr.c * CWS + ((c0 ^ (k & 1)) * KK) + (k >> 1)] = a.rhs[e.y + k];
    }
  }
  __syncthreads();

  // ---- red pass on the tile + 1-column apron (in place) ----
  const int sI = NJ * CWS;
  double acc_r = 0.0;
  {
    Walk w(KT);
    for (; w.c < nrc; w.next()) {
      const unsigned ex = (unsigned)tab[w.c].x;
      if (!(ex & (1u << 29))) continue;
      const int kp = (int)(((ex >> 28) & 1u) ^ 1u);  // red cells have k parity kp
      const int t = w.t;
      if (2 * t + 2 - kp > km) continue;
      const int sb = (int)(ex & FZ_BASE);
      const int sl = t + 1 - kp;
      const int s = sb + sl;
      const float* So = S + KK;  // black slots
      const float pc = S[s];
      const float pE = So[s + sI];
      const float pW = So[s - sI];
      const float pN = So[s + CWS];
      const float pS = So[s - CWS];
      const float pT = So[sb + t + 1];
      const float pB = So[sb + t];
      float nb = a.w2l * pE;
      nb = nb + a.w2s * pW;
      nb = nb + a.w3l * pN;
      nb = nb + a.w3s * pS;
      nb = nb + a.w4l * pT;
      nb = nb + a.w4s * pB;
      const float rh = R[w.c * CWS + sl];
      const float rel = a.om * (a.cn1 * (nb - rh) - pc);
      S[s] = pc + rel;
      if (ex & (1u << 30)) acc_r += (double)rel * (double)rel;
    }
  }
  __syncthreads();

  // ---- black pass on the tile (in place) ----
  double acc_b = 0.0;
  {
    Walk w(KT);
    for (; w.c < nrc; w.next()) {
      const unsigned ex = (unsigned)tab[w.c].x;
      if (!(ex & (1u << 30))) continue;
      const int kp = (int)((ex >> 28) & 1u);  // black cells have k parity kp
      const int t = w.t;
      if (2 * t + 2 - kp > km) continue;
      const int sb = (int)(ex & FZ_BASE);
      const int sl = t + 1 - kp;
      const int s = sb + sl;  // red slot at the same k; the black cell is s + KK
      const float pc = S[s + KK];
      const float pE = S[s + sI];
      const float pW = S[s - sI];
      const float pN = S[s + CWS];
      const float pS = S[s - CWS];
      const float pT = S[sb + t + 1];
      const float pB = S[sb + t];
      float nb = a.w2l * pE;
      nb = nb + a.w2s * pW;
      nb = nb + a.w3l * pN;
      nb = nb + a.w3s * pS;
      nb = nb + a.w4l * pT;
      nb = nb + a.w4s * pB;
      const float rh = R[w.c * CWS + KK + sl];
      const float rel = a.om * (a.cn1 * (nb - rh) - pc);
      S[s + KK] = pc + rel;
      acc_b += (double)rel * (double)rel;
    }
  }
  __syncthreads();

  // ---- write the tile (both colours) to pb ----
  const int ntc = TI * TJ;
  if (VEC) {
    const int NCH = (km + 2) >> 2;
    Walk w(NCH);
    for (; w.c < ntc; w.next()) {
      const int li = 2 + w.c / TJ, lj = 2 + w.c % TJ;
      const int gi = I0 - 2 + li, gj = J0 - 2 + lj;
      const int k0 = 4 * w.t;
      const int c0 = (gi + gj + 1) & 1;
      const float* col = S + sbase(li, lj);
      const float2 xa = *reinterpret_cast<const float2*>(col + c0 * KK + (k0 >> 1));
      const float2 xb = *reinterpret_cast<const float2*>(col + (c0 ^ 1) * KK + (k0 >> 1));
      const float4 o = make_float4(xa.x, xb.x, xa.y, xb.y);
      float* dst = a.pb + cidx(g, gi, gj, k0);
      if (k0 == 0 || k0 + 3 == km + 1) {
        // pb's own halo cells (k = 0, km + 1) keep their values
        if (k0 != 0) dst[0] = o.x;
        dst[1] = o.y;
        dst[2] = o.z;
        if (k0 + 3 != km + 1) dst[3] = o.w;
      } else {
        *reinterpret_cast<float4*>(dst) = o;
      }
    }
  } else {
    Walk w(km);
    for (; w.c < ntc; w.next()) {
      const int li = 2 + w.c / TJ, lj = 2 + w.c % TJ;
      const int gi = I0 - 2 + li, gj = J0 - 2 + lj;
      const int k = 1 + w.t;
      a.pb[cidx(g, gi, gj, k)] = S[sbase(li, lj) + (((gi + gj + k + 1) & 1) * KK) + (k >> 1)];
    }
  }
  const double sr = block_sum<FZ_WARPS>(acc_r, red);
  __syncthreads();
  const double sb_ = block_sum<FZ_WARPS>(acc_b, red);
  if (tid == 0) {
    a.partials[bt] = sr;
    a.partials[gridDim.x + bt] = sb_;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int fz_max_smem = -1;
static int fz_num_sms = -1;

struct FzPlan {
  int ti, tj, ntj, nblk, kk;
  size_t smem;
  bool ok;
};

static size_t fz_smem(int ti, int tj, int kk) {
  const size_t ncs = (size_t)(ti + 4) * (tj + 4), nrc = (size_t)(ti + 2) * (tj + 2);
  return 4ull * 2 * kk * (ncs + nrc) + 8 * ((nrc + 1) & ~(size_t)1) + 8 * ncs;
}

static FzPlan fz_plan(const Geo& g, int device) {
  FzPlan pl{};
  if (fz_max_smem < 0) {
    cudaDeviceGetAttribute(&fz_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&fz_num_sms, cudaDevAttrMultiProcessorCount, device);
  }
  pl.kk = (((g.km + 1) >> 1) + 2) & ~1;  // slots 0 .. (km+1)>>1, rounded up to even (8-byte stores)
  // square tiles: minimise (waves x staged columns per CTA), i.e. the time of
  // the slowest SM, counting up to two resident CTAs per SM
  double best = 1e300;
  for (int t = 16; t >= 2; --t) {
    const int ti = t < g.im ? t : g.im, tj = t < g.jm ? t : g.jm;
    const size_t smem = fz_smem(ti, tj, pl.kk);
    if (smem > (size_t)fz_max_smem - 1024) continue;
    int per_sm = (int)(((size_t)fz_max_smem) / (smem + 1024));
    if (per_sm > 2) per_sm = 2;
    if (per_sm < 1) per_sm = 1;
    const int nblk = ((g.im + ti - 1) / ti) * ((g.jm + tj - 1) / tj);
    const int waves = (nblk + fz_num_sms * per_sm - 1) / (fz_num_sms * per_sm);
    const double cost = (double)waves * per_sm * (ti + 4) * (tj + 4);
    if (cost < best) {
      best = cost;
      pl.ti = ti;
      pl.tj = tj;
      pl.smem = smem;
    }
  }
  if (best == 1e300) return pl;
  pl.ntj = (g.jm + pl.tj - 1) / pl.tj;
  pl.nblk = ((g.im + pl.ti - 1) / pl.ti) * pl.ntj;
  pl.ok = true;
  return pl;
}

int sor_blocks_fused(const Geo& g, int device) {
  FzPlan pl = fz_plan(g, device);
  return pl.ok ? pl.nblk : 0;
}

template <bool PRESS, bool VEC>
static cudaError_t fz_attr() {
  static bool set = false;
  if (set) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_sor_rbfused<PRESS, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       fz_max_smem - 2 * FZ_WARPS * 8);
  if (e == cudaSuccess) set = true;
  return e;
}

// One fused iteration pa -> pb; partials[0 .. 2 nblk) receive the red and
// black residual partial sums.
cudaError_t launch_rb_fused(const Geo& g, int device, const float* pa, float* pb, const float* rhs, const SorC& cf,
                            float om, int policy, double* partials, cudaStream_t st) {
  FzPlan pl = fz_plan(g, device);
  if (!pl.ok || !cf.uni || cf.cn1) return cudaErrorInvalidValue;
  const bool vec = ((g.km + 2) & 3) == 0;
  cudaError_t e = policy == 1 ? (vec ? fz_attr<true, true>() : fz_attr<true, false>())
                              : (vec ? fz_attr<false, true>() : fz_attr<false, false>());
  if (e != cudaSuccess) return e;
  FzArgs a{g, pa, pb, rhs, om, cf.cn1s, cf.w2l, cf.w2s, cf.w3l, cf.w3s, cf.w4l, cf.w4s,
           pl.ti, pl.tj, pl.ntj, pl.kk, partials};
  if (policy == 1) {
    if (vec) k_sor_rbfused<true, true><<<pl.nblk, FZ_THREADS, pl.smem, st>>>(a);
    else k_sor_rbfused<true, false><<<pl.nblk, FZ_THREADS, pl.smem, st>>>(a);
  } else {
    if (vec) k_sor_rbfused<false, true><<<pl.nblk, FZ_THREADS, pl.smem, st>>>(a);
    else k_sor_rbfused<false, false><<<pl.nblk, FZ_THREADS, pl.smem, st>>>(a);
  }
  return cudaGetLastError();
}

bool fused_supported(const Geo& g, const SorC& cf, int device) {
  return cf.uni && !cf.cn1 && g.west_bc && g.east_bc && g.ioff == 0 && fz_plan(g, device).ok;
}

}  // namespace lesb
