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
// colour c = (i+j+k+1)&1 at slot k>>1), computes r' in place for the tile
// plus a one-column apron (identical arithmetic to the neighbouring tile's,
// so the redundant values are bitwise equal), then computes b' for the tile
// and writes r' and b' to pb.  Each iteration moves p once in, p once out and
// rhs once (the apron re-reads hit L2): ~12 B per cell and iteration from HBM
// against the 16 B of two unfused colour passes.
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
  int policy;     // 0 STORED, 1 PRESS
  int ti, tj;     // tile extents (max)
  int ntj;        // tiles along j
  int kk;         // slots per colour column
  double* partials;  // [2][nblocks]: red sums, then black sums
};

__device__ __forceinline__ int fz_colour(int i, int j, int k) { return (i + j + k + 1) & 1; }

template <bool PRESS>
__global__ void __launch_bounds__(FZ_THREADS) k_sor_rbfused(FzArgs a) {
  extern __shared__ float sm[];
  __shared__ double red[FZ_WARPS];
  const Geo& g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bt = blockIdx.x;
  const int ti = bt / a.ntj, tj = bt - ti * a.ntj;
  const int I0 = 1 + ti * a.ti, J0 = 1 + tj * a.tj;
  const int TI = min(a.ti, g.im - I0 + 1), TJ = min(a.tj, g.jm - J0 + 1);
  const int km = g.km, KK = a.kk, KT = (km + 1) >> 1;
  const int CWS = 2 * KK;                    // floats per staged column (two colours)
  const int NJ = TJ + 4;                     // staged columns along j (2-column apron)
  float* S = sm;                             // p  [(TI+4)][(TJ+4)][2][KK]
  float* R = sm + (size_t)(a.ti + 4) * (a.tj + 4) * CWS;  // rhs [(TI+2)][(TJ+2)][2][KK]
  const int NJr = TJ + 2;
  auto sbase = [&](int li, int lj) { return (li * NJ + lj) * CWS; };     // li, lj in [0, TI+4)
  auto rbase = [&](int li, int lj) { return (li * NJr + lj) * CWS; };    // li, lj in [0, TI+2)

  // ---- stage pa (tile + 2 apron columns) and rhs (tile + 1 apron) ----
  // staged column (li, lj) is global (I0 - 2 + li, J0 - 2 + lj)
  const int ncs = (TI + 4) * NJ;
  for (int col = warp; col < ncs; col += FZ_WARPS) {
    const int li = col / NJ, lj = col - li * NJ;
    const int gi = I0 - 2 + li, gj = J0 - 2 + lj;
    // source cell identity after the press remap (i: 0 -> 1; j periodic)
    int si = gi, sj = gj;
    bool zero_col = false, skip = false;
    if (gi < 0 || gi > g.im + 1 || ((gj < 0 || gj > g.jm + 1) && !PRESS)) skip = true;
    if (PRESS) {
      if (gi > g.im) zero_col = true;                // east halo: 0
      if (gi == 0) si = 1;                           // west halo mirrors i = 1
      if (gj < 1 || gj > g.jm) sj = ((gj - 1) % g.jm + g.jm) % g.jm + 1;  // periodic y
    }
    float* dst = S + sbase(li, lj);
    const bool rcol = li >= 1 && li <= TI + 2 && lj >= 1 && lj <= TJ + 2;
    float* rdst = rcol ? R + rbase(li - 1, lj - 1) : nullptr;
    // rhs is needed where r' is computed: real cells and (PRESS) y images
    const bool rreal = gi >= 1 && gi <= g.im && ((gj >= 1 && gj <= g.jm) || PRESS);
    const int rj = PRESS ? sj : gj;
    for (int k = lane; k <= km + 1; k += 32) {
      float v = 0.0f;
      if (!skip && !zero_col) {
        if (PRESS) {
          const int sk = k == 0 ? 1 : k;             // bottom mirrors k = 1
          v = (k == km + 1) ? 0.0f : a.pa[cidx(g, si, sj, sk)];
        } else {
          v = a.pa[cidx(g, gi, gj, k)];
        }
      }
      // slot by the colour of the staged position
      const int c = fz_colour(gi, gj, k);
      dst[c * KK + (k >> 1)] = v;
      if (rdst && rreal && k >= 1 && k <= km) rdst[c * KK + (k >> 1)] = a.rhs[cidx(g, gi, rj, k)];
    }
  }
  __syncthreads();

  // ---- red pass on the tile + 1-column apron ----
  // positions (li, lj) in [1, TI+2] x [1, TJ+2] of the staged grid; a
  // position is updated when it is a real interior cell, or (PRESS, even jm)
  // a periodic y image of one
  const int nreg = (TI + 2) * (TJ + 2);
  double acc_r = 0.0;
  {
    const int nitems = nreg * KT;
    for (int w = tid; w < nitems; w += FZ_THREADS) {
      const int c = w / KT, t = w - c * KT;
      const int li = 1 + c / (TJ + 2), lj = 1 + c % (TJ + 2);
      const int gi = I0 - 2 + li, gj = J0 - 2 + lj;
      if (gi < 1 || gi > g.im) continue;
      const bool jreal = gj >= 1 && gj <= g.jm;
      if (!jreal && !(PRESS && !(g.jm & 1))) continue;
      const int kp = (0 + ((gi + gj) & 1) + 1) & 1;  // red (nrd = 0) cells have k parity kp
      const int k = 2 * t + 2 - kp;
      if (k > km) continue;
      const int sb = sbase(li, lj);
      const int sl = t + 1 - kp;
      const float* So = S + KK;           // black slots
      float* Sc = S;                      // red slots
      const int s = sb + sl;
      const float pc = Sc[s];
      const float pE = So[s + NJ * CWS];
      const float pW = So[s - NJ * CWS];
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
      const float rh = R[rbase(li - 1, lj - 1) + sl];
      const float rel = a.om * (a.cn1 * (nb - rh) - pc);
      Sc[s] = pc + rel;
      if (li >= 2 && li <= TI + 1 && lj >= 2 && lj <= TJ + 1) acc_r += (double)rel * (double)rel;
    }
  }
  __syncthreads();

  // ---- black pass on the tile; write r' and b' of the tile to pb ----
  double acc_b = 0.0;
  {
    const int ncol = TI * TJ;
    for (int col = warp; col < ncol; col += FZ_WARPS) {
      const int li = 2 + col / TJ, lj = 2 + col % TJ;
      const int gi = I0 - 2 + li, gj = J0 - 2 + lj;
      const int sb = sbase(li, lj);
      const int kpb = (1 + ((gi + gj) & 1) + 1) & 1;  // black cells' k parity
      for (int k = 1 + lane; k <= km; k += 32) {
        const int c = fz_colour(gi, gj, k);
        const int sl = k >> 1;
        float out;
        if (c == 0) {
          out = S[sb + sl];  // r'
        } else {
          const float* So = S;       // red slots (r') are the black cells' neighbours
          const float* Sc = S + KK;  // black slots (old)
          const int s = sb + sl;
          const float pc = Sc[s];
          const float pE = So[s + NJ * CWS];
          const float pW = So[s - NJ * CWS];
          const float pN = So[s + CWS];
          const float pS = So[s - CWS];
          const float pT = So[sb + ((k + 1) >> 1)];
          const float pB = So[sb + ((k - 1) >> 1)];
          float nb = a.w2l * pE;
          nb = nb + a.w2s * pW;
          nb = nb + a.w3l * pN;
          nb = nb + a.w3s * pS;
          nb = nb + a.w4l * pT;
          nb = nb + a.w4s * pB;
          const float rh = R[rbase(li - 1, lj - 1) + KK + sl];
          const float rel = a.om * (a.cn1 * (nb - rh) - pc);
          out = pc + rel;
          acc_b += (double)rel * (double)rel;
        }
        (void)kpb;
        a.pb[cidx(g, gi, gj, k)] = out;
      }
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

struct FzPlan {
  int ti, tj, ntj, nblk, kk;
  size_t smem;
  bool ok;
};

static size_t fz_smem(int ti, int tj, int kk) {
  return 4ull * 2 * kk * ((size_t)(ti + 4) * (tj + 4) + (size_t)(ti + 2) * (tj + 2));
}

static FzPlan fz_plan(const Geo& g, int device) {
  FzPlan pl{};
  if (fz_max_smem < 0) cudaDeviceGetAttribute(&fz_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  pl.kk = ((g.km + 1) >> 1) + 1;
  // largest square-ish tile that fits, capped at 16 x 16
  int best_ti = 0, best_tj = 0;
  for (int t = 16; t >= 1; --t) {
    const int ti = t, tj = t;
    if (fz_smem(ti, tj, pl.kk) <= (size_t)fz_max_smem - 1024) {
      best_ti = ti;
      best_tj = tj;
      break;
    }
  }
  if (best_ti == 0) return pl;
  pl.ti = best_ti < g.im ? best_ti : g.im;
  pl.tj = best_tj < g.jm ? best_tj : g.jm;
  pl.ntj = (g.jm + pl.tj - 1) / pl.tj;
  pl.nblk = ((g.im + pl.ti - 1) / pl.ti) * pl.ntj;
  pl.smem = fz_smem(pl.ti, pl.tj, pl.kk);
  pl.ok = true;
  return pl;
}

int sor_blocks_fused(const Geo& g, int device) {
  FzPlan pl = fz_plan(g, device);
  return pl.ok ? pl.nblk : 0;
}

template <bool PRESS>
static cudaError_t fz_attr(size_t smem) {
  static size_t set = 0;
  if (set >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_sor_rbfused<PRESS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       fz_max_smem - 2 * FZ_WARPS * 8);
  if (e == cudaSuccess) set = (size_t)fz_max_smem - 2 * FZ_WARPS * 8;
  return e;
}

// One fused iteration pa -> pb; partials[0 .. 2 nblk) receive the red and
// black residual partial sums.
cudaError_t launch_rb_fused(const Geo& g, int device, const float* pa, float* pb, const float* rhs, const SorC& cf,
                            float om, int policy, double* partials, cudaStream_t st) {
  FzPlan pl = fz_plan(g, device);
  if (!pl.ok || !cf.uni || cf.cn1) return cudaErrorInvalidValue;
  cudaError_t e = policy == 1 ? fz_attr<true>(pl.smem) : fz_attr<false>(pl.smem);
  if (e != cudaSuccess) return e;
  FzArgs a{g, pa, pb, rhs, om, cf.cn1s, cf.w2l, cf.w2s, cf.w3l, cf.w3s, cf.w4l, cf.w4s, policy,
           pl.ti, pl.tj, pl.ntj, pl.kk, partials};
  if (policy == 1) k_sor_rbfused<true><<<pl.nblk, FZ_THREADS, pl.smem, st>>>(a);
  else k_sor_rbfused<false><<<pl.nblk, FZ_THREADS, pl.smem, st>>>(a);
  return cudaGetLastError();
}

bool fused_supported(const Geo& g, const SorC& cf, int device) {
  return cf.uni && !cf.cn1 && g.west_bc && g.east_bc && g.ioff == 0 && fz_plan(g, device).ok;
}

}  // namespace lesb
