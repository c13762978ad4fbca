// i-marching, colour-fused, out-of-place red-black SOR iteration for large
// grids (reference semantics: gmcf_mini/sor.py:181-203 with the halo
// policies of sor.cu; the same pa -> pb contract as sor_fused.cu).
//
// A CTA owns a strip of TJ rows (j) with full k columns and marches along x
// over a chunk of planes.  At march step x it
//   * updates the red cells of plane x+1 (they need the old black values of
//     planes x, x+1, x+2),
//   * updates the black cells of plane x (they need the new red values of
//     planes x-1, x, x+1),
//   * writes plane x (both colours) to pb,
// while the next plane of p and rhs is already in flight (cp.async into a
// ring of shared-memory planes).  The strip carries a 2-row apron in j: red
// is recomputed redundantly on the first apron row (identical arithmetic, so
// bitwise equal to the neighbour strip's), which the black cells at the strip
// edge need.  A chunk starts two planes early so that its first black plane
// sees new red values on both sides.  Per iteration p and rhs cross HBM about
// once and pb is written once: ~12 B per cell, the algorithmic minimum with
// a scalar cn1.
//
// Shared-memory planes are colour split (cell (i,j,k) of colour
// (i+j+k+1)&1 at slot k>>1 of its row's colour array), so a warp's lanes
// touch consecutive words.  Boundary values follow each pass's halo_fn as in
// sor_fused.cu (stored halos, or the press remap applied while staging,
// including the periodic y images with the reference's snapshot semantics for
// odd jm).  Arithmetic per point is sor_point's (same op order,
// -fmad=false).
#include <cstdlib>

#include "lesb_common.cuh"
#include "lesb_kernels.h"

namespace lesb {

constexpr int MR_THREADS = 512;
constexpr int MR_WARPS = MR_THREADS / 32;
constexpr int MR_PSLOTS = 5;  // colour-split p planes x-1 .. x+3
constexpr int MR_RSLOTS = 4;  // colour-split rhs planes x .. x+3
constexpr int MR_LSLOTS = 3;  // plain landing planes x+3 .. x+5 (cp.async in flight)
constexpr int MR_ITEMS = 4;   // (row, k-pair) items per thread and step

struct MrArgs {
  Geo g;
  const float* pa;
  float* pb;
  const float* rhs;
  float om, cn1;
  float w2l, w2s, w3l, w3s, w4l, w4s;
  int tj, ch;      // strip rows, chunk planes
  int njt;         // strips along j
  int kk;          // slots per colour row (even)
  int kc;          // plain row pitch (floats): km + 2 rounded up to 4
  double* partials;  // [2][nblocks]
};

__device__ __forceinline__ void cp_async16(unsigned dst, const float* src, bool zero) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(zero ? 0u : 16u) : "memory");
}
__device__ __forceinline__ void cp_async4(unsigned dst, const float* src, bool zero) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(zero ? 0u : 4u) : "memory");
}

template <bool PRESS, bool VEC>
__global__ void __launch_bounds__(MR_THREADS) k_sor_rbmarch(MrArgs a) {
  extern __shared__ __align__(16) float sm[];
  __shared__ double red[MR_WARPS];
  const Geo& g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int jt = blockIdx.x % a.njt, ic = blockIdx.x / a.njt;
  const int J0 = 1 + jt * a.tj;
  const int TJ = min(a.tj, g.jm - J0 + 1);
  const int I0 = 1 + ic * a.ch;
  const int I1 = min(I0 + a.ch, g.im + 1);  // chunk planes [I0, I1)
  const int km = g.km, KK = a.kk, KP = (km + 1) >> 1, KC = a.kc;
  const int NR = TJ + 4;                      // staged p rows: J0-2 .. J0+TJ+1
  const int NRR = TJ + 2;                     // staged rhs rows: J0-1 .. J0+TJ
  const int RW = 2 * KK;                      // floats per colour-split row
  const int PS = (a.tj + 4) * RW;             // floats per split p plane
  const int RS = (a.tj + 2) * RW;             // floats per split rhs plane
  const int LS = (2 * a.tj + 6) * KC;         // floats per plain landing plane (p rows, then rhs rows)
  float* Pp = sm;                             // [MR_PSLOTS][PS]
  float* Rr = Pp + MR_PSLOTS * PS;            // [MR_RSLOTS][RS]
  float* Ll = Rr + MR_RSLOTS * RS;            // [MR_LSLOTS][LS]
  const unsigned lbase = (unsigned)__cvta_generic_to_shared(Ll);
  auto pslot = [&](int gi) { return Pp + ((gi + MR_PSLOTS * 4) % MR_PSLOTS) * PS; };
  auto rslot = [&](int gi) { return Rr + ((gi + MR_RSLOTS * 4) % MR_RSLOTS) * RS; };
  auto lslot = [&](int gi) { return ((gi + MR_LSLOTS * 4) % MR_LSLOTS) * LS; };

  // source row (k = 0) of staged p row gj of plane gi, or -1 for a zero row
  auto p_row = [&](int gi, int gj) -> long long {
    int si = gi, sj = gj;
    if (gi < 0 || gi > g.im + 1) return -1;
    if (PRESS) {
      if (gi > g.im) return -1;                     // east halo: 0
      if (gi == 0) si = 1;                          // west halo mirrors i = 1
      if (gj < 1 || gj > g.jm) sj = ((gj - 1) % g.jm + g.jm) % g.jm + 1;  // periodic y
    } else if (gj < 0 || gj > g.jm + 1) {
      return -1;
    }
    return cidx(g, si, sj, 0);
  };
  // source row of staged rhs row gj of plane gi, or -1
  auto r_row = [&](int gi, int gj) -> long long {
    if (gi < 1 || gi > g.im) return -1;
    int sj = gj;
    if (gj < 1 || gj > g.jm) {
      if (!PRESS) return -1;
      sj = ((gj - 1) % g.jm + g.jm) % g.jm + 1;
    }
    return cidx(g, gi, sj, 0);
  };

  // ---- land plane gi (p rows then rhs rows, plain layout) asynchronously:
  // warp per row, lanes over 16-byte chunks (VEC) or elements ----
  auto land = [&](int gi) {
    const unsigned dst0 = lbase + 4u * (unsigned)lslot(gi);
    const int nrows = NR + NRR;
    for (int rr = warp; rr < nrows; rr += MR_WARPS) {
      const bool isp = rr < NR;
      const int gj = isp ? J0 - 2 + rr : J0 - 1 + (rr - NR);
      const long long src = isp ? p_row(gi, gj) : r_row(gi, gj);
      const float* sp = src >= 0 ? (isp ? a.pa : a.rhs) + src : a.pa;
      const unsigned d = dst0 + 4u * (unsigned)(rr * KC);
      if (VEC) {
        for (int q = lane; q < KC / 4; q += 32) cp_async16(d + 16u * q, sp + 4 * q, src < 0);
      } else {
        for (int k = lane; k < km + 2; k += 32) cp_async4(d + 4u * k, sp + k, src < 0);
      }
    }
  };
  // ---- split landed plane gi into the colour arrays (shared to shared).
  // Items (row, pair q = (2q, 2q+1)) are the same every step: decoded once. ----
  constexpr int SPL = 6;
  const int npair = (km + 3) >> 1;  // pairs covering k = 0 .. km+1
  const int nsplit = (NR + NRR) * npair;
  int sp_src[SPL], sp_dst[SPL], sp_q[SPL];  // landing offset, split offset (-1: none), pair
#pragma unroll
  for (int u = 0; u < SPL; ++u) {
    const int w = tid + u * MR_THREADS;
    sp_dst[u] = -1;
    sp_src[u] = 0;
    sp_q[u] = 0;
    if (w < nsplit) {
      const int rr = w / npair, q = w - (w / npair) * npair;
      const bool isp = rr < NR;
      sp_src[u] = rr * KC + 2 * q;
      // split row base; bit 30 marks a rhs row, bit 29 the row's (gj) parity
      const int gj = isp ? J0 - 2 + rr : J0 - 1 + (rr - NR);
      sp_dst[u] = (isp ? rr * RW : (rr - NR) * RW) | (isp ? 0 : (1 << 30)) | ((gj & 1) << 29);
      sp_q[u] = q;
    }
  }
  auto split = [&](int gi) {
    const float* L = Ll + lslot(gi);
    float* P = pslot(gi);
    float* R = rslot(gi);
#pragma unroll
    for (int u = 0; u < SPL; ++u) {
      if (sp_dst[u] < 0) continue;
      const int q = sp_q[u];
      const bool isp = !(sp_dst[u] & (1 << 30));
      const int gjp = (sp_dst[u] >> 29) & 1;
      const float2 v = *reinterpret_cast<const float2*>(L + sp_src[u]);
      float v0 = v.x, v1 = v.y;
      if (isp && PRESS) {
        if (q == 0) v0 = v1;                      // bottom mirrors k = 1
        if (2 * q == km + 1) v0 = 0.0f;           // top: 0
        if (2 * q + 1 == km + 1) v1 = 0.0f;
      }
      // k = 2q has colour c0, k = 2q+1 the other; both at slot q
      const int c0 = (gi + gjp + 1) & 1;
      float* dst = (isp ? P : R) + (sp_dst[u] & 0x1FFFFFFF);
      dst[c0 * KK + q] = v0;
      if (2 * q + 1 <= km + 1) dst[(c0 ^ 1) * KK + q] = v1;
    }
  };

  // ---- this thread's fixed (row, k-pair) items ----
  // red rows: strip rows + 1 apron row each side (r = 0 .. TJ+1 <-> j = J0-1 ..
  // J0+TJ); black rows r = 1 .. TJ.  Item w -> r = w / KP, q = w % KP.
  int it_r[MR_ITEMS], it_q[MR_ITEMS];
  const int nitems = (TJ + 2) * KP;
#pragma unroll
  for (int u = 0; u < MR_ITEMS; ++u) {
    const int w = tid + u * MR_THREADS;
    it_r[u] = w < nitems ? w / KP : -1;
    it_q[u] = w < nitems ? w - (w / KP) * KP : 0;
  }
  // write-out items (strip row, pair)
  constexpr int WRL = 3;
  int wr_r[WRL], wr_q[WRL];
#pragma unroll
  for (int u = 0; u < WRL; ++u) {
    const int w = tid + u * MR_THREADS;
    wr_r[u] = w < TJ * npair ? w / npair : -1;
    wr_q[u] = w < TJ * npair ? w - (w / npair) * npair : 0;
  }
  // red images: periodic y images are updated (even jm) like real cells
  const bool img_ok = PRESS && !(g.jm & 1);

  double acc_r = 0.0, acc_b = 0.0;
  const int x0 = I0 - 2;
  // prologue: split planes x0-1 .. x0+2 (landed one by one), planes x0+3 ..
  // x0+5 in flight
  for (int gi = x0 - 1; gi <= x0 + 2; ++gi) {
    land(gi);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    split(gi);
    __syncthreads();
  }
  for (int gi = x0 + 3; gi <= x0 + 5; ++gi) {
    land(gi);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  for (int x = x0; x < I1; ++x) {
    // plane x+3 has landed (x+4, x+5 may still be in flight)
    asm volatile("cp.async.wait_group 2;" ::: "memory");
    __syncthreads();
    const float* P0 = pslot(x);      // plane x
    float* P1 = pslot(x + 1);        // plane x+1
    const float* P2 = pslot(x + 2);  // plane x+2
    // ---- red cells of plane x+1 ----
    const int xr = x + 1;
    if (xr >= 1 && xr <= g.im) {
      const float* R1 = rslot(xr);
#pragma unroll
      for (int u = 0; u < MR_ITEMS; ++u) {
        const int r = it_r[u];
        if (r < 0) continue;
        const int gj = J0 - 1 + r;
        const bool real = gj >= 1 && gj <= g.jm;
        if (!real && !img_ok) continue;
        // red at (xr, gj, k): k parity == (x + gj) parity
        const int k = 2 * it_q[u] + 2 - ((x + gj) & 1);
        if (k > km) continue;
        const int sl = k >> 1;
        const int row = (r + 1) * RW;  // staged row of gj (staged rows start at J0-2)
        const float pc = P1[row + sl];
        const float pE = P2[row + KK + sl];
        const float pW = P0[row + KK + sl];
        const float pN = P1[row + RW + KK + sl];
        const float pS = P1[row - RW + KK + sl];
        const float pT = P1[row + KK + ((k + 1) >> 1)];
        const float pB = P1[row + KK + ((k - 1) >> 1)];
        float nb = a.w2l * pE;
        nb = nb + a.w2s * pW;
        nb = nb + a.w3l * pN;
        nb = nb + a.w3s * pS;
        nb = nb + a.w4l * pT;
        nb = nb + a.w4s * pB;
        const float rh = R1[r * RW + sl];
        const float rel = a.om * (a.cn1 * (nb - rh) - pc);
        P1[row + sl] = pc + rel;
        if (xr >= I0 && xr < I1 && r >= 1 && r <= TJ) acc_r += (double)rel * (double)rel;
      }
    }
    // split plane x+3 into the slots of planes x-2 (p) and x-1 (rhs): free
    split(x + 3);
    __syncthreads();
    // ---- black cells of plane x (strip rows), then write plane x ----
    if (x >= I0) {
      const float* Pm = pslot(x - 1);  // plane x-1
      float* Pc = pslot(x);            // plane x
      const float* R0 = rslot(x);
#pragma unroll
      for (int u = 0; u < MR_ITEMS; ++u) {
        const int r = it_r[u];
        if (r < 1 || r > TJ) continue;
        const int gj = J0 - 1 + r;
        // black at (x, gj, k): k parity == (x + gj) parity
        const int k = 2 * it_q[u] + 2 - ((x + gj) & 1);
        if (k > km) continue;
        const int sl = k >> 1;
        const int row = (r + 1) * RW;
        const float pc = Pc[row + KK + sl];
        const float pE = P1[row + sl];
        const float pW = Pm[row + sl];
        const float pN = Pc[row + RW + sl];
        const float pS = Pc[row - RW + sl];
        const float pT = Pc[row + ((k + 1) >> 1)];
        const float pB = Pc[row + ((k - 1) >> 1)];
        float nb = a.w2l * pE;
        nb = nb + a.w2s * pW;
        nb = nb + a.w3l * pN;
        nb = nb + a.w3s * pS;
        nb = nb + a.w4l * pT;
        nb = nb + a.w4s * pB;
        const float rh = R0[r * RW + KK + sl];
        const float rel = a.om * (a.cn1 * (nb - rh) - pc);
        Pc[row + KK + sl] = pc + rel;
        acc_b += (double)rel * (double)rel;
      }
      __syncthreads();
      // write plane x rows J0 .. J0+TJ-1, k = 1 .. km (pb's halo cells keep
      // their values): pairs (2q, 2q+1) merged from the two colour arrays
#pragma unroll
      for (int u = 0; u < WRL; ++u) {
        if (wr_r[u] < 0) continue;
        const int r = wr_r[u], q = wr_q[u];
        const int gj = J0 + r;
        const int c0 = (x + gj + 1) & 1;
        const float* srow = Pc + (r + 2) * RW;
        float2 o;
        o.x = srow[c0 * KK + q];
        o.y = srow[(c0 ^ 1) * KK + q];
        float* d = a.pb + cidx(g, x, gj, 2 * q);
        if (VEC && 2 * q >= 1 && 2 * q + 1 <= km) {
          *reinterpret_cast<float2*>(d) = o;  // 8-byte aligned: VEC rows are 16-byte aligned
        } else {
          if (2 * q >= 1 && 2 * q <= km) d[0] = o.x;
          if (2 * q + 1 <= km) d[1] = o.y;
        }
      }
    }
    // land plane x+6 into the plain slot of plane x+3 (split above)
    land(x + 6);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  const double sr = block_sum<MR_WARPS>(acc_r, red);
  __syncthreads();
  const double sb = block_sum<MR_WARPS>(acc_b, red);
  if (tid == 0) {
    a.partials[blockIdx.x] = sr;
    a.partials[gridDim.x + blockIdx.x] = sb;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int mr_max_smem = -1, mr_num_sms = -1;

struct MrPlan {
  int tj, ch, njt, nblk, kk, kc;
  size_t smem;
  bool ok;
};

static size_t mr_smem(int tj, int kk, int kc) {
  return 4ull * (2 * kk * ((size_t)MR_PSLOTS * (tj + 4) + (size_t)MR_RSLOTS * (tj + 2)) +
                 (size_t)MR_LSLOTS * (2 * tj + 6) * kc);
}

static MrPlan mr_plan(const Geo& g, int device) {
  MrPlan pl{};
  if (mr_max_smem < 0) {
    cudaDeviceGetAttribute(&mr_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&mr_num_sms, cudaDevAttrMultiProcessorCount, device);
  }
  pl.kk = (((g.km + 1) >> 1) + 2) & ~1;
  pl.kc = (g.km + 2 + 3) & ~3;
  const int KP = (g.km + 1) >> 1;
  // strip rows: as many as the per-thread item budget allows (<= 16)
  int tj = 16;
  while (tj > 1 && (tj + 2) * KP > MR_ITEMS * MR_THREADS) --tj;
  if ((tj + 2) * KP > MR_ITEMS * MR_THREADS) return pl;
  tj = tj < g.jm ? tj : g.jm;
  const size_t smem = mr_smem(tj, pl.kk, pl.kc);
  if (smem > (size_t)mr_max_smem - 1024) return pl;
  int per_sm = (int)((size_t)mr_max_smem / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  pl.tj = tj;
  pl.njt = (g.jm + tj - 1) / tj;
  // chunk length: enough CTAs for ~2 waves, at least 8 planes per chunk
  const long long slots = (long long)mr_num_sms * per_sm;
  int nch = (int)((2 * slots + pl.njt - 1) / pl.njt);
  if (nch < 1) nch = 1;
  int ch = (g.im + nch - 1) / nch;
  if (ch < 8) ch = 8 < g.im ? 8 : g.im;
  pl.ch = ch;
  pl.nblk = pl.njt * ((g.im + ch - 1) / ch);
  pl.smem = smem;
  pl.ok = true;
  return pl;
}

int sor_blocks_march(const Geo& g, int device) {
  MrPlan pl = mr_plan(g, device);
  return pl.ok ? pl.nblk : 0;
}

bool march_supported(const Geo& g, const SorC& cf, int device) {
  return cf.uni && !cf.cn1 && g.west_bc && g.east_bc && g.ioff == 0 && mr_plan(g, device).ok;
}

template <bool PRESS, bool VEC>
static cudaError_t mr_attr() {
  static bool set = false;
  if (set) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_sor_rbmarch<PRESS, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       mr_max_smem - 2 * MR_WARPS * 8);
  if (e == cudaSuccess) set = true;
  return e;
}

cudaError_t launch_rb_march(const Geo& g, int device, const float* pa, float* pb, const float* rhs, const SorC& cf,
                            float om, int policy, double* partials, cudaStream_t st) {
  MrPlan pl = mr_plan(g, device);
  if (!pl.ok || !cf.uni || cf.cn1) return cudaErrorInvalidValue;
  // 16-byte row copies need rows that start on 16-byte boundaries
  const bool vec = ((g.km + 2) & 3) == 0 && (((size_t)pa | (size_t)rhs) & 15) == 0;
  cudaError_t e = policy == 1 ? (vec ? mr_attr<true, true>() : mr_attr<true, false>())
                              : (vec ? mr_attr<false, true>() : mr_attr<false, false>());
  if (e != cudaSuccess) return e;
  MrArgs a{g, pa, pb, rhs, om, cf.cn1s, cf.w2l, cf.w2s, cf.w3l, cf.w3s, cf.w4l, cf.w4s,
           pl.tj, pl.ch, pl.njt, pl.kk, pl.kc, partials};
  if (policy == 1) {
    if (vec) k_sor_rbmarch<true, true><<<pl.nblk, MR_THREADS, pl.smem, st>>>(a);
    else k_sor_rbmarch<true, false><<<pl.nblk, MR_THREADS, pl.smem, st>>>(a);
  } else {
    if (vec) k_sor_rbmarch<false, true><<<pl.nblk, MR_THREADS, pl.smem, st>>>(a);
    else k_sor_rbmarch<false, false><<<pl.nblk, MR_THREADS, pl.smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace lesb
