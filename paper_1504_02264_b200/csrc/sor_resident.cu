// Persistent, shared-memory-resident red-black SOR (reference semantics:
// gmcf_mini/sor.py:181-203 with the halo policies of sor.cu).
//
// One CTA per SM (cooperative launch, so every CTA is co-resident) owns an
// (i, j) tile of the grid with its full k columns.  The tile's pressure and
// rhs stay in shared memory for the whole solve; only tile faces move, through
// L2, once per colour pass:
//
//   for pass n (colour nrd = n & 1):
//     update the colour-nrd cells of the tile in shared memory
//     publish the colour-nrd cells of the 4 tile faces to a global face buffer
//     release-store flag[tile] = n + 1
//     acquire-wait until every neighbour's flag >= n + 1
//     copy the neighbours' published faces into the tile's halo slots
//
// Shared memory holds each colour separately ("colour split": cell (i,j,k)
// lives in array colour(i,j,k) at slot k >> 1), so a warp's 32 lanes touch 32
// consecutive words for the centre, all six neighbours and rhs (no bank
// conflicts).  Halo slots take the colour of their storage position; for the
// periodic wrap with odd jm the source cell has the other colour, which is
// exactly the reference's pre-pass snapshot of the y halo (the slot is only
// refreshed after the pass that updated its source).
//
// Arithmetic per point is sor_point's (same op order, -fmad=false), so the
// result is bitwise identical to the streaming kernels and the reference.
#include <cooperative_groups.h>

#include "lesb_common.cuh"
#include "lesb_kernels.h"

namespace lesb {

struct ResPlan {
  int ni, nj;       // tile grid
  int ti_max, tj_max;
  int kk;           // slots per colour column: ((km + 1) >> 1) + 1
  int nthreads;
  size_t smem;      // dynamic shared memory bytes
  long long xbuf;   // floats of the face exchange buffer
  bool ok;
};

struct ResArgs {
  Geo g;
  ResPlan pl;
  float* p;
  const float* rhs;
  SorC cf;
  float om;
  int n_iter;
  int policy;       // 0 STORED, 1 PRESS
  float* xbuf;      // [2][ntiles][4][fmax * kk]
  unsigned* flags;  // [ntiles], zero at entry
  double* partials; // [2 n_iter][ntiles]
  unsigned* err;    // set when a neighbour wait times out
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

__device__ __forceinline__ int tile_lo(int t, int n, int nt) { return 1 + (int)(((long long)t * n) / nt); }

// colour of global cell: the pass nrd updates cells with colour == nrd
// ((i-1)+(j-1)+(k-1)+nrd even, sor.py:174-178)
__device__ __forceinline__ int colour(int i, int j, int k) { return (i + j + k + 1) & 1; }

__global__ void __launch_bounds__(512, 1) k_sor_resident(ResArgs a) {
  extern __shared__ float smem[];
  const Geo& g = a.g;
  const ResPlan& pl = a.pl;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int tile = blockIdx.x;
  const int ti = tile / pl.nj, tj = tile % pl.nj;
  const int I0 = tile_lo(ti, g.im, pl.ni), I1 = tile_lo(ti + 1, g.im, pl.ni);
  const int J0 = tile_lo(tj, g.jm, pl.nj), J1 = tile_lo(tj + 1, g.jm, pl.nj);
  const int TI = I1 - I0, TJ = J1 - J0;
  const int KK = pl.kk;
  const int sJ = KK, sI = (pl.tj_max + 2) * KK;
  const int csz = (pl.ti_max + 2) * sI;  // floats per colour array
  float* S = smem;                       // [2][ti_max+2][tj_max+2][KK]
  float* R = smem + 2 * csz;             // same layout, interior used
  const int fmax = pl.ti_max > pl.tj_max ? pl.ti_max : pl.tj_max;
  const long long fstride = (long long)fmax * KK;
  const int ntiles = pl.ni * pl.nj;
  const bool press = a.policy == 1;

  // local (li, lj) in [0, TI+1] x [0, TJ+1]; global i = I0 - 1 + li
  auto sidx = [&](int li, int lj, int k) { return li * sI + lj * sJ + (k >> 1); };
  auto gval = [&](int i, int j, int k) { return a.p[cidx(g, i, j, k)]; };

  // ---- load tile interior, rhs and halo slots from global memory ----
  const int ncol_h = (TI + 2) * (TJ + 2);
  for (int idx = tid; idx < ncol_h * (g.km + 2); idx += nth) {
    const int col = idx / (g.km + 2), k = idx - col * (g.km + 2);
    const int li = col / (TJ + 2), lj = col - li * (TJ + 2);
    const int i = I0 - 1 + li, j = J0 - 1 + lj;
    const bool ih = li == 0 || li == TI + 1, jh = lj == 0 || lj == TJ + 1, kh = k == 0 || k == g.km + 1;
    if ((ih && jh) || (ih && kh) || (jh && kh)) continue;  // edges/corners are never read
    float v;
    if (!press) {
      v = gval(i, j, k);  // stored halo, or neighbour tile's initial value
    } else if (kh) {
      v = 0.0f;  // top: 0; bottom: remapped at read time
    } else if (ih && (i == 0 || i == g.im + 1)) {
      v = 0.0f;  // east: 0; west: remapped at read time
    } else if (jh) {
      const int jj = j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j);
      v = gval(i, jj, k);
    } else {
      v = gval(i, j, k);
    }
    S[colour(i, j, k) * csz + sidx(li, lj, k)] = v;
    if (!ih && !jh && !kh) R[colour(i, j, k) * csz + sidx(li, lj, k)] = a.rhs[cidx(g, i, j, k)];
  }
  // neighbour tiles (-1: physical boundary with a fixed / remapped halo)
  int nbr[4];
  nbr[0] = ti > 0 ? tile - pl.nj : -1;            // west  <- its i-hi face
  nbr[1] = ti < pl.ni - 1 ? tile + pl.nj : -1;    // east  <- its i-lo face
  nbr[2] = tj > 0 ? tile - 1 : (press ? ti * pl.nj + pl.nj - 1 : -1);  // south <- its j-hi face
  nbr[3] = tj < pl.nj - 1 ? tile + 1 : (press ? ti * pl.nj : -1);     // north <- its j-lo face
  const int wrap_flip = (g.jm & 1);  // periodic source parity differs from the slot's for odd jm
  __syncthreads();

  const int KH = (g.km + 1) >> 1;  // colour cells per column (upper bound)
  const int ncol = TI * TJ;
  const int nwork = ncol * KH;
  const bool wphys = press && g.west_bc && ti == 0;
  __shared__ double red[16];

  for (int n = 0; n < 2 * a.n_iter; ++n) {
    const int nrd = n & 1;
    float* Sc = S + nrd * csz;         // cells being updated
    const float* So = S + (1 - nrd) * csz;  // their neighbours
    const float* Rc = R + nrd * csz;
    double acc = 0.0;
    for (int w = tid; w < nwork; w += nth) {
      const int col = w / KH, t = w - col * KH;
      const int li = 1 + col / TJ, lj = 1 + (col - (li - 1) * TJ);
      const int i = I0 - 1 + li, j = J0 - 1 + lj;
      const int k = 1 + ((i + j + nrd) & 1) + 2 * t;  // colour(i,j,k) == nrd
      if (k > g.km) continue;
      const int s = sidx(li, lj, k);
      const int sk_lo = li * sI + lj * sJ + ((k - 1) >> 1);
      const int sk_hi = li * sI + lj * sJ + ((k + 1) >> 1);
      const float pc = Sc[s];
      const float pE = So[s + sI];
      const float pW = (wphys && li == 1) ? pc : So[s - sI];
      const float pN = So[s + sJ];
      const float pS = So[s - sJ];
      const float pT = So[sk_hi];
      const float pB = (press && k == 1) ? pc : So[sk_lo];
      float nb = a.cf.cn2l[i - 1] * pE;
      nb = nb + a.cf.cn2s[i - 1] * pW;
      nb = nb + a.cf.cn3l[j - 1] * pN;
      nb = nb + a.cf.cn3s[j - 1] * pS;
      nb = nb + a.cf.cn4l[k - 1] * pT;
      nb = nb + a.cf.cn4s[k - 1] * pB;
      const float rel = a.om * (a.cf.cn1s * (nb - Rc[s]) - pc);
      Sc[s] = pc + rel;
      acc += (double)rel * (double)rel;
    }
    __syncthreads();
    // publish this pass's colour on the 4 faces: [face][m][kk] with m along the face
    float* X = a.xbuf + ((long long)(n & 1) * ntiles + tile) * 4 * fstride;
    {
      const int nf0 = TJ * KK, nf2 = TI * KK;
      const int tot = 2 * nf0 + 2 * nf2;
      for (int idx = tid; idx < tot; idx += nth) {
        int f, m, kk;
        if (idx < 2 * nf0) {
          f = idx / nf0;
          const int r = idx - f * nf0;
          m = r / KK;
          kk = r - m * KK;
        } else {
          const int r0 = idx - 2 * nf0;
          f = 2 + r0 / nf2;
          const int r = r0 - (f - 2) * nf2;
          m = r / KK;
          kk = r - m * KK;
        }
        const int li = f == 0 ? 1 : (f == 1 ? TI : 1 + m);
        const int lj = f == 2 ? 1 : (f == 3 ? TJ : 1 + m);
        __stcg(X + f * fstride + m * KK + kk, Sc[li * sI + lj * sJ + kk]);
      }
    }
    const double bs = block_sum<16>(acc, red);
    if (tid == 0) a.partials[(long long)n * ntiles + tile] = bs;
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(a.flags + tile, (unsigned)(n + 1));
    if (tid < 4 && nbr[tid] >= 0) {
      const unsigned* fl = a.flags + nbr[tid];
      unsigned spins = 0;
      while (ld_acquire(fl) < (unsigned)(n + 1)) {
        if (++spins > (1u << 26)) {  // ~seconds: never hang the GPU
          atomicOr(a.err, 1u);
          break;
        }
        if (spins > 64) __nanosleep(32);
      }
    }
    __syncthreads();
    // receive: neighbour faces into this tile's halo slots
    {
      const int nf0 = TJ * KK, nf2 = TI * KK;
      const int tot = 2 * nf0 + 2 * nf2;
      for (int idx = tid; idx < tot; idx += nth) {
        int side, m, kk;
        if (idx < 2 * nf0) {
          side = idx / nf0;
          const int r = idx - side * nf0;
          m = r / KK;
          kk = r - m * KK;
        } else {
          const int r0 = idx - 2 * nf0;
          side = 2 + r0 / nf2;
          const int r = r0 - (side - 2) * nf2;
          m = r / KK;
          kk = r - m * KK;
        }
        const int src = nbr[side];
        if (src < 0) continue;
        // west reads the neighbour's east face (1), east its west face (0), ...
        const int sface = side ^ 1;
        const float* XS = a.xbuf + ((long long)(n & 1) * ntiles + src) * 4 * fstride + sface * fstride;
        const int li = side == 0 ? 0 : (side == 1 ? TI + 1 : 1 + m);
        const int lj = side == 2 ? 0 : (side == 3 ? TJ + 1 : 1 + m);
        const bool wrap = (side == 2 && tj == 0) || (side == 3 && tj == pl.nj - 1);
        const int slot_colour = nrd ^ (wrap ? wrap_flip : 0);
        const float v = __ldcg(XS + m * KK + kk);
        // only slots whose source cell has colour nrd changed in this pass
        const int i = I0 - 1 + li, j = J0 - 1 + lj;
        const int k_src_par = (i + j + 1 + slot_colour) & 1;  // k parity of slot-colour cells here
        const int k = 2 * kk + k_src_par;
        if (k < 1 || k > g.km) continue;
        S[slot_colour * csz + li * sI + lj * sJ + kk] = v;
      }
    }
    __syncthreads();
  }

  // ---- write the tile back ----
  for (int idx = tid; idx < ncol * g.km; idx += nth) {
    const int col = idx / g.km, k = 1 + (idx - col * g.km);
    const int li = 1 + col / TJ, lj = 1 + (col - (li - 1) * TJ);
    const int i = I0 - 1 + li, j = J0 - 1 + lj;
    a.p[cidx(g, i, j, k)] = S[colour(i, j, k) * csz + sidx(li, lj, k)];
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int g_num_sms = -1;
static int g_max_smem = -1;

ResPlan plan_resident(const Geo& g, int device) {
  ResPlan pl{};
  pl.ok = false;
  if (g_num_sms < 0) {
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&g_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  }
  if (g_num_sms <= 0 || !g.west_bc || !g.east_bc || g.ioff != 0) return pl;
  pl.kk = ((g.km + 1) >> 1) + 1;
  pl.nthreads = 512;
  size_t best = (size_t)-1;
  for (int ni = 1; ni <= g.im && ni <= g_num_sms; ++ni) {
    for (int nj = 1; nj <= g.jm && ni * nj <= g_num_sms; ++nj) {
      const int tim = (g.im + ni - 1) / ni, tjm = (g.jm + nj - 1) / nj;
      const size_t smem = 4 * (size_t)2 * 2 * (tim + 2) * (tjm + 2) * pl.kk;
      if (smem > (size_t)g_max_smem - 2048) continue;
      // cost: largest tile's cells plus a face-exchange term
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
  pl.xbuf = 2LL * pl.ni * pl.nj * 4 * fmax * pl.kk;
  pl.ok = true;
  return pl;
}

bool resident_supported(const Geo& g, const SorC& cf, int device) {
  if (cf.cn1 != nullptr) return false;  // cn1 must be a scalar
  return plan_resident(g, device).ok;
}

int resident_ntiles(const Geo& g, int device) {
  ResPlan pl = plan_resident(g, device);
  return pl.ok ? pl.ni * pl.nj : 0;
}

long long resident_xbuf_floats(const Geo& g, int device) {
  ResPlan pl = plan_resident(g, device);
  return pl.ok ? pl.xbuf : 0;
}

cudaError_t launch_sor_resident(const Geo& g, int device, float* p, const float* rhs, const SorC& cf, float om,
                                int n_iter, int policy, float* xbuf, unsigned* flags, double* partials,
                                unsigned* err, cudaStream_t st) {
  ResPlan pl = plan_resident(g, device);
  if (!pl.ok) return cudaErrorInvalidValue;
  static int attr_set = 0;
  if (attr_set < (int)pl.smem) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_sor_resident);
    if (e != cudaSuccess) return e;
    const int dyn_max = g_max_smem - (int)fa.sharedSizeBytes;
    e = cudaFuncSetAttribute(k_sor_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
    if (e != cudaSuccess) return e;
    attr_set = dyn_max;
  }
  const int ntiles = pl.ni * pl.nj;
  cudaError_t e = cudaMemsetAsync(flags, 0, ntiles * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  ResArgs a{g, pl, p, rhs, cf, om, n_iter, policy, xbuf, flags, partials, err};
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((const void*)k_sor_resident, dim3(ntiles), dim3(pl.nthreads), args, pl.smem,
                                     st);
}

}  // namespace lesb
