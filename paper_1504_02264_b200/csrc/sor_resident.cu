// Host side of the shared-memory-resident red-black SOR: tile plans, buffers
// and launches (the kernel and its device code: sor_resident_dev.cuh, also
// compiled at run time per geometry by jit.cu).
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "lesb_common.cuh"
#include "lesb_kernels.h"
#include "sor_resident_dev.cuh"

namespace lesb {

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int g_num_sms = -1;
static int g_max_smem = -1;

static size_t plan_smem(int tim, int tjm, int kk) {
  const int cw = 4 * kk + CW_EXTRA;
  const size_t arrays = 4ull * ((((size_t)cw * (tjm + 2) + ROW_PAD_MAX) * (tim + 2) + 3) & ~(size_t)3);  // p and rhs, 2 colours each
  const size_t coltab = 4ull * ((tim * tjm + 3) & ~3);
  const size_t pubcol = 8ull * ((tim * tjm + 1) & ~1);
  const size_t rcvtab = 16ull * 2 * (tim + tjm);
    // boundary-unit table: every column of a tile up to 3 x 3, else the ring
  const int nb = (tim <= 2 || tjm <= 2) ? tim * tjm : 2 * tjm + 2 * (tim - 2);
  const size_t btab = RES_BTAB ? 16ull * nb * (((kk + 1) & ~1) >> 1) : 0;
  return arrays + coltab + pubcol + rcvtab + btab;
}

// Shared-memory bank load of the interior runs for a row pad: warps of 32
// consecutive interior columns (the unit order of update_phase) touch
// column base + (1 - kp) (kp alternates with the column parity); the sum
// over warps and both colours of the most-loaded bank.
static int interior_bank_load(int TI, int TJ, int kk, int pad) {
  const int cw = 4 * kk + CW_EXTRA, sI = (TJ + 2) * cw + pad;
  const int nj = TJ - 2, nint = (TI - 2) * nj;
  int load = 0;
  for (int nrd = 0; nrd < 2; ++nrd)
    for (int w0 = 0; w0 < nint; w0 += 32) {
      int cnt[32] = {0};
      int mx = 0;
      if (RES_IPAIRS) {
        // pair runs: 64-bit accesses at the same slot of every lane's column,
        // one wavefront per half-warp when the 8-byte words hit distinct banks
        for (int h0 = w0; h0 < nint && h0 < w0 + 32; h0 += 16) {
          int c16[16] = {0}, m16 = 0;
          for (int r = h0; r < nint && r < h0 + 16; ++r) {
            const int li = 2 + r / nj, lj = 2 + r % nj;
            const int b = ((li * sI + lj * cw + nrd * kk) >> 1) & 15;
            m16 = ++c16[b] > m16 ? c16[b] : m16;
          }
          mx += m16;
        }
      } else {
        for (int r = w0; r < nint && r < w0 + 32; ++r) {
          const int li = 2 + r / nj, lj = 2 + r % nj;
          const int kp = (nrd + ((li + lj) & 1) + 1) & 1;
          const int b = (li * sI + lj * cw + nrd * kk + (1 - kp)) & 31;
          mx = ++cnt[b] > mx ? cnt[b] : mx;
        }
      }
      load += mx;
    }
  return load;
}

static int best_row_pad(int TI, int TJ, int kk) {
  if (TI <= 2 || TJ <= 2) return 0;
  int best = 0, bl = 1 << 30;
  for (int pad = 0; pad <= ROW_PAD_MAX; pad += RES_PAIRS ? 2 : 1) {
    const int l = interior_bank_load(TI, TJ, kk, pad);
    if (l < bl) {
      bl = l;
      best = pad;
    }
  }
  return best;
}

static ResPlan plan_resident_uncached(const Geo& g, int device, int max_tiles);

// plans are pure functions of (im, jm, km, max_tiles) on one GPU model; the
// row-pad search makes them worth caching (they are asked for on every solve)
ResPlan plan_resident(const Geo& g, int device, int max_tiles) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, ResPlan> cache;
  const auto key = std::make_tuple(g.im, g.jm, g.km, max_tiles);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  ResPlan pl = plan_resident_uncached(g, device, max_tiles);
  cache.emplace(key, pl);
  return pl;
}

static ResPlan plan_resident_uncached(const Geo& g, int device, int max_tiles) {
  ResPlan pl{};
  pl.ok = false;
  if (g_num_sms < 0) {
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&g_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  }
  if (g_num_sms <= 0) return pl;
  if (max_tiles <= 0 || max_tiles > g_num_sms) max_tiles = g_num_sms;
  pl.kk = ((g.km + 1) >> 1) + 1;
  if (RES_PAIRS) pl.kk = (pl.kk + 1) & ~1;
  pl.kt = (g.km + 1) >> 1;
  size_t best = (size_t)-1;
  // tiles of at least 2 x 2 columns: a column then lies on at most two faces
  for (int ni = 1; 2 * ni <= g.im && ni <= max_tiles; ++ni) {
    for (int nj = 1; 2 * nj <= g.jm && ni * nj <= max_tiles; ++nj) {
      const int tim = (g.im + ni - 1) / ni, tjm = (g.jm + nj - 1) / nj;
      const size_t smem = plan_smem(tim, tjm, pl.kk);
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
  pl.fstride = (long long)fmax * ((pl.kk + 1) & ~1);  // even words per face column (16-byte pairs)
  pl.bstride = (4LL * pl.ni * pl.nj + 2LL * pl.nj) * pl.fstride;  // tile faces + ghost slots
  pl.xbuf = 4 * pl.bstride;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) pl.pad[a][b] = best_row_pad(pl.ti_max - a, pl.tj_max - b, pl.kk);
  pl.ok = true;
  return pl;
}

bool resident_supported(const Geo& g, const SorC& cf, int device, int max_tiles) {
  if (cf.cn1 != nullptr || !cf.uni) return false;  // scalar cn1 and neighbour weights
  return plan_resident(g, device, max_tiles).ok;
}

int resident_ntiles(const Geo& g, int device, int max_tiles) {
  ResPlan pl = plan_resident(g, device, max_tiles);
  return pl.ok ? pl.ni * pl.nj : 0;
}

int resident_partials(const Geo& g, int device, int max_tiles) {
  ResPlan pl = plan_resident(g, device, max_tiles);
  return pl.ok ? pl.ni * pl.nj * RES_WARPS : 0;
}

long long resident_xbuf_words(const Geo& g, int device, int max_tiles) {
  ResPlan pl = plan_resident(g, device, max_tiles);
  return pl.ok ? pl.xbuf : 0;
}

static unsigned long long* g_tbuf = nullptr;  // LESB_RES_TRACE stamps of the last launch
static size_t g_tcap = 0, g_tlen = 0;

// the dynamic shared-memory ceiling of a kernel (ahead-of-time or runtime
// specialised), raised once per function
static cudaError_t set_smem_attr(const void* fn) {
  static std::mutex mu;
  static std::map<const void*, int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(fn)) return cudaSuccess;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  const int dyn_max = g_max_smem - (int)fa.sharedSizeBytes;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
  if (e != cudaSuccess) return e;
  done[fn] = dyn_max;
  return cudaSuccess;
}

static cudaError_t launch_group(ResGroup& grp, int policy, bool slab, size_t smem, cudaStream_t st) {
  const void* fn = policy == 1 ? (slab ? (const void*)k_sor_resident<true, true> : (const void*)k_sor_resident<true, false>)
                               : (slab ? (const void*)k_sor_resident<false, true> : (const void*)k_sor_resident<false, false>);
  // this geometry and tile plan as compile-time constants (jit.cu), when specialised
  if (cudaKernel_t k = jit_resident_kernel(grp.a[0].g, grp.a[0].pl, policy == 1, slab))
    fn = reinterpret_cast<const void*>(k);
  cudaError_t e = set_smem_attr(fn);
  if (e != cudaSuccess) return e;
  void* args[] = {&grp};
  // programmatic dependent launch: the CTAs may start (and build their
  // tables) while the step's fused kernel drains; griddepcontrol.wait in the
  // kernel orders every global access after it.  LESB_STEP_PDL=0: plain.
  static const bool pdl = !(std::getenv("LESB_STEP_PDL") && std::atoi(std::getenv("LESB_STEP_PDL")) == 0);
  if (!pdl) return cudaLaunchCooperativeKernel(fn, dim3(grp.n * grp.tps), dim3(RES_THREADS), args, smem, st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grp.n * grp.tps);
  cfg.blockDim = dim3(RES_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

static ResArgs make_args(const ResidentCall& c, const ResPlan& pl) {
  ResArgs a{};
  a.g = *c.g;
  a.pl = pl;
  a.p = c.p;
  a.rhs = c.rhs;
  a.om = c.om;
  a.cn1 = c.cf->cn1s;
  a.w2l = c.cf->w2l; a.w2s = c.cf->w2s; a.w3l = c.cf->w3l; a.w3s = c.cf->w3s; a.w4l = c.cf->w4l; a.w4s = c.cf->w4s;
  a.n_iter = c.n_iter;
  a.xbuf = (unsigned long long*)c.xbuf;
  a.epoch = c.epoch;
  a.partials = c.partials;
  a.res = c.res;
  a.pflags = c.pflags;
  a.err = c.err;
  a.peer_w = (unsigned long long*)c.peer_w;
  a.peer_e = (unsigned long long*)c.peer_e;
#ifdef LESB_RES_DEBUG_BUILD
  static const int dbg = getenv("LESB_RES_DEBUG") ? atoi(getenv("LESB_RES_DEBUG")) : 0;
  a.debug = dbg;
#else
  a.debug = 0;
#endif
  a.trace = nullptr;
  a.book = c.book;
  return a;
}

// One launch does the whole solve: n_iter iterations, the press halo (policy
// 1) with its non-finite check into pflags, and res[n_iter].  xbuf holds
// resident_xbuf_words() 64-bit words, zeroed once; *epoch starts at 0 and is
// advanced by every launch (both are reset after a timeout).  With peer_w /
// peer_e set the domain is an x-slab whose neighbours run the same plan on
// other GPUs (their face buffers mapped here), launched at the same time.
cudaError_t launch_sor_resident(const ResidentCall& c, cudaStream_t st) {
  ResPlan pl = plan_resident(*c.g, c.device, c.max_tiles);
  if (!pl.ok || !c.cf->uni || c.cf->cn1) return cudaErrorInvalidValue;
  ResGroup grp{};
  grp.a[0] = make_args(c, pl);
  grp.n = 1;
  grp.tps = pl.ni * pl.nj;
  static const bool trace = getenv("LESB_RES_TRACE") != nullptr;
  const size_t tneed = (size_t)grp.tps * 2 * c.n_iter * NST + (size_t)grp.tps * 8;  // + per-tile phase stamps
  if (trace) {
    if (g_tcap < tneed) {
      if (g_tbuf) cudaFree(g_tbuf);
      cudaMalloc(&g_tbuf, tneed * 8);
      g_tcap = tneed;
    }
    g_tlen = tneed;
    grp.a[0].trace = g_tbuf;
  }
  return launch_group(grp, c.policy, c.peer_w || c.peer_e, pl.smem, st);
}

// n in-process x-slabs of one device (west to east), one cooperative launch:
// each slab gets num_SMs / n tiles; the slabs' x faces move through each
// other's ghost slots like the cross-GPU case.  All slabs must share
// (im, jm, km) (so they share the plan) and one epoch word.
cudaError_t launch_sor_resident_group(int n, const ResidentCall* cs, cudaStream_t st) {
  if (n < 1 || n > RES_GROUP_MAX) return cudaErrorInvalidValue;
  ResPlan pl = plan_resident(*cs[0].g, cs[0].device, resident_group_tiles(n));
  if (!pl.ok) return cudaErrorInvalidValue;
  ResGroup grp{};
  for (int s = 0; s < n; ++s) {
    if (!cs[s].cf->uni || cs[s].cf->cn1) return cudaErrorInvalidValue;
    grp.a[s] = make_args(cs[s], pl);
  }
  grp.n = n;
  grp.tps = pl.ni * pl.nj;
  return launch_group(grp, cs[0].policy, true, pl.smem, st);
}

int resident_group_max() { return RES_GROUP_MAX; }

int resident_group_tiles(int n) {
  if (g_num_sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&g_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return g_num_sms > 0 && n > 0 ? (g_num_sms / n > 0 ? g_num_sms / n : 1) : 1;
}

}  // namespace lesb

// Debug only (not in the public header): copy the last traced launch's
// stamps ([tile][pass][NST]: before receive, after receive barrier, after
// the boundary phase (three copies), after interior runs) to host; returns
// the word count.
extern "C" long long lesb_debug_resident_trace(unsigned long long* host, long long cap) {
  using namespace lesb;
  if (!g_tbuf || !host) return 0;
  const long long n = (long long)g_tlen < cap ? (long long)g_tlen : cap;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_tbuf, n * 8, cudaMemcpyDeviceToHost);
  return n;
}
