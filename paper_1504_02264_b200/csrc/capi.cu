// C ABI of the B200 DPRI-LES library (declared in include/les_b200.h).
//
// A domain handle owns device-resident state: u, v, w (plus a second
// velocity set the fused step kernels ping-pong through), p (plus a second
// buffer for the twinned scheme), rhs, mask, fgh, fgh_old, spacings and SOR
// coefficients.  One time step is captured once into a CUDA graph per
// (n_iter, scheme, omega) and replayed.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <nccl.h>

#include "les_b200.h"
#include "lesb_common.cuh"
#include "lesb_kernels.h"

#include <nvtx3/nvToolsExt.h>

namespace {
// NVTX range around a C ABI entry point (tracing): shows the
// host-side step / solve calls in Nsight Systems; without a tool attached the
// calls are no-ops.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace lesb;

namespace {

thread_local std::string g_err;

std::mutex& g_solver_mu_fwd() {
  static std::mutex m;
  return m;
}
std::map<std::tuple<int, int, int, int>, lesb_domain*>& solver_map() {
  static std::map<std::tuple<int, int, int, int>, lesb_domain*> m;
  return m;
}

int default_sor_path() {
  static int v = [] {
    const char* e = std::getenv("LESB_SOR_PATH");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
int g_default_sor_path = -1;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) return fail(LESB_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

enum { MODE_SYNC = 0, MODE_ASYNC = 1 };

// device-side step bookkeeping for asynchronous runs: lesb::StepBook
// (lesb_kernels.h); the resident solver does it itself when it ends the step
__global__ void k_step_tail(StepBook* b) {
  if (threadIdx.x == 0 && blockIdx.x == 0) step_book_update(b);
}

// The synchronous step moves its inflow in and its residuals and flags out
// through host-mapped pinned memory with these kernels instead of copy-engine
// memcpys: the bulk copies of lesb_stage_upload / lesb_download_async run on
// the copy engines meanwhile, and a step's small copies would queue behind
// them (one direction's copies are served in order).
__global__ void k_step_head(float* __restrict__ in_d, const float* __restrict__ in_h, int n, StepBook* b) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) in_d[i] = in_h[i];
  if (threadIdx.x == 0) {
    b->flags = 0;
    b->err = 0;
  }
}

// the inflow as a kernel argument (launched before the step graph): the step
// then reads nothing from host memory -- a host read waits behind a bulk
// device-to-host copy's writes on the link
constexpr int INFLOW_ARG_MAX = 288;  // (3 km floats, km <= 96; the argument is rewritten every step)
struct InflowArg {
  float v[INFLOW_ARG_MAX];
};
__global__ void k_step_head_arg(float* __restrict__ in_d, const __grid_constant__ InflowArg in, int n, StepBook* b) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) in_d[i] = in.v[i];
  if (threadIdx.x == 0) {
    b->flags = 0;
    b->err = 0;
  }
}

bool inflow_by_arg(int km) {
  static const bool off = std::getenv("LESB_INFLOW_ARG") && std::atoi(std::getenv("LESB_INFLOW_ARG")) == 0;
  return !off && 3 * km <= INFLOW_ARG_MAX;
}

__global__ void k_step_out(double* __restrict__ res_h, const double* __restrict__ res_d, int n,
                           StepBook* __restrict__ book_h, const StepBook* __restrict__ book_d) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) res_h[i] = res_d[i];
  if (threadIdx.x == 0) *book_h = *book_d;
}

__global__ void k_word_out(unsigned* dst_h, const unsigned* src_d) { *dst_h = *src_d; }

__global__ void k_set_word(int* dst, int v) { *dst = v; }

// device-to-device field copy (staged commit, snapshot): a kernel, for the
// same reason
__global__ void k_copy_field(float* __restrict__ dst, const float* __restrict__ src, long long n) {
  const long long n4 = n >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  float4* d4 = reinterpret_cast<float4*>(dst);
  const float4* s4 = reinterpret_cast<const float4*>(src);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) d4[i] = s4[i];
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) dst[4 * n4 + threadIdx.x] = src[4 * n4 + threadIdx.x];
}

cudaError_t copy_field(float* dst, const float* src, long long n, int device, cudaStream_t st) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  k_copy_field<<<4 * sms, 512, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}

int first_stage(unsigned bits) {
  for (int s = 0; s < 7; ++s)
    if (bits & (1u << s)) return s;
  return -1;
}

}  // namespace

// Neighbours of an x-slab: in-process domains on the same
// device (plane copies), or ranks rank-1 / rank+1 of an NCCL communicator.
struct SlabLink {
  lesb_domain* west = nullptr;
  lesb_domain* east = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
};

struct lesb_domain {
  SlabLink link;
  int device = 0;
  cudaStream_t st = nullptr;
  Geo g{};
  float dt = 0.5f, vn = 1e-5f, cs = 0.14f, csd2s = 0.f;
  float* csd2 = nullptr;
  float *dx1 = nullptr, *dy1 = nullptr, *dzn = nullptr;
  float *u = nullptr, *v = nullptr, *w = nullptr, *ub = nullptr, *vb = nullptr, *wb = nullptr;
  float *p = nullptr, *pb = nullptr, *rhs = nullptr, *mask = nullptr, *fgh = nullptr, *fgh_old = nullptr;
  float* cn1 = nullptr;
  float* cn[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  float cn1s = 0.f;
  int cuni = 0;
  float cw[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  bool coeffs_set = false;
  float* inflow_d = nullptr;
  float* inflow_h = nullptr;  // pinned
  StepBook* book_d = nullptr;
  StepBook* book_h = nullptr;  // pinned
  double* partials = nullptr;
  long long partials_cap = 0;
  double* res_d = nullptr;
  double* res_h = nullptr;  // pinned
  int res_cap = 0;
  float* scratch = nullptr;  // im*jm*km
  std::map<std::tuple<int, int, int, unsigned>, cudaGraphExec_t> graphs;
  // synchronous step graphs with the inflow as a kernel argument: the head
  // node (its arguments set before every launch) and the captured graph it
  // belongs to
  std::map<std::tuple<int, int, int, unsigned>, std::pair<cudaGraph_t, cudaGraphNode_t>> heads;
  bool timing = false;
  int sor_path = 0;  // 0 auto, 1 streaming colour passes, 2 shared-memory-resident solver, 3 natural-layout passes
  float* split = nullptr;  // colour-split p / rhs of the streaming red-black passes (4 * SplitGeo::n floats)
  void* xbuf = nullptr;       // resident solver face exchange (64-bit words)
  int* coll_d = nullptr;      // NCCL slabs: scratch of the stage reductions
  int* coll_h = nullptr;      // (pinned, host-mapped: the reduced value)
  // x-slab streaming passes with the fused plane exchange (PassGhost):
  // ghost planes [from west: 4 slots][from east: 4 slots] of spi words, the
  // solve epoch, and (NCCL ranks) the neighbours' ghost buffers mapped
  unsigned long long* ghost = nullptr;
  unsigned* gh_epoch = nullptr;
  void* gpeer_w = nullptr;
  void* gpeer_e = nullptr;
  bool ghost_ready = false;
  unsigned* repoch = nullptr;  // resident solver tag epoch
  // x-slab on NCCL ranks: the neighbour ranks' face buffers mapped through
  // CUDA IPC (peer memory over NVLink) so the resident solver exchanges tile
  // faces inside its one launch; peer_ready once both sides are mapped
  void* peer_w = nullptr;
  void* peer_e = nullptr;
  bool peer_ready = false;
  bool peer_tried = false;
  // in-process slab group: face buffers sized for the group plan, shared epoch
  void* gxbuf = nullptr;
  unsigned* gepoch = nullptr;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // asynchronous state copies (lesb_stage_upload / lesb_download_async): an
  // upload and a download stream beside `st`, a device staging buffer and a
  // device snapshot buffer per field, events ordering their reuse
  cudaStream_t up_st = nullptr, dn_st = nullptr;
  float* staged[8] = {};
  float* snap[8] = {};
  unsigned staged_mask = 0;
  cudaEvent_t ev_up = nullptr, ev_commit = nullptr, ev_snap = nullptr;
  cudaEvent_t ev_dn[8] = {};  // per field: the last download from its snapshot buffer
  // the copies not yet enqueued: a synchronous step enqueues one chunk of
  // each direction after its launch (so the link carries at most one chunk
  // while the step's own transfers run); commit / a reused snapshot buffer /
  // lesb_copies_wait enqueue the rest at once
  struct Chunk {
    void* dst;
    const void* src;
    size_t bytes;
    int field;
    bool last;
  };
  std::vector<Chunk> pend_up, pend_dn;
  size_t pu = 0, pd = 0;  // next pending chunk
  size_t chunk_bytes = 0;
  bool known_finite = false;
  long long n_alloc = 0;  // (im+3)*si
  long long n_py = 0;     // (im+2)*si : the Python-visible array
  std::mutex mu;

  Spac sp{};  // spacings + exact reciprocals (set_spacing_info)
  Spac spac() const { return sp; }
  SorC sorc() const {
    return SorC{cn1, cn1s, cn[0], cn[1], cn[2], cn[3], cn[4], cn[5], cuni, cw[0], cw[1], cw[2], cw[3], cw[4], cw[5]};
  }
  ResidentBufs rbufs() const {
    // auto: the resident solver where the grid fits the SMs' shared memory,
    // else the streaming colour passes on the colour-split layout (path 3:
    // the same passes on the natural layout, also the fallback for
    // non-uniform coefficients)
    const bool res = resident_in_use();
    ResidentBufs rb{res, device, sor_path == 3 ? 1 : 0, xbuf, repoch, &book_d->err};
    rb.split = split;
    if (ghost_ready && !res) {  // NCCL slab on the streaming passes: exchange fused into the pass kernel
      const long long sp = split_geo(g).spi;
      rb.ghost.my_w = g.west_bc ? nullptr : ghost;
      rb.ghost.my_e = g.east_bc ? nullptr : ghost + 4 * sp;
      rb.ghost.to_w = gpeer_w ? (unsigned long long*)gpeer_w + 4 * sp : nullptr;  // the west rank's from-east planes
      rb.ghost.to_e = gpeer_e ? (unsigned long long*)gpeer_e : nullptr;           // the east rank's from-west planes
      rb.ghost.epoch = gh_epoch;
      rb.ghost.err = &book_d->err;
      rb.ghost.sys = 1;
    }
    if (res && !(g.west_bc && g.east_bc && g.ioff == 0)) {  // x-slab: faces through the neighbours' buffers
      rb.peer_w = peer_w;
      rb.peer_e = peer_e;
    }
    return rb;
  }
  long long n_int() const { return (long long)g.im * g.jm * g.km; }
  bool resident_in_use() const {
    const bool whole = g.west_bc && g.east_bc && g.ioff == 0;  // one domain (not an x-slab)
    return (sor_path == 0 || sor_path == 2) && xbuf != nullptr && (whole || peer_ready);
  }
};

namespace {

// x is a power of two (normal, positive): its reciprocal is exact.
bool pow2(float x) {
  if (!(x > 0.0f) || !std::isfinite(x)) return false;
  int e;
  const float m = std::frexp(x, &e);
  return m == 0.5f && x >= 1e-30f && x <= 1e30f;
}

// All n entries equal one power of two.
bool uniform_pow2(const float* a, int n, float* h) {
  for (int i = 1; i < n; ++i)
    if (a[i] != a[0]) return false;
  *h = a[0];
  return pow2(a[0]);
}

// Record the exact-reciprocal information of the spacings and dt (Spac).
void set_spacing_info(lesb_domain* h, const float* dx, const float* dy, const float* dz) {
  Spac& s = h->sp;
  s.dx1 = h->dx1;
  s.dy1 = h->dy1;
  s.dzn = h->dzn;
  float hx = 0, hy = 0, hz = 0;
  s.p2 = uniform_pow2(dx, h->g.im + 3, &hx) && uniform_pow2(dy, h->g.jm + 2, &hy) &&
         uniform_pow2(dz, h->g.km + 2, &hz);
  const float hs[3] = {hx, hy, hz};
  for (int a = 0; a < 3; ++a) {
    s.r1[a] = s.p2 ? 1.0f / hs[a] : 0.f;
    s.r2[a] = s.p2 ? 1.0f / (hs[a] + hs[a]) : 0.f;
    s.rsq[a] = s.p2 ? 1.0f / (hs[a] * hs[a]) : 0.f;
  }
  s.dtp2 = pow2(h->dt);
  s.rdt = s.dtp2 ? 1.0f / h->dt : 0.f;
}

// Exchange the face-buffer IPC handles of an NCCL slab with every rank (one
// all-gather, at the first solve: every rank takes it) and open the west /
// east neighbours' buffers.  All ranks run the same plan (same slab shape),
// so the ghost slots line up.  Returns false (and leaves the slab on the
// streaming path) when any step fails, e.g. without peer access.
void clear_graphs(lesb_domain* h);

// Collective: every rank shares a CUDA-IPC handle of `buf` (nullptr: it
// votes "no") with a signature, opens its west / east neighbours' buffers,
// and keeps them only when every rank mapped both of its neighbours (an
// all-reduce of the vote): a partial mapping would leave ranks on different
// exchange paths.
bool map_neighbour_bufs(lesb_domain* h, void* buf, long long sig, void** out_w, void** out_e) {
  const int nr = h->link.nranks, r = h->link.rank;
  struct Rec {
    cudaIpcMemHandle_t h;
    long long jm, km, sig, ok;
  } rec{};
  rec.ok = buf != nullptr && cudaIpcGetMemHandle(&rec.h, buf) == cudaSuccess;
  rec.jm = h->g.jm;
  rec.km = h->g.km;
  rec.sig = sig;
  *out_w = *out_e = nullptr;
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(Rec) * (nr + 1) + sizeof(int) * 2) != cudaSuccess) return false;
  std::vector<Rec> all(nr);
  int* flag = reinterpret_cast<int*>((char*)d + sizeof(Rec) * (nr + 1));
  bool ok = cudaMemcpy((char*)d + sizeof(Rec) * nr, &rec, sizeof(Rec), cudaMemcpyHostToDevice) == cudaSuccess &&
            ncclAllGather((char*)d + sizeof(Rec) * nr, d, sizeof(Rec), ncclChar, h->link.comm, h->st) == ncclSuccess &&
            cudaStreamSynchronize(h->st) == cudaSuccess &&
            cudaMemcpy(all.data(), d, sizeof(Rec) * nr, cudaMemcpyDeviceToHost) == cudaSuccess;
  for (int q = 0; ok && q < nr; ++q)
    ok = all[q].ok && all[q].jm == rec.jm && all[q].km == rec.km && all[q].sig == rec.sig;
  void* w = nullptr;
  void* e = nullptr;
  if (ok && r > 0) ok = cudaIpcOpenMemHandle(&w, all[r - 1].h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
  if (ok && r < nr - 1) ok = cudaIpcOpenMemHandle(&e, all[r + 1].h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
  int mine = ok ? 1 : 0, every = 0;
  const bool agreed = cudaMemcpy(flag, &mine, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
                      ncclAllReduce(flag, flag + 1, 1, ncclInt, ncclMin, h->link.comm, h->st) == ncclSuccess &&
                      cudaStreamSynchronize(h->st) == cudaSuccess &&
                      cudaMemcpy(&every, flag + 1, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
  cudaFree(d);
  if (!agreed || !every) {
    if (w) cudaIpcCloseMemHandle(w);
    if (e) cudaIpcCloseMemHandle(e);
    return false;
  }
  *out_w = w;
  *out_e = e;
  return true;
}

// Map the neighbours' exchange buffers of an NCCL slab at its first solve
// (every rank takes both handshakes): the resident solver's face buffers
// (one plan on every rank: same slab shape) and the streaming passes' ghost
// planes.
void map_slab_peers(lesb_domain* h) {
  void* w = nullptr;
  void* e = nullptr;
  const long long rsig = h->xbuf ? resident_xbuf_words(h->g, h->device) * 1000003LL + h->g.im : -1;
  if (map_neighbour_bufs(h, h->xbuf, rsig, &w, &e)) {
    h->peer_w = w;
    h->peer_e = e;
    h->peer_ready = true;
  }
  if (map_neighbour_bufs(h, h->ghost, split_geo(h->g).spi, &w, &e)) {
    h->gpeer_w = w;
    h->gpeer_e = e;
    h->ghost_ready = true;
  }
  clear_graphs(h);
}

int ensure_partials(lesb_domain* h, int n_iter) {
  int maxblk = std::max(std::max(sor_blocks_rb(h->g), sor_blocks_tw(h->g)),
                        std::max(resident_partials(h->g, h->device), sor_blocks_split(h->g)));
  if (tws_supported(h->g, h->sorc())) maxblk = std::max(maxblk, sor_blocks_tws(h->g));
  long long need = (long long)n_iter * 2 * maxblk + reduce_scratch(maxblk, n_iter);
  if (need > h->partials_cap) {
    if (h->partials) cudaFree(h->partials);
    h->partials = nullptr;
    CK(cudaMalloc(&h->partials, need * sizeof(double)));
    h->partials_cap = need;
  }
  if ((h->sor_path == 0 || h->sor_path == 2) && !h->xbuf && resident_supported(h->g, h->sorc(), h->device)) {
    const size_t xb = resident_xbuf_words(h->g, h->device) * sizeof(unsigned long long);
    CK(cudaMalloc(&h->xbuf, xb));
    CK(cudaMemset(h->xbuf, 0, xb));
    CK(cudaMalloc(&h->repoch, sizeof(unsigned)));
    CK(cudaMemset(h->repoch, 0, sizeof(unsigned)));
  }
  if ((h->link.comm || h->link.west || h->link.east) && !h->ghost && split_supported(h->g, h->sorc())) {
    const size_t gb = 8 * split_geo(h->g).spi * sizeof(unsigned long long);
    CK(cudaMalloc(&h->ghost, gb));
    CK(cudaMemset(h->ghost, 0, gb));
    CK(cudaMalloc(&h->gh_epoch, sizeof(unsigned)));
    CK(cudaMemset(h->gh_epoch, 0, sizeof(unsigned)));
  }
  if (h->link.comm && !h->peer_tried) {  // collective: every rank, whatever its own plan
    h->peer_tried = true;
    map_slab_peers(h);  // on failure the slab keeps the streaming colour passes
  }
  if (!h->split && h->sor_path != 3 && !h->resident_in_use() && split_supported(h->g, h->sorc())) {
    const size_t sb = 6 * split_geo(h->g).n * sizeof(float);
    CK(cudaMalloc(&h->split, sb));
    CK(cudaMemset(h->split, 0, sb));
  }
  if (n_iter > h->res_cap) {
    if (h->res_d) cudaFree(h->res_d);
    if (h->res_h) cudaFreeHost(h->res_h);
    h->res_d = nullptr;
    h->res_h = nullptr;
    CK(cudaMalloc(&h->res_d, n_iter * sizeof(double)));
    CK(cudaMallocHost(&h->res_h, n_iter * sizeof(double)));
    h->res_cap = n_iter;
  }
  return LESB_OK;
}

// A resident solve whose neighbour wait timed out leaves its tile flags set:
// clear them (and the error word) so the next solve starts clean.
int resident_timeout(lesb_domain* h) {
  cudaStreamSynchronize(h->st);
  if (h->xbuf) cudaMemset(h->xbuf, 0, resident_xbuf_words(h->g, h->device) * sizeof(unsigned long long));
  if (h->repoch) cudaMemset(h->repoch, 0, sizeof(unsigned));
  cudaMemset(&h->book_d->err, 0, sizeof(unsigned));
  cudaDeviceSynchronize();
  return fail(LESB_E_CUDA, "resident SOR: neighbour wait timed out");
}

// After a synchronous solve: report a resident-solver wait timeout.
int check_resident_err(lesb_domain* h) {
  unsigned e = 0;
  CK(cudaMemcpy(&e, &h->book_d->err, sizeof(unsigned), cudaMemcpyDeviceToHost));
  return e ? resident_timeout(h) : LESB_OK;
}

void clear_graphs(lesb_domain* h) {
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
  for (auto& kv : h->heads) cudaGraphDestroy(kv.second.first);
  h->heads.clear();
}

float* field_ptr(lesb_domain* h, int f) {
  switch (f) {
    case LESB_U: return h->u;
    case LESB_V: return h->v;
    case LESB_W: return h->w;
    case LESB_P: return h->p;
    case LESB_MASK: return h->mask;
    case LESB_FGH: return h->fgh;
    case LESB_FGH_OLD: return h->fgh_old;
    case LESB_RHS: return h->rhs;
    default: return nullptr;
  }
}

long long field_count(lesb_domain* h, int f) { return (f == LESB_FGH || f == LESB_FGH_OLD) ? 3 * h->n_py : h->n_py; }

// ---- x-slab halo exchange ----
// Halo planes are contiguous (jm+2)(km+2) runs.  The low halo (plane 0) takes
// the west neighbour's last interior plane; the high halo (planes im+1 ..
// im+depth) takes the east neighbour's first `depth` planes.  Velocities use
// depth 2 (velfg's shifted derivative at local i = im, les.py:100-110), the
// pressure depth 1.
ncclResult_t nccl_exchange(lesb_domain* h, float* f, int depth, cudaStream_t st, long long plane = 0) {
  const size_t si = plane ? (size_t)plane : (size_t)h->g.si;
  const int r = h->link.rank;
  ncclResult_t e = ncclGroupStart();
  if (e != ncclSuccess) return e;
  if (!h->g.west_bc) {
    ncclSend(f + si, depth * si, ncclFloat, r - 1, h->link.comm, st);
    ncclRecv(f, si, ncclFloat, r - 1, h->link.comm, st);
  }
  if (!h->g.east_bc) {
    ncclSend(f + (size_t)h->g.im * si, si, ncclFloat, r + 1, h->link.comm, st);
    ncclRecv(f + (size_t)(h->g.im + 1) * si, depth * si, ncclFloat, r + 1, h->link.comm, st);
  }
  return ncclGroupEnd();
}

// in-process neighbours: copy the neighbours' planes of field `which` into h
void local_exchange(lesb_domain* h, float* lesb_domain::*which, int depth, cudaStream_t st) {
  const size_t si = (size_t)h->g.si, fb = si * sizeof(float);
  float* f = h->*which;
  if (h->link.west) {
    const lesb_domain* w = h->link.west;
    cudaMemcpyAsync(f, w->*which + (size_t)w->g.im * si, fb, cudaMemcpyDeviceToDevice, st);
  }
  if (h->link.east) cudaMemcpyAsync(f + (size_t)(h->g.im + 1) * si, h->link.east->*which + si, depth * fb,
                                    cudaMemcpyDeviceToDevice, st);
}

void nccl_p_hook(void* ctx, float* p, long long plane) {
  lesb_domain* h = static_cast<lesb_domain*>(ctx);
  nccl_exchange(h, p, 1, h->st, plane);
}

// NCCL slabs: reductions over the ranks on the domain stream, synchronous
// (SURVEY 8(e) C4, C5).  coll_d: 2 ints of scratch.
int nccl_int_reduce(lesb_domain* h, int* v, ncclRedOp_t op) {
  // (the value in as a kernel argument and out through host-mapped memory:
  // no copy-engine work, which would queue behind asynchronous state copies)
  if (!h->coll_d) CK(cudaMalloc(&h->coll_d, 2 * sizeof(int)));
  if (!h->coll_h) CK(cudaMallocHost(&h->coll_h, sizeof(int)));
  k_set_word<<<1, 1, 0, h->st>>>(h->coll_d, *v);
  CK(cudaGetLastError());
  if (ncclAllReduce(h->coll_d, h->coll_d + 1, 1, ncclInt, op, h->link.comm, h->st) != ncclSuccess)
    return fail(LESB_E_CUDA, "ncclAllReduce (stage reduction) failed");
  k_word_out<<<1, 1, 0, h->st>>>(reinterpret_cast<unsigned*>(h->coll_h), reinterpret_cast<const unsigned*>(h->coll_d + 1));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->st));
  *v = *h->coll_h;
  return LESB_OK;
}

// C4: the residual history is the sum of the slabs' partial histories
// (in place on res_d; only when the caller asks for residuals -- inside a
// step nothing reads them)
int nccl_residuals(lesb_domain* h, int n_iter) {
  if (ncclAllReduce(h->res_d, h->res_d, n_iter, ncclDouble, ncclSum, h->link.comm, h->st) != ncclSuccess)
    return fail(LESB_E_CUDA, "ncclAllReduce (residuals) failed");
  return LESB_OK;
}

// in-process neighbours, one colour array of the split layout: planes 0 and
// im+1 of colour c take the neighbours' last / first interior planes
void local_exchange_split(lesb_domain* h, int c, cudaStream_t st) {
  const SplitGeo sg = split_geo(h->g);
  const size_t fb = sg.spi * sizeof(float);
  float* f = h->split + c * sg.n;
  if (h->link.west) {
    const lesb_domain* w = h->link.west;
    const SplitGeo sw = split_geo(w->g);
    cudaMemcpyAsync(f, w->split + c * sw.n + (size_t)w->g.im * sw.spi, fb, cudaMemcpyDeviceToDevice, st);
  }
  if (h->link.east)
    cudaMemcpyAsync(f + (size_t)(h->g.im + 1) * sg.spi, h->link.east->split + c * split_geo(h->link.east->g).n + sg.spi,
                    fb, cudaMemcpyDeviceToDevice, st);
}

// Enqueue the press stage on the stream: rhs = div(u)/dt, SOR, final halo.
cudaError_t enqueue_press(lesb_domain* h, int n_iter, int scheme, float omega, bool rhs_from_state,
                          unsigned* flags) {
  if (rhs_from_state) launch_divergence(h->g, h->spac(), h->u, h->v, h->w, h->rhs, h->dt, 1, h->st);
  ResidentBufs rb = h->rbufs();
  const bool res_slab = h->link.comm && rb.use && scheme == 0;  // resident solver exchanging through peer memory
  ExchangeHook hook{h->link.comm && !res_slab ? nccl_p_hook : nullptr, h};
  cudaError_t e = enqueue_sor(h->g, h->p, h->pb, h->rhs, h->sorc(), omega, n_iter, scheme, 1, h->partials, h->res_d,
                              flags, h->st, &hook, nullptr, &rb);
  if (e == cudaSuccess && res_slab) nccl_exchange(h, h->p, 1, h->st);  // inner x halo planes: the final values
  return e;
}

// The full step: velnw+bondv1 (A -> B), velfg+feedbf+les+adam+rhs (B -> A), press.
// With timing on, event records are captured between the phases:
// ev0 | velnw+bondv1 | ev1 | fused | ev2 | SOR passes | ev3 | halo + reduction | ev4
cudaError_t enqueue_step_body(lesb_domain* h, int n_iter, int scheme, float omega, StepBook* tail_book = nullptr,
                              bool* tail_done = nullptr) {
  unsigned* flags = &h->book_d->flags;
  auto mark = [&](int i) {
    if (h->timing) cudaEventRecordWithFlags(h->ev[i], h->st, cudaEventRecordExternal);
  };
  mark(0);
  launch_velnw_bondv1(h->g, h->spac(), h->u, h->v, h->w, h->p, h->fgh, h->dt, h->inflow_d, h->ub, h->vb, h->wb,
                      flags, h->st);
  if (h->link.comm) {  // x-slab: velocity halos after velnw + bondv1, one NCCL group
    ncclGroupStart();
    nccl_exchange(h, h->ub, 2, h->st);
    nccl_exchange(h, h->vb, 2, h->st);
    nccl_exchange(h, h->wb, 2, h->st);
    ncclGroupEnd();
  }
  mark(1);
  launch_fused_rhs(h->g, h->spac(), h->ub, h->vb, h->wb, h->mask, h->fgh, h->fgh_old, h->u, h->v, h->w, h->rhs,
                   h->vn, h->dt, h->cs != 0.0f, h->csd2, h->csd2s, flags, h->st);
  mark(2);
  SorMarks marks{h->timing ? h->ev[3] : nullptr};
  ResidentBufs rb = h->rbufs();
  const bool res_slab = h->link.comm && rb.use && scheme == 0;  // resident solver exchanging through peer memory
  if (!h->link.comm) {  // the solve ends the step: it may take over the bookkeeping
    rb.book = tail_book;
    rb.book_used = tail_done;
  }
  ExchangeHook hook{h->link.comm && !res_slab ? nccl_p_hook : nullptr, h};
  cudaError_t e = enqueue_sor(h->g, h->p, h->pb, h->rhs, h->sorc(), omega, n_iter, scheme, 1, h->partials,
                              h->res_d, flags, h->st, &hook, &marks, &rb);
  if (e == cudaSuccess && res_slab) nccl_exchange(h, h->p, 1, h->st);  // inner x halo planes: the final values
  mark(4);
  return e;
}

int get_graph(lesb_domain* h, int mode, int n_iter, int scheme, float omega, cudaGraphExec_t* out,
              cudaGraphNode_t* head = nullptr) {
  unsigned ob;
  std::memcpy(&ob, &omega, 4);
  auto key = std::make_tuple(mode | (h->timing ? 2 : 0), n_iter, scheme, ob);
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) {
    *out = it->second;
    if (head) {
      auto hn = h->heads.find(key);
      *head = hn == h->heads.end() ? nullptr : hn->second.second;
    }
    return LESB_OK;
  }
  const bool arg_head = mode == MODE_SYNC && inflow_by_arg(h->g.km);
  int rc = ensure_partials(h, n_iter);
  if (rc) return rc;
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  const int n_in = 3 * h->g.km, nt_in = std::min(1024, (n_in + 31) / 32 * 32);
  if (arg_head) {  // (its arguments are set before every launch: lesb_step)
    static const InflowArg zero{};
    k_step_head_arg<<<1, nt_in, 0, h->st>>>(h->inflow_d, zero, n_in, h->book_d);
  } else if (mode == MODE_SYNC) {
    // (every inflow word read in one round: host reads are slow under bulk copies)
    k_step_head<<<1, nt_in, 0, h->st>>>(h->inflow_d, h->inflow_h, n_in, h->book_d);
  }
  bool tail_done = false;
  cudaError_t body_err =
      enqueue_step_body(h, n_iter, scheme, omega, mode == MODE_ASYNC ? h->book_d : nullptr, &tail_done);
  if (mode == MODE_SYNC) {
    k_step_out<<<1, 256, 0, h->st>>>(h->res_h, h->res_d, n_iter, h->book_h, h->book_d);
  } else if (!tail_done) {
    k_step_tail<<<1, 32, 0, h->st>>>(h->book_d);
  }
  cudaError_t e = cudaStreamEndCapture(h->st, &graph);
  if (body_err != cudaSuccess) {
    if (e == cudaSuccess) cudaGraphDestroy(graph);
    cudaGetLastError();
    return fail(LESB_E_CUDA, std::string("step capture: ") + cudaGetErrorString(body_err));
  }
  if (e != cudaSuccess) return fail(LESB_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  cudaGraphNode_t head_node = nullptr;
  if (arg_head) {
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(graph, nodes.data(), &nn);
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      cudaKernelNodeParams kp;
      if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel &&
          cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func == (void*)k_step_head_arg) {
        head_node = nd;
        break;
      }
    }
    if (!head_node) {
      cudaGraphDestroy(graph);
      return fail(LESB_E_CUDA, "step capture: inflow node not found");
    }
  }
  cudaGraphExec_t exec;
  e = cudaGraphInstantiate(&exec, graph, 0);
  if (arg_head && e == cudaSuccess) h->heads[key] = {graph, head_node};
  else cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(LESB_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  h->graphs[key] = exec;
  *out = exec;
  if (head) *head = head_node;
  return LESB_OK;
}

// Full finiteness scan of the six state fields (les.py:387-390).
int scan_finite(lesb_domain* h, bool* ok) {
  CK(cudaMemsetAsync(&h->book_d->flags, 0, sizeof(unsigned), h->st));
  unsigned* fl = &h->book_d->flags;
  launch_check_finite(h->u, h->n_py, fl, 1, h->st);
  launch_check_finite(h->v, h->n_py, fl, 1, h->st);
  launch_check_finite(h->w, h->n_py, fl, 1, h->st);
  launch_check_finite(h->p, h->n_py, fl, 1, h->st);
  launch_check_finite(h->fgh, 3 * h->n_py, fl, 1, h->st);
  launch_check_finite(h->fgh_old, 3 * h->n_py, fl, 1, h->st);
  k_word_out<<<1, 1, 0, h->st>>>(&h->book_h->flags, fl);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->st));
  *ok = h->book_h->flags == 0;
  return LESB_OK;
}

int check_args_step(lesb_domain* h, int n_iter, int scheme) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  if (n_iter < 1) return fail(LESB_E_ARG, "n_iter must be >= 1");
  if (scheme != LESB_REDBLACK && scheme != LESB_TWINNED) return fail(LESB_E_ARG, "unknown scheme");
  if (!h->coeffs_set) return fail(LESB_E_STATE, "SOR coefficients not set (lesb_set_coeffs)");
  return LESB_OK;
}

// Reference behaviour when the state already holds a non-finite value: velnw
// runs and the check after it raises (velnw can never clear a non-finite).
int handle_dirty_state(lesb_domain* h, int* fail_stage, bool* failed) {
  *failed = false;
  bool ok = true;
  if (!h->known_finite) {
    int rc = scan_finite(h, &ok);
    if (rc) return rc;
  }
  // NCCL slabs decide together (a rank returning early would strand the
  // others' exchanges).  SPMD contract: every rank makes the same calls, so
  // known_finite -- made global after every step by the stage reduction --
  // is the same on every rank and they all reach this collective together.
  if (h->link.comm && !h->known_finite) {
    int bad = ok ? 0 : 1;
    int rc = nccl_int_reduce(h, &bad, ncclMax);
    if (rc) return rc;
    ok = bad == 0;
  }
  if (!ok) {
    launch_velnw(h->g, h->spac(), h->u, h->v, h->w, h->p, h->fgh, h->dt, h->st);
    CK(cudaStreamSynchronize(h->st));
    if (fail_stage) *fail_stage = LESB_STAGE_VELNW;
    *failed = true;
  }
  h->known_finite = ok;
  return LESB_OK;
}

}  // namespace

extern "C" {

const char* lesb_last_error(void) { return g_err.c_str(); }
int lesb_abi_version(void) { return LESB_ABI_VERSION; }

int lesb_create(const lesb_desc* d, lesb_handle* out) {
  if (!d || !out) return fail(LESB_E_ARG, "null argument");
  if (d->im < 1 || d->jm < 1 || d->km < 1) return fail(LESB_E_ARG, "grid dimensions must be >= 1");
  if (!d->dx1 || !d->dy1 || !d->dzn) return fail(LESB_E_ARG, "spacing arrays are required");
  auto* h = new lesb_domain();
  h->device = d->device;
  cudaError_t e = cudaSetDevice(d->device);
  if (e != cudaSuccess) {
    delete h;
    return fail(LESB_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  Geo& g = h->g;
  g.im = d->im;
  g.jm = d->jm;
  g.km = d->km;
  g.sj = d->km + 2;
  g.si = (long long)(d->jm + 2) * (d->km + 2);
  g.ioff = d->i_offset;
  g.west_bc = d->west_boundary ? 1 : 0;
  g.east_bc = d->east_boundary ? 1 : 0;
  h->n_py = (long long)(g.im + 2) * g.si;
  h->n_alloc = (long long)(g.im + 3) * g.si;
  h->dt = d->dt;
  h->vn = d->vn;
  h->cs = d->cs;
  h->csd2s = d->csd2_scalar;
  const size_t fb = h->n_alloc * sizeof(float);
  cudaError_t err = cudaSuccess;
  auto A = [&](float** ptr, size_t bytes) {
    if (err == cudaSuccess) err = cudaMalloc(ptr, bytes);
    if (err == cudaSuccess) err = cudaMemset(*ptr, 0, bytes);
  };
  A(&h->u, fb); A(&h->v, fb); A(&h->w, fb);
  A(&h->ub, fb); A(&h->vb, fb); A(&h->wb, fb);
  A(&h->p, fb); A(&h->pb, fb); A(&h->rhs, fb); A(&h->mask, fb);
  A(&h->fgh, 3 * fb); A(&h->fgh_old, 3 * fb);
  A(&h->dx1, (g.im + 3) * sizeof(float));
  A(&h->dy1, (g.jm + 2) * sizeof(float));
  A(&h->dzn, (g.km + 2) * sizeof(float));
  A(&h->inflow_d, 3 * g.km * sizeof(float));
  A(&h->scratch, h->n_int() * sizeof(float));
  if (err == cudaSuccess) err = cudaMalloc(&h->book_d, sizeof(StepBook));
  if (err == cudaSuccess) err = cudaMallocHost(&h->book_h, sizeof(StepBook));
  if (err == cudaSuccess) err = cudaMallocHost(&h->inflow_h, 3 * g.km * sizeof(float));
  if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaMemcpy(h->dx1, d->dx1, (g.im + 3) * sizeof(float), cudaMemcpyHostToDevice);
  if (err == cudaSuccess) err = cudaMemcpy(h->dy1, d->dy1, (g.jm + 2) * sizeof(float), cudaMemcpyHostToDevice);
  if (err == cudaSuccess) err = cudaMemcpy(h->dzn, d->dzn, (g.km + 2) * sizeof(float), cudaMemcpyHostToDevice);
  if (err == cudaSuccess) {
    StepBook b{0u, 0u, -1, 0u, 0u};
    err = cudaMemcpy(h->book_d, &b, sizeof(b), cudaMemcpyHostToDevice);
  }
  if (err == cudaSuccess && d->csd2) {
    err = cudaMalloc(&h->csd2, h->n_int() * sizeof(float));
    if (err == cudaSuccess)
      err = cudaMemcpy(h->csd2, d->csd2, h->n_int() * sizeof(float), cudaMemcpyHostToDevice);
  }
  if (err == cudaSuccess) set_spacing_info(h, d->dx1, d->dy1, d->dzn);
  if (err != cudaSuccess) {
    std::string m = std::string("lesb_create: ") + cudaGetErrorString(err);
    lesb_destroy(h);
    return fail(err == cudaErrorMemoryAllocation ? LESB_E_NOMEM : LESB_E_CUDA, m);
  }
  h->known_finite = true;  // all zero
  h->sor_path = g_default_sor_path >= 0 ? g_default_sor_path : default_sor_path();
  *out = h;
  return LESB_OK;
}

int lesb_destroy(lesb_handle h) {
  if (!h) return LESB_OK;
  cudaSetDevice(h->device);
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->peer_w) cudaIpcCloseMemHandle(h->peer_w);
  if (h->peer_e) cudaIpcCloseMemHandle(h->peer_e);
  if (h->link.comm) ncclCommDestroy(h->link.comm);
  if (h->link.west) h->link.west->link.east = nullptr;
  if (h->link.east) h->link.east->link.west = nullptr;
  clear_graphs(h);
  float* bufs[] = {h->u, h->v, h->w, h->ub, h->vb, h->wb, h->p, h->pb, h->rhs, h->mask, h->fgh, h->fgh_old,
                   h->dx1, h->dy1, h->dzn, h->inflow_d, h->scratch, h->csd2, h->cn1,
                   h->cn[0], h->cn[1], h->cn[2], h->cn[3], h->cn[4], h->cn[5]};
  for (float* b : bufs)
    if (b) cudaFree(b);
  if (h->partials) cudaFree(h->partials);
  if (h->xbuf) cudaFree(h->xbuf);
  if (h->repoch) cudaFree(h->repoch);
  if (h->gxbuf) cudaFree(h->gxbuf);
  if (h->gepoch) cudaFree(h->gepoch);
  if (h->split) cudaFree(h->split);
  if (h->coll_d) cudaFree(h->coll_d);
  if (h->coll_h) cudaFreeHost(h->coll_h);
  if (h->gpeer_w) cudaIpcCloseMemHandle(h->gpeer_w);
  if (h->gpeer_e) cudaIpcCloseMemHandle(h->gpeer_e);
  if (h->ghost) cudaFree(h->ghost);
  if (h->gh_epoch) cudaFree(h->gh_epoch);
  if (h->res_d) cudaFree(h->res_d);
  if (h->book_d) cudaFree(h->book_d);
  if (h->res_h) cudaFreeHost(h->res_h);
  if (h->book_h) cudaFreeHost(h->book_h);
  if (h->inflow_h) cudaFreeHost(h->inflow_h);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  if (h->up_st) cudaStreamSynchronize(h->up_st);
  if (h->dn_st) cudaStreamSynchronize(h->dn_st);
  for (int f = 0; f < 8; ++f) {
    if (h->staged[f]) cudaFree(h->staged[f]);
    if (h->snap[f]) cudaFree(h->snap[f]);
  }
  for (cudaEvent_t e : {h->ev_up, h->ev_commit, h->ev_snap})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_dn)
    if (e) cudaEventDestroy(e);
  if (h->up_st) cudaStreamDestroy(h->up_st);
  if (h->dn_st) cudaStreamDestroy(h->dn_st);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
  return LESB_OK;
}

int lesb_set_coeffs(lesb_handle h, const lesb_coeffs* c) {
  if (!h || !c) return fail(LESB_E_ARG, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  const Geo& g = h->g;
  const int lens[6] = {g.im, g.im, g.jm, g.jm, g.km, g.km};
  const float* src[6] = {c->cn2l, c->cn2s, c->cn3l, c->cn3s, c->cn4l, c->cn4s};
  h->cuni = 1;
  for (int a = 0; a < 6; ++a) {
    if (!src[a]) return fail(LESB_E_ARG, "cn2l/cn2s/cn3l/cn3s/cn4l/cn4s are required");
    h->cw[a] = src[a][0];
    for (int x = 1; x < lens[a]; ++x)
      if (std::memcmp(&src[a][x], &src[a][0], sizeof(float)) != 0) h->cuni = 0;
  }
  for (int a = 0; a < 6; ++a) {
    if (!src[a]) return fail(LESB_E_ARG, "cn2l/cn2s/cn3l/cn3s/cn4l/cn4s are required");
    if (!h->cn[a]) CK(cudaMalloc(&h->cn[a], lens[a] * sizeof(float)));
    CK(cudaMemcpy(h->cn[a], src[a], lens[a] * sizeof(float), cudaMemcpyHostToDevice));
  }
  if (c->cn1) {
    if (!h->cn1) CK(cudaMalloc(&h->cn1, h->n_int() * sizeof(float)));
    CK(cudaMemcpy(h->cn1, c->cn1, h->n_int() * sizeof(float), cudaMemcpyHostToDevice));
  } else if (h->cn1) {
    cudaFree(h->cn1);
    h->cn1 = nullptr;
  }
  h->cn1s = c->cn1_scalar;
  h->coeffs_set = true;
  clear_graphs(h);
  return LESB_OK;
}

int lesb_set_physics(lesb_handle h, float dt, float vn, float cs, const float* csd2, float csd2_scalar) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  h->dt = dt;
  h->vn = vn;
  h->cs = cs;
  h->csd2s = csd2_scalar;
  h->sp.dtp2 = pow2(dt);
  h->sp.rdt = h->sp.dtp2 ? 1.0f / dt : 0.f;
  if (csd2) {
    if (!h->csd2) CK(cudaMalloc(&h->csd2, h->n_int() * sizeof(float)));
    CK(cudaMemcpy(h->csd2, csd2, h->n_int() * sizeof(float), cudaMemcpyHostToDevice));
  } else if (h->csd2) {
    cudaFree(h->csd2);
    h->csd2 = nullptr;
  }
  clear_graphs(h);
  return LESB_OK;
}

int lesb_upload(lesb_handle h, int field, const float* host) {
  if (!h || !host) return fail(LESB_E_ARG, "null argument");
  float* d = field_ptr(h, field);
  if (!d) return fail(LESB_E_ARG, "unknown field id");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(d, host, field_count(h, field) * sizeof(float), cudaMemcpyHostToDevice));
  if (field != LESB_MASK && field != LESB_RHS) h->known_finite = false;
  return LESB_OK;
}

int lesb_download(lesb_handle h, int field, float* host) {
  if (!h || !host) return fail(LESB_E_ARG, "null argument");
  float* d = field_ptr(h, field);
  if (!d) return fail(LESB_E_ARG, "unknown field id");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(host, d, field_count(h, field) * sizeof(float), cudaMemcpyDeviceToHost));
  return LESB_OK;
}

// ---- asynchronous state copies ----
// The copies run on their own streams so they overlap the steps enqueued on
// `st`: a staged upload lands in a device staging buffer and becomes the
// state at lesb_stage_commit (a device-to-device copy ordered on `st`); an
// asynchronous download snapshots the field on `st` (device-to-device, so
// later steps may overwrite the field at once) and copies the snapshot to
// the host on the download stream.  Buffers are reused only after the copy
// that last read them (ev_commit / the field's ev_dn: one event for all
// fields would hold the domain stream until the previous field's download
// had finished).
static int ensure_copy_streams(lesb_domain* h) {
  if (h->up_st) return LESB_OK;
  CK(cudaStreamCreateWithFlags(&h->up_st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&h->dn_st, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&h->ev_up, &h->ev_commit, &h->ev_snap})
    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t& e : h->ev_dn) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const char* mb = std::getenv("LESB_COPY_CHUNK_MB");  // 0: every copy enqueued at once
  h->chunk_bytes = (size_t)((mb ? std::atof(mb) : 8.0) * (1 << 20));
  return LESB_OK;
}

static int enqueue_chunk(lesb_domain* h, bool up) {
  auto& q = up ? h->pend_up : h->pend_dn;
  size_t& i = up ? h->pu : h->pd;
  const lesb_domain::Chunk c = q[i++];
  if (i == q.size()) {
    q.clear();
    i = 0;
  }
  if (!c.dst) return LESB_OK;  // (superseded)
  CK(cudaMemcpyAsync(c.dst, c.src, c.bytes, up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                     up ? h->up_st : h->dn_st));
  if (!up && c.last) CK(cudaEventRecord(h->ev_dn[c.field], h->dn_st));
  return LESB_OK;
}

static int flush_copies(lesb_domain* h, bool up) {
  while (!(up ? h->pend_up : h->pend_dn).empty()) {
    int rc = enqueue_chunk(h, up);
    if (rc) return rc;
  }
  return LESB_OK;
}

// one chunk of each direction (after a step's launch)
static int pump_copies(lesb_domain* h) {
  for (bool up : {true, false}) {
    auto& q = up ? h->pend_up : h->pend_dn;
    size_t done = 0;
    while (!q.empty() && done < h->chunk_bytes) {
      done += q[up ? h->pu : h->pd].bytes;
      int rc = enqueue_chunk(h, up);
      if (rc) return rc;
    }
  }
  return LESB_OK;
}

static void split_copy(lesb_domain* h, bool up, void* dst, const void* src, size_t bytes, int field) {
  auto& q = up ? h->pend_up : h->pend_dn;
  const size_t cb = h->chunk_bytes ? h->chunk_bytes : bytes;
  for (size_t off = 0; off < bytes; off += cb) {
    const size_t n = std::min(cb, bytes - off);
    q.push_back({(char*)dst + off, (const char*)src + off, n, field, off + n == bytes});
  }
}

int lesb_stage_upload(lesb_handle h, int field, const float* host) {
  if (!h || !host) return fail(LESB_E_ARG, "null argument");
  if (!field_ptr(h, field)) return fail(LESB_E_ARG, "unknown field id");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  int rc = ensure_copy_streams(h);
  if (rc) return rc;
  const size_t bytes = field_count(h, field) * sizeof(float);
  if (!h->staged[field]) CK(cudaMalloc(&h->staged[field], bytes));
  CK(cudaStreamWaitEvent(h->up_st, h->ev_commit, 0));  // the last commit has read the staging buffer
  for (size_t q = h->pu; q < h->pend_up.size(); ++q)      // a pending copy into this buffer is superseded
    if (h->pend_up[q].field == field) h->pend_up[q].dst = nullptr;
  split_copy(h, true, h->staged[field], host, bytes, field);
  if (!h->chunk_bytes) rc = flush_copies(h, true);
  h->staged_mask |= 1u << field;
  return rc;
}

int lesb_stage_commit(lesb_handle h) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  if (!h->staged_mask) return LESB_OK;
  int rc = flush_copies(h, true);
  if (rc) return rc;
  CK(cudaEventRecord(h->ev_up, h->up_st));
  CK(cudaStreamWaitEvent(h->st, h->ev_up, 0));
  for (int f = 0; f < 8; ++f) {
    if (!(h->staged_mask & (1u << f))) continue;
    CK(copy_field(field_ptr(h, f), h->staged[f], field_count(h, f), h->device, h->st));
    if (f != LESB_MASK && f != LESB_RHS) h->known_finite = false;
  }
  CK(cudaEventRecord(h->ev_commit, h->st));
  h->staged_mask = 0;
  return LESB_OK;
}

int lesb_download_async(lesb_handle h, int field, float* host) {
  if (!h || !host) return fail(LESB_E_ARG, "null argument");
  float* d = field_ptr(h, field);
  if (!d) return fail(LESB_E_ARG, "unknown field id");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  int rc = ensure_copy_streams(h);
  if (rc) return rc;
  const size_t bytes = field_count(h, field) * sizeof(float);
  if (!h->snap[field]) CK(cudaMalloc(&h->snap[field], bytes));
  for (size_t q = h->pd; q < h->pend_dn.size(); ++q)  // this snapshot buffer still has copies pending
    if (h->pend_dn[q].field == field) {
      rc = flush_copies(h, false);
      if (rc) return rc;
      break;
    }
  CK(cudaStreamWaitEvent(h->st, h->ev_dn[field], 0));  // the last download has read this snapshot buffer
  CK(copy_field(h->snap[field], d, field_count(h, field), h->device, h->st));
  CK(cudaEventRecord(h->ev_snap, h->st));
  CK(cudaStreamWaitEvent(h->dn_st, h->ev_snap, 0));  // (ahead of every chunk queued from now on)
  split_copy(h, false, host, h->snap[field], bytes, field);
  if (!h->chunk_bytes) rc = flush_copies(h, false);
  return rc;
}

int lesb_copies_wait(lesb_handle h) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  for (bool up : {true, false}) {
    int rc = flush_copies(h, up);
    if (rc) return rc;
  }
  if (h->up_st) CK(cudaStreamSynchronize(h->up_st));
  if (h->dn_st) CK(cudaStreamSynchronize(h->dn_st));
  return LESB_OK;
}

void* lesb_device_ptr(lesb_handle h, int field) { return h ? (void*)field_ptr(h, field) : nullptr; }
void* lesb_stream(lesb_handle h) { return h ? (void*)h->st : nullptr; }

int lesb_synchronize(lesb_handle h) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  return LESB_OK;
}

int lesb_check_finite(lesb_handle h, int* all_finite) {
  if (!h || !all_finite) return fail(LESB_E_ARG, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  bool ok = false;
  int rc = scan_finite(h, &ok);
  if (rc) return rc;
  *all_finite = ok ? 1 : 0;
  h->known_finite = ok;
  return LESB_OK;
}

// ---- single stages ----
#define STAGE_PROLOGUE()                      \
  if (!h) return fail(LESB_E_ARG, "null handle"); \
  std::lock_guard<std::mutex> lk(h->mu);      \
  CK(cudaSetDevice(h->device));

#define STAGE_EPILOGUE()                      \
  CK(cudaGetLastError());                     \
  CK(cudaStreamSynchronize(h->st));           \
  h->known_finite = false;                    \
  return LESB_OK;

int lesb_velnw(lesb_handle h) {
  STAGE_PROLOGUE();
  launch_velnw(h->g, h->spac(), h->u, h->v, h->w, h->p, h->fgh, h->dt, h->st);
  STAGE_EPILOGUE();
}

int lesb_bondv1(lesb_handle h, const float* in_u, const float* in_v, const float* in_w) {
  STAGE_PROLOGUE();
  if (!in_u || !in_v || !in_w) return fail(LESB_E_ARG, "inflow arrays are required");
  const int km = h->g.km;
  std::memcpy(h->inflow_h, in_u, km * sizeof(float));
  std::memcpy(h->inflow_h + km, in_v, km * sizeof(float));
  std::memcpy(h->inflow_h + 2 * km, in_w, km * sizeof(float));
  CK(cudaMemcpyAsync(h->inflow_d, h->inflow_h, 3 * km * sizeof(float), cudaMemcpyHostToDevice, h->st));
  launch_bondv1(h->g, h->u, h->v, h->w, h->inflow_d, h->st);
  STAGE_EPILOGUE();
}

int lesb_velfg(lesb_handle h) {
  STAGE_PROLOGUE();
  launch_velfg(h->g, h->spac(), h->u, h->v, h->w, h->fgh, h->vn, h->st);
  STAGE_EPILOGUE();
}

int lesb_feedbf(lesb_handle h) {
  STAGE_PROLOGUE();
  launch_feedbf(h->g, h->u, h->v, h->w, h->fgh, h->mask, h->dt, h->st);
  STAGE_EPILOGUE();
}

int lesb_les_viscosity(lesb_handle h) {
  STAGE_PROLOGUE();
  if (h->cs != 0.0f) launch_les(h->g, h->spac(), h->u, h->v, h->w, h->fgh, h->csd2, h->csd2s, h->st);
  STAGE_EPILOGUE();
}

int lesb_adam(lesb_handle h) {
  STAGE_PROLOGUE();
  launch_adam(h->fgh, h->fgh_old, 3 * h->n_py, h->st);
  STAGE_EPILOGUE();
}

int lesb_divergence(lesb_handle h, float* out_host) {
  STAGE_PROLOGUE();
  if (!out_host) return fail(LESB_E_ARG, "null output");
  launch_divergence(h->g, h->spac(), h->u, h->v, h->w, h->scratch, 1.0f, 0, h->st);
  CK(cudaMemcpyAsync(out_host, h->scratch, h->n_int() * sizeof(float), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return LESB_OK;
}

int lesb_strain_magnitude(lesb_handle h, float* out_host) {
  STAGE_PROLOGUE();
  if (!out_host) return fail(LESB_E_ARG, "null output");
  launch_strain(h->g, h->spac(), h->u, h->v, h->w, h->scratch, h->st);
  CK(cudaMemcpyAsync(out_host, h->scratch, h->n_int() * sizeof(float), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return LESB_OK;
}

int lesb_press(lesb_handle h, int n_iter, int scheme, float omega, double* residuals_out) {
  NvtxRange nvtx_range_("lesb_press");
  int rc = check_args_step(h, n_iter, scheme);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  rc = ensure_partials(h, n_iter);
  if (rc) return rc;
  CK(enqueue_press(h, n_iter, scheme, omega, true, nullptr));
  CK(cudaGetLastError());
  if (residuals_out && h->link.comm) {
    rc = nccl_residuals(h, n_iter);
    if (rc) return rc;
  }
  if (residuals_out)
    CK(cudaMemcpyAsync(residuals_out, h->res_d, n_iter * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  rc = check_resident_err(h);
  if (rc) return rc;
  h->known_finite = false;
  return LESB_OK;
}

int lesb_sor_solve(lesb_handle h, int n_iter, int scheme, float omega, int halo_policy, double* residuals_out) {
  NvtxRange nvtx_range_("lesb_sor_solve");
  int rc = check_args_step(h, n_iter, scheme);
  if (rc) return rc;
  if (halo_policy != LESB_HALO_STORED && halo_policy != LESB_HALO_PRESS) return fail(LESB_E_ARG, "unknown halo policy");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  rc = ensure_partials(h, n_iter);
  if (rc) return rc;
  if (scheme == LESB_TWINNED)
    CK(cudaMemcpyAsync(h->pb, h->p, h->n_py * sizeof(float), cudaMemcpyDeviceToDevice, h->st));
  ResidentBufs rb = h->rbufs();
  const bool res_slab = h->link.comm && rb.use && scheme == LESB_REDBLACK;
  ExchangeHook hook{h->link.comm && !res_slab ? nccl_p_hook : nullptr, h};
  CK(enqueue_sor(h->g, h->p, h->pb, h->rhs, h->sorc(), omega, n_iter, scheme, halo_policy, h->partials, h->res_d,
                 nullptr, h->st, &hook, nullptr, &rb));
  if (res_slab) nccl_exchange(h, h->p, 1, h->st);  // inner x halo planes: the final values
  CK(cudaGetLastError());
  if (residuals_out && h->link.comm) {
    rc = nccl_residuals(h, n_iter);
    if (rc) return rc;
  }
  if (residuals_out)
    CK(cudaMemcpyAsync(residuals_out, h->res_d, n_iter * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  rc = check_resident_err(h);
  if (rc) return rc;
  h->known_finite = false;
  return LESB_OK;
}

// ---- the time step ----
int lesb_step(lesb_handle h, const float* in_u, const float* in_v, const float* in_w, int n_iter, int scheme,
              float omega, double* residuals_out, int* fail_stage) {
  NvtxRange nvtx_range_("lesb_step");
  int rc = check_args_step(h, n_iter, scheme);
  if (rc) return rc;
  if (!in_u || !in_v || !in_w) return fail(LESB_E_ARG, "inflow arrays are required");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  if (fail_stage) *fail_stage = -1;
  bool failed = false;
  rc = handle_dirty_state(h, fail_stage, &failed);
  if (rc) return rc;
  if (failed) return LESB_NONFINITE;
  cudaGraphExec_t ge;
  cudaGraphNode_t head = nullptr;
  rc = get_graph(h, MODE_SYNC, n_iter, scheme, omega, &ge, &head);
  if (rc) return rc;
  const int km = h->g.km;
  std::memcpy(h->inflow_h, in_u, km * sizeof(float));
  std::memcpy(h->inflow_h + km, in_v, km * sizeof(float));
  std::memcpy(h->inflow_h + 2 * km, in_w, km * sizeof(float));
  if (head) {  // the inflow as the head node's argument (no host read in the step)
    InflowArg arg;
    std::memcpy(arg.v, h->inflow_h, 3 * km * sizeof(float));
    int n_in = 3 * km;
    void* args[] = {&h->inflow_d, &arg, &n_in, &h->book_d};
    cudaKernelNodeParams kp = {};
    kp.func = (void*)k_step_head_arg;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(std::min(1024, (n_in + 31) / 32 * 32));
    kp.kernelParams = args;
    CK(cudaGraphExecKernelNodeSetParams(ge, head, &kp));
  }
  CK(cudaGraphLaunch(ge, h->st));
  if (h->up_st) {
    rc = pump_copies(h);
    if (rc) return rc;
  }
  CK(cudaStreamSynchronize(h->st));
  if (residuals_out && h->link.comm) {  // C4: the global residual history
    rc = nccl_residuals(h, n_iter);
    if (rc) return rc;
    k_step_out<<<1, 256, 0, h->st>>>(h->res_h, h->res_d, n_iter, h->book_h, h->book_d);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->st));
  }
  if (residuals_out) std::memcpy(residuals_out, h->res_h, n_iter * sizeof(double));
  if (h->book_h->err) return resident_timeout(h);
  int stage = h->book_h->flags ? first_stage(h->book_h->flags) : 99;
  if (h->link.comm) {  // C5: the first failing stage anywhere in the grid (step order), on every rank
    rc = nccl_int_reduce(h, &stage, ncclMin);
    if (rc) return rc;
  }
  if (stage < 99) {
    h->known_finite = false;
    if (fail_stage) *fail_stage = stage;
    return LESB_NONFINITE;
  }
  return LESB_OK;
}

int lesb_set_inflow(lesb_handle h, const float* in_u, const float* in_v, const float* in_w) {
  if (!h || !in_u || !in_v || !in_w) return fail(LESB_E_ARG, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  const int km = h->g.km;
  CK(cudaMemcpyAsync(h->inflow_d, in_u, km * sizeof(float), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->inflow_d + km, in_v, km * sizeof(float), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->inflow_d + 2 * km, in_w, km * sizeof(float), cudaMemcpyHostToDevice, h->st));
  return LESB_OK;
}

int lesb_step_async(lesb_handle h, int n_iter, int scheme, float omega) {
  NvtxRange nvtx_range_("lesb_step_async");
  int rc = check_args_step(h, n_iter, scheme);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  if (!h->known_finite) {
    bool failed = false;
    rc = handle_dirty_state(h, nullptr, &failed);
    if (rc) return rc;
    if (failed) return fail(LESB_E_STATE, "state holds non-finite values");
    StepBook b{0u, 0u, -1, 0u, 0u};
    CK(cudaMemcpyAsync(h->book_d, &b, sizeof(b), cudaMemcpyHostToDevice, h->st));
  }
  cudaGraphExec_t ge;
  rc = get_graph(h, MODE_ASYNC, n_iter, scheme, omega, &ge);
  if (rc) return rc;
  CK(cudaGraphLaunch(ge, h->st));
  return LESB_OK;
}

int lesb_poll_failure(lesb_handle h, int* steps_done, int* fail_step, int* fail_stage) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(h->book_h, h->book_d, sizeof(StepBook), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  const StepBook b = *h->book_h;
  if (steps_done) *steps_done = (int)b.steps;
  if (fail_step) *fail_step = b.fail_step;
  if (fail_stage) *fail_stage = b.fail_step >= 0 ? first_stage(b.fail_flags) : -1;
  if (b.err) return resident_timeout(h);
  // reset the counters for the next run
  StepBook z{0u, 0u, -1, 0u, 0u};
  CK(cudaMemcpyAsync(h->book_d, &z, sizeof(z), cudaMemcpyHostToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (b.fail_step >= 0) h->known_finite = false;
  return LESB_OK;
}

int lesb_run_steps(lesb_handle h, int n_steps, const float* inflow, int n_profiles, int n_iter, int scheme,
                   float omega, int* steps_done, int* fail_stage) {
  NvtxRange nvtx_range_("lesb_run_steps");
  if (!h || !inflow || n_profiles < 1 || n_steps < 0) return fail(LESB_E_ARG, "bad argument");
  int rc = check_args_step(h, n_iter, scheme);
  if (rc) return rc;
  const int km = h->g.km;
  float* prof_d = nullptr;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    CK(cudaSetDevice(h->device));
    CK(cudaMalloc(&prof_d, (size_t)n_profiles * 3 * km * sizeof(float)));
    CK(cudaMemcpyAsync(prof_d, inflow, (size_t)n_profiles * 3 * km * sizeof(float), cudaMemcpyHostToDevice,
                       h->st));
  }
  int done = 0;
  for (int s = 0; s < n_steps; ++s) {
    const int pi = s < n_profiles ? s : n_profiles - 1;
    if (s == 0 || n_profiles > 1) {
      std::lock_guard<std::mutex> lk(h->mu);
      CK(cudaMemcpyAsync(h->inflow_d, prof_d + (size_t)pi * 3 * km, 3 * km * sizeof(float),
                         cudaMemcpyDeviceToDevice, h->st));
    }
    rc = lesb_step_async(h, n_iter, scheme, omega);
    if (rc) {
      cudaFree(prof_d);
      return rc;
    }
  }
  int fstep = -1, fstage = -1;
  rc = lesb_poll_failure(h, &done, &fstep, &fstage);
  cudaFree(prof_d);
  if (rc) return rc;
  if (fstep >= 0) {
    if (steps_done) *steps_done = fstep;
    if (fail_stage) *fail_stage = fstage;
    return LESB_NONFINITE;
  }
  if (steps_done) *steps_done = done;
  if (fail_stage) *fail_stage = -1;
  return LESB_OK;
}

int lesb_copy_state(lesb_handle dst, lesb_handle src) {
  if (!dst || !src) return fail(LESB_E_ARG, "null handle");
  if (dst->n_alloc != src->n_alloc || dst->device != src->device) return fail(LESB_E_ARG, "domains differ");
  std::lock_guard<std::mutex> lk(dst->mu);
  CK(cudaSetDevice(dst->device));
  CK(cudaStreamSynchronize(src->st));
  const size_t fb = dst->n_alloc * sizeof(float);
  CK(cudaMemcpyAsync(dst->u, src->u, fb, cudaMemcpyDeviceToDevice, dst->st));
  CK(cudaMemcpyAsync(dst->v, src->v, fb, cudaMemcpyDeviceToDevice, dst->st));
  CK(cudaMemcpyAsync(dst->w, src->w, fb, cudaMemcpyDeviceToDevice, dst->st));
  CK(cudaMemcpyAsync(dst->p, src->p, fb, cudaMemcpyDeviceToDevice, dst->st));
  CK(cudaMemcpyAsync(dst->mask, src->mask, fb, cudaMemcpyDeviceToDevice, dst->st));
  CK(cudaMemcpyAsync(dst->fgh, src->fgh, 3 * fb, cudaMemcpyDeviceToDevice, dst->st));
  CK(cudaMemcpyAsync(dst->fgh_old, src->fgh_old, 3 * fb, cudaMemcpyDeviceToDevice, dst->st));
  dst->known_finite = src->known_finite;
  return LESB_OK;
}

int lesb_set_sor_path(lesb_handle h, int path) {
  if (!h || path < 0 || path > 3) return fail(LESB_E_ARG, "bad argument");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  h->sor_path = path;
  clear_graphs(h);
  return LESB_OK;
}

int lesb_set_default_sor_path(int path) {
  if (path < 0 || path > 3) return fail(LESB_E_ARG, "bad argument");
  g_default_sor_path = path;
  std::lock_guard<std::mutex> lk(g_solver_mu_fwd());
  for (auto& kv : solver_map()) lesb_set_sor_path(kv.second, path);
  return LESB_OK;
}

int lesb_sor_path_in_use(lesb_handle h, int scheme) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  if (scheme != LESB_REDBLACK || !h->coeffs_set) return 1;  // twinned: streaming sweeps
  const bool whole = h->g.west_bc && h->g.east_bc && h->g.ioff == 0;
  const bool res = (h->sor_path == 0 || h->sor_path == 2) && resident_supported(h->g, h->sorc(), h->device) &&
                   (whole || h->peer_ready);
  if (res) return 2;
  if (h->sor_path == 3 || !split_supported(h->g, h->sorc())) return 3;
  return 1;
}

int lesb_set_timing(lesb_handle h, int on) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  for (auto& e : h->ev)
    if (!e) CK(cudaEventCreate(&e));
  h->timing = on != 0;
  return LESB_OK;
}

int lesb_last_step_times(lesb_handle h, float* ms) {
  if (!h || !ms) return fail(LESB_E_ARG, "null argument");
  if (!h->timing) return fail(LESB_E_STATE, "timing is off (lesb_set_timing)");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  for (int i = 0; i < 4; ++i) CK(cudaEventElapsedTime(&ms[i], h->ev[i], h->ev[i + 1]));
  return LESB_OK;
}

int lesb_kernels_per_step(lesb_handle h, int n_iter, int scheme) {
  if (!h) return fail(LESB_E_ARG, "null handle");
  const int path = lesb_sor_path_in_use(h, scheme);
  // + the asynchronous step's bookkeeping kernel, unless the resident solver
  // ends the step and does it (single domain)
  const int tail = (path == 2 && !h->link.comm) ? 0 : 1;
  return 2 + sor_kernels_per_solve(h->g, h->sorc(), n_iter, scheme, 1, path == 2, path == 3) + tail;
}

// ---- solver on host buffers ----
}  // extern "C"

namespace {

// Solver domains for the host-buffer entry points, cached per (shape,
// device).  Cached domains are never destroyed while the library is loaded
// (a caller on another thread may hold one); once the cache holds
// kMaxSolvers shapes, further shapes get a private domain that the call
// destroys when it returns.
constexpr size_t kMaxSolvers = 8;

int get_solver(int im, int jm, int km, int device, lesb_domain** out, bool* owned) {
  std::lock_guard<std::mutex> lk(g_solver_mu_fwd());
  auto& g_solvers = solver_map();
  auto key = std::make_tuple(im, jm, km, device);
  auto it = g_solvers.find(key);
  *owned = false;
  if (it != g_solvers.end()) {
    *out = it->second;
    return LESB_OK;
  }
  std::vector<float> dx(im + 3, 1.f), dy(jm + 2, 1.f), dz(km + 2, 1.f);
  lesb_desc d{};
  d.im = im; d.jm = jm; d.km = km;
  d.west_boundary = 1; d.east_boundary = 1;
  d.dx1 = dx.data(); d.dy1 = dy.data(); d.dzn = dz.data();
  d.dt = 1.f; d.device = device;
  lesb_domain* h = nullptr;
  int rc = lesb_create(&d, &h);
  if (rc) return rc;
  if (g_solvers.size() < kMaxSolvers) g_solvers[key] = h;
  else *owned = true;
  *out = h;
  return LESB_OK;
}

// destroys a private (uncached) solver domain at scope exit
struct SolverLease {
  lesb_domain* h = nullptr;
  bool owned = false;
  ~SolverLease() {
    if (owned && h) lesb_destroy(h);
  }
};

int solver_prepare(int im, int jm, int km, const float* rhs, const lesb_coeffs* c, int device, SolverLease* out) {
  if (im < 1 || jm < 1 || km < 1) return fail(LESB_E_ARG, "grid dimensions must be >= 1");
  if (!rhs || !c) return fail(LESB_E_ARG, "null argument");
  int rc = get_solver(im, jm, km, device, &out->h, &out->owned);
  if (rc) return rc;
  rc = lesb_set_coeffs(out->h, c);
  if (rc) return rc;
  return lesb_upload(out->h, LESB_RHS, rhs);
}

}  // namespace

extern "C" {

int lesb_solve_pressure(int im, int jm, int km, const float* p0, const float* rhs, const lesb_coeffs* c,
                        float omega, int n_iter, int scheme, int halo_policy, float* p_out, double* residuals,
                        int device) {
  NvtxRange nvtx_range_("lesb_solve_pressure");
  if (n_iter < 1) return fail(LESB_E_ARG, "n_iter must be >= 1");
  if (scheme != LESB_REDBLACK && scheme != LESB_TWINNED) return fail(LESB_E_ARG, "unknown scheme");
  if (halo_policy != LESB_HALO_STORED && halo_policy != LESB_HALO_PRESS) return fail(LESB_E_ARG, "unknown halo policy");
  if (!p0 || !p_out) return fail(LESB_E_ARG, "null argument");
  SolverLease lease;
  int rc = solver_prepare(im, jm, km, rhs, c, device, &lease);
  if (rc) return rc;
  lesb_domain* h = lease.h;
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  rc = ensure_partials(h, n_iter);
  if (rc) return rc;
  const size_t bytes = h->n_py * sizeof(float);
  CK(cudaMemcpyAsync(h->p, p0, bytes, cudaMemcpyHostToDevice, h->st));
  if (scheme == LESB_TWINNED) CK(cudaMemcpyAsync(h->pb, h->p, bytes, cudaMemcpyDeviceToDevice, h->st));
  ResidentBufs rb = h->rbufs();
  CK(enqueue_sor(h->g, h->p, h->pb, h->rhs, h->sorc(), omega, n_iter, scheme, halo_policy, h->partials, h->res_d,
                 nullptr, h->st, nullptr, nullptr, &rb));
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(p_out, h->p, bytes, cudaMemcpyDeviceToHost, h->st));
  if (residuals) CK(cudaMemcpyAsync(residuals, h->res_d, n_iter * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return check_resident_err(h);
}

int lesb_redblack_iteration(int im, int jm, int km, float* p, const float* rhs, const lesb_coeffs* c, float omega,
                            int halo_policy, double* residual, int device) {
  return lesb_solve_pressure(im, jm, km, p, rhs, c, omega, 1, LESB_REDBLACK, halo_policy, p, residual, device);
}

int lesb_twinned_sweep(int im, int jm, int km, const float* src, float* dst, const float* rhs, const lesb_coeffs* c,
                       float omega, double* residual, int device) {
  if (!src || !dst) return fail(LESB_E_ARG, "null argument");
  SolverLease lease;
  int rc = solver_prepare(im, jm, km, rhs, c, device, &lease);
  if (rc) return rc;
  lesb_domain* h = lease.h;
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  rc = ensure_partials(h, 1);
  if (rc) return rc;
  const size_t bytes = h->n_py * sizeof(float);
  CK(cudaMemcpyAsync(h->p, src, bytes, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->pb, dst, bytes, cudaMemcpyHostToDevice, h->st));
  const int nblk = sor_blocks_tw(h->g);
  launch_tw_sweep(h->g, h->p, h->pb, h->rhs, h->sorc(), omega, 0, h->partials, h->st);
  // single-pass reduction: zero the second pass slot, reuse the 2-pass reducer
  CK(cudaMemsetAsync(h->partials + nblk, 0, nblk * sizeof(double), h->st));
  launch_reduce_res(h->partials, nblk, 1, h->res_d, h->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(dst, h->pb, bytes, cudaMemcpyDeviceToHost, h->st));
  if (residual) CK(cudaMemcpyAsync(residual, h->res_d, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return LESB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// x-slab decomposition
// ---------------------------------------------------------------------------
extern "C" {

int lesb_nccl_unique_id(void* out, int nbytes) {
  if (!out || nbytes < (int)sizeof(ncclUniqueId)) return fail(LESB_E_ARG, "unique-id buffer too small");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return fail(LESB_E_CUDA, "ncclGetUniqueId failed");
  std::memcpy(out, &id, sizeof(id));
  return (int)sizeof(ncclUniqueId);
}

int lesb_link_nccl(lesb_handle h, const void* id, int nranks, int rank) {
  if (!h || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(LESB_E_ARG, "bad argument");
  if ((rank > 0) == (bool)h->g.west_bc || (rank < nranks - 1) == (bool)h->g.east_bc)
    return fail(LESB_E_ARG, "slab boundaries do not match the rank's position");
  std::lock_guard<std::mutex> lk(h->mu);
  CK(cudaSetDevice(h->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  const ncclResult_t e = ncclCommInitRank(&comm, nranks, uid, rank);
  if (e != ncclSuccess) return fail(LESB_E_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(e));
  h->link.comm = comm;
  h->link.rank = rank;
  h->link.nranks = nranks;
  clear_graphs(h);
  return LESB_OK;
}

int lesb_link_local(lesb_handle* hs, int n) {
  if (!hs || n < 1) return fail(LESB_E_ARG, "bad argument");
  for (int s = 0; s < n; ++s) {
    if (!hs[s]) return fail(LESB_E_ARG, "null handle");
    if (hs[s]->device != hs[0]->device) return fail(LESB_E_ARG, "in-process slabs must share a device");
    if ((s > 0) == (bool)hs[s]->g.west_bc || (s < n - 1) == (bool)hs[s]->g.east_bc)
      return fail(LESB_E_ARG, "slab boundaries do not match the slab's position");
    if (s > 0 && (hs[s]->g.jm != hs[0]->g.jm || hs[s]->g.km != hs[0]->g.km ||
                  hs[s]->g.ioff != hs[s - 1]->g.ioff + hs[s - 1]->g.im))
      return fail(LESB_E_ARG, "slabs must tile the x axis in order");
    hs[s]->link.west = s > 0 ? hs[s - 1] : nullptr;
    hs[s]->link.east = s < n - 1 ? hs[s + 1] : nullptr;
  }
  return LESB_OK;
}

// The SOR solve of n in-process slabs on h0's stream (policy 1: press
// halo, 0: stored halo), residual histories left in each slab's res_h and
// flags in book_h (synchronised).  Red-black on slabs of one shape that fit:
// the resident solver for the whole group in one cooperative launch;
// otherwise the streaming passes (colour-split layout where supported) with
// a plane copy after every pass / sweep.
static int group_sor(lesb_domain** hs, int n, int n_iter, int scheme, float omega, int policy, cudaStream_t st) {
  lesb_domain* h0 = hs[0];
  // Red-black on slabs of one shape: the resident solver for the whole group
  // in one cooperative launch, tile faces crossing slab boundaries through
  // the neighbours' ghost slots (the in-process form of the NVLink peer path)
  bool group_res = scheme == LESB_REDBLACK && n <= resident_group_max() &&
                   (h0->sor_path == 0 || h0->sor_path == 2) && !std::getenv("LESB_GROUP_PASSES");
  for (int s = 0; s < n && group_res; ++s)
    group_res = hs[s]->g.im == h0->g.im && hs[s]->g.jm == h0->g.jm && hs[s]->g.km == h0->g.km &&
                resident_supported(hs[s]->g, hs[s]->sorc(), hs[s]->device, resident_group_tiles(n));
  if (group_res) {
    for (int s = 0; s < n; ++s) {
      lesb_domain* h = hs[s];
      if (!h->gxbuf) {
        const size_t xb = resident_xbuf_words(h->g, h->device, resident_group_tiles(n)) * sizeof(unsigned long long);
        CK(cudaMalloc(&h->gxbuf, xb));
        CK(cudaMemset(h->gxbuf, 0, xb));
        CK(cudaMalloc(&h->gepoch, sizeof(unsigned)));
        CK(cudaMemset(h->gepoch, 0, sizeof(unsigned)));
      }
    }
    std::vector<ResidentCall> calls(n);
    std::vector<SorC> cfs(n);
    for (int s = 0; s < n; ++s) {
      lesb_domain* h = hs[s];
      cfs[s] = h->sorc();
      calls[s] = ResidentCall{&h->g,        h->device,  h->p,        h->rhs,   &cfs[s],
                              omega,        n_iter,     policy,      h->gxbuf, h0->gepoch,
                              h->partials,  h->res_d,   &h->book_d->flags,     &h0->book_d->err,
                              s > 0 ? hs[s - 1]->gxbuf : nullptr, s < n - 1 ? hs[s + 1]->gxbuf : nullptr};
    }
    if (!std::getenv("LESB_GROUP_SEPARATE")) {
      CK(launch_sor_resident_group(n, calls.data(), st));
    } else {
      // Test form of the multi-GPU path: every slab its own cooperative launch
      // on its own stream with its own epoch, exchanging through the
      // neighbours' ghost slots -- as NCCL ranks do across GPUs (each launch
      // keeps num_SMs / n tiles so the n launches can be co-resident).
      cudaEvent_t ev_in;
      CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
      CK(cudaEventRecord(ev_in, st));
      std::vector<cudaEvent_t> ev_out(n);
      for (int s = 0; s < n; ++s) {
        lesb_domain* h = hs[s];
        calls[s].epoch = h->gepoch;
        calls[s].max_tiles = resident_group_tiles(n);
        CK(cudaStreamWaitEvent(h->st, ev_in, 0));
        CK(launch_sor_resident(calls[s], h->st));
        CK(cudaEventCreateWithFlags(&ev_out[s], cudaEventDisableTiming));
        CK(cudaEventRecord(ev_out[s], h->st));
      }
      for (int s = 0; s < n; ++s) {
        CK(cudaStreamWaitEvent(st, ev_out[s], 0));
        cudaEventDestroy(ev_out[s]);
      }
      cudaEventDestroy(ev_in);
    }
  }
  // streaming passes: the colour-split layout where every slab supports it
  bool split = !group_res && scheme == LESB_REDBLACK && h0->sor_path != 3;
  for (int s = 0; s < n && split; ++s) split = hs[s]->split && split_supported(hs[s]->g, hs[s]->sorc());
  // the plane exchange fused into the pass kernel through the slabs' ghost
  // planes (LESB_GHOST=0: a plane copy after every pass instead)
  std::vector<PassGhost> gh(n);
  bool ghosts = split && !(std::getenv("LESB_GHOST") && std::atoi(std::getenv("LESB_GHOST")) == 0);
  for (int s = 0; s < n && ghosts; ++s) ghosts = hs[s]->ghost && ghost_supported(hs[s]->g, n_iter);
  if (ghosts)
    for (int s = 0; s < n; ++s) {
      const long long sp = split_geo(hs[s]->g).spi;
      gh[s].my_w = s > 0 ? hs[s]->ghost : nullptr;
      gh[s].my_e = s < n - 1 ? hs[s]->ghost + 4 * sp : nullptr;
      gh[s].to_w = s > 0 ? hs[s - 1]->ghost + 4 * sp : nullptr;
      gh[s].to_e = s < n - 1 ? hs[s + 1]->ghost : nullptr;
      gh[s].epoch = hs[s]->gh_epoch;
      gh[s].err = &h0->book_d->err;
    }
  if (split)
    for (int s = 0; s < n; ++s) {
      launch_split_pack(hs[s]->g, hs[s]->p, hs[s]->rhs, hs[s]->split, policy, st);
      if (ghosts) launch_ghost_prologue(hs[s]->g, hs[s]->split, gh[s], st);
    }
  // With the fused exchange every slab runs its passes on its own stream,
  // nothing ordering the slabs but the ghost tags -- what one rank per GPU
  // does (the in-process test form of the multi-GPU path), and the slabs'
  // half-size kernels then fill the device together (600x300x90 on two
  // slabs: +4% over one domain, +39% serialised on one stream).
  // LESB_GROUP_STREAMS=0 serialises them on the first slab's stream.
  const bool sep = ghosts && !(std::getenv("LESB_GROUP_STREAMS") && std::atoi(std::getenv("LESB_GROUP_STREAMS")) == 0);
  if (sep) {
    cudaEvent_t ev_in;
    CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    CK(cudaEventRecord(ev_in, st));
    std::vector<cudaEvent_t> ev_out(n);
    for (int s = 0; s < n; ++s) {
      lesb_domain* h = hs[s];
      CK(cudaStreamWaitEvent(h->st, ev_in, 0));
      const int nblk = sor_blocks_split(h->g);
      for (int it = 0; it < n_iter; ++it)
        for (int nrd = 0; nrd < 2; ++nrd) {
          PassGhost gp = gh[s];
          gp.pass = 2 * it + nrd;
          launch_rbs_pass(h->g, h->split, h->sorc(), omega, nrd, policy,
                          h->partials + ((long long)it * 2 + nrd) * nblk, h->st, &gp);
        }
      CK(cudaEventCreateWithFlags(&ev_out[s], cudaEventDisableTiming));
      CK(cudaEventRecord(ev_out[s], h->st));
    }
    for (int s = 0; s < n; ++s) {
      CK(cudaStreamWaitEvent(st, ev_out[s], 0));
      cudaEventDestroy(ev_out[s]);
    }
    cudaEventDestroy(ev_in);
  }
  for (int it = 0; it < (group_res || sep ? 0 : n_iter); ++it) {
    for (int nrd = 0; nrd < 2; ++nrd) {
      for (int s = 0; s < n; ++s) {
        lesb_domain* h = hs[s];
        const int nblk = split ? sor_blocks_split(h->g)
                               : (scheme == LESB_REDBLACK ? sor_blocks_rb(h->g) : sor_blocks_tw(h->g));
        double* part = h->partials + ((long long)it * 2 + nrd) * nblk;
        if (split) {
          PassGhost gp = gh[s];
          gp.pass = 2 * it + nrd;
          launch_rbs_pass(h->g, h->split, h->sorc(), omega, nrd, policy, part, st, ghosts ? &gp : nullptr);
        } else if (scheme == LESB_REDBLACK) {
          launch_rb_pass(h->g, h->p, h->rhs, h->sorc(), omega, nrd, policy, part, st);
        } else {
          launch_tw_sweep(h->g, nrd == 0 ? h->p : h->pb, nrd == 0 ? h->pb : h->p, h->rhs, h->sorc(), omega, policy,
                          part, st);
        }
      }
      for (int s = 0; s < n; ++s) {
        if (ghosts) continue;  // the pass kernels exchanged their edge planes themselves
        if (split) local_exchange_split(hs[s], nrd, st);
        else local_exchange(hs[s], (scheme == LESB_TWINNED && nrd == 0) ? &lesb_domain::pb : &lesb_domain::p, 1, st);
      }
    }
  }
  for (int s = 0; s < n; ++s) {
    if (split) launch_split_unpack(hs[s]->g, hs[s]->split, hs[s]->p, policy, &hs[s]->book_d->flags, st);
    else if (policy == 1) launch_press_halo(hs[s]->g, hs[s]->p, &hs[s]->book_d->flags, st);
  }
  for (int s = 0; s < n; ++s) local_exchange(hs[s], &lesb_domain::p, 1, st);
  for (int s = 0; s < n; ++s) {
    lesb_domain* h = hs[s];
    if (!group_res)  // (the resident solver reduces its residuals itself)
      launch_reduce_res(h->partials,
                        split ? sor_blocks_split(h->g)
                              : (scheme == LESB_REDBLACK ? sor_blocks_rb(h->g) : sor_blocks_tw(h->g)),
                        n_iter, h->res_d, st);
    CK(cudaMemcpyAsync(h->res_h, h->res_d, n_iter * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&h->book_h->flags, &h->book_d->flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  if (group_res) {  // a neighbour wait that timed out: reset the group's face buffers and report
    unsigned e = 0;
    CK(cudaMemcpy(&e, &h0->book_d->err, sizeof(unsigned), cudaMemcpyDeviceToHost));
    if (e) {
      for (int s = 0; s < n; ++s) {
        cudaMemset(hs[s]->gxbuf, 0, resident_xbuf_words(hs[s]->g, hs[s]->device, resident_group_tiles(n)) * 8);
        cudaMemset(hs[s]->gepoch, 0, sizeof(unsigned));
      }
      cudaMemset(&h0->book_d->err, 0, sizeof(unsigned));
      cudaDeviceSynchronize();
      return fail(LESB_E_CUDA, "resident SOR (slab group): neighbour wait timed out");
    }
  }
  return LESB_OK;
}

// One step of n in-process slabs, all enqueued on the first slab's stream:
// each phase runs on every slab before the halo planes move.  Red-black and
// twinned use the streaming kernels (the resident / fused solvers need the
// whole grid).  Results equal one domain's step bitwise; residuals (summed
// over slabs in order) agree to summation-order tolerance.
int lesb_group_step(lesb_handle* hs, int n, const float* in_u, const float* in_v, const float* in_w, int n_iter,
                    int scheme, float omega, double* residuals_out, int* fail_stage) {
  NvtxRange nvtx_range_("lesb_group_step");
  if (!hs || n < 1 || !in_u || !in_v || !in_w) return fail(LESB_E_ARG, "bad argument");
  for (int s = 0; s < n; ++s) {
    int rc = check_args_step(hs[s], n_iter, scheme);
    if (rc) return rc;
  }
  lesb_domain* h0 = hs[0];
  CK(cudaSetDevice(h0->device));
  cudaStream_t st = h0->st;
  for (int s = 0; s < n; ++s) {
    lesb_domain* h = hs[s];
    CK(cudaStreamSynchronize(h->st));
    int rc = ensure_partials(h, n_iter);
    if (rc) return rc;
    const int km = h->g.km;
    std::memcpy(h->inflow_h, in_u, km * sizeof(float));
    std::memcpy(h->inflow_h + km, in_v, km * sizeof(float));
    std::memcpy(h->inflow_h + 2 * km, in_w, km * sizeof(float));
    CK(cudaMemcpyAsync(h->inflow_d, h->inflow_h, 3 * km * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(&h->book_d->flags, 0, sizeof(unsigned), st));
  }
  for (int s = 0; s < n; ++s) {
    lesb_domain* h = hs[s];
    launch_velnw_bondv1(h->g, h->spac(), h->u, h->v, h->w, h->p, h->fgh, h->dt, h->inflow_d, h->ub, h->vb, h->wb,
                        &h->book_d->flags, st);
  }
  for (int s = 0; s < n; ++s) {
    local_exchange(hs[s], &lesb_domain::ub, 2, st);
    local_exchange(hs[s], &lesb_domain::vb, 2, st);
    local_exchange(hs[s], &lesb_domain::wb, 2, st);
  }
  for (int s = 0; s < n; ++s) {
    lesb_domain* h = hs[s];
    launch_fused_rhs(h->g, h->spac(), h->ub, h->vb, h->wb, h->mask, h->fgh, h->fgh_old, h->u, h->v, h->w, h->rhs,
                     h->vn, h->dt, h->cs != 0.0f, h->csd2, h->csd2s, &h->book_d->flags, st);
    if (scheme == LESB_TWINNED)
      CK(cudaMemcpyAsync(h->pb, h->p, h->n_py * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  int rc = group_sor(hs, n, n_iter, scheme, omega, 1, st);
  if (rc) return rc;
  unsigned bits = 0;
  for (int s = 0; s < n; ++s) {
    bits |= hs[s]->book_h->flags;
    hs[s]->known_finite = false;
  }
  if (residuals_out)
    for (int it = 0; it < n_iter; ++it) {
      double t = 0.0;
      for (int s = 0; s < n; ++s) t += hs[s]->res_h[it];
      residuals_out[it] = t;
    }
  if (fail_stage) *fail_stage = bits ? first_stage(bits) : -1;
  return bits ? LESB_NONFINITE : LESB_OK;
}

// solve_pressure (sor.py:255-309) on n in-process slabs: p and rhs are
// the slabs' own buffers (lesb_upload of LESB_P / LESB_RHS); the residual
// history is the sum of the slabs' histories, in slab order.
int lesb_group_sor_solve(lesb_handle* hs, int n, int n_iter, int scheme, float omega, int halo_policy,
                         double* residuals_out) {
  NvtxRange nvtx_range_("lesb_group_sor_solve");
  if (!hs || n < 1) return fail(LESB_E_ARG, "bad argument");
  if (halo_policy != LESB_HALO_STORED && halo_policy != LESB_HALO_PRESS) return fail(LESB_E_ARG, "unknown halo policy");
  for (int s = 0; s < n; ++s) {
    int rc = check_args_step(hs[s], n_iter, scheme);
    if (rc) return rc;
  }
  lesb_domain* h0 = hs[0];
  CK(cudaSetDevice(h0->device));
  cudaStream_t st = h0->st;
  for (int s = 0; s < n; ++s) {
    lesb_domain* h = hs[s];
    CK(cudaStreamSynchronize(h->st));
    int rc = ensure_partials(h, n_iter);
    if (rc) return rc;
    CK(cudaMemsetAsync(&h->book_d->flags, 0, sizeof(unsigned), st));
    if (scheme == LESB_TWINNED)
      CK(cudaMemcpyAsync(h->pb, h->p, h->n_py * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  int rc = group_sor(hs, n, n_iter, scheme, omega, halo_policy, st);
  if (rc) return rc;
  for (int s = 0; s < n; ++s) hs[s]->known_finite = false;
  if (residuals_out)
    for (int it = 0; it < n_iter; ++it) {
      double t = 0.0;
      for (int s = 0; s < n; ++s) t += hs[s]->res_h[it];
      residuals_out[it] = t;
    }
  return LESB_OK;
}

}  // extern "C"

/* ---------------------------------------------------------------------------
 * Boundary-range launch geometry (sor.py:312-349, cli.py:286-320)
 * ------------------------------------------------------------------------- */
int lesb_boundary_decode(int ip, int jp, int kp, long long gid0, long long n, int* face, int* c0, int* c1) {
  using namespace lesb;
  if (ip < 1 || jp < 1 || kp < 1) return fail(LESB_E_ARG, "ip, jp, kp must be >= 1");
  if (gid0 < 0) return fail(LESB_E_ARG, "gid must be >= 0");
  if (n < 0 || (n > 0 && (!face || !c0 || !c1))) return fail(LESB_E_ARG, "output arrays are required");
  if (n == 0) return LESB_OK;
  int* d = nullptr;
  CK(cudaMalloc(&d, 3 * n * sizeof(int)));
  cudaError_t e = launch_boundary_decode(gid0, n, ip, jp, kp, d, d + n, d + 2 * n, 0);
  if (e == cudaSuccess) e = cudaMemcpy(face, d, n * sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(c0, d + n, n * sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(c1, d + 2 * n, n * sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LESB_E_CUDA, std::string("boundary decode: ") + cudaGetErrorString(e));
  return LESB_OK;
}

int lesb_boundary_audit(int ip, int jp, int kp, int nthreads, int nunits, long long* stats) {
  using namespace lesb;
  if (ip < 1 || jp < 1 || kp < 1) return fail(LESB_E_ARG, "ip, jp, kp must be >= 1");
  if (nthreads < 1 || nunits < 1) return fail(LESB_E_ARG, "nthreads and nunits must be >= 1");
  if (nthreads > 1024) return fail(LESB_E_ARG, "nthreads must be <= 1024 (one launch block)");
  if (!stats) return fail(LESB_E_ARG, "stats array is required");
  const long long br = boundary_range(ip, jp, kp);
  const long long pr = padded_range(br, nthreads, nunits);
  unsigned* hits = nullptr;
  unsigned long long* buf = nullptr;  // stats[5], first[3]
  CK(cudaMalloc(&hits, br * sizeof(unsigned)));
  cudaError_t e = cudaMalloc(&buf, 8 * sizeof(unsigned long long));
  unsigned long long hb[8] = {0, 0, 0, 0, 0, ~0ull, ~0ull, ~0ull};
  if (e == cudaSuccess) e = cudaMemset(hits, 0, br * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemcpy(buf, hb, sizeof hb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_boundary_audit(ip, jp, kp, nthreads, nunits, hits, buf, buf + 5, 0);
  if (e == cudaSuccess) e = cudaMemcpy(hb, buf, sizeof hb, cudaMemcpyDeviceToHost);
  cudaFree(hits);
  cudaFree(buf);
  if (e != cudaSuccess) return fail(LESB_E_CUDA, std::string("boundary audit: ") + cudaGetErrorString(e));
  stats[0] = br;
  stats[1] = pr;
  stats[2] = (long long)hb[0];  // in-range gids decoded to padding
  stats[3] = (long long)hb[1];  // padding gids that escaped the guard
  stats[4] = (long long)hb[2];  // points covered exactly once
  stats[5] = (long long)hb[3];  // points covered more than once
  stats[6] = (long long)hb[4];  // points never covered
  const unsigned long long f0 = hb[5] < hb[6] ? hb[5] : hb[6];
  stats[7] = f0 == ~0ull ? -1 : (long long)f0;  // smallest violating gid
  return LESB_OK;
}

int lesb_boundp_faces(lesb_handle h) {
  STAGE_PROLOGUE();
  launch_boundp_faces(h->g, h->p, h->st);
  STAGE_EPILOGUE();
}

