// Host-side launchers of the B200 DPRI-LES kernels (internal interface).
#pragma once

#include <cuda_runtime.h>

#include "lesb_common.cuh"

namespace lesb {

// Called after every SOR pass / sweep and after the final halo
// materialisation with the freshly written pressure buffer (x-slab halo
// exchange for multi-GPU runs; unused on one GPU).
// plane: floats per x plane of the buffer (natural p: Geo::si; one colour
// array of the split layout: SplitGeo::spi).
struct ExchangeHook {
  void (*fn)(void* ctx, float* p, long long plane);
  void* ctx;
};

// Colour-split layout of p / rhs for the streaming red-black solver
// (sor_split.cu): per colour (im+2) x (jm+2) rows of khp slots.
struct SplitGeo {
  int khp;        // slots per row: ceil((km+2)/2) rounded up to a multiple of 4
  int kh4;        // khp / 4
  long long spi;  // floats per x plane of one colour array: (jm+2) * khp
  long long n;    // floats per colour array: (im+2) * spi
};

// Optional event recorded after the last SOR pass (stage timing).
struct SorMarks {
  cudaEvent_t after_passes;
};

// Buffers of the shared-memory-resident red-black solver (sor_resident.cu);
// use == 0 forces the streaming kernels.
// Streaming passes on x-slabs: the plane exchange fused into the pass
// kernel (sor_split.cu).  Each slab keeps two ghost planes (from the west,
// from the east) of 4 slots x SplitGeo::spi (value, tag) 64-bit words; the
// tiles of a slab's edge planes write their new values straight into the
// neighbour's ghost slot of the pass (peer memory over NVLink across GPUs)
// and read their own ghost slot of the neighbour's previous pass, spinning
// on the tag -- no copy and no collective between passes.
struct PassGhost {
  unsigned long long* my_w = nullptr;  // ghost planes from the west neighbour [4][spi], or nullptr (physical face)
  unsigned long long* my_e = nullptr;  // from the east neighbour
  unsigned long long* to_w = nullptr;  // the west neighbour's my_e (peer memory on another GPU)
  unsigned long long* to_e = nullptr;  // the east neighbour's my_w
  unsigned* epoch = nullptr;           // solve counter of this slab (launch_ghost_epoch), tags are unique per solve
  unsigned* err = nullptr;             // set when a wait times out
  int pass = 0;                        // pass of the solve (0 .. 2 n_iter - 1)
  int sys = 0;                         // the neighbours are on other GPUs: system-scope accesses
  bool on() const { return my_w || my_e; }
};

struct ResidentBufs {
  int use;
  int device;
  int natural;       // streaming passes on the natural layout (k_sor_rb) instead of the split one
  void* xbuf;        // resident_xbuf_words() 64-bit words, zero-initialised
  unsigned* epoch;   // one word, zero-initialised
  unsigned* err;
  void* peer_w = nullptr;  // x-slab: neighbour slabs' face buffers (peer memory)
  void* peer_e = nullptr;
  // asynchronous step: the resident solver, the step's last kernel, also does
  // the end-of-step bookkeeping (*book_used is set when it took it over)
  StepBook* book = nullptr;
  bool* book_used = nullptr;
  float* split = nullptr;  // 6 * SplitGeo::n floats: p (colour 0, 1), rhs (colour 0, 1), p' (twinned ping-pong)
  PassGhost ghost;         // x-slab streaming passes: fused plane exchange (ghost.on())
};

// stages.cu
void launch_velnw(const Geo& g, const Spac& s, float* u, float* v, float* w, const float* p, const float* fgh,
                  float dt, cudaStream_t st);
void launch_bondv1(const Geo& g, float* u, float* v, float* w, const float* inflow, cudaStream_t st);
void launch_velnw_bondv1(const Geo& g, const Spac& s, const float* u, const float* v, const float* w,
                         const float* p, const float* fgh, float dt, const float* inflow, float* ub, float* vb,
                         float* wb, unsigned* flags, cudaStream_t st);
void launch_velfg(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* fgh,
                  float vn, cudaStream_t st);
void launch_feedbf(const Geo& g, float* u, float* v, float* w, float* fgh, const float* mask, float dt,
                   cudaStream_t st);
void launch_les(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* fgh,
                const float* csd2f, float csd2s, cudaStream_t st);
void launch_strain(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* out,
                   cudaStream_t st);
void launch_adam(float* fgh, float* fgh_old, long long n, cudaStream_t st);
void launch_divergence(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* out,
                       float dt, int to_rhs, cudaStream_t st);
void launch_fused_rhs(const Geo& g, const Spac& s, const float* ub, const float* vb, const float* wb,
                      const float* mask, float* fgh, float* fgh_old, float* ua, float* va, float* wa, float* rhs,
                      float vn, float dt, int do_les, const float* csd2f, float csd2s, unsigned* flags,
                      cudaStream_t st);
void launch_check_finite(const float* a, long long n, unsigned* flags, unsigned bit, cudaStream_t st);

// Runtime-specialised step kernels (jit.cu): the kernel compiled with this
// geometry as constants, or nullptr (small domain, LESB_JIT=0, no NVRTC) --
// then the ahead-of-time kernel runs.
enum { JIT_VELNW_BONDV1 = 0, JIT_FUSED_RHS = 1 };
bool jit_enabled(const Geo& g);
cudaKernel_t jit_stage_kernel(int kind, const Geo& g, int p2);
struct ResPlan;
// the resident solver with this geometry and tile plan as constants, or nullptr
cudaKernel_t jit_resident_kernel(const Geo& g, const ResPlan& pl, bool press, bool slab);

// sor.cu
int sor_blocks_rb(const Geo& g);
int sor_blocks_tw(const Geo& g);
void launch_rb_pass(const Geo& g, float* p, const float* rhs, const SorC& cf, float om, int nrd, int policy,
                    double* partials, cudaStream_t st);
void launch_tw_sweep(const Geo& g, const float* src, float* dst, const float* rhs, const SorC& cf, float om,
                     int policy, double* partials, cudaStream_t st);
void launch_press_halo(const Geo& g, float* p, unsigned* flags, cudaStream_t st);
void launch_press_halo_copy(const Geo& g, const float* src, float* dst, unsigned* flags, cudaStream_t st);
void launch_reduce_res(const double* partials, int nblk, int n_iter, double* out, cudaStream_t st);
int reduce_scratch(int nblk, int n_iter);  // extra doubles launch_reduce_res needs after the partials
int sor_kernels_per_solve(const Geo& g, const SorC& cf, int n_iter, int scheme, int policy, bool resident,
                          bool natural);
cudaError_t enqueue_sor(const Geo& g, float* p, float* pb, const float* rhs, const SorC& cf, float om, int n_iter,
                        int scheme, int policy, double* partials, double* res_dev, unsigned* flags, cudaStream_t st,
                        const ExchangeHook* hook, const SorMarks* marks, const ResidentBufs* res = nullptr);

// sor_split.cu
SplitGeo split_geo(const Geo& g);
bool split_supported(const Geo& g, const SorC& cf);
int sor_blocks_split(const Geo& g);
// p_copy: a second destination of the split p (the twinned sweeps' second buffer)
void launch_split_pack(const Geo& g, const float* p, const float* rhs, float* split, int policy, cudaStream_t st,
                       float* p_copy = nullptr);
void launch_rbs_pass(const Geo& g, float* split, const SorC& cf, float om, int c, int policy, double* partials,
                     cudaStream_t st, const PassGhost* gh = nullptr);
// before the passes of a solve: bump the slab's epoch, then publish its
// initial colour-1 edge planes (what the neighbours' pass 0 reads)
void launch_ghost_prologue(const Geo& g, const float* split, const PassGhost& gh, cudaStream_t st);
bool ghost_supported(const Geo& g, int n_iter);
// twinned sweeps on the colour-split layout (single domains): src -> dst, both colours
bool tws_supported(const Geo& g, const SorC& cf);
int sor_blocks_tws(const Geo& g);
void launch_tws_sweep(const Geo& g, const float* src, float* dst, const float* rhs_split, const SorC& cf, float om,
                      int policy, double* partials, cudaStream_t st);
void launch_split_unpack(const Geo& g, const float* split, float* p, int policy, unsigned* flags, cudaStream_t st);

// sor_resident.cu
// max_tiles: 0 for every SM (one domain or one slab per GPU); num_SMs / n for
// a group of n in-process slabs launched together
bool resident_supported(const Geo& g, const SorC& cf, int device, int max_tiles = 0);
int resident_ntiles(const Geo& g, int device, int max_tiles = 0);
int resident_partials(const Geo& g, int device, int max_tiles = 0);  // per-pass residual partials
long long resident_xbuf_words(const Geo& g, int device, int max_tiles = 0);
struct ResidentCall {
  const Geo* g;
  int device;
  float* p;
  const float* rhs;
  const SorC* cf;
  float om;
  int n_iter, policy;
  void* xbuf;
  unsigned* epoch;
  double* partials;
  double* res;
  unsigned* pflags;
  unsigned* err;
  void* peer_w;  // x-slab neighbours' face buffers (another GPU's, mapped), or nullptr
  void* peer_e;
  int max_tiles = 0;  // tiles of the plan (0: every SM); slabs sharing a device use num_SMs / n
  StepBook* book = nullptr;  // single domain: end-of-step bookkeeping after the solve (ResidentBufs::book)
};
cudaError_t launch_sor_resident(const ResidentCall& c, cudaStream_t st);
cudaError_t launch_sor_resident_group(int n, const ResidentCall* cs, cudaStream_t st);
int resident_group_max();
int resident_group_tiles(int n);  // tiles per slab when n slabs share one launch

// boundary.cu: boundary-range launch geometry (sor.py:312-349)
long long boundary_range(int ip, int jp, int kp);
long long padded_range(long long range, int nthreads, int nunits);
cudaError_t launch_boundary_decode(long long gid0, long long n, int ip, int jp, int kp, int* face, int* c0, int* c1,
                                   cudaStream_t st);
cudaError_t launch_boundary_audit(int ip, int jp, int kp, int nthreads, int nunits, unsigned* hits,
                                  unsigned long long* stats, unsigned long long* first, cudaStream_t st);
void launch_boundp_faces(const Geo& g, float* p, cudaStream_t st);

}  // namespace lesb
