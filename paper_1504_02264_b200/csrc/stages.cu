// Stage kernels of the DPRI-LES step (reference: gmcf_mini/les.py).
//
// Two families:
//  * in-place single-stage kernels, one per reference stage function, used by
//    the per-stage API (les.velnw(state), ...);
//  * the two fused kernels of the time step:
//      k_velnw_bondv1 : velnw + bondv1 over the whole array, A -> B buffers
//      k_fused_rhs    : velfg + feedbf + les + adam + divergence/dt, B -> A
//    Each computes, per cell, the value the reference holds after every stage
//    it covers, and raises that stage's non-finite bit when the value is not
//    finite (les.py:384-390 semantics, checked inductively: all six fields are
//    finite when a step starts).
#include <cstdlib>

#include "lesb_common.cuh"
#include "lesb_kernels.h"
#include "stages_dev.cuh"

namespace lesb {

// ---------------------------------------------------------------------------
// finiteness of a whole buffer (les.py:387-390)
// ---------------------------------------------------------------------------
__global__ void k_check_finite(const float* __restrict__ a, long long n, unsigned* flags, unsigned bit) {
  unsigned bits = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    if (!finite32(a[t])) bits = bit;
  flag_or(flags, bits);
}

// ---------------------------------------------------------------------------
// host-side launch helpers
// ---------------------------------------------------------------------------
static void box_launch(int nk, int nj, int ni, dim3& grid, dim3& block) {
  int bx = ((nk + 31) / 32) * 32;
  if (bx > 128) bx = 128;
  int by = 256 / bx;
  block = dim3(bx, by, 1);
  grid = dim3((nk + bx - 1) / bx, (nj + by - 1) / by, ni);
}

void launch_velnw(const Geo& g, const Spac& s, float* u, float* v, float* w, const float* p, const float* fgh,
                  float dt, cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km + 1, g.jm + 1, g.im + 1, gr, bl);
  k_velnw_inplace<<<gr, bl, 0, st>>>(g, s, u, v, w, p, fgh, dt);
}

void launch_bondv1(const Geo& g, float* u, float* v, float* w, const float* inflow, cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km + 2, g.jm + 2, g.im + 2, gr, bl);
  k_bondv1_inplace<<<gr, bl, 0, st>>>(g, u, v, w, inflow);
}

void launch_velnw_bondv1(const Geo& g, const Spac& s, const float* u, const float* v, const float* w,
                         const float* p, const float* fgh, float dt, const float* inflow, float* ub, float* vb,
                         float* wb, unsigned* flags, cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km + 2, g.jm + 2, g.im + 2, gr, bl);
  if (cudaKernel_t k = jit_stage_kernel(JIT_VELNW_BONDV1, g, s.p2)) {  // this geometry as constants (jit.cu)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = gr;
    cfg.blockDim = bl;
    cfg.stream = st;
    Geo ga = g;
    Spac sa = s;
    void* args[] = {&ga, &sa, &u, &v, &w, &p, &fgh, &dt, &inflow, &ub, &vb, &wb, &flags};
    cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), args);
    return;
  }
  if (s.p2) k_velnw_bondv1<true><<<gr, bl, 0, st>>>(g, s, u, v, w, p, fgh, dt, inflow, ub, vb, wb, flags);
  else k_velnw_bondv1<false><<<gr, bl, 0, st>>>(g, s, u, v, w, p, fgh, dt, inflow, ub, vb, wb, flags);
}

void launch_velfg(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* fgh,
                  float vn, cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km, g.jm, g.im, gr, bl);
  k_velfg<<<gr, bl, 0, st>>>(g, s, u, v, w, fgh, vn);
}

void launch_feedbf(const Geo& g, float* u, float* v, float* w, float* fgh, const float* mask, float dt,
                   cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km, g.jm, g.im, gr, bl);
  k_feedbf<<<gr, bl, 0, st>>>(g, u, v, w, fgh, mask, dt);
}

void launch_les(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* fgh,
                const float* csd2f, float csd2s, cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km, g.jm, g.im, gr, bl);
  k_les<<<gr, bl, 0, st>>>(g, s, u, v, w, fgh, csd2f, csd2s);
}

void launch_strain(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* out,
                   cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km, g.jm, g.im, gr, bl);
  k_strain<<<gr, bl, 0, st>>>(g, s, u, v, w, out);
}

void launch_adam(float* fgh, float* fgh_old, long long n, cudaStream_t st) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_adam<<<(unsigned)blocks, 256, 0, st>>>(fgh, fgh_old, n);
}

void launch_divergence(const Geo& g, const Spac& s, const float* u, const float* v, const float* w, float* out,
                       float dt, int to_rhs, cudaStream_t st) {
  dim3 gr, bl;
  box_launch(g.km, g.jm, g.im, gr, bl);
  k_divergence<<<gr, bl, 0, st>>>(g, s, u, v, w, out, dt, to_rhs);
}

void launch_fused_rhs(const Geo& g, const Spac& s, const float* ub, const float* vb, const float* wb,
                      const float* mask, float* fgh, float* fgh_old, float* ua, float* va, float* wa, float* rhs,
                      float vn, float dt, int do_les, const float* csd2f, float csd2s, unsigned* flags,
                      cudaStream_t st) {
  // one-warp-wide blocks, 4 rows: measured fastest on B200 for 150x150x90
  // (64.0 us vs 73.7 us for 96x2 blocks; the kernel is latency bound and
  // small blocks retire without waiting on a slow sibling warp)
  const dim3 bl(32, 4, 1);
  const dim3 gr((g.km + 2 + 31) / 32, (g.jm + 2 + 3) / 4, g.im + 2);
  // programmatic dependent launch after velnw + bondv1 (LESB_STEP_PDL=0: plain)
  static const bool pdl = !(std::getenv("LESB_STEP_PDL") && std::atoi(std::getenv("LESB_STEP_PDL")) == 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = gr;
  cfg.blockDim = bl;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (cudaKernel_t k = jit_stage_kernel(JIT_FUSED_RHS, g, s.p2)) {  // this geometry as constants (jit.cu)
    Geo ga = g;
    Spac sa = s;
    void* args[] = {&ga, &sa, &ub, &vb, &wb, &mask, &fgh, &fgh_old, &ua, &va, &wa, &rhs, &vn, &dt, &do_les,
                    &csd2f, &csd2s, &flags};
    cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), args);
    return;
  }
  if (s.p2)
    cudaLaunchKernelEx(&cfg, k_fused_rhs<true>, g, s, ub, vb, wb, mask, fgh, fgh_old, ua, va, wa, rhs, vn, dt, do_les,
                       csd2f, csd2s, flags);
  else
    cudaLaunchKernelEx(&cfg, k_fused_rhs<false>, g, s, ub, vb, wb, mask, fgh, fgh_old, ua, va, wa, rhs, vn, dt,
                       do_les, csd2f, csd2s, flags);
}

void launch_check_finite(const float* a, long long n, unsigned* flags, unsigned bit, cudaStream_t st) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_check_finite<<<(unsigned)blocks, 256, 0, st>>>(a, n, flags, bit);
}

}  // namespace lesb
