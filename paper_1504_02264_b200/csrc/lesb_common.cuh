// Shared device-side definitions for the B200 DPRI-LES kernels.
//
// Bitwise parity with the numpy reference rests on three rules (SURVEY
// Appendix A): every float op rounds once (compiled with -fmad=false, no
// fast-math, IEEE div/sqrt), operations are evaluated in the reference's
// order, and boundary values are read through the closed-form halo maps of
// SURVEY Appendix B.
#pragma once

#ifndef __CUDACC_RTC__  // (NVRTC, jit.cu: the device types are built in)
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace lesb {

// Stage bits for the non-finite flag word (les.py:401-409 order).
enum : unsigned {
  F_VELNW = 1u << 0, F_BONDV1 = 1u << 1, F_VELFG = 1u << 2, F_FEEDBF = 1u << 3,
  F_LES = 1u << 4, F_ADAM = 1u << 5, F_PRESS = 1u << 6
};

// Geometry of one (slab) domain.  Device arrays are (im+3, jm+2, km+2): the
// extra high-x plane holds the depth-2 velocity halo an x-slab needs for the
// shifted derivative at local i = im (les.py:100-110).
struct Geo {
  int im, jm, km;
  int sj;            // km + 2
  long long si;      // (jm + 2) * (km + 2)
  int ioff;          // global i = local i + ioff
  int west_bc;       // local i = 0 plane is the physical west face
  int east_bc;       // local i = im+1 plane is the physical east face
};

struct Spac {
  const float* dx1;  // im + 3
  const float* dy1;  // jm + 2
  const float* dzn;  // km + 2
  // p2 != 0: every spacing of each axis equals one power of two h_a.  Every
  // divisor on the path is then a power of two (h, 2h, h*h, and dt when
  // dtp2), and x / 2^n == x * 2^-n exactly (both are the correctly rounded
  // value of the same real number), so the kernels multiply by these exact
  // reciprocals instead of dividing: bitwise identical, far fewer instructions.
  int p2;
  float r1[3], r2[3], rsq[3];  // 1/h, 1/(2h), 1/(h*h) per axis
  int dtp2;
  float rdt;                   // 1/dt
};

struct SorC {
  const float* cn1;  // im*jm*km (interior, C order) or nullptr -> cn1s
  float cn1s;
  const float *cn2l, *cn2s, *cn3l, *cn3s, *cn4l, *cn4s;
  // uni != 0: every entry of each neighbour-weight vector equals the scalar
  // below (build_uniform_coeffs, sor.py:121-137), so kernels may use them.
  int uni;
  float w2l, w2s, w3l, w3s, w4l, w4s;
};

__device__ __forceinline__ bool finite32(float x) {
  return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}

__device__ __forceinline__ long long cidx(const Geo& g, int i, int j, int k) {
  return (long long)i * g.si + (long long)j * g.sj + k;
}

// OR the per-thread stage bits into the flag word: one atomic per warp at most.
// All 32 lanes of every warp must call this (kernels never return early).
// One atomic per warp that has a bit to add -- and none once the word holds
// them all: a field that went non-finite everywhere must not turn every warp
// of a whole-array kernel into an atomic on one address.
__device__ __forceinline__ void flag_or(unsigned* flags, unsigned bits) {
  unsigned any = __reduce_or_sync(0xffffffffu, bits);
  unsigned tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  if (any && (tid & 31u) == 0 && (*(volatile unsigned*)flags & any) != any) atomicOr(flags, any);
}

// Deterministic block reduction of a double (fixed shuffle tree, fixed warp order).
template <int NWARPS>
__device__ __forceinline__ double block_sum(double v, double* smem) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  int lane = (threadIdx.x + threadIdx.y * blockDim.x) & 31;
  int wid = (threadIdx.x + threadIdx.y * blockDim.x) >> 5;
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = (lane < NWARPS) ? smem[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// device-side step bookkeeping for asynchronous runs (capi.cu)
struct StepBook {
  unsigned flags;       // stage bits of the current (or first failing) step
  unsigned steps;       // steps enqueued and completed on the device
  int fail_step;        // -1 while no step failed
  unsigned fail_flags;  // stage bits of the first failing step
  unsigned err;         // device-side solver error (neighbour wait timed out)
};

// the end-of-step update (one thread, after every stage's flags are final)
__device__ __forceinline__ void step_book_update(StepBook* b) {
  if (b->flags && b->fail_step < 0) {
    b->fail_step = (int)b->steps;
    b->fail_flags = b->flags;
  }
  b->steps += 1;
}


// The geometry a step kernel works with: its launch parameter, or in a
// runtime-specialised build the same values as constants, so every neighbour
// offset folds into the load instructions (the ahead-of-time kernels spend a
// tenth of their instructions on 64-bit address arithmetic).
__device__ __forceinline__ Geo jit_geo(const Geo& g_in) {
  Geo g = g_in;
#ifdef LESB_JIT_IM
  g.im = LESB_JIT_IM;
  g.jm = LESB_JIT_JM;
  g.km = LESB_JIT_KM;
  g.sj = LESB_JIT_KM + 2;
  g.si = (long long)(LESB_JIT_JM + 2) * (LESB_JIT_KM + 2);
#endif
  return g;
}

}  // namespace lesb
