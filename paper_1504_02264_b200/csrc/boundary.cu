// Boundary-range launch geometry (reference: gmcf_mini/sor.py:312-349, the
// paper's §2.4 one-launch enumeration of the three boundary face families,
// PAPER.md:292-341) on the device, and the pressure face refresh (boundp,
// les.py:341-355) launched over it.
//
// A global id gid in [0, boundary_range) decodes, exactly as
// map_boundary_gid does (sor.py:319-338), to one point of
//   YZ: (j, k) = (gid % jp, gid / jp),              gid < jp*kp
//   ZX: (k, i) = (r / ip, r % ip),  r = gid - jp*kp, r < kp*ip
//   XY: (j, i) = (r / ip, r % ip),  r = ... - kp*ip, r < jp*ip
// and every gid at or beyond the range (the padding up to a multiple of
// nthreads * nunits, padded_range sor.py:341-349) takes the guarded branch.
//
// The face refresh touches the face-interior halo cells only -- exactly the
// cells the 6-point SOR stencil reads.  For those cells the reference's
// sequential slice assignments (x faces, then y, then z) reduce to one copy
// from an interior cell (or a constant 0), so the parallel launch is exact.
// Edges and corners are not in the three families; the time step keeps the
// closed-form whole-array halo kernels, which also materialise them.
#include "lesb_common.cuh"
#include "lesb_kernels.h"

namespace lesb {

// face: 0 YZ, 1 ZX, 2 XY, -1 padding (Face enum order of sor.py:34-37)
__device__ __forceinline__ int decode_gid(long long gid, int ip, int jp, int kp, int& a, int& b) {
  const long long n_yz = (long long)jp * kp, n_zx = (long long)kp * ip, n_xy = (long long)jp * ip;
  if (gid < n_yz) {
    a = (int)(gid % jp);
    b = (int)(gid / jp);
    return 0;
  }
  if (gid < n_yz + n_zx) {
    const long long r = gid - n_yz;
    a = (int)(r / ip);
    b = (int)(r % ip);
    return 1;
  }
  if (gid < n_yz + n_zx + n_xy) {
    const long long r = gid - n_yz - n_zx;
    a = (int)(r / ip);
    b = (int)(r % ip);
    return 2;
  }
  return -1;
}

__global__ void k_boundary_decode(long long gid0, long long n, int ip, int jp, int kp, int* face, int* c0, int* c1) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int a = -1, b = -1;
  const int f = decode_gid(gid0 + t, ip, jp, kp, a, b);
  face[t] = f;
  c0[t] = f < 0 ? -1 : a;
  c1[t] = f < 0 ? -1 : b;
}

// The audit launch: blocks of nthreads threads, each thread nunits gids
// (gid = (block * nunits + u) * nthreads + thread), over the padded range.
// hits[p] counts the gids decoding to boundary point p; stats[0] counts
// in-range gids that fell into padding, stats[1] padding gids that escaped
// the guard; first[0] / first[1] keep the smallest such gid.
__global__ void k_boundary_audit(int ip, int jp, int kp, int nunits, long long br, unsigned* hits,
                                 unsigned long long* stats, unsigned long long* first) {
  for (int u = 0; u < nunits; ++u) {
    const long long gid = ((long long)blockIdx.x * nunits + u) * blockDim.x + threadIdx.x;
    int a, b;
    const int f = decode_gid(gid, ip, jp, kp, a, b);
    if (gid < br) {
      if (f < 0) {
        atomicAdd(&stats[0], 1ull);
        atomicMin(&first[0], (unsigned long long)gid);
        continue;
      }
      // point index: YZ (j, k) -> k jp + j; ZX (k, i) -> jp kp + k ip + i; XY (j, i) -> ... + j ip + i
      const long long p = f == 0 ? (long long)b * jp + a
                          : f == 1 ? (long long)jp * kp + (long long)a * ip + b
                                   : (long long)jp * kp + (long long)kp * ip + (long long)a * ip + b;
      atomicAdd(&hits[p], 1u);
    } else if (f >= 0) {
      atomicAdd(&stats[1], 1ull);
      atomicMin(&first[1], (unsigned long long)gid);
    }
  }
}

// stats[2] points hit exactly once, stats[3] points hit more than once,
// stats[4] points never hit; first[2] smallest repeated point
__global__ void k_boundary_count(const unsigned* hits, long long br, unsigned long long* stats,
                                 unsigned long long* first) {
  unsigned long long once = 0, dup = 0, miss = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < br; p += (long long)gridDim.x * blockDim.x) {
    const unsigned h = hits[p];
    if (h == 1) ++once;
    else if (h == 0) ++miss;
    else {
      ++dup;
      atomicMin(&first[2], (unsigned long long)p);
    }
  }
  if (once) atomicAdd(&stats[2], once);
  if (dup) atomicAdd(&stats[3], dup);
  if (miss) atomicAdd(&stats[4], miss);
}

// boundp over the face families (les.py:341-355 on face-interior cells):
//   YZ (j, k): p[0] = p[1] (physical west), p[im+1] = 0 (physical east)
//   ZX (k, i): p[i, 0] = p[i, jm], p[i, jm+1] = p[i, 1]
//   XY (j, i): p[i, j, 0] = p[i, j, 1], p[i, j, km+1] = 0
__global__ void k_boundp_faces(Geo g, float* __restrict__ p) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int a, b;
  const int f = decode_gid(gid, g.im, g.jm, g.km, a, b);
  if (f < 0) return;  // the padding branch
  if (f == 0) {
    const int j = a + 1, k = b + 1;
    if (g.west_bc) p[cidx(g, 0, j, k)] = p[cidx(g, 1, j, k)];
    if (g.east_bc) p[cidx(g, g.im + 1, j, k)] = 0.0f;
  } else if (f == 1) {
    const int k = a + 1, i = b + 1;
    p[cidx(g, i, 0, k)] = p[cidx(g, i, g.jm, k)];
    p[cidx(g, i, g.jm + 1, k)] = p[cidx(g, i, 1, k)];
  } else {
    const int j = a + 1, i = b + 1;
    p[cidx(g, i, j, 0)] = p[cidx(g, i, j, 1)];
    p[cidx(g, i, j, g.km + 1)] = 0.0f;
  }
}

long long boundary_range(int ip, int jp, int kp) {
  return (long long)jp * kp + (long long)kp * ip + (long long)jp * ip;
}

long long padded_range(long long range, int nthreads, int nunits) {
  const long long m = (long long)nthreads * nunits;
  const long long rem = range % m;
  return rem == 0 ? range : range + (m - rem);
}

cudaError_t launch_boundary_decode(long long gid0, long long n, int ip, int jp, int kp, int* face, int* c0, int* c1,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_boundary_decode<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gid0, n, ip, jp, kp, face, c0, c1);
  return cudaGetLastError();
}

cudaError_t launch_boundary_audit(int ip, int jp, int kp, int nthreads, int nunits, unsigned* hits,
                                  unsigned long long* stats, unsigned long long* first, cudaStream_t st) {
  const long long br = boundary_range(ip, jp, kp);
  const long long pr = padded_range(br, nthreads, nunits);
  const long long nblk = pr / ((long long)nthreads * nunits);
  if (nblk > 0) k_boundary_audit<<<(unsigned)nblk, nthreads, 0, st>>>(ip, jp, kp, nunits, br, hits, stats, first);
  k_boundary_count<<<148, 256, 0, st>>>(hits, br, stats, first);
  return cudaGetLastError();
}

void launch_boundp_faces(const Geo& g, float* p, cudaStream_t st) {
  // one launch over padded_range(boundary_range, 256, 1)
  const long long pr = padded_range(boundary_range(g.im, g.jm, g.km), 256, 1);
  k_boundp_faces<<<(unsigned)(pr / 256), 256, 0, st>>>(g, p);
}

}  // namespace lesb
