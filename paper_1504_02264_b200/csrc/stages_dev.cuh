// Device code of the step's stage kernels (reference: gmcf_mini/les.py),
// shared by the ahead-of-time build (stages.cu) and the runtime-specialised
// build (jit.cu: NVRTC compiles this header with the domain's geometry as
// compile-time constants, LESB_JIT_IM / _JM / _KM; LESB_JIT leaves out the
// per-stage kernels, which are not specialised).
#pragma once

#include "lesb_common.cuh"

namespace lesb {


// ---------------------------------------------------------------------------
// velnw point updates (les.py:226-241):  f + dt*(fgh_a - ((p[+a]-p)*2)/(s[n]+s[n+1]))
// ---------------------------------------------------------------------------
template <bool P2 = false>
__device__ __forceinline__ float velnw_u(const Geo& g, const Spac& s, const float* u, const float* p,
                                         const float* fgh, float dt, long long c, int i) {
  const float num = (p[c + g.si] - p[c]) * 2.0f;
  const float gx = P2 ? num * s.r2[0] : num / (s.dx1[i] + s.dx1[i + 1]);
  return u[c] + dt * (fgh[3 * c + 0] - gx);
}
template <bool P2 = false>
__device__ __forceinline__ float velnw_v(const Geo& g, const Spac& s, const float* v, const float* p,
                                         const float* fgh, float dt, long long c, int j) {
  const float num = (p[c + g.sj] - p[c]) * 2.0f;
  const float gy = P2 ? num * s.r2[1] : num / (s.dy1[j] + s.dy1[j + 1]);
  return v[c] + dt * (fgh[3 * c + 1] - gy);
}
template <bool P2 = false>
__device__ __forceinline__ float velnw_w(const Geo& g, const Spac& s, const float* w, const float* p,
                                         const float* fgh, float dt, long long c, int k) {
  const float num = (p[c + 1] - p[c]) * 2.0f;
  const float gz = P2 ? num * s.r2[2] : num / (s.dzn[k] + s.dzn[k + 1]);
  return w[c] + dt * (fgh[3 * c + 2] - gz);
}

// u is updated on faces i = 0..im (the low face only where it is physical),
// v on j = 0..jm, w on k = 0..km; the other two coordinates interior.
__device__ __forceinline__ bool in_velnw_u(const Geo& g, int i, int j, int k) {
  return (i >= 1 || g.west_bc) && i <= g.im && j >= 1 && j <= g.jm && k >= 1 && k <= g.km;
}
__device__ __forceinline__ bool in_velnw_v(const Geo& g, int i, int j, int k) {
  return i >= 1 && i <= g.im && j <= g.jm && k >= 1 && k <= g.km;
}
__device__ __forceinline__ bool in_velnw_w(const Geo& g, int i, int j, int k) {
  return i >= 1 && i <= g.im && j >= 1 && j <= g.jm && k <= g.km;
}

#ifndef LESB_JIT
__global__ void k_velnw_inplace(Geo g, Spac s, float* __restrict__ u, float* __restrict__ v,
                                float* __restrict__ w, const float* __restrict__ p,
                                const float* __restrict__ fgh, float dt) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y * blockDim.y + threadIdx.y;
  int i = blockIdx.z;
  if (k > g.km || j > g.jm) return;
  long long c = cidx(g, i, j, k);
  if (in_velnw_u(g, i, j, k)) u[c] = velnw_u(g, s, u, p, fgh, dt, c, i);
  if (in_velnw_v(g, i, j, k)) v[c] = velnw_v(g, s, v, p, fgh, dt, c, j);
  if (in_velnw_w(g, i, j, k)) w[c] = velnw_w(g, s, w, p, fgh, dt, c, k);
}
#endif  // LESB_JIT

// ---------------------------------------------------------------------------
// bondv1 closed form (les.py:254-266): resolve k (w -> 0 at
// k in {0, km+1}; u, v clamp), then j (periodic), then i (0 -> inflow at the
// resolved k, im+1 -> im).  Returns false when the cell belongs to a
// neighbouring slab (internal x face): the halo exchange fills it.
// ---------------------------------------------------------------------------
struct BondSrc {
  int kind;  // 0 zero, 1 inflow, 2 interior cell
  int kk;
  int ii, jj;  // source cell (ii, jj, kk) when kind == 2
  long long src;
};

__device__ __forceinline__ bool bond_source(const Geo& g, int comp, int i, int j, int k, BondSrc& b) {
  if ((i == 0 && !g.west_bc) || (i >= g.im + 1 && !g.east_bc)) return false;
  if (comp == 2 && (k == 0 || k == g.km + 1)) { b.kind = 0; return true; }
  int kk = k < 1 ? 1 : (k > g.km ? g.km : k);
  int jj = j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j);
  if (i == 0) { b.kind = 1; b.kk = kk; return true; }
  int ii = i == g.im + 1 ? g.im : i;
  b.kind = 2;
  b.ii = ii;
  b.jj = jj;
  b.src = cidx(g, ii, jj, kk);
  return true;
}

#ifndef LESB_JIT
__global__ void k_bondv1_inplace(Geo g, float* __restrict__ u, float* __restrict__ v,
                                 float* __restrict__ w, const float* __restrict__ inflow) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y * blockDim.y + threadIdx.y;
  int i = blockIdx.z;
  if (k > g.km + 1 || j > g.jm + 1) return;
  bool halo = i == 0 || i == g.im + 1 || j == 0 || j == g.jm + 1 || k == 0 || k == g.km + 1;
  if (!halo) return;
  long long c = cidx(g, i, j, k);
  float* f[3] = {u, v, w};
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    BondSrc b;
    if (!bond_source(g, m, i, j, k, b)) continue;
    f[m][c] = b.kind == 0 ? 0.0f : (b.kind == 1 ? inflow[m * g.km + b.kk - 1] : f[m][b.src]);
  }
}
#endif  // LESB_JIT

// Fused velnw + bondv1 over the whole array: reads state A, writes B.
template <bool P2>
__global__ void k_velnw_bondv1(Geo g_in, Spac s, const float* __restrict__ u, const float* __restrict__ v,
                               const float* __restrict__ w, const float* __restrict__ p,
                               const float* __restrict__ fgh, float dt, const float* __restrict__ inflow,
                               float* __restrict__ ub, float* __restrict__ vb, float* __restrict__ wb,
                               unsigned* flags) {
  const Geo g = jit_geo(g_in);
  // the fused kernel that follows may be scheduled now (it waits for this
  // grid's completion before its first access: programmatic dependent launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y * blockDim.y + threadIdx.y;
  int i = blockIdx.z;
  unsigned bits = 0;
  if (k <= g.km + 1 && j <= g.jm + 1) {
    long long c = cidx(g, i, j, k);
    // a warp is a run of k in one (i, j) column (box_launch: blockDim.x a
    // multiple of 32), so this test is warp uniform
    const bool column = i >= 1 && i <= g.im && j >= 1 && j <= g.jm;
    if (column) {
      // every k of an interior column, k halo included, on one path (the
      // halo lanes at k = 0 and km + 1 share a warp with interior lanes: a
      // branch per cell made those warps run both paths).  bondv1 there
      // (les.py:254-258): u, v = velnw at the clamped k, w = 0; velnw's own
      // check covers its w face at k = 0 (les.py:413-415, in_velnw_w).
      const int kb = k < 1 ? 1 : (k > g.km ? g.km : k);
      const int kw = k > g.km ? g.km : k;
      const float a = velnw_u<P2>(g, s, u, p, fgh, dt, c + (kb - k), i);
      const float b = velnw_v<P2>(g, s, v, p, fgh, dt, c + (kb - k), j);
      const float d = velnw_w<P2>(g, s, w, p, fgh, dt, c + (kw - k), kw);
      const bool kh = k == 0 || k == g.km + 1;
      const bool ab = finite32(a) && finite32(b);
      if (!kh) {
        if (!(ab && finite32(d))) bits |= F_VELNW;
      } else {
        if (k == 0 && !finite32(d)) bits |= F_VELNW;
        if (!ab) bits |= F_BONDV1;
      }
      ub[c] = a; vb[c] = b; wb[c] = kh ? 0.0f : d;
    } else {
      // velnw's own writes to halo faces are overwritten by bondv1 but are
      // still checked after the velnw stage (les.py:413-415).
      if (in_velnw_u(g, i, j, k) && !finite32(velnw_u<P2>(g, s, u, p, fgh, dt, c, i))) bits |= F_VELNW;
      if (in_velnw_v(g, i, j, k) && !finite32(velnw_v<P2>(g, s, v, p, fgh, dt, c, j))) bits |= F_VELNW;
      if (in_velnw_w(g, i, j, k) && !finite32(velnw_w<P2>(g, s, w, p, fgh, dt, c, k))) bits |= F_VELNW;
      float* out[3] = {ub, vb, wb};
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        BondSrc b;
        if (!bond_source(g, m, i, j, k, b)) continue;
        float val;
        if (b.kind == 0) {
          val = 0.0f;
        } else if (b.kind == 1) {
          val = inflow[m * g.km + b.kk - 1];
        } else {
          val = m == 0 ? velnw_u<P2>(g, s, u, p, fgh, dt, b.src, b.ii)
              : (m == 1 ? velnw_v<P2>(g, s, v, p, fgh, dt, b.src, b.jj)
                        : velnw_w<P2>(g, s, w, p, fgh, dt, b.src, b.kk));
        }
        if (!finite32(val)) bits |= F_BONDV1;
        out[m][c] = val;
      }
    }
  }
  flag_or(flags, bits);
}

// ---------------------------------------------------------------------------
// velfg (les.py:90-192, _combine_force 128-175).  Component M at interior P.
// ---------------------------------------------------------------------------
template <int M, bool P2 = false>
__device__ __forceinline__ float velfg_point(const Geo& g, const Spac& s, const float* __restrict__ u,
                                             const float* __restrict__ v, const float* __restrict__ w,
                                             float vn, long long c, int i, int j, int k) {
  const float* V[3] = {u, v, w};
  const float* vm = V[M];
  float avg[3], term[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const long long sd = d == 0 ? g.si : (d == 1 ? (long long)g.sj : 1LL);
    const int pd = d == 0 ? i : (d == 1 ? j : k);
    const int nd = d == 0 ? g.im : (d == 1 ? g.jm : g.km);
    const float* sa = d == 0 ? s.dx1 : (d == 1 ? s.dy1 : s.dzn);
    const float lo = sa[pd], hi = sa[pd + 1];
    // D_d(v_m, P): central (les.py:100-110)
    const float n0 = vm[c + sd] - vm[c - sd];
    const float d0 = P2 ? n0 * s.r2[d] : n0 / (lo + hi);
    // D_d(v_m, P + e_d): central, or one-sided at the global index N+1 (111-117)
    float d1;
    const bool onesided = (pd + 1 > nd) && (d != 0 || g.east_bc);
    if (onesided) {
      const float n1 = vm[c + sd] - vm[c];
      d1 = P2 ? n1 * s.r1[d] : n1 / sa[nd + 1];
    } else {
      const float n1 = vm[c + 2 * sd] - vm[c];
      d1 = P2 ? n1 * s.r2[d] : n1 / (hi + sa[pd + 2]);
    }
    const float cov = V[d][c] * d0;
    const float cp = V[d][c + sd] * d1;
    if (d == M) {
      const float na = hi * cov + lo * cp, nt = 2.0f * (-d0 + d1);
      avg[d] = P2 ? na * s.r2[d] : na / (lo + hi);
      term[d] = P2 ? nt * s.r2[d] : nt / (lo + hi);
    } else {
      avg[d] = (cov + cp) * 0.5f;  // x / 2 == x * 0.5 exactly
      const float nt = -d0 + d1;
      term[d] = P2 ? nt * s.r1[d] : nt / lo;
    }
  }
  const float df = (term[0] + term[1]) + term[2];
  const float covc = (avg[0] + avg[1]) + avg[2];
  return -covc + vn * df;
}

#ifndef LESB_JIT
__global__ void k_velfg(Geo g, Spac s, const float* __restrict__ u, const float* __restrict__ v,
                        const float* __restrict__ w, float* __restrict__ fgh, float vn) {
  int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  int j = blockIdx.y * blockDim.y + threadIdx.y + 1;
  int i = blockIdx.z + 1;
  if (k > g.km || j > g.jm) return;
  long long c = cidx(g, i, j, k);
  fgh[3 * c + 0] = velfg_point<0>(g, s, u, v, w, vn, c, i, j, k);
  fgh[3 * c + 1] = velfg_point<1>(g, s, u, v, w, vn, c, i, j, k);
  fgh[3 * c + 2] = velfg_point<2>(g, s, u, v, w, vn, c, i, j, k);
}
#endif  // LESB_JIT

// ---------------------------------------------------------------------------
// feedbf (les.py:269-282)
// ---------------------------------------------------------------------------
#ifndef LESB_JIT
__global__ void k_feedbf(Geo g, float* __restrict__ u, float* __restrict__ v, float* __restrict__ w,
                         float* __restrict__ fgh, const float* __restrict__ mask, float dt) {
  int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  int j = blockIdx.y * blockDim.y + threadIdx.y + 1;
  int i = blockIdx.z + 1;
  if (k > g.km || j > g.jm) return;
  long long c = cidx(g, i, j, k);
  const float m = mask[c];
  const float coef = m / dt;
  const float keep = 1.0f - m;
  float* V[3] = {u, v, w};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float x = V[a][c];
    fgh[3 * c + a] = fgh[3 * c + a] - coef * x;
    V[a][c] = x * keep;
  }
}
#endif  // LESB_JIT

// ---------------------------------------------------------------------------
// les_viscosity (les.py:285-320).  Reader R gives the velocity the stage
// sees: the stored arrays (stand-alone) or, inside the fused step kernel, the
// post-feedbf values computed on the fly from the pre-feedbf ones.
// ---------------------------------------------------------------------------
struct PlainReader {
  const float* V[3];
  __device__ __forceinline__ float operator()(int m, long long q, int, int) const { return V[m][q]; }
  __device__ __forceinline__ void all(long long q, int, int, float out[3]) const {
#pragma unroll
    for (int m = 0; m < 3; ++m) out[m] = V[m][q];
  }
};

// feedbf masks interior cells only (les.py:281-282); halo cells keep their
// bondv1 values.  An x-slab's internal halo planes are interior cells of the
// global grid and are masked like any other interior cell.
struct MaskedReader {
  const float* V[3];
  const float* mask;
  Geo g;
  __device__ __forceinline__ float operator()(int m, long long q, int iq, int on_axis_halo) const {
    bool interior = !on_axis_halo && (iq >= 1 || !g.west_bc) && (iq <= g.im || !g.east_bc);
    float x = V[m][q];
    return interior ? x * (1.0f - mask[q]) : x;
  }
  // the three components at one cell: one mask load and one 1 - mask (the
  // compiler did not merge them across three operator() calls)
  __device__ __forceinline__ void all(long long q, int iq, int on_axis_halo, float out[3]) const {
    const bool interior = !on_axis_halo && (iq >= 1 || !g.west_bc) && (iq <= g.im || !g.east_bc);
    const float keep = interior ? 1.0f - mask[q] : 0.0f;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const float x = V[m][q];
      out[m] = interior ? x * keep : x;
    }
  }
};

template <class R, bool P2 = false>
__device__ __forceinline__ void les_point(const Geo& g, const Spac& s, const R& rd, float csd2, long long c,
                                          int i, int j, int k, float lap_out[3]) {
  // neighbour reads: (m, axis, +/-).  on_axis_halo marks a j or k halo cell.
  float d[3][3];
  float ctr[3], nb_hi[3][3], nb_lo[3][3];
  {
    float t[7][3];
    rd.all(c, i, 0, t[0]);
    rd.all(c + g.si, i + 1, 0, t[1]);
    rd.all(c - g.si, i - 1, 0, t[2]);
    rd.all(c + g.sj, i, j + 1 > g.jm, t[3]);
    rd.all(c - g.sj, i, j - 1 < 1, t[4]);
    rd.all(c + 1, i, k + 1 > g.km, t[5]);
    rd.all(c - 1, i, k - 1 < 1, t[6]);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      ctr[m] = t[0][m];
      nb_hi[m][0] = t[1][m];
      nb_lo[m][0] = t[2][m];
      nb_hi[m][1] = t[3][m];
      nb_lo[m][1] = t[4][m];
      nb_hi[m][2] = t[5][m];
      nb_lo[m][2] = t[6][m];
    }
  }
  const float hx = s.dx1[i], hy = s.dy1[j], hz = s.dzn[k];
  const float den[3] = {hx + s.dx1[i + 1], hy + s.dy1[j + 1], hz + s.dzn[k + 1]};
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float nd_ = nb_hi[m][a] - nb_lo[m][a];
      d[m][a] = P2 ? nd_ * s.r2[a] : nd_ / den[a];
    }
  const float s11 = d[0][0], s22 = d[1][1], s33 = d[2][2];
  const float s12 = 0.5f * (d[0][1] + d[1][0]);
  const float s13 = 0.5f * (d[0][2] + d[2][0]);
  const float s23 = 0.5f * (d[1][2] + d[2][1]);
  const float sq = ((s11 * s11 + s22 * s22) + s33 * s33) + 2.0f * ((s12 * s12 + s13 * s13) + s23 * s23);
  const float nu = csd2 * sqrtf(sq);
  const float hh[3] = {hx * hx, hy * hy, hz * hz};
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    float lap = 0.0f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float nl = (nb_hi[m][a] - 2.0f * ctr[m]) + nb_lo[m][a];
      lap = lap + (P2 ? nl * s.rsq[a] : nl / hh[a]);
    }
    lap_out[m] = nu * lap;
  }
}

__device__ __forceinline__ long long icompact(const Geo& g, int i, int j, int k) {
  return ((long long)(i - 1) * g.jm + (j - 1)) * g.km + (k - 1);
}

#ifndef LESB_JIT
__global__ void k_les(Geo g, Spac s, const float* __restrict__ u, const float* __restrict__ v,
                      const float* __restrict__ w, float* __restrict__ fgh, const float* __restrict__ csd2f,
                      float csd2s) {
  int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  int j = blockIdx.y * blockDim.y + threadIdx.y + 1;
  int i = blockIdx.z + 1;
  if (k > g.km || j > g.jm) return;
  long long c = cidx(g, i, j, k);
  PlainReader rd{{u, v, w}};
  float add[3];
  les_point(g, s, rd, csd2f ? csd2f[icompact(g, i, j, k)] : csd2s, c, i, j, k, add);
#pragma unroll
  for (int m = 0; m < 3; ++m) fgh[3 * c + m] = fgh[3 * c + m] + add[m];
}
#endif  // LESB_JIT

#ifndef LESB_JIT
__global__ void k_strain(Geo g, Spac s, const float* __restrict__ u, const float* __restrict__ v,
                         const float* __restrict__ w, float* __restrict__ out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  int j = blockIdx.y * blockDim.y + threadIdx.y + 1;
  int i = blockIdx.z + 1;
  if (k > g.km || j > g.jm) return;
  long long c = cidx(g, i, j, k);
  const float* V[3] = {u, v, w};
  const long long st[3] = {g.si, g.sj, 1};
  const float den[3] = {s.dx1[i] + s.dx1[i + 1], s.dy1[j] + s.dy1[j + 1], s.dzn[k] + s.dzn[k + 1]};
  float d[3][3];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int a = 0; a < 3; ++a) d[m][a] = (V[m][c + st[a]] - V[m][c - st[a]]) / den[a];
  const float s12 = 0.5f * (d[0][1] + d[1][0]);
  const float s13 = 0.5f * (d[0][2] + d[2][0]);
  const float s23 = 0.5f * (d[1][2] + d[2][1]);
  const float sq = ((d[0][0] * d[0][0] + d[1][1] * d[1][1]) + d[2][2] * d[2][2]) +
                   2.0f * ((s12 * s12 + s13 * s13) + s23 * s23);
  out[icompact(g, i, j, k)] = sqrtf(sq);
}
#endif  // LESB_JIT

// ---------------------------------------------------------------------------
// adam (les.py:323-327): whole array including halos.
// ---------------------------------------------------------------------------
#ifndef LESB_JIT
__global__ void k_adam(float* __restrict__ fgh, float* __restrict__ fgh_old, long long n) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; t < n; t += (long long)gridDim.x * blockDim.x) {
    const float f = fgh[t];
    fgh[t] = 1.5f * f - 0.5f * fgh_old[t];
    fgh_old[t] = f;
  }
}
#endif  // LESB_JIT

// ---------------------------------------------------------------------------
// divergence (les.py:330-338); rhs = divergence / dt (les.py:374-375)
// ---------------------------------------------------------------------------
template <bool P2 = false>
__device__ __forceinline__ float div_point(const Geo& g, const Spac& s, float uc, float um, float vc, float vm,
                                           float wc, float wm, int i, int j, int k) {
  if (P2) return ((uc - um) * s.r1[0] + (vc - vm) * s.r1[1]) + (wc - wm) * s.r1[2];
  return ((uc - um) / s.dx1[i] + (vc - vm) / s.dy1[j]) + (wc - wm) / s.dzn[k];
}

#ifndef LESB_JIT
__global__ void k_divergence(Geo g, Spac s, const float* __restrict__ u, const float* __restrict__ v,
                             const float* __restrict__ w, float* __restrict__ out, float dt, int to_rhs) {
  int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  int j = blockIdx.y * blockDim.y + threadIdx.y + 1;
  int i = blockIdx.z + 1;
  if (k > g.km || j > g.jm) return;
  long long c = cidx(g, i, j, k);
  float d = div_point(g, s, u[c], u[c - g.si], v[c], v[c - g.sj], w[c], w[c - 1], i, j, k);
  if (to_rhs) out[c] = d / dt;
  else out[icompact(g, i, j, k)] = d;
}
#endif  // LESB_JIT

// ---------------------------------------------------------------------------
// Fused velfg -> feedbf -> les -> adam -> rhs over the whole array.
// Reads the post-bondv1 velocities B; writes masked velocities to A, fgh,
// fgh_old (interior: full chain; halo: adam only), and rhs (interior).
// ---------------------------------------------------------------------------
// (128, 8): 64 registers; measured fastest ahead of time (62.6 us at
// 150^2x90 against 68-72 us at 48-94 registers); the specialised build
// (jit.cu) uses 10
#ifndef FUSED_MINB
#define FUSED_MINB 8
#endif
template <bool P2>
__global__ void __launch_bounds__(128, FUSED_MINB) k_fused_rhs(Geo g_in, Spac s, const float* __restrict__ ub, const float* __restrict__ vb,
                            const float* __restrict__ wb, const float* __restrict__ mask,
                            float* __restrict__ fgh, float* __restrict__ fgh_old, float* __restrict__ ua,
                            float* __restrict__ va, float* __restrict__ wa, float* __restrict__ rhs, float vn,
                            float dt, int do_les, const float* __restrict__ csd2f, float csd2s,
                            unsigned* flags) {
  const Geo g = jit_geo(g_in);
  // programmatic dependent launch (launch_fused_rhs): every input is the
  // previous kernel's output or follows it in stream order
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y * blockDim.y + threadIdx.y;
  int i = blockIdx.z;
  unsigned bits = 0;
  if (k <= g.km + 1 && j <= g.jm + 1) {
    long long c = cidx(g, i, j, k);
    bool interior = i >= 1 && i <= g.im && j >= 1 && j <= g.jm && k >= 1 && k <= g.km;
    // adam and the stores are common to interior and halo cells (a warp's
    // k-halo lanes share it with interior lanes: only the loads differ)
    float fo[3], f[3], vk[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) fo[a] = fgh_old[3 * c + a];
    if (interior) {
      // the last-used operands first: their DRAM latency overlaps velfg / les
      const float m = mask[c];
      f[0] = velfg_point<0, P2>(g, s, ub, vb, wb, vn, c, i, j, k);
      f[1] = velfg_point<1, P2>(g, s, ub, vb, wb, vn, c, i, j, k);
      f[2] = velfg_point<2, P2>(g, s, ub, vb, wb, vn, c, i, j, k);
      if (!(finite32(f[0]) && finite32(f[1]) && finite32(f[2]))) bits |= F_VELFG;
      // feedbf
      const float coef = (P2 && s.dtp2) ? m * s.rdt : m / dt;
      const float keep = 1.0f - m;
      const float vel[3] = {ub[c], vb[c], wb[c]};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        f[a] = f[a] - coef * vel[a];
        vk[a] = vel[a] * keep;
      }
      if (!(finite32(f[0]) && finite32(f[1]) && finite32(f[2]) && finite32(vk[0]) && finite32(vk[1]) &&
            finite32(vk[2])))
        bits |= F_FEEDBF;
      // les on the post-feedbf velocities
      MaskedReader rd{{ub, vb, wb}, mask, g};
      if (do_les) {
        float add[3];
        les_point<MaskedReader, P2>(g, s, rd, csd2f ? csd2f[icompact(g, i, j, k)] : csd2s, c, i, j, k, add);
#pragma unroll
        for (int a = 0; a < 3; ++a) f[a] = f[a] + add[a];
        if (!(finite32(f[0]) && finite32(f[1]) && finite32(f[2]))) bits |= F_LES;
      }
      // divergence of the post-feedbf velocities, / dt
      const float um = rd(0, c - g.si, i - 1, 0);
      const float vm_ = rd(1, c - g.sj, i, j - 1 < 1);
      const float wm = rd(2, c - 1, i, k - 1 < 1);
      const float dv = div_point<P2>(g, s, vk[0], um, vk[1], vm_, vk[2], wm, i, j, k);
      rhs[c] = (P2 && s.dtp2) ? dv * s.rdt : dv / dt;
    } else {
      // halo: velfg / feedbf / les leave fgh and the velocities as they are;
      // adam runs on the whole array (les.py:323-327)
#pragma unroll
      for (int a = 0; a < 3; ++a) f[a] = fgh[3 * c + a];
      vk[0] = ub[c];
      vk[1] = vb[c];
      vk[2] = wb[c];
    }
    // adam
    float nf[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) nf[a] = 1.5f * f[a] - 0.5f * fo[a];
    if (!(finite32(nf[0]) && finite32(nf[1]) && finite32(nf[2]))) bits |= F_ADAM;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      fgh[3 * c + a] = nf[a];
      fgh_old[3 * c + a] = f[a];
    }
    ua[c] = vk[0]; va[c] = vk[1]; wa[c] = vk[2];
  }
  flag_or(flags, bits);
}

}  // namespace lesb
