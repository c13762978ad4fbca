// Persistent, shared-memory-resident red-black SOR (reference semantics:
// gmcf_mini/sor.py:181-203 with the halo policies of sor.cu, plus the final
// halo_fn call of the press policy, les.py:341-355, and the residual sums of
// sor.py:199-203).
//
// One CTA per SM (cooperative launch, so every CTA is co-resident) owns an
// (i, j) tile of the grid with its full k columns.  The tile's pressure and
// rhs stay in shared memory for the whole solve; only tile faces move, through
// L2, once per colour pass:
//
//   for pass n (colour nrd = n & 1):
//     receive: the neighbours' pass n-1 faces (self-validating LL words, one
//       16-byte load per slot pair, issued during pass n-1's interior runs)
//       into this tile's halo columns; barrier
//     update the colour-nrd cells of the tile's BOUNDARY columns, two slots
//       per work unit (decoded once per solve into a per-unit table),
//       publishing each pair of new values with one 16-byte store into the
//       tile's face slots (or, on an x-slab edge, straight into the neighbour
//       slab's ghost slot -- NVLink peer memory across GPUs)
//     update the colour-nrd cells of the tile's INTERIOR columns, in runs of
//       slot pairs, while the published faces travel
//
// Layout ("colour split"): cell (i,j,k) lives in colour array
// colour(i,j,k) = (i+j+k+1)&1 at slot k>>1 of its column, so for a fixed
// column the colour-c cells are consecutive slots: slot s of the colour-nrd
// array holds k = 2 s + kp (kp the parity of the colour's k values in the
// column), its E/W/N/S neighbours sit at slot s of the neighbour columns'
// other-colour arrays and its top/bottom at slots s + kp, s + kp - 1 of its
// own column's other-colour array.  A warp's lanes work on the same slot
// pair of consecutive columns (64-bit shared accesses at one offset).
//
// Work units are walked with an incremental decode (no integer division in
// the pass loop) over a column table whose boundary columns come first.  Halo slots take the colour of their storage position; for the
// periodic wrap with odd jm the source cell has the other colour, which is
// exactly the reference's pre-pass snapshot of the y halo (the slot is only
// refreshed after the pass that updated its source).
//
// After the last pass each tile writes its columns back, materialising the
// press halo in closed form for the halo cells whose
// source it owns and raising the press non-finite bit; after a grid-wide
// barrier tile b reduces the residual of iteration b in a fixed order.
//
// Arithmetic per point is sor_point's (same op order, -fmad=false), so the
// result is bitwise identical to the streaming kernels and the reference.
#pragma once

#include <cooperative_groups.h>

#include "lesb_common.cuh"


namespace cg = cooperative_groups;

// Timing experiments that drop waits / updates / receives (results wrong):
// compiled only into experiment builds (scripts/build_variant.sh NAME WORK
// -DLESB_RES_DEBUG_BUILD), never into the product library.
#ifdef LESB_RES_DEBUG_BUILD
#define RES_DBG(a, bit) ((a).debug & (bit))
#else
#define RES_DBG(a, bit) 0
#endif

namespace lesb {

#ifndef RES_NTHREADS
#define RES_NTHREADS 512
#endif
constexpr int RES_THREADS = RES_NTHREADS;
constexpr int RES_WARPS = RES_THREADS / 32;
constexpr int NST = 6;   // LESB_RES_TRACE stamps per pass
#ifndef RES_RU
#define RES_RU 4
#endif
#ifndef RES_RCVP
#define RES_RCVP 3
#endif
constexpr int RCVP = RES_RCVP;  // receive slot pairs each thread keeps in registers

struct ResPlan {
  int ni, nj;       // tile grid
  int ti_max, tj_max;
  int kk;           // slots per colour column: ((km + 1) >> 1) + 1
  int kt;           // work items per column and pass: (km + 1) >> 1
  size_t smem;      // dynamic shared memory bytes
  long long fstride;  // words per face slot
  long long bstride;  // words per ring buffer: ntiles * 4 faces + 2 * nj ghost slots
  long long xbuf;   // words of the face exchange buffer (4 ring buffers)
  int pad[2][2];    // row pad by (TI == ti_max ? 0 : 1, TJ == tj_max ? 0 : 1)
  bool ok;
};

// The tile plan the kernel works with: its launch parameter, or in a
// runtime-specialised build (jit.cu) the same plan as compile-time constants.
__device__ __forceinline__ ResPlan jit_res_plan(const ResPlan& p_in) {
  ResPlan p = p_in;
#ifdef LESB_JIT_RES_NI
  p.ni = LESB_JIT_RES_NI;
  p.nj = LESB_JIT_RES_NJ;
  p.ti_max = LESB_JIT_RES_TIM;
  p.tj_max = LESB_JIT_RES_TJM;
  p.kk = LESB_JIT_RES_KK;
  p.kt = LESB_JIT_RES_KT;
  p.fstride = LESB_JIT_RES_FSTRIDE;
  p.bstride = LESB_JIT_RES_BSTRIDE;
  p.pad[0][0] = LESB_JIT_RES_PAD00;
  p.pad[0][1] = LESB_JIT_RES_PAD01;
  p.pad[1][0] = LESB_JIT_RES_PAD10;
  p.pad[1][1] = LESB_JIT_RES_PAD11;
#endif
  return p;
}

struct ResArgs {
  Geo g;
  ResPlan pl;
  float* p;
  const float* rhs;
  float om, cn1;
  float w2l, w2s, w3l, w3s, w4l, w4s;
  int n_iter;
  unsigned long long* xbuf;  // [4 ring][ntiles * 4 faces + 2 nj ghost slots][fstride] (value, tag) words
  // x-slabs: the face buffers of the neighbouring slabs (same
  // plan), or nullptr at a physical x face.  An edge tile writes its x face
  // straight into the neighbour's ghost slot for its tj (west peer: ghost-E
  // slot, east peer: ghost-W slot) and reads its own ghost slots; on another
  // GPU the peer buffer is NVLink peer memory and those words use .sys scope.
  unsigned long long* peer_w;
  unsigned long long* peer_e;
  unsigned* epoch;   // launch counter: tags of this launch are unique across launches
  double* partials;  // [n_iter][ntiles][RES_WARPS] per-warp residual partials (both colour passes)
  double* res;       // [n_iter] residual per iteration
  unsigned* pflags;  // stage flag word (F_PRESS) or nullptr
  unsigned* err;     // set when a neighbour wait times out
  int debug;         // timing experiments only (LESB_RES_DEBUG): 1 no waits, 2 no updates, 4 no receive
  unsigned long long* trace;  // LESB_RES_TRACE: [ntiles][2 n_iter][NST] %globaltimer stamps, or nullptr
  StepBook* book;             // end-of-step bookkeeping after the grid barrier (single domain), or nullptr
};

// Face exchange in the "LL" style: every published value travels with the
// tag of its pass in one 64-bit word, written and read with single-copy-atomic
// 64-bit accesses, so a reader that sees the right tag also sees the right
// value -- no fences, counters or flag round trips.
__device__ __forceinline__ void st_ll_word(unsigned long long* a, unsigned long long w) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(w));
}
__device__ __forceinline__ void st_ll_sys(unsigned long long* a, unsigned long long w) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(a), "l"(w));
}
__device__ __forceinline__ unsigned long long ld_ll_sys(const unsigned long long* a) {
  unsigned long long w;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(a));
  return w;
}
__device__ __forceinline__ void st_ll_pair(unsigned long long* a, unsigned long long x, unsigned long long y) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(a), "l"(x), "l"(y));
}
__device__ __forceinline__ void st_ll_pair_sys(unsigned long long* a, unsigned long long x, unsigned long long y) {
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(a), "l"(x), "l"(y));
}
__device__ __forceinline__ void ld_ll2(const unsigned long long* a, unsigned long long& x, unsigned long long& y) {
  // two LL words in one 16-byte load (each 8-byte element single-copy atomic)
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(a));
}
__device__ __forceinline__ void ld_ll2_sys(const unsigned long long* a, unsigned long long& x,
                                           unsigned long long& y) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(a));
}
__device__ __forceinline__ unsigned long long ld_ll(const unsigned long long* a) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(a));
  return w;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int ROW_PAD_MAX = 31;  // row padding of the column grid (chosen per tile shape by the plan)
// Pair layout (RES_PAIRS): KK even, column stride CW = 4 KK + 2 and even row
// pads, so every column base is 8-byte aligned and the boundary walk's slot
// pairs move with 64-bit shared accesses (16 lanes on consecutive pairs of a
// column: conflict free).  The interior runs stay scalar: the checkerboard's
// alternating slot offset keeps their bank load at the odd-stride layout's
// (the plan's row-pad model; measured: pair-wise runs diverge between the
// two column parities and were slower).  RES_PAIRS=0: CW = 4 KK + 1.
#ifndef RES_PAIRS
#define RES_PAIRS 1
#endif
constexpr int CW_EXTRA = RES_PAIRS ? 2 : 1;

__device__ __forceinline__ int tile_lo(int t, int n, int nt) { return 1 + (int)(((long long)t * n) / nt); }

// colour of a cell: the pass nrd updates cells with colour == nrd
// ((i-1)+(j-1)+(k-1)+nrd even, sor.py:174-178), i GLOBAL (an x-slab adds ioff)
__device__ __forceinline__ int colour(int i, int j, int k) { return (i + j + k + 1) & 1; }

// Shared-memory column layout: [p colour 0 | p colour 1 | rhs colour 0 |
// rhs colour 1], KK slots each, so one column is 4 KK floats and every
// operand of a point update is (column base + slot + a per-pass constant).
// Column-table entry: column base | parity(i+j) << 28 | west-physical << 29.
constexpr unsigned CB_MASK = 0x0FFFFFFFu;
// publish-table flags: the face word lives in the west / east peer slab's buffer
constexpr int PUB_RW = 1 << 30, PUB_RE = 1 << 29, PUB_OFF = PUB_RE - 1;

// One run of work: colour-nrd cells t0 <= t < t1 of one column.  The
// addresses of consecutive cells differ by one slot, and the bottom neighbour
// of cell t+1 is the top neighbour of cell t, so a run costs 7 shared loads
// and 1 store per cell with no per-cell index arithmetic.
template <bool PRESS>
__device__ __forceinline__ double update_run(const ResArgs& a, float* S, unsigned ci, int t0, int t1, int nrd,
                                             int KK, int CW, int sI, int km) {
  const int cb = (int)(ci & CB_MASK);
  const int kp = (nrd + (int)((ci >> 28) & 1u) + 1) & 1;
  const bool wphys = PRESS && (ci & (1u << 29));
  // cells k = 2t + 2 - kp <= km
  const int tmax = (km + kp - 2) >> 1;  // last valid t
  if (t1 > tmax + 1) t1 = tmax + 1;
  float* cur = S + cb + nrd * KK + (1 - kp) + t0;           // centre, slot t + 1 - kp
  const float* oth = S + cb + (1 - nrd) * KK + (1 - kp) + t0;  // other colour, same k
  const float* tb = S + cb + (1 - nrd) * KK + t0;             // other colour, slot t (bottom)
  const float* rr = cur + 2 * KK;
  double acc = 0.0;
  if (t0 >= t1) return acc;
  float pB = tb[0];
  int t = t0;
  // Groups of RU cells: every load of the group is issued before the first
  // store (the colour-nrd stores never alias the other-colour and rhs loads,
  // which the compiler cannot prove), so RU point updates overlap.
  constexpr int RU = RES_RU;
  for (; t + RU <= t1; t += RU) {
    float pc[RU], pE[RU], pW[RU], pN[RU], pS[RU], pT[RU], r[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      pc[u] = cur[u];
      pE[u] = oth[sI + u];
      pW[u] = oth[-sI + u];
      pN[u] = oth[CW + u];
      pS[u] = oth[-CW + u];
      pT[u] = tb[1 + u];
      r[u] = rr[u];
    }
    double d[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      float pb = u == 0 ? pB : pT[u - 1];
      float pw = pW[u];
      if (PRESS) {
        if (wphys) pw = pc[u];                          // physical west: p[0] -> p[1]
        if (u == 0 && t == 0 && kp == 1) pb = pc[u];    // bottom: p[.,.,0] -> p[.,.,1]
      }
      // sor.py:164-171: E, W, N, S, T, B summed left to right
      float nb = a.w2l * pE[u];
      nb = nb + a.w2s * pw;
      nb = nb + a.w3l * pN[u];
      nb = nb + a.w3s * pS[u];
      nb = nb + a.w4l * pT[u];
      nb = nb + a.w4s * pb;
      // sor.py:197: reltmp = omega * (cn1 * (nb - rhs) - p)
      const float rel = a.om * (a.cn1 * (nb - r[u]) - pc[u]);
      cur[u] = pc[u] + rel;
      d[u] = (double)rel * (double)rel;
    }
    double gsum = 0.0;
#pragma unroll
    for (int u = 0; u < RU; ++u) gsum += d[u];
    acc += gsum;
    pB = pT[RU - 1];
    cur += RU;
    oth += RU;
    tb += RU;
    rr += RU;
  }
  for (; t < t1; ++t) {
    const float pc = *cur;
    const float pE = oth[sI];
    float pW = oth[-sI];
    const float pN = oth[CW];
    const float pS = oth[-CW];
    const float pT = tb[1];
    const float r = *rr;
    float pb = pB;
    if (PRESS) {
      if (wphys) pW = pc;
      if (t == 0 && kp == 1) pb = pc;
    }
    float nb = a.w2l * pE;
    nb = nb + a.w2s * pW;
    nb = nb + a.w3l * pN;
    nb = nb + a.w3s * pS;
    nb = nb + a.w4l * pT;
    nb = nb + a.w4s * pb;
    const float rel = a.om * (a.cn1 * (nb - r) - pc);
    *cur = pc + rel;
    acc += (double)rel * (double)rel;
    pB = pT;
    ++cur;
    ++oth;
    ++tb;
    ++rr;
  }
  return acc;
}

// One run of slot PAIRS j0 <= j < j1 of one column (slots 2j, 2j + 1 of the
// colour-nrd array): six 64-bit shared loads (centre, E, W, N, S, rhs) and
// three words of the other colour's top/bottom chain per pair.  Every lane
// of a warp is at the same slot offset of its column, so the 64-bit accesses
// are parity independent and conflict free for the plan's row pad
// (interior_bank_load), unlike the per-cell walk (update_run) whose centre
// slot alternates with the column parity (measured there: 2.1x the ideal
// shared-memory wavefronts, the kernel's bound at 150^2x90; pair runs
// 383 -> 345 us per 50-iteration solve).
#ifndef RES_IPAIRS
#define RES_IPAIRS RES_PAIRS  // (64-bit accesses need the pair layout)
#endif

template <bool PRESS>
__device__ __forceinline__ double update_prun(const ResArgs& a, float* S, unsigned ci, int j0, int j1, int nrd,
                                              int KK, int CW, int sI, int km) {
  const int cb = (int)(ci & CB_MASK);
  const int kp = (nrd + (int)((ci >> 28) & 1u) + 1) & 1;
  const bool wphys = PRESS && (ci & (1u << 29));
  // slot s holds k = 2 s + kp: pair j has a cell while 4 j + kp <= km
  const int jmax = (km - kp) >> 2;
  if (j1 > jmax + 1) j1 = jmax + 1;
  double acc = 0.0;
  if (j0 >= j1) return acc;
  float* const ce0 = S + cb + nrd * KK;             // colour-nrd array of the column
  const float* const ob = S + cb + (1 - nrd) * KK;  // the other colour's
  // the other colour's slot s holds k = 2 s + 1 - kp: for the pair at slot
  // s0 the chain bottom, k+-1 between the cells, top is ob[s0 + kp - 1 + 0..2]
  auto pair = [&](int s0, float pB0, float pTB, float pT1, bool v0, bool v1, bool bottom) -> double {
    float* ce = ce0 + s0;
    const float* o = ob + s0;
    const float2 c2 = *reinterpret_cast<const float2*>(ce);
    const float2 e2 = *reinterpret_cast<const float2*>(o + sI);
    const float2 w2 = *reinterpret_cast<const float2*>(o - sI);
    const float2 n2 = *reinterpret_cast<const float2*>(o + CW);
    const float2 s2 = *reinterpret_cast<const float2*>(o - CW);
    const float2 r2 = *reinterpret_cast<const float2*>(ce + 2 * KK);
    float pW0 = w2.x, pW1 = w2.y;
    if (PRESS) {
      if (wphys) {  // physical west: p[0] -> p[1]
        pW0 = c2.x;
        pW1 = c2.y;
      }
      if (bottom) pB0 = c2.x;  // bottom: p[.,.,0] -> p[.,.,1]
    }
    // sor.py:164-171: E, W, N, S, T, B summed left to right
    float nb0 = a.w2l * e2.x, nb1 = a.w2l * e2.y;
    nb0 = nb0 + a.w2s * pW0;
    nb1 = nb1 + a.w2s * pW1;
    nb0 = nb0 + a.w3l * n2.x;
    nb1 = nb1 + a.w3l * n2.y;
    nb0 = nb0 + a.w3s * s2.x;
    nb1 = nb1 + a.w3s * s2.y;
    nb0 = nb0 + a.w4l * pTB;
    nb1 = nb1 + a.w4l * pT1;
    nb0 = nb0 + a.w4s * pB0;
    nb1 = nb1 + a.w4s * pTB;
    // sor.py:197: reltmp = omega * (cn1 * (nb - rhs) - p)
    const float rel0 = a.om * (a.cn1 * (nb0 - r2.x) - c2.x);
    const float rel1 = a.om * (a.cn1 * (nb1 - r2.y) - c2.y);
    *reinterpret_cast<float2*>(ce) = make_float2(v0 ? c2.x + rel0 : c2.x, v1 ? c2.y + rel1 : c2.y);
    return (v0 ? (double)rel0 * (double)rel0 : 0.0) + (v1 ? (double)rel1 * (double)rel1 : 0.0);
  };
  // every pair in the checked form (measured: a separate unchecked loop for
  // the pairs between the column ends, with the chain carried in registers,
  // was 2% slower, and one with pointer increments 4%)
  for (int j = j0; j < j1; ++j) {
    const int s0 = 2 * j;
    const int lo = s0 + kp - 1;  // (clamped into the array: a clamped word is never used)
    const float pB0 = ob[max(lo, 0)], pTB = ob[lo + 1], pT1 = ob[min(lo + 2, KK - 1)];
    acc += pair(s0, pB0, pTB, pT1, s0 + kp >= 1, 2 * s0 + 2 + kp <= km, s0 == 0 && kp == 1);
  }
  return acc;
}

// Boundary phase from a per-unit table (RES_BTAB): unit w = c HP + j goes to
// thread w % nth as in update_boundary, but everything about the unit that
// does not change between passes -- column base + slot, column parity and
// west-physical bits, the pair's cell validity and chain clamps for either
// colour, the two face word offsets -- sits in one 16-byte entry, written by
// the thread that uses it before the pass loop.  (The per-pass decode of
// update_boundary cost as many instructions as the arithmetic.)
#ifndef RES_BTAB
#define RES_BTAB RES_PAIRS
#endif
// entry.w bits, per kp = 0 / 1 (shift 4 kp): v0, v1, far end of the chain clamped
constexpr int BT_V0 = 1, BT_V1 = 2, BT_CL = 4, BT_BOT = 1 << 8;  // BT_BOT: slot 0 (press bottom when kp = 1)

__device__ __forceinline__ int4 btab_entry(unsigned ci, int2 pub, int j, int KK, int km) {
  const int s0 = 2 * j;
  int bits = (s0 == 0) ? BT_BOT : 0;
#pragma unroll
  for (int kp = 0; kp < 2; ++kp) {
    int b = 0;
    if (s0 + kp >= 1 && 2 * s0 + kp <= km) b |= BT_V0;
    if (2 * s0 + 2 + kp <= km) b |= BT_V1;
    if (kp ? s0 + 2 >= KK : s0 == 0) b |= BT_CL;
    bits |= b << (4 * kp);
  }
  return make_int4((int)(ci + (unsigned)s0), pub.x >= 0 ? pub.x + s0 : -1, pub.y >= 0 ? pub.y + s0 : -1, bits);
}

template <bool PRESS, bool SLAB>
__device__ __forceinline__ double update_boundary_tab(const ResArgs& a, float* S, const int4* __restrict__ btab,
                                                   int nbu, unsigned long long* X, unsigned long long* XRw,
                                                   unsigned long long* XRe, unsigned tag, int nrd, int KK, int CW,
                                                   int sI) {
  double acc = 0.0;
  float* const Sc = S + nrd * KK;
  const float* const So = S + (1 - nrd) * KK;
  const unsigned long long tagw = (unsigned long long)tag << 32;
  for (int w = threadIdx.x; w < nbu; w += RES_THREADS) {
    const int4 d = btab[w];
    const unsigned ci = (unsigned)d.x;
    const int kp = (nrd + (int)((ci >> 28) & 1u) + 1) & 1;
    const int vb = d.w >> (4 * kp);
    const bool v0 = vb & BT_V0, v1 = vb & BT_V1;
    if (!(v0 || v1)) continue;
    const int off = (int)(ci & CB_MASK);  // column base + s0
    float* ce = Sc + off;
    const float* o = So + off;            // other colour, same k as slot s0
    const float2 c2 = *reinterpret_cast<const float2*>(ce);
    const float2 e2 = *reinterpret_cast<const float2*>(o + sI);
    const float2 w2 = *reinterpret_cast<const float2*>(o - sI);
    const float2 n2 = *reinterpret_cast<const float2*>(o + CW);
    const float2 s2 = *reinterpret_cast<const float2*>(o - CW);
    const float2 o2 = *reinterpret_cast<const float2*>(o);
    // far end of the chain, kept inside the column's colour array (a clamped word is unused)
    const float ox = o[kp ? ((vb & BT_CL) ? 1 : 2) : ((vb & BT_CL) ? 0 : -1)];
    const float2 r2 = *reinterpret_cast<const float2*>(ce + 2 * KK);
    float pW0 = w2.x, pW1 = w2.y;
    float pB0 = kp ? o2.x : ox;          // k - 1 of the first cell
    const float pTB = kp ? o2.y : o2.x;  // k + 1 of the first = k - 1 of the second
    const float pT1 = kp ? ox : o2.y;
    if (PRESS) {
      if (ci & (1u << 29)) {  // physical west: p[0] -> p[1]
        pW0 = c2.x;
        pW1 = c2.y;
      }
      if (kp && (d.w & BT_BOT)) pB0 = c2.x;  // bottom: p[.,.,0] -> p[.,.,1]
    }
    // sor.py:164-171: E, W, N, S, T, B summed left to right
    float nb0 = a.w2l * e2.x, nb1 = a.w2l * e2.y;
    nb0 = nb0 + a.w2s * pW0;
    nb1 = nb1 + a.w2s * pW1;
    nb0 = nb0 + a.w3l * n2.x;
    nb1 = nb1 + a.w3l * n2.y;
    nb0 = nb0 + a.w3s * s2.x;
    nb1 = nb1 + a.w3s * s2.y;
    nb0 = nb0 + a.w4l * pTB;
    nb1 = nb1 + a.w4l * pT1;
    nb0 = nb0 + a.w4s * pB0;
    nb1 = nb1 + a.w4s * pTB;
    // sor.py:197: reltmp = omega * (cn1 * (nb - rhs) - p)
    const float rel0 = a.om * (a.cn1 * (nb0 - r2.x) - c2.x);
    const float rel1 = a.om * (a.cn1 * (nb1 - r2.y) - c2.y);
    const float np0 = v0 ? c2.x + rel0 : c2.x;
    const float np1 = v1 ? c2.y + rel1 : c2.y;
    *reinterpret_cast<float2*>(ce) = make_float2(np0, np1);  // (an unused slot keeps its value)
    const unsigned long long w0 = tagw | __float_as_uint(np0), w1 = tagw | __float_as_uint(np1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int v = h ? d.z : d.y;  // a column lies on at most two faces
      if (v < 0) continue;
      if (!SLAB) {
        st_ll_pair(X + (unsigned)v, w0, w1);
      } else {
        const unsigned fo = (unsigned)(v & PUB_OFF);
        if (v & PUB_RW) st_ll_pair_sys(XRw + fo, w0, w1);
        else if (v & PUB_RE) st_ll_pair_sys(XRe + fo, w0, w1);
        else st_ll_pair(X + fo, w0, w1);
      }
    }
    if (v0) acc += (double)rel0 * (double)rel0;
    if (v1) acc += (double)rel1 * (double)rel1;
  }
  return acc;
}

// Boundary phase over slot PAIRS: unit w = (c - c0) * HP + j goes to thread
// w % nth and updates the colour-nrd cells in slots 2j, 2j + 1 of column c
// (one column decode per two cells, the bottom neighbour of the second cell
// is the top one of the first), then publishes both words with one 16-byte
// store (face columns have an even number of words; the word of a slot
// holding no cell is never read by the receiver).
template <bool PRESS, bool SLAB>
__device__ __forceinline__ double update_boundary(const ResArgs& a, float* S, const unsigned* __restrict__ coltab,
                                               const int2* __restrict__ pubcol, unsigned long long* X,
                                               unsigned long long* XRw, unsigned long long* XRe, unsigned tag,
                                               int c, int j, int dq, int dr, int c1, int HP, int nrd, int KK,
                                               int CW, int sI, int km) {
  // (c, j): this thread's first unit; (dq, dr): RES_THREADS units on, in
  // (columns, pairs) -- pass invariants, decoded once before the pass loop
  double acc = 0.0;
  float* Sc = S + nrd * KK;
  const float* So = S + (1 - nrd) * KK;
  const unsigned long long tagw = (unsigned long long)tag << 32;
  while (c < c1) {
    const unsigned ci = coltab[c];
    const int cb = (int)(ci & CB_MASK);
    const int kp = (nrd + (int)((ci >> 28) & 1u) + 1) & 1;
    const int s0 = 2 * j;
    // slot s holds k = 2 s + kp; a cell when 1 <= k <= km
    const bool v0 = s0 + kp >= 1 && 2 * s0 + kp <= km;
    const bool v1 = 2 * (s0 + 1) + kp <= km;
    if (v0 || v1) {
      const float* o = So + (cb + s0);  // other colour, same k as slot s0
      float* ce = Sc + (cb + s0);
#if RES_PAIRS
      // (8-byte aligned: cb, KK and s0 are even)
      const float2 c2 = *reinterpret_cast<const float2*>(ce);
      const float2 e2 = *reinterpret_cast<const float2*>(o + sI);
      const float2 w2 = *reinterpret_cast<const float2*>(o - sI);
      const float2 n2 = *reinterpret_cast<const float2*>(o + CW);
      const float2 s2 = *reinterpret_cast<const float2*>(o - CW);
      const float2 o2 = *reinterpret_cast<const float2*>(o);
      // (kept inside the column's colour array: at the ends the value is unused)
      const float ox = o[kp ? (s0 + 2 < KK ? 2 : 1) : (s0 > 0 ? -1 : 0)];
      const float2 r2 = *reinterpret_cast<const float2*>(ce + 2 * KK);
      const float pc0 = c2.x, pc1 = c2.y;
      const float pE0 = e2.x, pE1 = e2.y;
      float pW0 = w2.x, pW1 = w2.y;
      const float pN0 = n2.x, pN1 = n2.y;
      const float pS0 = s2.x, pS1 = s2.y;
      float pB0 = kp ? o2.x : ox;        // k - 1 of the first cell
      const float pTB = kp ? o2.y : o2.x;  // k + 1 of the first = k - 1 of the second
      const float pT1 = kp ? ox : o2.y;
      const float r0 = r2.x, r1 = r2.y;
#else
      const float pc0 = ce[0], pc1 = ce[1];
      const float pE0 = o[sI], pE1 = o[sI + 1];
      float pW0 = o[-sI], pW1 = o[-sI + 1];
      const float pN0 = o[CW], pN1 = o[CW + 1];
      const float pS0 = o[-CW], pS1 = o[-CW + 1];
      float pB0 = o[kp - 1];             // k - 1 of the first cell
      const float pTB = o[kp];           // k + 1 of the first = k - 1 of the second
      const float pT1 = o[kp + 1];
      const float r0 = ce[2 * KK], r1 = ce[2 * KK + 1];
#endif
      float pB1 = pTB;
      if (PRESS) {
        if (ci & (1u << 29)) {  // physical west: p[0] -> p[1]
          pW0 = pc0;
          pW1 = pc1;
        }
        if (2 * s0 + kp == 1) pB0 = pc0;  // bottom: p[.,.,0] -> p[.,.,1]
      }
      // sor.py:164-171: E, W, N, S, T, B summed left to right
      float nb0 = a.w2l * pE0, nb1 = a.w2l * pE1;
      nb0 = nb0 + a.w2s * pW0;
      nb1 = nb1 + a.w2s * pW1;
      nb0 = nb0 + a.w3l * pN0;
      nb1 = nb1 + a.w3l * pN1;
      nb0 = nb0 + a.w3s * pS0;
      nb1 = nb1 + a.w3s * pS1;
      nb0 = nb0 + a.w4l * pTB;
      nb1 = nb1 + a.w4l * pT1;
      nb0 = nb0 + a.w4s * pB0;
      nb1 = nb1 + a.w4s * pB1;
      // sor.py:197: reltmp = omega * (cn1 * (nb - rhs) - p)
      const float rel0 = a.om * (a.cn1 * (nb0 - r0) - pc0);
      const float rel1 = a.om * (a.cn1 * (nb1 - r1) - pc1);
      const float np0 = v0 ? pc0 + rel0 : pc0;
      const float np1 = v1 ? pc1 + rel1 : pc1;
#if RES_PAIRS
      *reinterpret_cast<float2*>(ce) = make_float2(np0, np1);  // (an unused slot keeps its value)
#else
      if (v0) ce[0] = np0;
      if (v1) ce[1] = np1;
#endif
      const unsigned long long w0 = tagw | __float_as_uint(np0), w1 = tagw | __float_as_uint(np1);
      const int2 pub = pubcol[c];  // a column lies on at most two faces
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int v = h ? pub.y : pub.x;
        if (v < 0) continue;
        if (!SLAB) {
          st_ll_pair(X + (unsigned)(v + s0), w0, w1);
        } else {
          const unsigned off = (unsigned)((v & PUB_OFF) + s0);
          if (v & PUB_RW) st_ll_pair_sys(XRw + off, w0, w1);
          else if (v & PUB_RE) st_ll_pair_sys(XRe + off, w0, w1);
          else st_ll_pair(X + off, w0, w1);
        }
      }
      if (v0) acc += (double)rel0 * (double)rel0;
      if (v1) acc += (double)rel1 * (double)rel1;
    }
    j += dr;
    c += dq;
    if (j >= HP) {
      j -= HP;
      ++c;
    }
  }
  return acc;
}

// All runs of this thread in columns [c0, c1): the columns are cut into nseg
// runs of L work items (the last run of a column the shortest) and run
// u = g * (c1 - c0) + (c - c0) goes to thread (u - rot) mod U, U = nseg (c1 - c0):
// rot = (nseg - 1)(c1 - c0) hands the short last runs to the lowest threads,
// which are the ones with an extra boundary pair.  Column-fastest numbering
// puts a warp's lanes in consecutive columns at the same slot offset.
// (g, cc): the segment and column of this thread's first run, nu its run
// count; (dg, dcc): RES_THREADS runs on -- decoded once before the pass loop.
// mid() runs once, part-way through the thread's first run (or first, when
// the thread has none): it issues the next pass's receive loads, so their
// L2 round trip overlaps the rest of the interior.
#ifndef RES_MID
#define RES_MID 1
#endif
template <bool PRESS, class F>
__device__ __forceinline__ double update_phase(const ResArgs& a, float* S, const unsigned* __restrict__ coltab,
                                               int c0, int c1, int nseg, int g, int cc, int nu, int dg, int dcc,
                                               int L, int KT, int nrd, int KK, int CW, int sI, int km, F&& mid) {
  double acc = 0.0;
  const int ncc = c1 - c0;
  bool issued = false;
  for (; nu > 0; --nu) {
    const int t0 = g * L;
    const int t1 = min(t0 + L, KT);
    const unsigned ci = coltab[c0 + cc];
#if RES_IPAIRS
    // (t0, t1): slot pairs
    if (!issued) {
      const int tm = t0 + ((t1 - t0) >> 1);
      acc += update_prun<PRESS>(a, S, ci, t0, tm, nrd, KK, CW, sI, km);
      mid();
      issued = true;
      acc += update_prun<PRESS>(a, S, ci, tm, t1, nrd, KK, CW, sI, km);
    } else {
      acc += update_prun<PRESS>(a, S, ci, t0, t1, nrd, KK, CW, sI, km);
    }
#else
    if (!issued) {
      constexpr int RU = RES_RU;
      const int h = (t1 - t0) >> 1;
      const int tm = min(t1, t0 + (RES_MID ? (h + RU - 1) / RU * RU : h / RU * RU));
      acc += update_run<PRESS>(a, S, ci, t0, tm, nrd, KK, CW, sI, km);
      mid();
      issued = true;
      acc += update_run<PRESS>(a, S, ci, tm, t1, nrd, KK, CW, sI, km);
    } else {
      acc += update_run<PRESS>(a, S, ci, t0, t1, nrd, KK, CW, sI, km);
    }
#endif
    g += dg;
    cc += dcc;
    if (cc >= ncc) {
      cc -= ncc;
      ++g;
    }
    if (g >= nseg) g -= nseg;
  }
  if (!issued) mid();
  return acc;
}

// One launch: a single domain, or (SLAB) every in-process x-slab of a group
// on one device -- block b works on tile b % tps of slab b / tps.  Across
// GPUs each rank launches its own slab with peer_w / peer_e mapped.
constexpr int RES_GROUP_MAX = 4;
struct ResGroup {
  ResArgs a[RES_GROUP_MAX];
  int n;    // slabs in this launch
  int tps;  // tiles per slab
};

// a receive that finds a neighbour's word not yet published waits this many
// ns before reading it again (0: spin)
#ifndef RES_SPIN_NS
#define RES_SPIN_NS 0
#endif

template <bool PRESS, bool SLAB>
__global__ void __launch_bounds__(RES_THREADS, 1) k_sor_resident(const __grid_constant__ ResGroup grp) {
  extern __shared__ float smem[];
  __shared__ double red[RES_WARPS];
  const int slab = SLAB ? (int)blockIdx.x / grp.tps : 0;
  const ResArgs& a = grp.a[slab];
#ifdef LESB_JIT_RES_NI  // runtime-specialised build (jit.cu): geometry and plan as compile-time constants
  const Geo g = jit_geo(a.g);
  const ResPlan pl = jit_res_plan(a.pl);
#else  // (references into the grid-constant parameter: no local copies)
  const Geo& g = a.g;
  const ResPlan& pl = a.pl;
#endif
  const int tid = threadIdx.x, nth = RES_THREADS;
  const int lane = tid & 31, warp = tid >> 5;
  const int tile = SLAB ? (int)blockIdx.x - slab * grp.tps : (int)blockIdx.x;
  const int ntiles = pl.ni * pl.nj;
  const int ti = tile / pl.nj, tj = tile % pl.nj;
  const int I0 = tile_lo(ti, g.im, pl.ni), I1 = tile_lo(ti + 1, g.im, pl.ni);
  const int J0 = tile_lo(tj, g.jm, pl.nj), J1 = tile_lo(tj + 1, g.jm, pl.nj);
  const int TI = I1 - I0, TJ = J1 - J0;
  const int KK = pl.kk, KT = pl.kt, km = g.km;
  const int KKF = (KK + 1) & ~1;  // face-buffer words per column: even, so slot pairs are 16-byte aligned
  const int CW = 4 * KK + CW_EXTRA;          // floats per column (see RES_PAIRS)
  // column stride along i, padded so that sI = (TJ - 2) CW (mod 32): the
  // interior columns then sit at CW * (ordinal) + const modulo the 32 banks,
  // and a warp's lanes on 32 consecutive interior columns never conflict
  // column stride along i: (TJ + 2) CW plus the row pad the plan chose for
  // this tile shape (fewest shared-memory bank conflicts in the interior runs)
  // (selects, not an indexed load: a local plan copy would go to local memory)
  const bool fti = TI == pl.ti_max, ftj = TJ == pl.tj_max;
  const int PADI = fti ? (ftj ? pl.pad[0][0] : pl.pad[0][1]) : (ftj ? pl.pad[1][0] : pl.pad[1][1]);
  const int sI = (TJ + 2) * CW + PADI;
  float* S = smem;                           // [ti+2][sI]: columns of [4][KK] (+1), rows padded
  const long long s_floats = (long long)(pl.ti_max + 2) * ((pl.tj_max + 2) * CW + ROW_PAD_MAX);
  unsigned* coltab = reinterpret_cast<unsigned*>(smem + ((s_floats + 3) & ~3LL));   // [TI*TJ]
  int2* pubcol = reinterpret_cast<int2*>(coltab + ((pl.ti_max * pl.tj_max + 3) & ~3)); // [TI*TJ]
  int4* rcvtab = reinterpret_cast<int4*>(pubcol + ((pl.ti_max * pl.tj_max + 1) & ~1));  // [2TI+2TJ]
  int4* btab = rcvtab + 2 * (pl.ti_max + pl.tj_max);  // [boundary units] (RES_BTAB)
  const long long fstride = pl.fstride;
  const long long tstride = 4 * fstride;     // words per tile in one face buffer
  const long long bstride = pl.bstride;      // words per face buffer (tiles, then 2 nj ghost slots)
  const long long ghost_w = ntiles * tstride + (long long)tj * fstride;           // this tile's ghost-W slot
  const long long ghost_e = ntiles * tstride + (long long)(pl.nj + tj) * fstride;  // ... and ghost-E slot

  auto colbase = [&](int li, int lj) { return li * sI + lj * CW; };

  // neighbour tiles (-1: physical boundary with a fixed / remapped halo;
  // -2 / -3: the west / east neighbour slab, through this tile's ghost slot)
  const bool pw = SLAB && a.peer_w != nullptr, pe = SLAB && a.peer_e != nullptr;
  int nbr[4];
  nbr[0] = ti > 0 ? tile - pl.nj : (pw ? -2 : -1);                        // west  <- its east face (1)
  nbr[1] = ti < pl.ni - 1 ? tile + pl.nj : (pe ? -3 : -1);                // east  <- its west face (0)
  nbr[2] = tj > 0 ? tile - 1 : (PRESS ? ti * pl.nj + pl.nj - 1 : -1);     // south <- its north face (3)
  nbr[3] = tj < pl.nj - 1 ? tile + 1 : (PRESS ? ti * pl.nj : -1);         // north <- its south face (2)
  const int wrap_flip = g.jm & 1;  // periodic source parity differs from the slot's for odd jm

  // ---- tables: columns (boundary first) with their face slots; receive list ----
  const bool wtile = PRESS && g.west_bc && ti == 0;
  const int ncol = TI * TJ;
  const int nbnd = (TI <= 2 || TJ <= 2) ? ncol : 2 * TJ + 2 * (TI - 2);
  for (int c = tid; c < ncol; c += nth) {
    int li, lj;
    if (nbnd == ncol) {
      li = 1 + c / TJ;
      lj = 1 + c % TJ;
    } else if (c < TJ) {
      li = 1; lj = 1 + c;
    } else if (c < 2 * TJ) {
      li = TI; lj = 1 + (c - TJ);
    } else if (c < nbnd) {
      const int r = c - 2 * TJ;
      li = 2 + (r >> 1);
      lj = (r & 1) ? TJ : 1;
    } else {
      const int r = c - nbnd;  // interior (li, lj) in [2, TI-1] x [2, TJ-1]
      li = 2 + r / (TJ - 2);
      lj = 2 + r % (TJ - 2);
    }
    const int i = I0 - 1 + li, j = J0 - 1 + lj;
    coltab[c] = (unsigned)colbase(li, lj) | ((unsigned)((i + g.ioff + j) & 1) << 28) |
                ((wtile && li == 1) ? (1u << 29) : 0u);
    // face words of the column: west / east face (x), south / north face (y)
    // (an x face of an edge tile goes to the neighbour slab's ghost slot)
    const int fx = li == 1 ? ((ti == 0 && pw) ? (PUB_RW | ((lj - 1) * KKF)) : (int)(0 * fstride + (lj - 1) * KKF))
                           : (li == TI ? ((ti == pl.ni - 1 && pe) ? (PUB_RE | ((lj - 1) * KKF))
                                                                  : (int)(1 * fstride + (lj - 1) * KKF))
                                       : -1);
    const int fy = lj == 1 ? (int)(2 * fstride + (li - 1) * KKF) : (lj == TJ ? (int)(3 * fstride + (li - 1) * KKF) : -1);
    // (tiles are at least 2 x 2 columns, so no column lies on more faces)
    pubcol[c] = fx >= 0 ? make_int2(fx, fy) : make_int2(fy, -1);
  }
  const int nfc = 2 * TJ + 2 * TI;
  for (int q = tid; q < nfc; q += nth) {
    int f, m;
    if (q < 2 * TJ) { f = q / TJ; m = q - f * TJ; }
    else { f = 2 + (q - 2 * TJ) / TI; m = (q - 2 * TJ) - (f - 2) * TI; }
    // receive: halo column on side f <- neighbour's face f^1
    const int rli = f == 0 ? 0 : (f == 1 ? TI + 1 : 1 + m);
    const int rlj = f == 2 ? 0 : (f == 3 ? TJ + 1 : 1 + m);
    const bool wrap = (f == 2 && tj == 0) || (f == 3 && tj == pl.nj - 1);
    // parity of the source column (the neighbour's cell, across the wrap for y)
    const int si_ = I0 - 1 + rli, sj0 = J0 - 1 + rlj;
    const int sj_ = sj0 == 0 ? g.jm : (sj0 == g.jm + 1 ? 1 : sj0);
    // (halo column, source word, wrap flip | ghost << 1, source parity)
    const int nf = nbr[f];
    const long long src_off = nf >= 0 ? nf * tstride + (f ^ 1) * fstride + m * KKF
                              : nf == -2 ? ghost_w + m * KKF
                              : nf == -3 ? ghost_e + m * KKF
                                         : -1;
    rcvtab[q] = make_int4(colbase(rli, rlj), (int)src_off, (wrap ? wrap_flip : 0) | (nf < -1 ? 2 : 0),
                          (si_ + g.ioff + sj_) & 1);
  }

  // (programmatic dependent launch: everything above used only the launch
  // parameters; p and rhs are the previous kernel's output)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // ---- load tile columns, rhs and halo columns from global memory (warp per
  // column).  Every element is an asynchronous 4-byte copy (cp.async, zero-fill
  // where the value is a constant 0), so all of a thread's loads are in flight
  // at once instead of one L2 round trip per column chunk. ----
  // LESB_RES_TRACE: per-tile stamps of the phases around the pass loop
  unsigned long long* tx = a.trace ? a.trace + ((long long)ntiles * 2 * a.n_iter) * NST + (long long)tile * 8 : nullptr;
  if (tx && tid == 0) tx[0] = gtimer();
  const unsigned sm_s = (unsigned)__cvta_generic_to_shared(S);
  const int ncol_h = (TI + 2) * (TJ + 2);
  for (int col = warp; col < ncol_h; col += RES_WARPS) {
    const int li = col / (TJ + 2), lj = col - li * (TJ + 2);
    const bool ih = li == 0 || li == TI + 1, jh = lj == 0 || lj == TJ + 1;
    if (ih && jh) continue;  // corner columns are never read
    const int i = I0 - 1 + li, j = J0 - 1 + lj;
    const int jj = j == 0 ? g.jm : (j == g.jm + 1 ? 1 : j);
    const bool xphys = ih && ((i == 0 && g.west_bc) || (i == g.im + 1 && g.east_bc));
    // stored halo / neighbour tile's initial value, or (press) the periodic y
    // halo's pre-pass snapshot of its source
    const float* src = a.p + cidx(g, i, PRESS ? jj : j, 0);
    const float* rsrc = a.rhs + cidx(g, i, j, 0);
    const bool inner = !ih && !jh;
    const int cb = colbase(li, lj);
    const int c0 = colour(i + g.ioff, j, 0);
    for (int k = lane; k <= km + 1; k += 32) {
      const bool kh = k == 0 || k == km + 1;
      // press: top / east are 0; bottom / west are remapped at read time
      const bool zero = PRESS && (kh || xphys);
      const unsigned slot = (unsigned)(cb + (c0 ^ (k & 1)) * KK + (k >> 1));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sm_s + 4u * slot), "l"(src + k),
                   "r"(zero ? 0u : 4u)
                   : "memory");
      if (inner && !kh)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sm_s + 4u * (slot + 2u * KK)), "l"(rsrc + k)
                     : "memory");
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (tx && tid == 0) tx[6] = gtimer();
#if RES_BTAB
  // boundary-unit table: each thread writes the entries it will walk
  const int nbu = nbnd * (KKF >> 1);
  for (int w = tid; w < nbu; w += nth) {
    const int c = w / (KKF >> 1);
    btab[w] = btab_entry(coltab[c], pubcol[c], w - c * (KKF >> 1), KK, km);
  }
#endif

  // tags: pass n of this launch is tag0 + n + 2; *epoch advances by the tags
  // a launch uses, so tags never repeat across launches and stale words can
  // never match.  No initial publish: pass 0 needs the neighbours' initial
  // colour-1 faces and pass 1 (across an odd-jm wrap) their initial colour-0
  // faces -- exactly the values the halo columns were just loaded with (from
  // p, whose x-halo planes hold the neighbour slab's values), so those
  // receives are skipped.
  const unsigned tag0 = 1u + *a.epoch;

  if (tx && tid == 0) tx[7] = gtimer();
  // runs: every thread gets about one boundary run and one interior run
  const int nint = ncol - nbnd;
  // interior work items per column: cells (update_run) or slot pairs (update_prun)
  const int KTI = RES_IPAIRS ? (KK >> 1) : KT;
  const int nseg_i = max(1, min(KTI, nint > 0 ? nth / nint : 1));
  const int L_i = (KTI + nseg_i - 1) / nseg_i;
  // pass-invariant decode of this thread's first interior run / boundary pair
  const int nint1 = max(nint, 1);
  const int U_i = nseg_i * nint;  // interior runs
  const int iu0 = tid + (nseg_i - 1) * nint >= U_i ? tid + (nseg_i - 1) * nint - U_i : tid + (nseg_i - 1) * nint;
  const int inu = tid < U_i ? (U_i - 1 - tid) / nth + 1 : 0;
  const int ig0 = iu0 / nint1, icc0 = iu0 - ig0 * nint1;
  const int idg = nth / nint1, idcc = nth - idg * nint1;
#if !RES_BTAB
  const int HPb = KKF >> 1;
  const int bc0 = tid / HPb, bj0 = tid - bc0 * HPb, bdq = nth / HPb, bdr = nth - bdq * HPb;
#endif
  // receive walk over slot PAIRS (face column q, slots sl, sl + 1; sl even):
  // pair w = tid + nth u, one 16-byte load each (two LL words).  The first
  // RCVP pairs of every thread keep their descriptors in registers for the
  // whole solve (source word, halo slot, wrap / ghost bits, and per colour
  // which of the two slots hold a published cell); further pairs are decoded
  // per pass.
  const int HP = KKF >> 1;  // pairs per face column
  const int nrcv = nfc * HP;
  int roff[RCVP], rdst[RCVP];
  unsigned rwrap = 0, rsys = 0, rval0 = 0, rval1 = 0;
#pragma unroll
  for (int u = 0; u < RCVP; ++u) {
    const int w = tid + nth * u;
    const int q = w / HP, sl = 2 * (w - (w / HP) * HP);
    roff[u] = 0;
    rdst[u] = -1;
    if (q < nfc) {
      const int4 e = rcvtab[q];
      if (e.y >= 0) {
        roff[u] = e.y + sl;
        rdst[u] = e.x + sl;
        if (e.z & 1) rwrap |= 1u << u;
        if (e.z & 2) rsys |= 1u << u;  // a ghost slot, written by a neighbour slab
        // only slots holding cells of the source colour were published
        // (bits 2u, 2u+1 of rval<c>: slot sl / sl+1 valid in passes of colour c)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int kps = (((1 - c) ^ (e.z & 1)) + e.w + 1) & 1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int s2 = sl + h;
            const bool valid = kps ? s2 <= ((km - 1) >> 1) : (s2 >= 1 && s2 <= ((km - 2) >> 1) + 1);
            if (valid) (c ? rval1 : rval0) |= 1u << (2 * u + h);
          }
        }
      }
    }
  }
  bool timed_out = false;
  unsigned rwrapm = 0;  // slot-pair bits (2u, 2u + 1) of the wrap pairs
#pragma unroll
  for (int u = 0; u < RCVP; ++u)
    if ((rwrap >> u) & 1u) rwrapm |= 3u << (2 * u);
  double acc = 0.0;

  unsigned long long* tr = a.trace ? a.trace + ((long long)tile * 2 * a.n_iter) * NST : nullptr;
  if (tx && tid == 0) tx[1] = gtimer();
  // the receive loads of pass n (register-held pairs), issued during pass n-1
  unsigned long long v[RCVP][2];
  auto issue_receive = [&](int n) {
    if (RES_DBG(a, 4)) return;
    const unsigned long long* XB1 = a.xbuf + ((n + 3) & 3) * bstride;
    const unsigned long long* XB2 = a.xbuf + ((n + 2) & 3) * bstride;
    const unsigned vm = ((n & 1) ? rval1 : rval0) & (n == 1 ? ~rwrapm : ~0u);
#pragma unroll
    for (int u = 0; u < RCVP; ++u)
      if ((vm >> (2 * u)) & 3u) {
        const unsigned long long* src = (((rwrap >> u) & 1u) ? XB2 : XB1) + roff[u];
        if (SLAB && ((rsys >> u) & 1u)) ld_ll2_sys(src, v[u][0], v[u][1]);
        else ld_ll2(src, v[u][0], v[u][1]);
      }
  };
  for (int n = 0; n < 2 * a.n_iter; ++n) {
    const int nrd = n & 1;
    if (tr && tid == 0) tr[NST * n + 0] = gtimer();
    // Receive the neighbours' faces into this tile's colour-(1-nrd) halo
    // slots: pass n-1's publish, or pass n-2's across an odd-jm periodic wrap.
    // Those slots were last read in pass n-2, which every thread finished
    // before the barrier of pass n-1, so no barrier is needed before this.
    if (n > 0 && !RES_DBG(a, 4)) {
      const unsigned long long* XB1 = a.xbuf + ((n + 3) & 3) * bstride;
      const unsigned long long* XB2 = a.xbuf + ((n + 2) & 3) * bstride;
      const unsigned t1 = tag0 + (unsigned)(n + 1), t2 = tag0 + (unsigned)n;
      float* Sd = S + (1 - nrd) * KK;
      const unsigned vm = (nrd ? rval1 : rval0) & (n == 1 ? ~rwrapm : ~0u);
#pragma unroll
      for (int u = 0; u < RCVP; ++u) {
        const bool w2 = (rwrap >> u) & 1u;
        const unsigned want = w2 ? t2 : t1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!((vm >> (2 * u + h)) & 1u)) continue;
          unsigned spins = 0;
          while ((unsigned)(v[u][h] >> 32) != want && !timed_out && !RES_DBG(a, 1)) {
            if (++spins > (1u << 24)) {  // ~seconds: never hang the GPU
              atomicOr(a.err, 1u);
              timed_out = true;
            }
            if (RES_SPIN_NS) __nanosleep(RES_SPIN_NS);  // (leave the issue slots to warps still updating)
            const unsigned long long* src = (w2 ? XB2 : XB1) + roff[u] + h;
            v[u][h] = (SLAB && ((rsys >> u) & 1u)) ? ld_ll_sys(src) : ld_ll(src);
          }
          if (!RES_PAIRS) Sd[rdst[u] + h] = __uint_as_float((unsigned)v[u][h]);
        }
        // pair layout: both slots in one 8-byte store (a slot without a
        // published cell is a k halo slot of a halo column, never read)
        if (RES_PAIRS && ((vm >> (2 * u)) & 3u))
          *reinterpret_cast<float2*>(Sd + rdst[u]) =
              make_float2(__uint_as_float((unsigned)v[u][0]), __uint_as_float((unsigned)v[u][1]));
      }
      // pairs beyond the register-held ones (large tiles / deep columns), one
      // word at a time
      for (int w0 = RCVP * nth; w0 < nrcv; w0 += nth) {
        const int w = w0 + tid;
        const int q = w / HP, sl0 = 2 * (w - (w / HP) * HP);
        if (q >= nfc) continue;
        const int4 e = rcvtab[q];
        if (e.y < 0) continue;
        const int kps = (((1 - nrd) ^ (e.z & 1)) + e.w + 1) & 1;
        const bool w2 = e.z & 1;
        if (w2 && n == 1) continue;  // initial values, already loaded
        const unsigned want = w2 ? t2 : t1;
        for (int h = 0; h < 2; ++h) {
          const int sl = sl0 + h;
          const bool valid = kps ? sl <= ((km - 1) >> 1) : (sl >= 1 && sl <= ((km - 2) >> 1) + 1);
          if (!valid) continue;
          const unsigned long long* src = (w2 ? XB2 : XB1) + e.y + sl;
          unsigned long long x = (SLAB && (e.z & 2)) ? ld_ll_sys(src) : ld_ll(src);
          unsigned spins = 0;
          while ((unsigned)(x >> 32) != want && !timed_out && !RES_DBG(a, 1)) {
            if (++spins > (1u << 24)) {
              atomicOr(a.err, 1u);
              timed_out = true;
            }
            if (RES_SPIN_NS) __nanosleep(RES_SPIN_NS);
            x = (SLAB && (e.z & 2)) ? ld_ll_sys(src) : ld_ll(src);
          }
          Sd[e.x + sl] = __uint_as_float((unsigned)x);
        }
      }
    }
    __syncthreads();
    if (tr && tid == 0) tr[NST * n + 1] = gtimer();
    unsigned long long* X = a.xbuf + (n & 3) * bstride + (long long)tile * tstride;
    const unsigned tag = tag0 + (unsigned)(n + 2);
    if (nrd == 0) acc = 0.0;  // one residual per iteration: both colour passes
    unsigned long long* XRw = pw ? a.peer_w + (n & 3) * bstride + ghost_e : nullptr;  // west peer's ghost-E slot tj
    unsigned long long* XRe = pe ? a.peer_e + (n & 3) * bstride + ghost_w : nullptr;  // east peer's ghost-W slot tj
    if (!RES_DBG(a, 2))
#if RES_BTAB
      acc += update_boundary_tab<PRESS, SLAB>(a, S, btab, nbu, X, XRw, XRe, tag, nrd, KK, CW, sI);
#else
      acc += update_boundary<PRESS, SLAB>(a, S, coltab, pubcol, X, XRw, XRe, tag, bc0, bj0, bdq, bdr, nbnd, HPb, nrd,
                                         KK, CW, sI, km);
#endif
    if (tr && tid == 0) tr[NST * n + 2] = tr[NST * n + 3] = tr[NST * n + 4] = gtimer();
    if (!RES_DBG(a, 2))
      acc += update_phase<PRESS>(a, S, coltab, nbnd, ncol, nseg_i, ig0, icc0, inu, idg, idcc, L_i, KTI, nrd, KK, CW, sI,
                                 km,
                                 [&] {
                                   if (n + 1 < 2 * a.n_iter) issue_receive(n + 1);
                                 });
    if (tr && tid == 0) tr[NST * n + 5] = gtimer();
    if (nrd == 1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
      if (lane == 0) a.partials[((long long)(n >> 1) * ntiles + tile) * RES_WARPS + warp] = acc;
    }
  }
  __syncthreads();

  if (tx && tid == 0) tx[2] = gtimer();
  // ---- write the tile back (warp per column); press: closed-form halo ----
  unsigned bad = 0;
  for (int c = warp; c < ncol; c += RES_WARPS) {
    const int li = 1 + c / TJ, lj = 1 + (c - (c / TJ) * TJ);
    const int i = I0 - 1 + li, j = J0 - 1 + lj;
    const int cb = colbase(li, lj);
    // targets: the column itself, plus the halo columns whose closed-form
    // source is this column (les.py:341-355: k first, then j, then i)
    int ti_[2] = {i, (PRESS && i == 1 && g.west_bc) ? 0 : -1};  // (a slab's inner x halo is the neighbour's)
    int tj_[3] = {j, (PRESS && j == 1) ? g.jm + 1 : -1, (PRESS && j == g.jm) ? 0 : -1};
    if (!(PRESS && ((i == 1 && g.west_bc) || j == 1 || j == g.jm || (i == g.im && g.east_bc)))) {
      // (warp-uniform) no halo column takes its value from this one: the
      // column itself, with the press k halo (p[0] = p[1], p[km+1] = 0)
      float* dst = a.p + cidx(g, i, j, 0);
      const int c0 = colour(i + g.ioff, j, 0);
      // a column's shared-memory reads first, then its stores (one round of
      // read latency per column instead of one per 32 cells)
      constexpr int WB = 4;
      for (int k0 = 0; k0 <= km + 1; k0 += 32 * WB) {
        float vv[WB];
#pragma unroll
        for (int r = 0; r < WB; ++r) {
          const int k = k0 + lane + 32 * r;
          const int kr = k == 0 ? 1 : (k > km ? km : k);
          vv[r] = k <= km + 1 ? S[cb + (c0 ^ (kr & 1)) * KK + (kr >> 1)] : 0.0f;
        }
#pragma unroll
        for (int r = 0; r < WB; ++r) {
          const int k = k0 + lane + 32 * r;
          if (k > km + 1) continue;
          const float v = vv[r];
          const bool own = k >= 1 && k <= km;
          if (own && !finite32(v)) bad = F_PRESS;
          if (own) dst[k] = v;
          else if (PRESS) dst[k] = (k == km + 1) ? 0.0f : v;
        }
      }
    } else {
      for (int k = lane; k <= km + 1; k += 32) {
        const int kr = k == 0 ? 1 : (k > km ? km : k);
        const float v = S[cb + colour(i + g.ioff, j, kr) * KK + (kr >> 1)];
        const bool own = k >= 1 && k <= km;
        if (own && !finite32(v)) bad = F_PRESS;
        const float hv = (k == km + 1) ? 0.0f : v;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (ti_[x] < 0) continue;
#pragma unroll
          for (int y = 0; y < 3; ++y) {
            if (tj_[y] < 0) continue;
            const bool self = x == 0 && y == 0;
            if (self && !own && !PRESS) continue;  // stored halo: untouched
            a.p[cidx(g, ti_[x], tj_[y], k)] = self && own ? v : hv;
          }
        }
        if (PRESS && i == g.im && g.east_bc) {  // east face is Dirichlet 0 for every j' mapped here
#pragma unroll
          for (int y = 0; y < 3; ++y)
            if (tj_[y] >= 0) a.p[cidx(g, g.im + 1, tj_[y], k)] = 0.0f;
        }
      }
    }
  }
  if (a.pflags) flag_or(a.pflags, bad);

  // ---- residuals: tile b sums iteration b over tiles and warps in a fixed order ----
  if (tx && tid == 0) tx[3] = gtimer();
  cg::this_grid().sync();
  if (tx && tid == 0) tx[4] = gtimer();
  // fresh tags for the next launch (a group's slabs share one epoch word)
  if (tid == 0 && blockIdx.x == 0) {
    *a.epoch += (unsigned)(2 * a.n_iter + 2);
    // every stage's flags are final here (the tiles raised theirs before the barrier)
    if (!SLAB && a.book) step_book_update(a.book);
  }
  const int per_pass = ntiles * RES_WARPS;
  for (int it = tile; it < a.n_iter; it += ntiles) {
    const double* q = a.partials + (long long)it * per_pass;
    double v = 0.0;
    for (int b = tid; b < per_pass; b += nth) v += q[b];
    v = block_sum<RES_WARPS>(v, red);
    __syncthreads();
    if (tid == 0) a.res[it] = v;
  }
  if (tx && tid == 0) tx[5] = gtimer();
}

}  // namespace lesb
