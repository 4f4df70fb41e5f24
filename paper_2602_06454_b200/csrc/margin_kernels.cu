// margin_kernels.cu — K1 relay_margin_rows and K4 relay_step_switch (sm_100a).
//
// One streaming pass over each logit row (§3.2): the softmax
// normaliser in fp32 against a lazily raised exp reference (MUFU.EX2 via
// ex2.approx; FFMA2/FADD2 on element pairs) and the exact top-2 (value desc,
// index asc) behind a CTA-shared threshold, so that only the rare stages that
// can still enter the row's top-2 take the exact per-element path
// (DESIGN.md §6).  HBM-bound by design: algorithmic bytes = vocab *
// sizeof(elem) per row; no tensor cores (a scan, not a contraction).
//
// K1 is a persistent warp-specialised kernel: one producer warp streams row
// bodies into shared-memory rings with 1-D TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx), consumer warps reduce them, an epilogue warp merges
// and finishes each row.  The consumer warps form two groups (NG = 2), each
// with its own ring and barriers, so a CTA streams two rows at once and the
// per-row work is paid by half the warps.  Ring-slot release and the hand-off of a row's
// partials use named barriers (bar.arrive by the consumers, bar.sync by the
// producer / epilogue warp: descheduled, no polling), so the two helper warps
// take no issue slots.  The ring runs across row boundaries, so a row's
// epilogue overlaps the next row's loads.  Steady-state stage per thread: the
// 32 terms, ONE comparison of their sum against the thread's guard T
// (consume_fast), a warp-uniform exact path only when some lane trips.  K4 is
// the same kernel with 12 consumer warps at 2 CTAs/SM, launched with
// programmatic dependent launch: whole rows per CTA when the batch fills the
// SMs, otherwise equal slices of the flattened batch merged by the last
// arriving CTA; its epilogue warp runs RelayGen's switch state machine
// on-device (switch.cuh).  In relay_step_sample it also bounds each row's
// top-k for the sampling kernel (sample_kernels.cu).  Opt-in, measured slower
// and kept for the record: K4 with consumer groups
// (RELAY_K4_GROUPS=1) and K4 drawing the token itself (RELAY_K4_FUSE=1).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "p2p.cuh"
#include "relay_device.cuh"
#include "relay_internal.h"
#include "draw.cuh"
#include "switch.cuh"

namespace relay {

#ifdef RELAY_TRACE
// Tuning-only timeline (tools/trace_rows.py): %globaltimer stamps per CTA.
// Slots: 0 entry, 1-14 ring stage n landed (consumer thread 0), 15 first
// TMA issued, 16-23 consumer item ends, 24-30 epilogue item ends, 31 exit.
constexpr int kTraceSlots = 32;
__device__ unsigned long long g_trace[4096][kTraceSlots];
__device__ __forceinline__ void stamp(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (blockIdx.x < 4096 && k < kTraceSlots) g_trace[blockIdx.x][k] = t;
}
extern "C" int relay_debug_trace_copy(unsigned long long* host, int n_ctas) {
  return static_cast<int>(
      cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * kTraceSlots * n_ctas));
}
extern "C" int relay_debug_trace_reset(const unsigned long long* zeros, int n_ctas) {
  return static_cast<int>(
      cudaMemcpyToSymbol(g_trace, zeros, sizeof(unsigned long long) * kTraceSlots * n_ctas));
}
__device__ unsigned long long g_fuse_stats[4];  // fused draw: rows drawn, rows to K5, candidates
extern "C" int relay_debug_fuse_stats(unsigned long long* host, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(host, g_fuse_stats, sizeof(unsigned long long) * 4);
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_fuse_stats, z, sizeof(z));
  }
  return static_cast<int>(e);
}
#define TRACE(k) stamp(k)
#else
#define TRACE(k) ((void)0)
#endif

#ifndef RELAY_STEADY_UNROLL
#define RELAY_STEADY_UNROLL 1
#endif
constexpr int kSteadyUnroll = RELAY_STEADY_UNROLL;  // steady-stage loop unroll (tuning)

// An opaque copy of a value: the compiler keeps it in a register instead of
// recomputing it in every stage (K1's 64-register budget makes ptxas
// rematerialise addresses it could keep).
__device__ __forceinline__ uint32_t pin_u32(uint32_t v) {
  uint32_t r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

constexpr float kHuge = 268435456.0f;  // 2^28: beyond it fp32 y = z*c is too coarse

struct ThreadState {
  Top2 t;
  float g2;    // own skip guard: NaN until t.i2 holds a real index, then t.v2
  float mref;  // exp reference in the y = z*c domain (never above the row max)
  float acc[4];
  int flags;   // kFlagHuge | kFlagNan
};

__device__ __forceinline__ void state_init(ThreadState& st) {
  st.t = top2_empty();
  st.g2 = qnan();
  st.mref = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < 4; k++) st.acc[k] = 0.0f;
  st.flags = 0;
}

__device__ __forceinline__ void rescale(ThreadState& st, float ymax) {
  if (ymax > st.mref + kSlack) {
    if (fabsf(ymax) >= kHuge) st.flags |= kFlagHuge;
    const float r = ex2(st.mref - ymax);
#pragma unroll
    for (int k = 0; k < 4; k++) st.acc[k] *= r;
    st.mref = ymax;
  }
}

// Exact path for one element (misaligned head/tail of a row range).
__device__ __forceinline__ void consume_scalar(float x, int j, ThreadState& st, float c) {
  if (x != x) st.flags |= kFlagNan;
  top2_push(st.t, x, j);
  st.g2 = (st.t.i2 == INT_MAX) ? qnan() : st.t.v2;
  rescale(st, x * c);
  st.acc[0] += ex2(fmaf(x, c, -st.mref));
}

// Maxima of two disjoint halves of the UV vectors' elements (NaN-propagating):
// lo/hi 16-bit lanes for packed formats, even/odd words for fp32.
template <class E, int UV>
__device__ __forceinline__ float2 stage_max2(const uint4 (&raw)[UV]) {
  if constexpr (E::SZ == 2) {
    uint32_t m[UV];
#pragma unroll
    for (int u = 0; u < UV; u++) m[u] = E::pmax(E::pmax(raw[u].x, raw[u].y), E::pmax(raw[u].z, raw[u].w));
#pragma unroll
    for (int w = 1; w < UV; w <<= 1)
#pragma unroll
      for (int u = 0; u + w < UV; u += 2 * w) m[u] = E::pmax(m[u], m[u + w]);
    float lo, hi;
    E::unpack2(m[0], lo, hi);
    return make_float2(lo, hi);
  } else {
    float a = max_nan(__uint_as_float(raw[0].x), __uint_as_float(raw[0].z));
    float b = max_nan(__uint_as_float(raw[0].y), __uint_as_float(raw[0].w));
#pragma unroll
    for (int u = 1; u < UV; u++) {
      a = max3_nan(a, __uint_as_float(raw[u].x), __uint_as_float(raw[u].z));
      b = max3_nan(b, __uint_as_float(raw[u].y), __uint_as_float(raw[u].w));
    }
    return make_float2(a, b);
  }
}

// Exact top-2 update from the vectors u < nvalid of a stage: only the
// elements that can still enter the row's top-2 are pushed (usually one):
// >= theta (a lower bound of the row's 2nd-best) and above this thread's own
// 2nd-best (indices only grow along a thread's walk).
template <class E, int UV>
__device__ __forceinline__ void exact_top2(const uint4 (&raw)[UV], int nvalid, int j0, int jstep, ThreadState& st,
                                           float theta) {
  constexpr int VEC = 16 / E::SZ;
#pragma unroll
  for (int u = 0; u < UV; u++) {
    const float vm = vec_max<E>(raw[u]);
    if (u < nvalid && vm >= theta && !(vm <= st.g2)) {
      float f[VEC];
      unpack16<E>(raw[u], f);
      unsigned m = 0;
#pragma unroll
      for (int k = 0; k < VEC; k++) m |= (f[k] >= theta && !(f[k] <= st.g2)) ? (1u << k) : 0u;
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        top2_push(st.t, elem_at<E>(raw[u], k), j0 + u * jstep + k);
      }
      st.g2 = (st.t.i2 == INT_MAX) ? qnan() : st.t.v2;
    }
  }
}

// One stage of UV 16-byte vectors; vector u holds elements j0 + u*jstep ..
// + VEC-1, and a thread's vectors are visited in increasing index order.
// The max-guarded form (a row's first stage, where the probe needs the half
// maxima h anyway, and short rows); consume_fast below is the steady state.
template <class E, int UV>
__device__ __forceinline__ void consume_stage(const uint4 (&raw)[UV], float2 h, int j0, int jstep,
                                              ThreadState& st, float c, float theta, bool& slow) {
  constexpr int VEC = 16 / E::SZ;
  const float gm = max_nan(h.x, h.y);
  if (gm != gm) st.flags |= kFlagNan;  // a NaN anywhere in the stage (status 1)
  // A vector can change the row's top-2 only if it holds a value >= theta
  // that also beats this thread's own 2nd-best.
  if (gm >= theta && !(gm <= st.g2)) {
    exact_top2<E, UV>(raw, UV, j0, jstep, st, theta);
    slow = true;
  }
#ifdef RELAY_K1_NULL
  st.acc[0] += gm;  // tuning only: streaming ceiling without the exp work
  return;
#endif
  rescale(st, gm * c);
  const float2 cc = make_float2(c, c);
  const float2 nm = make_float2(-st.mref, -st.mref);
#pragma unroll
  for (int u = 0; u < UV; u++) {
    float f[VEC];
    unpack16<E>(raw[u], f);
#pragma unroll
    for (int k = 0; k < VEC; k += 2) {
      const float2 y = __ffma2_rn(make_float2(f[k], f[k + 1]), cc, nm);
      const float2 e = make_float2(ex2(y.x), ex2(y.y));
      const int a = (((u * VEC + k) >> 1) & 1) * 2;
      const float2 s = __fadd2_rn(make_float2(st.acc[a], st.acc[a + 1]), e);
      st.acc[a] = s.x;
      st.acc[a + 1] = s.y;
    }
  }
}

// Warp top-2 of (a, b) value pairs (a >= b, distinct elements): the result's
// second value bounds the row's 2nd-best from below.
__device__ __forceinline__ float warp_second(float a, float b) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float oa = __shfl_xor_sync(kFull, a, off);
    const float ob = __shfl_xor_sync(kFull, b, off);
    b = fmaxf(fminf(a, oa), fmaxf(b, ob));
    a = fmaxf(a, oa);
  }
  return b;
}

// The CTA-shared threshold key, addressed by its 32-bit shared-window address
// (kept in a register: a generic pointer would re-derive the window base from
// SR_CgaCtaId at every stage).
__device__ __forceinline__ int theta_load(uint32_t a) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ float theta_raise(float b, uint32_t s_theta) {
  if ((threadIdx.x & 31) == 0 && b > unkey(theta_load(s_theta)))
    asm volatile("red.shared.max.s32 [%0], %1;" ::"r"(s_theta), "r"(fkey(b)) : "memory");
  return b;
}

// Sum of the stage's terms 2^(fl(z c - mref)) as two packed partial sums
// (unpack, FFMA2, 2 x MUFU.EX2, FADD2 per element pair: the whole per-element
// cost of the steady state).
// 2^y for an element pair on the FMA pipe (FlashAttention-4's trick: the
// MUFU.EX2 unit, 16 lanes/clk/SM, is the K1 ceiling; the FMA pipe has room).
// y clamped to [-125, 64] (a term below 2^-125 of the reference is 0 to fp32
// accuracy here; above 2^16 the guard trips and the stage is redone, so the
// clamp only keeps the exponent arithmetic in range); n = rint(y) by the
// 1.5*2^23 shifter, 2^(y-n) by a degree-5 minimax polynomial on [-1/2, 1/2]
// (max relative error 2.3e-7 in fp32 Horner, MUFU.EX2's ~2^-22 class), the
// exponent added to the bits.
#ifndef RELAY_K1_POLY_PAIRS
#define RELAY_K1_POLY_PAIRS 0  // K1: element pairs per 16 of a stage on the FMA pipe (power-capped: 0 best)
#endif
#ifndef RELAY_K4_POLY_PAIRS
#define RELAY_K4_POLY_PAIRS 0  // K4: the same for the decode step (XU-bound on the SMs with two rows)
#endif
__device__ __forceinline__ float2 exp2_poly2(float2 y) {
  y.x = fminf(fmaxf(y.x, -125.0f), 64.0f);
  y.y = fminf(fmaxf(y.y, -125.0f), 64.0f);
  const float2 t = __fadd2_rn(y, make_float2(12582912.0f, 12582912.0f));
  const float2 tm = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __fadd2_rn(y, make_float2(-tm.x, -tm.y));
  float2 h = __ffma2_rn(make_float2(1.327647129073739e-3f, 1.327647129073739e-3f), f,
                        make_float2(9.675541892647743e-3f, 9.675541892647743e-3f));
  h = __ffma2_rn(h, f, make_float2(5.550713092088699e-2f, 5.550713092088699e-2f));
  h = __ffma2_rn(h, f, make_float2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  h = __ffma2_rn(h, f, make_float2(6.931469440460205e-1f, 6.931469440460205e-1f));
  h = __ffma2_rn(h, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__uint_as_float(__float_as_uint(h.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(h.y) + (__float_as_uint(t.y) << 23)));
}

template <class E, int UV, int POLY>
__device__ __forceinline__ float2 stage_sum(const uint4 (&raw)[UV], int nvalid, float c, float mref) {
  constexpr int VEC = 16 / E::SZ;
  constexpr int NP = VEC / 2;  // element pairs per vector
  constexpr int kPoly = POLY * UV * NP / 16;  // the stage's last kPoly pairs on the FMA pipe
  const float2 cc = make_float2(c, c);
  const float2 nm = make_float2(-mref, -mref);
  // a sum tree, not accumulator chains: each vector's exps are independent of
  // the previous vector's adds, so the scheduler keeps many MUFU.EX2 in flight
  // (with chains it serialised unpack -> FFMA2 -> MUFU -> FADD2 pair by pair)
#ifdef RELAY_K1_NULL
  // tuning only: the streaming ceiling without the exp work (a 0/1 term per
  // stage from the words, so nothing is optimised away)
  uint32_t x = 0;
#pragma unroll
  for (int u = 0; u < UV; u++) x ^= raw[u].x ^ raw[u].y ^ raw[u].z ^ raw[u].w;
  return make_float2(static_cast<float>(x & 1u), 0.0f);
#endif
  float2 t[UV];
#pragma unroll
  for (int u = 0; u < UV; u++) {
    if (u >= nvalid) {  // a partial stage's missing vectors (nvalid == UV otherwise: folded away)
      t[u] = make_float2(0.0f, 0.0f);
      continue;
    }
    float f[VEC];
    unpack16<E>(raw[u], f);
    float2 e[NP];
#pragma unroll
    for (int k = 0; k < NP; k++) {
      const float2 y = __ffma2_rn(make_float2(f[2 * k], f[2 * k + 1]), cc, nm);
      if (u * NP + k >= UV * NP - kPoly)
        e[k] = exp2_poly2(y);
      else
        e[k] = make_float2(ex2(y.x), ex2(y.y));
    }
#pragma unroll
    for (int w = 1; w < NP; w <<= 1)
#pragma unroll
      for (int k = 0; k + w < NP; k += 2 * w) e[k] = __fadd2_rn(e[k], e[k + w]);
    t[u] = e[0];
  }
#pragma unroll
  for (int w = 1; w < UV; w <<= 1)
#pragma unroll
    for (int u = 0; u + w < UV; u += 2 * w) t[u] = __fadd2_rn(t[u], t[u + w]);
  return t[0];
}

// The steady-state guard of a thread: every term of a stage is below
// T = 2^(fl(max(theta, g2) c - mref) - eps) iff no element reaches
// max(theta, own 2nd-best) — then nothing in the stage can enter the row's
// top-2 — and T <= 2^16 also keeps every term under the lazy reference's
// slack.  fl(z c - mref) is monotone in z and MUFU.EX2's relative error
// (~2^-22) is far below eps, so an element >= the bound always gives a term
// >= T; a term can only trip the guard falsely, which costs one exact check.
constexpr float kGuardEps = 1.0f / 1024.0f;
constexpr float kGuardCap = 65536.0f;  // 2^kSlack

__device__ __forceinline__ float guard_T(float theta, const ThreadState& st, float c) {
  return fminf(ex2(fmaf(fmaxf(theta, st.g2), c, -st.mref) - kGuardEps), kGuardCap);
}

// Steady-state stage: the terms first, then ONE comparison of their sum
// against the thread's guard T (the sum is >= every term, exactly: rounding
// is monotone).  Only when it trips does the thread take the stage maxima,
// the exact top-2 update and the reference raise, so the common stage costs
// the exp work plus ~0.2 instructions per element (no per-stage max tree).
// nvalid < UV on a row's last, partial stage: the missing vectors hold -inf
// (no term, never pushed).
template <class E, int UV, int POLY>
__device__ __forceinline__ void consume_fast(const uint4 (&raw)[UV], int nvalid, int j0, int jstep,
                                             ThreadState& st, float c, float& T, int& tkey, float& theta_w,
                                             int key, uint32_t theta_p) {
  float2 s2 = stage_sum<E, UV, POLY>(raw, nvalid, c, st.mref);
  const float s = s2.x + s2.y;
#ifndef RELAY_K1_KEY_PRED
  // T follows the shared threshold (key: loaded with the stage, before the
  // ring words, so its latency hides under the sum): a stale (lower) T stays
  // correct, but every thread would trip on the elements between the old and
  // the new theta.  The key test joins the guard's vote, so the common stage
  // issues no T update at all (a predicated update cost 9 instructions per
  // stage, MUFU included: profiles/r02/k1_sass_lines.txt).
  if (!__any_sync(kFull, !(s < T) || key != tkey)) {
    const float2 acc = __fadd2_rn(make_float2(st.acc[0], st.acc[1]), s2);
    st.acc[0] = acc.x;
    st.acc[1] = acc.y;
    return;
  }
  if (key != tkey) {
    tkey = key;
    T = guard_T(fmaxf(theta_w, unkey(key)), st, c);
  }
#else
  if (key != tkey) {
    tkey = key;
    T = guard_T(fmaxf(theta_w, unkey(key)), st, c);
  }
#endif
  // warp-uniform: when any lane trips, the whole warp takes the exact path
  // (it would execute it anyway) and the warp's threshold raise joins it
  if (__any_sync(kFull, !(s < T))) {
    // the raw words again, opaque: the unpacked values of the sum above are
    // not kept live across it for the rare exact path (register spills)
    uint4 rw[UV];
#pragma unroll
    for (int u = 0; u < UV; u++) rw[u] = opaque(raw[u]);
    const float theta = fmaxf(theta_w, unkey(key));
    const float2 h = stage_max2<E, UV>(rw);
    const float gm = max_nan(h.x, h.y);
    if (gm != gm) st.flags |= kFlagNan;
    bool pushed = false;
    if (gm >= theta && !(gm <= st.g2)) {
      exact_top2<E, UV>(rw, nvalid, j0, jstep, st, theta);
      pushed = true;
    }
    // raise the reference to the stage maximum when a term passed the slack,
    // or when the stage sum alone is large (terms bunched near the slack:
    // every later stage would trip the guard again)
    const float ym = gm * c;
    if (ym > st.mref + kSlack || (ym > st.mref && !(s < 0.5f * kGuardCap))) {
      if (fabsf(ym) >= kHuge) st.flags |= kFlagHuge;
      const float r = ex2(st.mref - ym);
#pragma unroll
      for (int k = 0; k < 4; k++) st.acc[k] *= r;
      st.mref = ym;
      s2 = stage_sum<E, UV, POLY>(rw, nvalid, c, ym);  // the old terms may have overflowed (or been clamped)
    }
    if (__any_sync(kFull, pushed)) theta_w = fmaxf(theta_w, theta_raise(warp_second(st.t.v1, st.t.v2), theta_p));
    T = guard_T(fmaxf(theta_w, unkey(key)), st, c);  // mref, g2 or theta_w may have moved
  }
  const float2 acc = __fadd2_rn(make_float2(st.acc[0], st.acc[1]), s2);
  st.acc[0] = acc.x;
  st.acc[1] = acc.y;
}

__device__ __forceinline__ Partial thread_partial(const ThreadState& st) {
  return Partial{st.t, Norm{st.mref, (st.acc[0] + st.acc[1]) + (st.acc[2] + st.acc[3])}, st.flags};
}

__device__ __forceinline__ Partial partial_empty() {
  return Partial{top2_empty(), Norm{-FLT_MAX, 0.0f}, 0};
}

// Row geometry: `head` scalar elements up to the first 16-byte boundary, a
// 16-byte-aligned body, then scalar tail elements from `tail`.
struct Geom {
  int head;
  int body;  // bytes, multiple of 16 (< 2^31: validated on the host)
  int tail;
};

template <class E>
__device__ __forceinline__ Geom row_geom(const typename E::T* row, int j0, int j1) {
  Geom g;
  const uintptr_t a = reinterpret_cast<uintptr_t>(row + j0);
  int head = static_cast<int>(((16 - (a & 15)) & 15) / E::SZ);
  if (head > j1 - j0) head = j1 - j0;
  g.head = head;
  g.body = ((j1 - j0 - head) * E::SZ) & ~15;
  g.tail = j0 + head + g.body / E::SZ;
  return g;
}

// Exact normaliser pass for rows flagged huge: S = sum_j 2^((z_j - z1) c),
// the difference taken first (exact near the maximum by Sterbenz).
template <class E>
__device__ __forceinline__ float exact_sum_thread(const typename E::T* row, int vocab, float z1,
                                                  float c, int tid, int nthreads) {
  float s = 0.0f;
  for (int j = tid; j < vocab; j += nthreads) {
    const float z = E::load1(row + j);
    s += ex2((z - z1) * c);
  }
  return s;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  return v;
}

// ------------------------------------------- fused top-k draw (N2, K4)
constexpr int kFuseCap = 512;  // candidates per row held in shared memory (more: the row goes to K5)
static_assert(kFuseCap >= 128, "fuse_raise reads the first 128 entries");
constexpr int kFuseSeed = 8;   // first-stage seeds per warp (NCW * kFuseSeed >= kMaxTopK)
constexpr int kFuseRank = 128; // candidates >= the final bound that the epilogue ranks (more: K5)

// Every finite element >= B of the vectors u < nvalid into the row's
// candidate list (one slot reservation per vector; NaN never qualifies).
constexpr int kFuseRaise = 48;  // the list raises its bound each time it grows past a multiple of this

template <class E, int UV>
__device__ __forceinline__ bool fuse_push(const uint4 (&raw)[UV], int nvalid, int j0, int jstep, float B,
                                          float* fv, int* fi, int* fcnt) {
  constexpr int VEC = 16 / E::SZ;
  bool crossed = false;
#pragma unroll
  for (int u = 0; u < UV; u++) {
    if (u < nvalid && vec_max<E>(raw[u]) >= B) {
      float f[VEC];
      unpack16<E>(raw[u], f);
      unsigned m = 0;
#pragma unroll
      for (int k = 0; k < VEC; k++) m |= (f[k] >= B && f[k] > -INFINITY) ? (1u << k) : 0u;
      if (m) {
        int p = atomicAdd(fcnt, __popc(m));
        crossed |= p / kFuseRaise != (p + __popc(m)) / kFuseRaise;
        while (m) {
          const int k = __ffs(m) - 1;  // (elem_at: no local-memory copy of f[])
          m &= m - 1;
          if (p < kFuseCap) { fv[p] = elem_at<E>(raw[u], k); fi[p] = j0 + u * jstep + k; }
          p++;
        }
      }
    }
  }
  return crossed;
}

// Raise the list's shared bound to the topk-th largest of its first 128
// entries (distinct elements of the row; slots reserved but not yet written
// still hold -inf, so the result never exceeds a true lower bound).  One warp.
__device__ __forceinline__ void fuse_raise(const float* fv, int topk, int* bkey) {
  const int lane = threadIdx.x & 31;
  const volatile float* v = fv;
  float x0 = v[lane], x1 = v[lane + 32], x2 = v[lane + 64], x3 = v[lane + 96];
  float m = -INFINITY;
  for (int i = 0; i < topk; i++) {
    const float lm = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
    m = unkey(__reduce_max_sync(kFull, fkey(lm)));
    if (m == -INFINITY) return;
    const unsigned holders = __ballot_sync(kFull, lm == m);
    if (lane == __ffs(holders) - 1) {
      if (x0 == m) x0 = -INFINITY; else if (x1 == m) x1 = -INFINITY; else if (x2 == m) x2 = -INFINITY;
      else x3 = -INFINITY;
    }
  }
  if (lane == 0) atomicMax(bkey, fkey(m));
}

// The warp's kFuseSeed largest of its lanes' two (distinct) first-stage half
// maxima into seed[] (NaN read as -inf).
__device__ __forceinline__ void fuse_seeds(float2 h, float* seed) {
  const int lane = threadIdx.x & 31;
  float x0 = h.x == h.x ? h.x : -INFINITY, x1 = h.y == h.y ? h.y : -INFINITY;
#pragma unroll 1
  for (int i = 0; i < kFuseSeed; i++) {
    const float lm = fmaxf(x0, x1);
    const float m = unkey(__reduce_max_sync(kFull, fkey(lm)));
    const unsigned holders = __ballot_sync(kFull, lm == m);
    if (lane == __ffs(holders) - 1) {
      if (x0 == m) x0 = -INFINITY; else x1 = -INFINITY;
    }
    if (lane == 0) seed[i] = m;
  }
}

// The topk-th largest of the n <= 96 seeds (distinct elements of the row): a
// lower bound on the row's topk-th largest logit (-inf with fewer than topk
// finite).  Lane l holds seeds l, l + 32, l + 64; topk rounds of a warp max
// with one holder removing its entry.
__device__ __forceinline__ float fuse_bound(const float* seeds, int n, int topk) {
  const int lane = threadIdx.x & 31;
  float x0 = lane < n ? seeds[lane] : -INFINITY;
  float x1 = lane + 32 < n ? seeds[lane + 32] : -INFINITY;
  float x2 = lane + 64 < n ? seeds[lane + 64] : -INFINITY;
  float m = -INFINITY;
  for (int i = 0; i < topk; i++) {
    const float lm = fmaxf(fmaxf(x0, x1), x2);
    m = unkey(__reduce_max_sync(kFull, fkey(lm)));
    if (m == -INFINITY) break;
    const unsigned holders = __ballot_sync(kFull, lm == m);
    if (lane == __ffs(holders) - 1) {
      if (x0 == m) x0 = -INFINITY; else if (x1 == m) x1 = -INFINITY; else x2 = -INFINITY;
    }
  }
  return m;
}

// ------------------------------------------------- K1 / K4 row kernel
// Work items are (row, element range, part) triples (Item, ItemIter below).
// K1 takes whole rows; K4 whole rows or, for small batches, parts of rows
// merged by the last arriving CTA (arrival counter, reset after use so CUDA
// graph replays need no reset).
struct RowsArgs {
  const void* logits;
  long long n_rows;
  int vocab;
  long long stride;
  float c, iota;
  int flat;       // 0: one item per row, rows strided over CTAs (K1)
                  // 1: each CTA takes an equal slice of the flattened rows
                  // 3: hybrid: n_whole CTAs take one whole row each, the
                  //    others equal slices of the remaining rows (K4)
                  // 4: cluster: rows dealt to thread-block clusters, each
                  //    cluster's rows sliced equally over its CTAs; row parts
                  //    merged in the owner CTA's shared memory over DSMEM (K4)
                  // 2: rows cut into `chunk`-element chunks handed out by an
                  //    atomic work counter (K4; balances uneven SM service)
  float* margin;
  int* top1;
  int* top2;
  float* lse;
  uint8_t* status;
  int* counter;   // [n_rows] arrival counters (flat)
  float* part;    // [n_rows][kMaxSplit][kPartWords] row-part partials (flat)
  int* work;      // [2] dynamic mode: next chunk, CTAs done (zero between launches)
  int chunk;      // dynamic mode: elements per chunk (a multiple of a ring stage)
  long long n_whole;  // hybrid mode: rows taken whole (one per CTA)
  int csize;          // cluster mode (flat == 4): CTAs per thread-block cluster
  int cpr;        // dynamic mode: chunks per row (<= kMaxSplit)
  // vocabulary-parallel partials (kModePartial)
  long long col_offset;  // global index of the shard's first column
  float* tp_part;        // [n_rows][kPartWords] (or NULL with tp_peers)
  TpPeers tp;            // relay_margin_rows_tp: the partial goes straight to every rank (tp.world > 0)
  // decode-step switch (kModeStep)
  const int* sampled;
  uint8_t* state;
  int* hist;
  int* small_run;
  float gate;
  int max_seg;
  uint8_t* flag;
  int16_t* cue_id;
  // fused-sampler margin pass (relay_step_sample, N2): per row a lower bound
  // on the topk-th largest logit; the switch is left to the sampling kernel
  float* thk;     // [n_rows] or NULL
  float* zmax;    // [n_rows] with thk: the row maximum (the sampler's reference)
  int topk;       // 0 = off
  int keep_l2;    // L2 evict_last: the sampling kernel reads the rows again
  int* ready_q;   // relay_step_sample: rows pushed in completion order (release), so
  int* q_ctl;     // K5 samples a row as soon as its margin pass is done (q_ctl[0]: head)
  // relay_step_sample with a top-k, whole rows: the draw fused into this pass
  // (every finite logit >= a first-stage bound on the top_k-th largest is
  // collected in shared memory; the epilogue ranks, draws and switches); rows
  // whose candidates overflow go to K5 as before (queue entry r + 1; fused
  // rows are queued as -(r + 1), which K5 skips)
  int fuse;
  float s_c;             // log2(e) / temperature
  float topp;
  const float* uniform;  // [n_rows]
  int* sampled_out;      // [n_rows] the drawn tokens
};

// The epilogue's view of a row's candidate list (fused top-k draw).
struct FuseIn {
  bool on;
  int n;             // candidates pushed (> kFuseCap: overflowed)
  float thk;         // the final lower bound on the top_k-th largest logit
  float u;           // the row's uniform
  const float* fv;
  const int* fi;
  float* rv;         // [kFuseRank] scratch
  int* ri;
  float* topv;       // [kMaxTopK] the ranked top-k
  int* topi;
};

// The drawn token of a row from its candidate list (one warp, R20 as in K5:
// the exact top-k in (value desc, index asc) order, temperature, top-p,
// inverse CDF), -1 for a row that is not sampled (status != 0), INT_MIN when
// the list cannot give the top-k (overflow, or too many candidates at or
// above the final bound): K5 samples that row from the logits.
__device__ __forceinline__ int fused_draw(const RowsArgs& a, int status, const FuseIn& f) {
  const int lane = threadIdx.x & 31;
  if (status != 0) return -1;
  if (f.n > kFuseCap) return INT_MIN;
  // the candidates >= thk, compacted in list order
  int m = 0;
  for (int base = 0; base < f.n; base += 32) {
    const int e = base + lane;
    const bool take = e < f.n && f.fv[e] >= f.thk;
    const unsigned b = __ballot_sync(kFull, take);
    if (take) {
      const int p = m + __popc(b & ((1u << lane) - 1u));
      if (p < kFuseRank) { f.rv[p] = f.fv[e]; f.ri[p] = f.fi[e]; }
    }
    m += __popc(b);
  }
  if (m > kFuseRank) return INT_MIN;
  __syncwarp();
  // rank of each: the entries before it (distinct indices: distinct ranks)
  const int K = min(a.topk, m);
  for (int e = lane; e < m; e += 32) {
    const float v = f.rv[e];
    const int i = f.ri[e];
    int rank = 0;
    for (int g = 0; g < m; g++) rank += better(f.rv[g], f.ri[g], v, i);
    if (rank < K) { f.topv[rank] = v; f.topi[rank] = i; }
  }
  __syncwarp();
  if (K == 0) return -1;
  return draw_topk_warp(a.s_c, a.topp, f.u, K, f.topv, f.topi);
}

constexpr int kPartWords = 8;  // v1 v2 i1 i2 m s flags pad
constexpr int kXSlots = 4;     // cluster mode: rows a CTA owns at once (consecutive: distinct mod 4)
constexpr int kXParts = 8;     // cluster mode: parts per row (<= CTAs per cluster)
constexpr int kModeRows = 0;     // K1: margins of whole rows
constexpr int kModeStep = 1;     // K4: margins + the decode-step switch
constexpr int kModePartial = 2;  // N1: per-row partials of a vocabulary shard

// Arrival counter increment with acquire-release semantics at GPU scope: the
// part written before it is visible to the last arriver, which then reads
// every part after it (one fused fence + atomic).
__device__ __forceinline__ int atomic_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ SwitchIn load_switch_in(const RowsArgs& a, long long r) {
  return load_switch_in(a.hist, a.state, a.small_run, a.sampled, r);
}

// Warp-level finish of row r from its merged partial (lane 0 writes).
template <class E, int MODE>
__device__ __forceinline__ void finish_item(const RowsArgs& a, const CueDev& cs, const SmemCue& sc,
                                            long long r, const Partial& q, bool exact, float S,
                                            const SwitchIn& in, int best = -2, const FuseIn* fuse = nullptr,
                                            bool* drawn = nullptr) {
  const int lane = threadIdx.x & 31;
  if constexpr (MODE == kModePartial) {
    // vocabulary shard: top-2 with GLOBAL indices and the normaliser relative
    // to the shard maximum, S_rel = sum_j 2^((z_j - v1) c), shift removed
    // (every lane holds the merged partial)
    float srel = 0.0f;
    if (exact) {
      srel = S;
    } else if (q.t.v1 != -INFINITY && q.t.v1 != INFINITY) {
      const float My = q.t.v1 * a.c;
      srel = q.n.s * ex2((q.n.m - My) - fmaf(q.t.v1, a.c, -My));
    }
    float w[kPartWords];
    w[0] = q.t.v1;
    w[1] = q.t.v2;
    w[2] = __int_as_float(q.t.i1 == INT_MAX ? INT_MAX : static_cast<int>(q.t.i1 + a.col_offset));
    w[3] = __int_as_float(q.t.i2 == INT_MAX ? INT_MAX : static_cast<int>(q.t.i2 + a.col_offset));
    w[4] = srel;
    w[5] = __int_as_float(q.flags & kFlagNan);
    w[6] = 0.0f;
    w[7] = 0.0f;
    if (a.tp.world > 0) {
      // the exchange fused into the epilogue: lane k stores the row's partial
      // into rank k's receive buffer (NVLink P2P stores for peers), the tag
      // last with release semantics, so the transfer overlaps the stream
      if (lane < a.tp.world) {
        const unsigned tag = static_cast<unsigned>(*reinterpret_cast<const volatile int*>(a.tp.epoch)) + 1u;
        float* dst = a.tp.recv[lane] +
                     ((static_cast<long long>(tag & 1u) * a.tp.world + a.tp.rank) * a.tp.rows_cap + r) * kPartWords;
        reinterpret_cast<float4*>(dst)[0] = make_float4(w[0], w[1], w[2], w[3]);
        reinterpret_cast<float2*>(dst)[2] = make_float2(w[4], w[5]);
        dst[6] = 0.0f;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst + 7), "r"(tag) : "memory");
      }
      return;
    }
    if (lane == 0) {
      float* pw = a.tp_part + static_cast<size_t>(r) * kPartWords;
#pragma unroll
      for (int k = 0; k < kPartWords; k++) pw[k] = w[k];
    }
    return;
  }
  const RowOut o = finish_row(q, a.c, a.iota, exact, S);
  if (lane == 0) {
    a.margin[r] = o.margin;
    if (a.top1) a.top1[r] = o.i1;
    if (a.top2) a.top2[r] = o.i2;
    if (a.lse) a.lse[r] = o.lse;
    if (a.status) a.status[r] = static_cast<uint8_t>(o.status);
  }
  if constexpr (MODE == kModeStep) {
    int tok;
    if (a.thk) {
      // relay_step_sample: the fused draw, else the sampling kernel (K5)
      // draws and runs the switch
      if (!fuse || !fuse->on) return;
      tok = fused_draw(a, o.status, *fuse);
#ifdef RELAY_TRACE
      if (lane == 0 && blockIdx.x < 4096 && g_trace[blockIdx.x][23] == 0) TRACE(23);
#endif
      if (tok == INT_MIN) return;
      *drawn = true;
      if (lane == 0) a.sampled_out[r] = tok;
      best = -2;
    } else {
      tok = a.sampled ? in.sampled : o.i1;
    }
    switch_warp(cs, sc, tok, o.margin, in, a.state + r, a.hist + r * kHist,
                a.small_run ? a.small_run + r : nullptr, a.gate, a.max_seg, a.flag + r, a.cue_id + r, a.sampled ? best : -2);
  }
}

// Work items.  Strided mode: item i of a CTA is row blockIdx.x + i*gridDim.x,
// whole.  Flat mode: the n_rows*vocab elements are cut into gridDim.x equal
// slices (boundaries on 64-element multiples); a CTA's slice splits at row
// boundaries into 1-3 row parts, so every CTA streams the same number of bytes
// however few rows there are.  A row's parts are merged by the last arriver.
struct Item {
  long long r;
  int j0, j1;     // element range of the row
  int part, nparts;
};

// FLAT = false (K1, the TP partials: always whole rows, strided) lets the
// compiler drop the 64-bit slice state from the consumer loop's live set.
// SPLIT: 0 whole rows only, 1 flat slices only (K4's balanced split: no
// dynamic / hybrid / cluster code in the instantiation), 2 every mode (tuning).
template <int SPLIT>
__device__ __forceinline__ int flat_mode(const RowsArgs& a) {
  if constexpr (SPLIT == 0) return 0;
  else if constexpr (SPLIT == 1) return a.flat ? 1 : 0;
  else return a.flat;
}

template <int SPLIT>
struct ItemIter {
  static constexpr bool FLAT = SPLIT != 0;
  long long next_w;  // strided: next row
  long long e, E1;   // flat: next element, end of this CTA's slice
  long long row0;    // flat: first row of the sliced region (hybrid: the rows after the whole ones)
  long long T, G, b; // flat: elements of the sliced region, its CTAs, this CTA's index among them

  // Slice boundaries by floating point (no 64-bit integer division on the
  // producer's critical path): any monotone rounding gives consistent slices,
  // because every warp and CTA evaluates the same expression and owner()
  // corrects its estimate against slice_start itself.  T < 2^51 (host-checked).
  __device__ static long long slice_start(long long b, long long T, long long G, double Tg) {
    if (b >= G) return T;
    return static_cast<long long>(static_cast<double>(b) * Tg) & ~63LL;
  }
  // the CTA whose (non-empty) slice holds element e
  __device__ static long long owner(long long e, long long T, long long G, double Tg) {
    long long b = static_cast<long long>(static_cast<double>(e) / Tg);
    if (b >= G) b = G - 1;
    while (b > 0 && slice_start(b, T, G, Tg) > e) b--;
    while (b + 1 < G && slice_start(b + 1, T, G, Tg) <= e) b++;
    return b;
  }
  __device__ void init(const RowsArgs& a) {
    next_w = blockIdx.x;
    e = E1 = 0;
    if (!FLAT) return;
    if (flat_mode<SPLIT>(a) == 4) {
      // cluster c = blockIdx / csize takes rows [c R / C, (c + 1) R / C)
      const long long C = gridDim.x / a.csize, c = blockIdx.x / a.csize;
      row0 = c * a.n_rows / C;
      const long long row1 = (c + 1) * a.n_rows / C;
      T = (row1 - row0) * a.vocab;
      G = a.csize;
      b = blockIdx.x % a.csize;
      const double Tg = static_cast<double>(T) / static_cast<double>(G);
      e = slice_start(b, T, G, Tg);
      E1 = slice_start(b + 1, T, G, Tg);
    } else if (flat_mode<SPLIT>(a) == 1 || flat_mode<SPLIT>(a) == 3) {
      // hybrid (3): CTAs [0, n_whole) take rows [0, n_whole) whole; the rest
      // slice rows [n_whole, n_rows) equally (one whole row plus an equal
      // share of the rest per SM, instead of one or two whole rows)
      const long long nw = flat_mode<SPLIT>(a) == 3 ? a.n_whole : 0;
      row0 = nw;
      T = (a.n_rows - nw) * a.vocab;
      G = gridDim.x - nw;
      b = static_cast<long long>(blockIdx.x) - nw;
      if (b >= 0) {
        const double Tg = static_cast<double>(T) / static_cast<double>(G);
        e = slice_start(b, T, G, Tg);
        E1 = slice_start(b + 1, T, G, Tg);
      }
    }
  }
  // dynamic mode: chunk k of the n_rows * cpr chunks
  __device__ static Item from_k(const RowsArgs& a, long long k) {
    // k < 2^31 (host-checked): 32-bit division
    const long long r = static_cast<unsigned>(k) / static_cast<unsigned>(a.cpr);
    const int ch = static_cast<int>(k - r * a.cpr);
    const int j0 = ch * a.chunk;
    return Item{r, j0, min(a.vocab, j0 + a.chunk), ch, a.cpr};
  }
  __device__ bool next(const RowsArgs& a, Item& it) {
    if (!FLAT || !flat_mode<SPLIT>(a) || (flat_mode<SPLIT>(a) == 3 && b < 0)) {
      const bool hyb = FLAT && flat_mode<SPLIT>(a) == 3;
      if (next_w >= (hyb ? a.n_whole : a.n_rows)) return false;
      it = Item{next_w, 0, a.vocab, 0, 1};
      next_w = hyb ? a.n_whole : next_w + gridDim.x;  // hybrid: one whole row
      return true;
    }
    if (e >= E1) return false;
    const long long V = a.vocab;
    const double Tg = static_cast<double>(T) / static_cast<double>(G);
    long long r = static_cast<long long>(static_cast<double>(e) / static_cast<double>(V));
    while (r * V > e) r--;
    while ((r + 1) * V <= e) r++;
    it.r = row0 + r;
    it.j0 = static_cast<int>(e - r * V);
    it.j1 = static_cast<int>(min(V, E1 - r * V));
    const long long first = owner(r * V, T, G, Tg);
    it.part = static_cast<int>(b - first);
    it.nparts = static_cast<int>(owner(r * V + V - 1, T, G, Tg) - first + 1);
    e = (r + 1) * V;
    return true;
  }
};

// Next item of a consumer / epilogue warp.  Static modes compute it; in the
// dynamic mode the producer publishes each chunk it claimed in s_item[slot]
// (-1 = no more) and completes ifull[slot].  The producer refills a slot only
// after the epilogue released it (rempty), which happens after every consumer
// and the epilogue read it, so no waiter can miss a phase.
template <int SPLIT>
__device__ __forceinline__ bool fetch_item(const RowsArgs& a, ItemIter<SPLIT>& iter, int it, int nslots,
                                           const long long* s_item, uint32_t ifull_s, Item& item) {
  if (flat_mode<SPLIT>(a) != 2) return iter.next(a, item);
  const int slot = it % nslots;
  mbar_wait(ifull_s + 8 * slot, (it / nslots) & 1);
  const long long k = *reinterpret_cast<const volatile long long*>(s_item + slot);
  if (k < 0) return false;
  item = ItemIter<SPLIT>::from_k(a, k);
  return true;
}

// Warp roles: NCW consumer warps stream stages; warp NCW is the TMA producer;
// warp NCW+1 is the epilogue warp, which merges an item's partials, finishes
// the row (or publishes a part and, as last arriver, merges the row) and runs
// the decode-step switch — so consumer warps never wait for an epilogue.
// Items rotate over NSLOT reduction slots guarded by mbarriers.
constexpr int kSlots = 4;


template <class E, int NCW, int NS, int UV, int MINB, int MODE, int SPLIT, bool FUSE = false, int NG = 1>
__global__ void __launch_bounds__((NCW + 2) * 32, MINB) rows_kernel(RowsArgs a, CueDev cs) {
  using T = typename E::T;
  constexpr int VEC = 16 / E::SZ;          // elements per 16-byte vector
  constexpr int NCT = NCW * 32;             // consumer threads
  // NG consumer groups (K4 with more rows than SMs: one CTA per SM streams
  // its rows b and b + grid CONCURRENTLY, one group each, so an SM's two rows
  // finish together instead of one CTA of a co-resident pair being starved
  // of issue slots and HBM share until the other is done); each group has
  // its own ring of NS stages, its own barriers and its own items
  static_assert(NG == 1 || (SPLIT == 0 && !FUSE && NCW % NG == 0 && kSlots % NG == 0), "consumer groups");
  constexpr int NCWG = NCW / NG;            // consumer warps per group
  constexpr int NCTG = NCWG * 32;           // consumer threads per group
  constexpr int SB = UV * NCTG * 16;        // bytes per ring stage (one group's)
  // partials handed to the epilogue per consumer warp: 8 after two shuffle
  // rounds (K1: the epilogue is off the critical path), 1 after a full warp
  // reduction (K4: the epilogue is the tail of a ~30 us kernel)
  constexpr int RPW = (MODE == kModeStep) ? 1 : 8;
  constexpr int NRED = NCW * RPW;
  // named barriers: 0 __syncthreads, 1 the consumers' row-start probe,
  // kBarRing0 + s ring stage s released (consumers arrive, the producer warp
  // syncs), kBarRed0 + k reduction slot k filled (consumers arrive, the
  // epilogue warp syncs)
  constexpr int kBarRing0 = 2;              // + g * NS + s: group g's stage s
  constexpr int kBarRed0 = kBarRing0 + NG * NS;
  // SPLIT: the work-split modes that cut rows across CTAs (K4 small batches
  // and tuning modes); the whole-row instantiations carry none of that code
  const int fmode = flat_mode<SPLIT>(a);  // compile-time constant unless SPLIT == 2
  constexpr int kPolyPairs = MODE == kModeStep ? RELAY_K4_POLY_PAIRS : RELAY_K1_POLY_PAIRS;
  static_assert(kBarRed0 + kSlots <= 16, "named barriers");
  static_assert(!FUSE || NCW * kFuseSeed <= 96, "fuse_bound holds three seeds per lane");
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[NG * NS];
  __shared__ __align__(8) uint64_t red_empty[kSlots];
  __shared__ __align__(8) uint64_t ifull[kSlots];
  __shared__ long long s_item[kSlots];
  __shared__ int s_theta[kSlots];
  __shared__ float s_thk[kSlots][NCW];
  // fused top-k draw (FUSE instantiation only): two candidate lists (item it
  // uses it & 1; the epilogue releases a list before the consumers reach item
  // it + 2), the first-stage seeds, the ranked top-k
  constexpr int kFC = FUSE ? kFuseCap : 1;
  constexpr int kFS = FUSE ? NCW * kFuseSeed : 1;
  constexpr int kFR = FUSE ? kFuseRank : 1;
  __shared__ float s_fv[2][kFC];
  __shared__ int s_fi[2][kFC];
  __shared__ int s_fcnt[2];
  __shared__ int s_fbk[2];  // the lists' shared bounds (fkey), raised as they grow
  __shared__ float s_seed[2][kFS];  // by item parity, like the lists
  __shared__ float s_rv[kFR];
  __shared__ int s_ri[kFR];
  __shared__ float s_topv[FUSE ? kMaxTopK : 1];
  __shared__ int s_topi[FUSE ? kMaxTopK : 1];
  __shared__ Partial s_red[kSlots][NRED];
  __shared__ SmemCue sc;
  // cluster mode: row parts of the rows this CTA owns (it holds their first
  // part), written by the other CTAs of the cluster over DSMEM
  __shared__ __align__(16) float s_xpart[kXSlots][kXParts][kPartWords];
  __shared__ __align__(8) uint64_t s_xbar[kXSlots];

  const T* logits = static_cast<const T*>(a.logits);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) TRACE(0);
#ifdef RELAY_TRACE
  if (tid == 0 && blockIdx.x < 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_trace[blockIdx.x][29] = smid + 1;  // slot 29: the SM (+1: 0 means no stamp)
  }
#endif
  const uint32_t ring_s = smem_u32_pinned(ring);
  const uint32_t full_s = smem_u32_pinned(full);
  const uint32_t rempty_s = smem_u32_pinned(red_empty);
  const uint32_t ifull_s = smem_u32_pinned(ifull);
  const uint32_t theta_s = smem_u32_pinned(s_theta);
  if (tid == 0) {
    // Every consumer thread arrives on `empty` after its own shared-memory reads
    // and on `red_full` after its last threshold read / partial write, so each
    // thread's accesses are released to the TMA producer / epilogue warp.
    for (int s = 0; s < NG * NS; s++) {
      mbar_init(full_s + 8 * s, 1);
    }
    for (int s = 0; s < kSlots; s++) {
      mbar_init(rempty_s + 8 * s, 32);      // every reading lane of the epilogue warp
      mbar_init(ifull_s + 8 * s, 1);        // the producer (dynamic mode)
      s_theta[s] = fkey(-INFINITY);
    }
    s_fcnt[0] = 0;
    s_fcnt[1] = 0;
    s_fbk[0] = fkey(-INFINITY);
    s_fbk[1] = fkey(-INFINITY);
    if (fmode == 4) {
      // one mbarrier per owned split row, expecting its other parts
      ItemIter<SPLIT> it0;
      it0.init(a);
      Item x;
      while (it0.next(a, x))
        if (x.nparts > 1 && x.part == 0)
          mbar_init(smem_u32(&s_xbar[(x.r - it0.row0) % kXSlots]), x.nparts - 1);
    }
    fence_barrier_init();
  }
  if constexpr (FUSE)  // list slots hold -inf until written (fuse_raise reads reserved slots)
    for (int e = tid; e < 2 * kFC; e += blockDim.x) s_fv[e / kFC][e % kFC] = -INFINITY;
  __syncthreads();
  if (fmode == 4) cluster_sync_all();  // every owner's barriers exist before any remote arrive
  const float c = a.c;
  // K4 is launched with programmatic dependent launch: its prologue (barrier
  // init, item math, pattern staging) overlaps the previous kernel's tail;
  // every warp waits for that kernel's completion (griddepcontrol.wait)
  // before touching global data it may have produced.  Outside a PDL launch
  // both instructions are no-ops.
  if constexpr (MODE == kModeStep) {
    // with ready_q (relay_step_sample) the dependent K5 is released only
    // after every CTA passed griddepcontrol.wait (the epilogue warp below):
    // K5 then takes rows from the queue as they finish, every earlier kernel done
    if (tid == 0 && !a.ready_q) pdl_launch_dependents();
  }

  if (warp == NCW) {
    // ------------------------------------------------ producer warp
    // The whole warp waits for the consumers' release of a ring stage on that
    // stage's named barrier (bar.sync: the warp is descheduled, no polling);
    // lane 0 issues the copies.  One bar.sync per chunk, drained at the end.
    const uint64_t pol = a.keep_l2 == 1 ? policy_evict_last()
                         : a.keep_l2 == 2 ? policy_evict_normal() : policy_evict_first();
    int stage = 0;
    long long n_issued = 0;
#ifdef RELAY_TRACE
    bool first_issue = true;
#endif
    auto issue = [&](const Item& item) {
      const T* row = logits + item.r * a.stride;
      const Geom g = row_geom<E>(row, item.j0, item.j1);
      const char* src = reinterpret_cast<const char*>(row + item.j0 + g.head);
      for (int off = 0; off < g.body; off += SB) {
        const uint32_t bytes = static_cast<uint32_t>(min(SB, g.body - off));
        if (n_issued >= NS) named_bar(kBarRing0 + stage, NCT + 32);
        if (lane == 0) {
          fence_proxy_async_smem();  // the consumers' reads precede the async-proxy refill
          mbar_expect_tx(full_s + 8 * stage, bytes);
          bulk_g2s(ring_s + stage * SB, src + off, bytes, full_s + 8 * stage, pol);
#ifdef RELAY_TRACE
          if (first_issue) { TRACE(15); first_issue = false; }
#endif
        }
        ++n_issued;
        if (++stage == NS) stage = 0;
      }
    };
    if (fmode == 2) {
      const long long total = a.n_rows * a.cpr;
      if constexpr (MODE == kModeStep) pdl_wait();
      long long k = 0;
      if (lane == 0) k = atomicAdd(a.work, 1);
      k = __shfl_sync(kFull, k, 0);
      for (int it = 0;; ++it) {
        const int slot = it % kSlots;
        mbar_wait_sleep(rempty_s + 8 * slot, ((it / kSlots) & 1) ^ 1);
        const bool done = k >= total;
        long long kn = 0;
        if (lane == 0) {
          s_item[slot] = done ? -1 : k;
          mbar_arrive(ifull_s + 8 * slot);
          if (!done) kn = atomicAdd(a.work, 1);  // claimed while this chunk streams
        }
        __syncwarp();
        if (done) break;
        kn = __shfl_sync(kFull, kn, 0);
        issue(ItemIter<SPLIT>::from_k(a, k));
        k = kn;
      }
    } else if constexpr (NG > 1) {
      // groups: group g streams rows b + (g + k NG) grid; one stage per group
      // in turn (each group's stages land in its own ring)
      if constexpr (MODE == kModeStep) pdl_wait();
      long long gr[NG] = {};
      int goff[NG] = {}, gbody[NG] = {}, gstage[NG] = {};
      long long gn[NG] = {};
      const char* gsrc[NG] = {};
      auto open = [&](int g) {
        for (; gr[g] < a.n_rows; gr[g] += static_cast<long long>(NG) * gridDim.x) {
          const T* row = logits + gr[g] * a.stride;
          const Geom ge = row_geom<E>(row, 0, a.vocab);
          if (ge.body == 0) continue;  // scalars only: nothing to stream
          gsrc[g] = reinterpret_cast<const char*>(row + ge.head);
          gbody[g] = ge.body;
          goff[g] = 0;
          return;
        }
      };
#pragma unroll
      for (int g = 0; g < NG; g++) {
        gr[g] = blockIdx.x + static_cast<long long>(g) * gridDim.x;
        gstage[g] = 0;
        gn[g] = 0;
        open(g);
      }
      for (bool any = true; any;) {
        any = false;
#pragma unroll
        for (int g = 0; g < NG; g++) {
          if (gr[g] >= a.n_rows) continue;
          any = true;
          const uint32_t bytes = static_cast<uint32_t>(min(SB, gbody[g] - goff[g]));
          const int st = gstage[g];
          if (gn[g] >= NS) named_bar(kBarRing0 + g * NS + st, NCTG + 32);
          if (lane == 0) {
            const uint32_t fb = full_s + 8 * (g * NS + st);
            fence_proxy_async_smem();
            mbar_expect_tx(fb, bytes);
            bulk_g2s(ring_s + (g * NS + st) * SB, gsrc[g] + goff[g], bytes, fb, pol);
          }
          ++gn[g];
          if (++gstage[g] == NS) gstage[g] = 0;
          goff[g] += SB;
          if (goff[g] >= gbody[g]) {
            gr[g] += static_cast<long long>(NG) * gridDim.x;
            open(g);
          }
        }
      }
#pragma unroll
      for (int g = 0; g < NG; g++)
        for (long long k = gn[g] > NS ? gn[g] - NS : 0; k < gn[g]; ++k)
          named_bar(kBarRing0 + g * NS + static_cast<int>(k % NS), NCTG + 32);
      return;
    } else {
      ItemIter<SPLIT> iter;
      iter.init(a);
      Item item;
      bool more = iter.next(a, item);
      if constexpr (MODE == kModeStep) pdl_wait();
      for (; more; more = iter.next(a, item)) issue(item);
    }
    // drain: the stages still in flight are released once more each
    for (long long k = n_issued > NS ? n_issued - NS : 0; k < n_issued; ++k)
      named_bar(kBarRing0 + static_cast<int>(k % NS), NCT + 32);
    return;
  }

  if (warp == NCW + 1) {
    // ------------------------------------------------ epilogue warp
    if constexpr (MODE == kModeStep) {  // the switch patterns, for this warp only
      load_smem_cue(cs, sc);
      pdl_wait();
      if (lane == 0 && a.ready_q) pdl_launch_dependents();
    }
    ItemIter<SPLIT> iter;
    iter.init(a);
    Item item;
    for (int it = 0; fetch_item(a, iter, it, kSlots, s_item, ifull_s, item); ++it) {
      const int slot = it % kSlots;
      const long long r = item.r;
      const T* row = logits + r * a.stride;
      SwitchIn in{};
      int best = -2;
      if constexpr (MODE == kModeStep) {
        in = load_switch_in(a, r);
        // a sampled token is known now: its pattern test runs while the
        // consumers stream, off the step's tail
        if (a.sampled && !a.thk) best = switch_match(cs, sc, in.sampled, in);
      }
      const bool fuse = FUSE && MODE == kModeStep && a.fuse;
      const float fu = fuse ? a.uniform[r] : 0.0f;
      // the consumers' partials: a named barrier (a spinning epilogue warp took
      // issue slots from the consumers for the whole row, 0.45 per element)
      named_bar(kBarRed0 + slot, NCTG + 32);  // the item's group
      if (lane == 0 && it == 0) TRACE(20);
      Partial q = partial_empty();
#pragma unroll
      for (int e = lane; e < NCWG * RPW; e += 32) q = partial_merge(q, s_red[slot][e]);
      // full butterfly: every lane ends with the merged partial (the switch
      // below reads the row's top-1 on all lanes)
      q = warp_merge_all(q);
      if (lane == 0 && it == 0) TRACE(21);
      float thk = INFINITY;
      if (a.thk) {
#pragma unroll
        for (int w = 0; w < NCWG; w++) thk = fminf(thk, s_thk[slot][w]);
      }
      if (lane == 0) s_theta[slot] = fkey(-INFINITY);  // for item it + kSlots
      if (!fuse) mbar_arrive(rempty_s + 8 * slot);  // (fused draw: after the list is read)
      if (item.nparts == 1) {
        bool exact = false;
        float S = 0.0f;
        if (q.flags & kFlagHuge) {  // rare: exact normaliser over the row by this warp
          S = warp_sum(exact_sum_thread<E>(row, a.vocab, q.t.v1, c, lane, 32));
          exact = true;
        }
        if (a.thk && lane == 0) {
          a.thk[r] = thk;
          a.zmax[r] = q.t.v1;
        }
        if (lane == 0 && it == 0) TRACE(22);
        FuseIn fz{};
        bool drawn = false;
        if (fuse) {
          const int fb = it & 1;
          fz = FuseIn{true, s_fcnt[fb], thk, fu, s_fv[fb], s_fi[fb], s_rv, s_ri, s_topv, s_topi};
        }
        finish_item<E, MODE>(a, cs, sc, r, q, exact, S, in, best, &fz, &drawn);
#ifdef RELAY_TRACE
        if (fuse && lane == 0) {
          atomicAdd(&g_fuse_stats[drawn ? 0 : 1], 1ull);
          atomicAdd(&g_fuse_stats[2], static_cast<unsigned long long>(fz.n));
        }
#endif
        if (a.ready_q && lane == 0) {  // lane 0 wrote thk/zmax/margin/top1/top2/status: publish
          // (a row drawn here is queued as -(r + 1): K5 only takes its ticket)
          const int pos = atomicAdd(a.q_ctl, 1);
          const int v = drawn ? -(static_cast<int>(r) + 1) : static_cast<int>(r) + 1;
          asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(a.ready_q + pos), "r"(v) : "memory");
        }
        if (fuse) {
          __syncwarp();
          {
            const int fb = it & 1;
            const int n = min(s_fcnt[fb], kFC);
            for (int e = lane; e < n; e += 32) s_fv[fb][e] = -INFINITY;
            if (lane == 0) {
              s_fcnt[fb] = 0;
              s_fbk[fb] = fkey(-INFINITY);
            }
          }
          mbar_arrive(rempty_s + 8 * slot);  // the list is free for item it + 2
        }
        if (lane == 0 && it < 7) TRACE(24 + it);
        continue;
      }
      if (fmode == 4) {
        // cluster mode: the CTA holding the row's FIRST part owns it (its
        // last item: the other parts are the first items of the following
        // CTAs, long done, so no CTA waits on a chain of predecessors); the
        // others store their partial into its shared memory (DSMEM) and
        // arrive on its barrier; the owner merges once all have arrived
        const int xs = static_cast<int>((r - iter.row0) % kXSlots);
        if (item.part != 0) {
          if (lane == 0) {
            const uint32_t owner = static_cast<uint32_t>(iter.b - item.part);
            const uint32_t dst = mapa_cluster(smem_u32(&s_xpart[xs][item.part][0]), owner);
            st_cluster_v4(dst, __float_as_uint(q.t.v1), __float_as_uint(q.t.v2), static_cast<uint32_t>(q.t.i1),
                          static_cast<uint32_t>(q.t.i2));
            st_cluster_v4(dst + 16, __float_as_uint(q.n.m), __float_as_uint(q.n.s), static_cast<uint32_t>(q.flags),
                          0u);
            mbar_arrive_remote(mapa_cluster(smem_u32(&s_xbar[xs]), owner));
          }
          if (lane == 0 && it < 7) TRACE(24 + it);
          continue;
        }
        mbar_wait_cluster(smem_u32(&s_xbar[xs]), 0);
        Partial m = q;
        for (int k = 1; k < item.nparts; k++) {
          const float* pr = s_xpart[xs][k];
          Partial o;
          o.t.v1 = pr[0]; o.t.v2 = pr[1];
          o.t.i1 = __float_as_int(pr[2]); o.t.i2 = __float_as_int(pr[3]);
          o.n.m = pr[4]; o.n.s = pr[5];
          o.flags = __float_as_int(pr[6]);
          m = partial_merge(m, o);
        }
        bool exact = false;
        float S = 0.0f;
        if (m.flags & kFlagHuge) {
          S = warp_sum(exact_sum_thread<E>(row, a.vocab, m.t.v1, c, lane, 32));
          exact = true;
        }
        finish_item<E, MODE>(a, cs, sc, r, m, exact, S, in, best);
        if (lane == 0 && it < 7) TRACE(24 + it);
        continue;
      }
      // publish this part; the last part of the row to arrive finishes it
      int last = 0;
      if (lane == 0) {
        float* pw = a.part + (static_cast<size_t>(r) * kMaxSplit + item.part) * kPartWords;
        __stcg(pw + 0, q.t.v1); __stcg(pw + 1, q.t.v2);
        __stcg(pw + 2, __int_as_float(q.t.i1)); __stcg(pw + 3, __int_as_float(q.t.i2));
        __stcg(pw + 4, q.n.m); __stcg(pw + 5, q.n.s);
        __stcg(pw + 6, __int_as_float(q.flags));
        last = atomic_add_acq_rel(a.counter + r, 1) == item.nparts - 1;
      }
      if (!__shfl_sync(kFull, last, 0)) {
        if (lane == 0 && it < 7) TRACE(24 + it);
        continue;
      }
      Partial m = partial_empty();
      for (int k = lane; k < item.nparts; k += 32) {
        const float* pr = a.part + (static_cast<size_t>(r) * kMaxSplit + k) * kPartWords;
        Partial o;
        o.t.v1 = __ldcg(pr + 0); o.t.v2 = __ldcg(pr + 1);
        o.t.i1 = __float_as_int(__ldcg(pr + 2)); o.t.i2 = __float_as_int(__ldcg(pr + 3));
        o.n.m = __ldcg(pr + 4); o.n.s = __ldcg(pr + 5);
        o.flags = __float_as_int(__ldcg(pr + 6));
        m = partial_merge(m, o);
      }
      m = warp_merge_all(m);
      bool exact = false;
      float S = 0.0f;
      if (m.flags & kFlagHuge) {
        S = warp_sum(exact_sum_thread<E>(row, a.vocab, m.t.v1, c, lane, 32));
        exact = true;
      }
      if (lane == 0) a.counter[r] = 0;  // ready for the next launch / graph replay
      finish_item<E, MODE>(a, cs, sc, r, m, exact, S, in, best);
      if (lane == 0 && it < 7) TRACE(24 + it);
    }
    if (fmode == 2 && lane == 0) {
      // the last CTA out re-arms the work counter for the next launch / replay
      // (every producer's final claim precedes its CTA's arrival here)
      if (atomic_add_acq_rel(a.work + 1, 1) == static_cast<int>(gridDim.x) - 1) {
        a.work[0] = 0;
        a.work[1] = 0;
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  if constexpr (MODE == kModeStep) pdl_wait();  // head/tail scalars are read directly
#ifdef RELAY_TRACE
  int n_stage = 0;
#endif
  // this warp's group: its ring, its stage barriers, its items it = grp, grp + NG, ...
  const int grp = NG > 1 ? warp / NCWG : 0;
  const int ctid = tid - grp * NCTG;       // thread index within the group
  const int cwarp = warp - grp * NCWG;     // warp index within the group
  // stage: the ring position as an index over every group's stages (this
  // group's are [grp NS, grp NS + NS)), so that one register addresses the
  // stage's buffer, its full mbarrier and its release barrier
  const int st_beg = grp * NS, st_end = grp * NS + NS;
  int stage = st_beg;   // ring position, carried across items
  uint32_t phase = 0;
  // this thread's vector in stage 0's buffer (pinned: not recomputed from
  // %tid in every stage; with theta_p below, -2.7% K1 instructions)
  const uint32_t ring_t = pin_u32(ring_s + static_cast<uint32_t>(ctid) * 16);
  ItemIter<SPLIT> iter;
  iter.init(a);
  Item item;
  auto next_item = [&](int it) -> bool {
    if constexpr (NG == 1) {
      return fetch_item(a, iter, it, kSlots, s_item, ifull_s, item);
    } else {  // strided whole rows: item it is row blockIdx + it * grid
      const long long r = blockIdx.x + static_cast<long long>(it) * gridDim.x;
      if (r >= a.n_rows) return false;
      item = Item{r, 0, a.vocab, 0, 1};
      return true;
    }
  };
  for (int it = grp; next_item(it); it += NG) {
    const int slot = it % kSlots;
    const long long r = item.r;
    const int j0 = item.j0;
    const int j1 = item.j1;
    if (ctid == 0 && it == 1) TRACE(11);
    // the slot (threshold + partials) is free once the epilogue took item it - kSlots
    mbar_wait(rempty_s + 8 * slot, ((it / kSlots) & 1) ^ 1);
    if (ctid == 0 && it == 1) TRACE(12);
    const uint32_t theta_p = pin_u32(theta_s + 4 * slot);
    const T* row = logits + r * a.stride;
    const Geom g = row_geom<E>(row, j0, j1);
    const int nst = g.body / SB;             // full ring stages of the item
    const int rem = g.body - nst * SB;       // bytes of its last, partial stage
    const int jt = j0 + g.head + ctid * VEC;  // element index of this thread's first vector
    ThreadState st;
    state_init(st);
    float theta_w = -INFINITY;  // warp-local lower bound of the row's 2nd-best
    float T = 0.0f;             // consume_fast's guard (set by the row's first stage)
    int tkey = INT_MIN;         // the threshold key T was computed from
    float tmax = -INFINITY;     // this thread's maximum (relay_step_sample's bound)
    // fused draw: this item's candidate list (released by the epilogue once it
    // drew item it - 2) and bound (-inf until the first stage's seeds are in)
    const bool fuse = FUSE && MODE == kModeStep && a.fuse;
    const int fb = it & 1;
    float fB = -INFINITY;
    if (fuse && it >= 2) mbar_wait(rempty_s + 8 * ((it - 2) % kSlots), ((it - 2) / kSlots) & 1);
    if (ctid < g.head) {
      const float x = E::load1(row + j0 + ctid);
      consume_scalar(x, j0 + ctid, st, c);
      if constexpr (MODE == kModeStep) tmax = fmaxf(tmax, x);
      if (fuse && x > -INFINITY) {  // (NaN fails the test)
        const int p = atomicAdd(&s_fcnt[fb], 1);
        if (p < kFuseCap) { s_fv[fb][p] = x; s_fi[fb][p] = j0 + ctid; }
      }
    }
    if (nst > 0) {
      // the item's first stage: the row-start probe.  The two half maxima of
      // a thread are two distinct elements, so the warp's second-best of them
      // bounds the row's 2nd-best from below and raises the shared threshold;
      // no barrier: each warp goes on with its own bound and whatever the
      // others have published (any of them is a valid lower bound), so the
      // steady state starts mostly on the fast path without a CTA-wide wait.
      mbar_wait(full_s + 8 * stage, phase);
#ifdef RELAY_TRACE
      if (ctid == 0 && n_stage < 10) TRACE(1 + n_stage);
      ++n_stage;
#endif
      uint4 raw[UV];
#pragma unroll
      for (int u = 0; u < UV; u++) raw[u] = lds128(ring_t + stage * SB + u * NCTG * 16);
      bar_arrive_pinned<UV>(kBarRing0 + stage, NCTG + 32, raw);  // release: the loads precede the refill
      const float2 h = stage_max2<E, UV>(raw);
      theta_w = theta_raise(warp_second(fmaxf(h.x, h.y), fminf(h.x, h.y)), theta_p);
#ifdef RELAY_PROBE_BAR
      named_bar(1, NCT);  // tuning: wait for every warp's probe (r02: 1.5% slower without gain)
#endif
      if (ctid == 0 && it == 1) TRACE(13);
      tkey = theta_load(theta_p);
      const float theta = fmaxf(theta_w, unkey(tkey));
      bool slow = false;
      consume_stage<E, UV>(raw, h, jt, NCTG * VEC, st, c, theta, slow);
      if (__any_sync(kFull, slow)) theta_w = fmaxf(theta_w, theta_raise(warp_second(st.t.v1, st.t.v2), theta_p));
      T = guard_T(fmaxf(theta, theta_w), st, c);
      if constexpr (MODE == kModeStep) {
        tmax = fmaxf(tmax, fmaxf(h.x, h.y));
        if (fuse) {
          // the bound: the top_k-th largest of every warp's kFuseSeed
          // largest first-stage half maxima (distinct elements of the row)
          fuse_seeds(h, s_seed[fb] + warp * kFuseSeed);
          named_bar(1, NCT);
          fB = fuse_bound(s_seed[fb], NCW * kFuseSeed, a.topk);
          if (ctid == 0 && it == 0) TRACE(11);
          if (lane == 0) atomicMax(&s_fbk[fb], fkey(fB));
          if (__any_sync(kFull, fmaxf(h.x, h.y) >= fB)) {
            const bool x = fuse_push<E, UV>(raw, UV, jt, NCTG * VEC, fB, s_fv[fb], s_fi[fb], &s_fcnt[fb]);
            if (__any_sync(kFull, x)) fuse_raise(s_fv[fb], a.topk, &s_fbk[fb]);
          }
        }
      }
      if (ctid == 0 && it <= 1) TRACE(14);
      if (++stage == st_end) { stage = st_beg; phase ^= 1; }
    }
    // steady state: per stage the wait, the words, one release, the terms and
    // one guard comparison (consume_fast)
#pragma unroll kSteadyUnroll
    for (int k = 1; k < nst; ++k) {
      mbar_wait(full_s + 8 * stage, phase);
#ifdef RELAY_TRACE
      if (ctid == 0 && n_stage < 10) TRACE(1 + n_stage);
      ++n_stage;
#endif
      const int key = theta_load(theta_p);  // before the words: its latency hides under the sum
      uint4 raw[UV];
#pragma unroll
      for (int u = 0; u < UV; u++) raw[u] = lds128(ring_t + stage * SB + u * NCTG * 16);
      bar_arrive_pinned<UV>(kBarRing0 + stage, NCTG + 32, raw);
      if constexpr (MODE == kModeStep) {
        // (before the terms: the words are dead after consume_fast)
        if (a.topk > 0) {
          const float2 h = stage_max2<E, UV>(raw);
          tmax = fmaxf(tmax, fmaxf(h.x, h.y));
          if (fuse) {
            fB = fmaxf(fB, unkey(*reinterpret_cast<volatile int*>(&s_fbk[fb])));  // raised by any warp
            if (__any_sync(kFull, fmaxf(h.x, h.y) >= fB)) {
              const bool x = fuse_push<E, UV>(raw, UV, jt + k * (SB / E::SZ), NCTG * VEC, fB, s_fv[fb], s_fi[fb],
                                              &s_fcnt[fb]);
              if (__any_sync(kFull, x)) fuse_raise(s_fv[fb], a.topk, &s_fbk[fb]);
            }
          }
        }
      }
      consume_fast<E, UV, kPolyPairs>(raw, UV, jt + k * (SB / E::SZ), NCTG * VEC, st, c, T, tkey, theta_w, key, theta_p);
      if (++stage == st_end) { stage = st_beg; phase ^= 1; }
    }
    if (rem > 0) {
      mbar_wait(full_s + 8 * stage, phase);
      const uint32_t buf = ring_s + stage * SB;
      const int jb = j0 + g.head + nst * (SB / E::SZ);
      if (nst > 0) {
        // the last, partial stage: the missing vectors read as -inf (no term,
        // never pushed)
        const int key = theta_load(theta_p);
        const int nvalid = min(UV, max(0, (rem / 16 - ctid + NCTG - 1) / NCTG));
        uint4 raw[UV];
#pragma unroll
        for (int u = 0; u < UV; u++) raw[u] = u < nvalid ? lds128(ring_t + stage * SB + u * NCTG * 16) : E::neg_inf16();
        bar_arrive_pinned<UV>(kBarRing0 + stage, NCTG + 32, raw);
        if constexpr (MODE == kModeStep) {
          if (a.topk > 0) {
            const float2 h = stage_max2<E, UV>(raw);
            tmax = fmaxf(tmax, fmaxf(h.x, h.y));
            if (fuse) {
              fB = fmaxf(fB, unkey(*reinterpret_cast<volatile int*>(&s_fbk[fb])));
              if (__any_sync(kFull, fmaxf(h.x, h.y) >= fB))
                fuse_push<E, UV>(raw, nvalid, jb + ctid * VEC, NCTG * VEC, fB, s_fv[fb], s_fi[fb], &s_fcnt[fb]);
            }
          }
        }
        consume_fast<E, UV, kPolyPairs>(raw, nvalid, jb + ctid * VEC, NCTG * VEC, st, c, T, tkey, theta_w, key, theta_p);
      } else {  // a row shorter than one stage: vector by vector, max-guarded
        const float theta = fmaxf(theta_w, unkey(theta_load(theta_p)));
        const int nvec = rem / 16;
        bool slow = false;
        for (int v = ctid; v < nvec; v += NCTG) {
          const uint4 raw1[1] = {lds128(buf + v * 16)};
          const float2 h1 = stage_max2<E, 1>(raw1);
          consume_stage<E, 1>(raw1, h1, jb + v * VEC, 0, st, c, theta, slow);
          if constexpr (MODE == kModeStep) {
            tmax = fmaxf(tmax, fmaxf(h1.x, h1.y));
            if (fuse) fuse_push<E, 1>(raw1, 1, jb + v * VEC, 0, fB, s_fv[fb], s_fi[fb], &s_fcnt[fb]);
          }
        }
        bar_arrive(kBarRing0 + stage, NCTG + 32);
      }
      if (++stage == st_end) { stage = st_beg; phase ^= 1; }
    }
    if (ctid < j1 - g.tail) {
      const float x = E::load1(row + g.tail + ctid);
      consume_scalar(x, g.tail + ctid, st, c);
      if constexpr (MODE == kModeStep) tmax = fmaxf(tmax, x);
      if (fuse && x >= fB && x > -INFINITY) {
        const int p = atomicAdd(&s_fcnt[fb], 1);
        if (p < kFuseCap) { s_fv[fb][p] = x; s_fi[fb][p] = g.tail + ctid; }
      }
    }
    if (a.topk > 0) {
      // N2: the warp's kw-th largest thread maximum, kw = ceil(topk / NCW);
      // the minimum over warps bounds the row's topk-th largest value from
      // below (NCW * kw >= topk distinct elements are at least as large)
      const int kw = (a.topk + NCWG - 1) / NCWG;
      float v = tmax, kth = -INFINITY;
      for (int i = 0; i < kw; i++) {
        float m = v;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, off));
        kth = m;
        const unsigned holders = __ballot_sync(kFull, v == m);
        if (lane == __ffs(holders) - 1) v = -INFINITY;
      }
      if (lane == 0) s_thk[slot][cwarp] = kth;
    }
    // hand the warp's 8 partials (after two shuffle rounds) to the epilogue warp
    Partial p = thread_partial(st);
    if constexpr (RPW == 1) {
      p = warp_merge_all(p);
    } else {
#pragma unroll
      for (int off = 16; off >= RPW; off >>= 1) p = partial_merge(p, shfl_xor_partial(p, off));
    }
    if (lane < RPW) s_red[slot][cwarp * RPW + lane] = p;
    bar_arrive(kBarRed0 + slot, NCTG + 32);
    if (ctid == 0 && it < 8) TRACE(16 + it);
  }
  if (ctid == 0) TRACE(31);
}

static int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// Row-kernel launch shape (overridable at build time for tuning sweeps,
// tools/k1_sweep.py).
#ifndef RELAY_K1_NCW
#define RELAY_K1_NCW 8
#endif
#ifndef RELAY_K1_STAGES
#define RELAY_K1_STAGES 4
#endif
#ifndef RELAY_K1_UV
#define RELAY_K1_UV 4
#endif
#ifndef RELAY_K1_MINB
#define RELAY_K1_MINB 3
#endif
constexpr int kNCW = RELAY_K1_NCW;        // consumer warps per CTA
constexpr int kStages = RELAY_K1_STAGES;  // ring depth
constexpr int kUV = RELAY_K1_UV;          // 16-byte vectors per consumer thread per stage
constexpr int kMinBlocks = RELAY_K1_MINB; // CTAs per SM the registers must allow
#ifndef RELAY_K4_STAGES
#define RELAY_K4_STAGES 4
#endif
#ifndef RELAY_K4_MINB
#define RELAY_K4_MINB 2
#endif
#ifndef RELAY_K4_NCW
#define RELAY_K4_NCW 12   // 12 consumer warps x 4 stages of 24 KB (tools/k4_sweep.py: 20.5 vs 21.2 us at 8 x 6 x 16 KB)
#endif
constexpr int kStepStages = RELAY_K4_STAGES;
constexpr int kStepMinBlocks = RELAY_K4_MINB;
constexpr int kStepNCW = RELAY_K4_NCW;     // consumer warps per CTA in K4
#ifndef RELAY_K4_UV
#define RELAY_K4_UV 4
#endif
constexpr int kStepUV = RELAY_K4_UV;       // 16-byte vectors per consumer thread per stage in K4

// K4 work split (RELAY_K4_MODE=strided|flat|dynamic overrides, for tuning
// and tests): strided = one whole row per CTA, no cross-CTA merge (default
// when the batch fills every SM at least once); flat = equal slices of the
// flattened batch merged by the last arriving CTA (default for small
// batches); dynamic = chunks of RELAY_K4_CHUNK_STAGES ring stages claimed from
// an atomic counter (measured slower).
static int k4_mode(int batch) {
  const char* e = getenv("RELAY_K4_MODE");
  if (e && !strcmp(e, "strided")) return 0;
  if (e && !strcmp(e, "flat")) return 1;
  if (e && !strcmp(e, "dynamic")) return 2;
  if (e && !strcmp(e, "hybrid")) return batch > num_sms() ? 3 : 1;
  if (e && !strcmp(e, "cluster")) return 4;
  return batch >= num_sms() ? 0 : 1;
}
static int k4_chunk_stages() {
  const char* e = getenv("RELAY_K4_CHUNK_STAGES");
  const int x = e ? atoi(e) : 0;
  return x > 0 ? x : 4;
}

// K4 with more rows than SMs, opt-in (RELAY_K4_GROUPS=1): one CTA per SM,
// two consumer groups of 12 warps streaming rows b and b + grid concurrently
// (rows_kernel NG = 2).  Measured slower than two CTAs per SM (19.6 vs 18.8
// us at configs[2]): an SM's two rows end at ~16 us either way (its HBM
// share and the exp rate at ~71% of MUFU peak bound it), and the shared
// producer / epilogue warps add to the tail (profiles/r02/k4_tail.txt).
#ifndef RELAY_K4_GROUP_NCW
#define RELAY_K4_GROUP_NCW 24
#endif
static bool k4_groups() {
  const char* e = getenv("RELAY_K4_GROUPS");
  return e && !strcmp(e, "1");
}

template <class E>
static cudaError_t launch_step_groups(RowsArgs a, const CueDev& cs, cudaStream_t st) {
  constexpr int NCW = RELAY_K4_GROUP_NCW, NS = kStepStages, UV = kStepUV;
  auto kern = rows_kernel<E, NCW, NS, UV, 1, kModeStep, 0, false, 2>;
  const int smem = NS * UV * NCW * 32 * 16;  // two rings of NS stages
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NCW + 2) * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    if (getenv("RELAY_DEBUG_LAUNCH"))
      fprintf(stderr, "relay rows_kernel K4 groups: %d CTAs/SM, smem %d B dynamic\n", per_sm, smem);
  }
  long long grid = static_cast<long long>(per_sm) * num_sms();
  if (grid > a.n_rows) grid = a.n_rows;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3((NCW + 2) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, cs);
}

// K1 with consumer groups (the default; RELAY_K1_GROUPS=0 for one row per CTA
// at a time): each CTA streams two rows at once, four consumer warps per row,
// so the per-row work (row-start probe, partial last stage, partial hand-off,
// ~510 instructions per warp per row) is paid by half the warps: configs[1]
// K1 1.518 -> 1.494 ms burst, 1.794 -> 1.779 ms sustained (profiles/r02/k1_v9_ab.txt).
#ifndef RELAY_K1_GROUPS_DEFAULT
#define RELAY_K1_GROUPS_DEFAULT 1
#endif
static bool k1_groups() {
  const char* e = getenv("RELAY_K1_GROUPS");
  return e ? !strcmp(e, "1") : RELAY_K1_GROUPS_DEFAULT != 0;
}

#ifndef RELAY_K1_NG
#define RELAY_K1_NG 2          // consumer groups per K1 CTA (rows streamed at once)
#endif
#ifndef RELAY_K1_GROUP_NS
#define RELAY_K1_GROUP_NS RELAY_K1_STAGES  // ring stages per group
#endif
template <class E>
static cudaError_t launch_rows_groups(RowsArgs a, const CueDev& cs, cudaStream_t st) {
  constexpr int NCW = kNCW, NS = RELAY_K1_GROUP_NS, UV = kUV, NG = RELAY_K1_NG;
  auto kern = rows_kernel<E, NCW, NS, UV, kMinBlocks, kModeRows, 0, false, NG>;
  const int smem = NS * UV * NCW * 32 * 16;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NCW + 2) * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  long long grid = static_cast<long long>(per_sm) * num_sms();
  if (grid > (a.n_rows + NG - 1) / NG) grid = (a.n_rows + NG - 1) / NG;
  kern<<<static_cast<unsigned>(grid), (NCW + 2) * 32, smem, st>>>(a, cs);
  return cudaGetLastError();
}

template <class E, int MODE>
static cudaError_t launch_rows_t(RowsArgs a, const CueDev& cs, cudaStream_t st) {
  if constexpr (MODE == kModeStep) {
    if (a.flat == 0 && !a.fuse && a.n_rows > num_sms() && k4_groups()) return launch_step_groups<E>(a, cs, st);
  }
  if constexpr (MODE == kModeRows) {
    if (a.flat == 0 && k1_groups()) return launch_rows_groups<E>(a, cs, st);
  }
  // K4 runs ~1-2 CTAs per SM: a deeper ring keeps more bytes in flight per CTA
  constexpr int NS = (MODE == kModeStep) ? kStepStages : kStages;
  constexpr int MINB = (MODE == kModeStep) ? kStepMinBlocks : kMinBlocks;
  constexpr int NCW = (MODE == kModeStep) ? kStepNCW : kNCW;
  constexpr int UV = (MODE == kModeStep) ? kStepUV : kUV;
  // instantiation: whole rows (0), flat slices only (1), every split mode (2)
  const int split = MODE != kModeStep || a.flat == 0 ? 0 : a.flat == 1 ? 1 : 2;
  // (the fused top-k draw is its own whole-row instantiation: its candidate
  // lists and pushes stay out of the decode-step switch's registers)
  const bool fz = MODE == kModeStep && a.fuse && split == 0;
  auto kern = fz ? rows_kernel<E, NCW, NS, UV, MINB, MODE, 0, MODE == kModeStep>
              : split == 0 ? rows_kernel<E, NCW, NS, UV, MINB, MODE, 0>
              : split == 1 ? rows_kernel<E, NCW, NS, UV, MINB, MODE, MODE == kModeStep ? 1 : 0>
                           : rows_kernel<E, NCW, NS, UV, MINB, MODE, MODE == kModeStep ? 2 : 0>;
  const int smem = NS * UV * NCW * 32 * 16;
  static int per_sm_of[4] = {0, 0, 0, 0};   // per instantiation (the attribute is per function)
  int& per_sm = per_sm_of[fz ? 3 : split];
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NCW + 2) * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    if (getenv("RELAY_DEBUG_LAUNCH"))
      fprintf(stderr, "relay rows_kernel mode %d split %d fuse %d: %d CTAs/SM, smem %d B dynamic\n", MODE, split,
              fz ? 1 : 0, per_sm, smem);
  }
  const long long slots = static_cast<long long>(per_sm) * num_sms();
  long long grid = slots;
  if (a.flat == 2) {
    const long long total = a.n_rows * a.cpr;
    if (total >= (1LL << 31)) return cudaErrorInvalidValue;  // int work counter
    if (grid > total) grid = total;
  } else if (a.flat == 4) {
    // clusters of csize CTAs, as many as fit at once; rows dealt to clusters
    {
      const char* e = getenv("RELAY_K4_CSIZE");
      a.csize = e && atoi(e) >= 2 && atoi(e) <= kXParts ? atoi(e) : 8;
    }
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(static_cast<unsigned>(slots / a.csize * a.csize));
    q.blockDim = dim3((NCW + 2) * 32);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = a.csize; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int nclusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, kern, &q);
    if (e != cudaSuccess) return e;
    long long C = nclusters;
    if (C > slots / a.csize) C = slots / a.csize;
    if (C > a.n_rows) C = a.n_rows;  // every cluster at least one row
    // every slice of a cluster >= 128 elements: no empty slice (an owner would
    // wait for a part that never comes)
    const long long cap = a.n_rows * a.vocab / (128LL * a.csize);
    if (C > cap) C = cap;
    if (C < 1) {  // too small for clusters: plain flat slices
      a.flat = 1;
      grid = slots;
      const long long T = a.n_rows * a.vocab;
      if (grid > T / 128) grid = T / 128 > 0 ? T / 128 : 1;
      if (grid > a.n_rows * (kMaxSplit - 2)) grid = a.n_rows * (kMaxSplit - 2);
    } else {
      grid = C * a.csize;
    }
  } else if (a.flat == 3) {
    // hybrid: one whole row per SM, the other slots slice the remaining rows
    a.n_whole = num_sms();
    if (a.n_rows <= a.n_whole || slots <= a.n_whole) {
      a.flat = 0;
      if (grid > a.n_rows) grid = a.n_rows;
    } else {
      const long long rest = (a.n_rows - a.n_whole) * a.vocab;
      long long g2 = slots - a.n_whole;
      if (rest >= (1LL << 51)) return cudaErrorInvalidValue;
      if (g2 > rest / 128) g2 = rest / 128 > 0 ? rest / 128 : 1;
      if (g2 > (a.n_rows - a.n_whole) * (kMaxSplit - 2)) g2 = (a.n_rows - a.n_whole) * (kMaxSplit - 2);
      grid = a.n_whole + g2;
    }
  } else if (a.flat) {
    // every slice at least 128 elements and a row in at most kMaxSplit parts
    const long long T = a.n_rows * a.vocab;
    if (T >= (1LL << 51)) return cudaErrorInvalidValue;  // slice math is 64-bit
    if (grid > 4096) grid = 4096;
    if (grid > T / 128) grid = T / 128 > 0 ? T / 128 : 1;
    if (grid > a.n_rows * (kMaxSplit - 2)) grid = a.n_rows * (kMaxSplit - 2);
  } else if (grid > a.n_rows) {
    grid = a.n_rows;
  }
  if constexpr (MODE == kModeStep) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3((NCW + 2) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (a.flat == 4) {
      attr[1].id = cudaLaunchAttributeClusterDimension;
      attr[1].val.clusterDim.x = a.csize; attr[1].val.clusterDim.y = 1; attr[1].val.clusterDim.z = 1;
      cfg.numAttrs = 2;
    }
    return cudaLaunchKernelEx(&cfg, kern, a, cs);
  }
  kern<<<static_cast<unsigned>(grid), (NCW + 2) * 32, smem, st>>>(a, cs);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_rows(int dt, const RowsArgs& a, const CueDev& cs, cudaStream_t st) {
  switch (dt) {
    case 0: return launch_rows_t<EBf16, MODE>(a, cs, st);
    case 1: return launch_rows_t<EF16, MODE>(a, cs, st);
    default: return launch_rows_t<EF32, MODE>(a, cs, st);
  }
}

cudaError_t launch_margin_rows(const void* logits, int dt, long long n_rows, int vocab,
                               long long stride, float iota, float* margin, int* top1, int* top2,
                               float* lse, uint8_t* status, cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  RowsArgs a{};
  a.logits = logits; a.n_rows = n_rows; a.vocab = vocab; a.stride = stride;
  a.c = iota * kLog2e; a.iota = iota; a.flat = 0;
  a.margin = margin; a.top1 = top1; a.top2 = top2; a.lse = lse; a.status = status;
  return launch_rows<kModeRows>(dt, a, CueDev{}, st);
}

cudaError_t launch_step_switch(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                               long long stride, float iota, const int* sampled, uint8_t* state,
                               int* hist, int* small_run, float gate, int max_seg, float* margin,
                               int* top1, int* top2, uint8_t* flag, int16_t* cue_id,
                               const StepWs& ws, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  RowsArgs a{};
  a.logits = logits; a.n_rows = batch; a.vocab = vocab; a.stride = stride;
  a.c = iota * kLog2e; a.iota = iota;
  a.margin = margin; a.top1 = top1; a.top2 = top2;
  a.counter = ws.counter; a.part = ws.part; a.work = ws.work;
  {
    // dynamic mode: chunks of k4_chunk_stages() ring stages (fewer, larger
    // chunks if a row would need more than kMaxSplit parts)
    const int esz = dt == 2 ? 4 : 2;
    const int stage_elems = kStepUV * kStepNCW * 32 * 16 / esz;
    int chunk = k4_chunk_stages() * stage_elems;
    if ((vocab + chunk - 1) / chunk > kMaxSplit) {
      const int per = (vocab + kMaxSplit - 1) / kMaxSplit;
      chunk = (per + stage_elems - 1) / stage_elems * stage_elems;
    }
    a.chunk = chunk;
    a.cpr = (vocab + chunk - 1) / chunk;
    a.flat = k4_mode(batch);
  }
  a.sampled = sampled; a.state = state; a.hist = hist; a.small_run = small_run;
  a.gate = gate; a.max_seg = max_seg; a.flag = flag; a.cue_id = cue_id;
  return launch_rows<kModeStep>(dt, a, cs, st);
}

cudaError_t launch_step_rows(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                             long long stride, float iota, uint8_t* state, int* hist, int* small_run,
                             float gate, int max_seg, float* margin, int* top1, int* top2,
                             const StepWs& ws, int topk, cudaStream_t st, const StepDraw* draw) {
  if (batch <= 0) return cudaSuccess;
  RowsArgs a{};
  a.logits = logits; a.n_rows = batch; a.vocab = vocab; a.stride = stride;
  a.c = iota * kLog2e; a.iota = iota;
  a.margin = margin; a.top1 = top1; a.top2 = top2; a.status = ws.status;
  a.counter = ws.counter; a.part = ws.part; a.work = ws.work;
  a.flat = 0;  // whole rows: the bound needs every thread maximum of the row
  a.state = state; a.hist = hist; a.small_run = small_run; a.gate = gate; a.max_seg = max_seg;
  a.thk = ws.thk; a.zmax = ws.zmax; a.topk = topk; a.ready_q = ws.ready_q; a.q_ctl = ws.q_ctl;
  // the fused top-k draw: opt-in (RELAY_K4_FUSE=1).  Parity-green, but measured
  // slower at configs[2] (49.6 vs 40.8 us per step: ~146 candidates per row
  // make most warp-stages take the push path, and the epilogue's ranking and
  // draw add ~8 us to the row's tail, profiles/r02/k4_fused_draw.txt)
  if (draw) {
    const char* e = getenv("RELAY_K4_FUSE");
    a.fuse = e && !strcmp(e, "1");
    a.s_c = draw->s_c; a.topp = draw->topp; a.uniform = draw->uniform; a.sampled_out = draw->sampled;
    a.flag = draw->flag; a.cue_id = draw->cue_id;
  }
  {  // tuning knob (RELAY_K4_L2 = last | normal | first): the L2 policy of the margin pass
     // (K5 reads the rows again: all of them, or with the fused draw only the overflowed ones)
    const char* e = getenv("RELAY_K4_L2");
    a.keep_l2 = (e && !strcmp(e, "normal")) ? 2 : (e && !strcmp(e, "first")) ? 0
              : (e && !strcmp(e, "last")) ? 1 : (a.fuse ? 0 : 1);
  }
  return launch_rows<kModeStep>(dt, a, cs, st);
}

cudaError_t launch_margin_partials(const void* logits, int dt, long long n_rows, int vocab,
                                  long long stride, long long col_offset, float iota, float* part,
                                  cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  RowsArgs a{};
  a.logits = logits; a.n_rows = n_rows; a.vocab = vocab; a.stride = stride;
  a.c = iota * kLog2e; a.iota = iota; a.flat = 0;
  a.col_offset = col_offset; a.tp_part = part;
  return launch_rows<kModePartial>(dt, a, CueDev{}, st);
}

// N1 combine: merge the vocabulary shards' partials of each row (one thread
// per row): top-2 by (value desc, global index asc); S = sum_k S_k 2^((v1_k -
// M) c); the margin as in finish_row's exact form.
__global__ void margin_combine_kernel(const float* __restrict__ part, int n_shards, long long n_rows,
                                      float c, float iota, float* __restrict__ margin,
                                      int* __restrict__ top1, int* __restrict__ top2,
                                      float* __restrict__ lse, uint8_t* __restrict__ status) {
  const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (r >= n_rows) return;
  Top2 t = top2_empty();
  int nan = 0;
  for (int k = 0; k < n_shards; k++) {
    const float* p = part + (static_cast<size_t>(k) * n_rows + r) * kPartWords;
    Top2 o{p[0], p[1], __float_as_int(p[2]), __float_as_int(p[3])};
    t = top2_merge(t, o);
    nan |= __float_as_int(p[5]);
  }
  int st = 0;
  if (nan || t.v1 == INFINITY) st = 1;
  else if (t.v1 == -INFINITY) st = 2;
  if (st) {
    margin[r] = qnan();
    if (top1) top1[r] = -1;
    if (top2) top2[r] = -1;
    if (lse) lse[r] = qnan();
    if (status) status[r] = static_cast<uint8_t>(st);
    return;
  }
  float S = 0.0f;
  for (int k = 0; k < n_shards; k++) {
    const float* p = part + (static_cast<size_t>(k) * n_rows + r) * kPartWords;
    if (p[4] > 0.0f) S += p[4] * ex2((p[0] - t.v1) * c);
  }
  margin[r] = (1.0f - ex2((t.v2 - t.v1) * c)) / S;
  if (top1) top1[r] = t.i1;
  if (top2) top2[r] = t.i2;
  if (lse) lse[r] = t.v1 * iota + logf(S);
  if (status) status[r] = 0;
}

cudaError_t launch_margin_combine(const float* part, int n_shards, long long n_rows, float iota,
                                  float* margin, int* top1, int* top2, float* lse, uint8_t* status,
                                  cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  const long long blocks = (n_rows + 127) / 128;
  margin_combine_kernel<<<static_cast<unsigned>(blocks), 128, 0, st>>>(part, n_shards, n_rows, iota * kLog2e,
                                                                        iota, margin, top1, top2, lse, status);
  return cudaGetLastError();
}

// Measurement utility (not on the path): a read-only stream of `bytes` the
// way K1 reads — 1-D TMA bulk copies (cp.async.bulk) of 32 KB into a 3-stage
// shared-memory ring, one contiguous slice per CTA, 2 CTAs per SM — without
// any compute; one word per CTA is folded into out so nothing is optimised
// away.  bench.py times it over the logits buffer as the read-only HBM
// ceiling that K1's fraction is also quoted against.
constexpr int kProbeStages = 3;
constexpr int kProbeChunk = 32768;

__global__ void __launch_bounds__(32) read_probe_kernel(const char* __restrict__ p, long long bytes,
                                                        unsigned* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[kProbeStages];
  if (threadIdx.x != 0) return;
  const uint32_t ring_s = smem_u32(ring), full_s = smem_u32(full);
  for (int k = 0; k < kProbeStages; k++) mbar_init(full_s + 8 * k, 1);
  fence_barrier_init();
  const long long chunks = (bytes + kProbeChunk - 1) / kProbeChunk;
  const long long per = (chunks + gridDim.x - 1) / gridDim.x;
  const long long c0 = blockIdx.x * per, c1 = min(chunks, c0 + per);
  const uint64_t pol = policy_evict_first();
  for (long long c = c0; c < c1; c++) {
    const int k = static_cast<int>((c - c0) % kProbeStages);
    const long long it = (c - c0) / kProbeStages;
    if (it > 0) mbar_wait(full_s + 8 * k, static_cast<uint32_t>((it - 1) & 1));
    const uint32_t n = static_cast<uint32_t>(min(static_cast<long long>(kProbeChunk), bytes - c * kProbeChunk));
    mbar_expect_tx(full_s + 8 * k, n);
    bulk_g2s(ring_s + k * kProbeChunk, p + c * kProbeChunk, n, full_s + 8 * k, pol);
  }
  const long long n_it = c1 - c0;
  for (int k = 0; k < kProbeStages && k < n_it; k++) {  // drain: the last copy of each stage
    const long long last = ((n_it - 1 - k) / kProbeStages) * kProbeStages + k;
    mbar_wait(full_s + 8 * k, static_cast<uint32_t>((last / kProbeStages) & 1));
  }
  atomicXor(out + blockIdx.x, *reinterpret_cast<const unsigned*>(ring));
}

cudaError_t launch_read_probe(const void* buf, long long bytes, unsigned* out, cudaStream_t st) {
  const int smem = kProbeStages * kProbeChunk;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(read_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  read_probe_kernel<<<2 * num_sms(), 32, smem, st>>>(static_cast<const char*>(buf), bytes, out);
  return cudaGetLastError();
}

cudaError_t launch_margin_partials_p2p(const void* logits, int dt, long long n_rows, int vocab, long long stride,
                                       long long col_offset, float iota, const TpPeers& peers, cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  RowsArgs a{};
  a.logits = logits; a.n_rows = n_rows; a.vocab = vocab; a.stride = stride;
  a.c = iota * kLog2e; a.iota = iota; a.flat = 0;
  a.col_offset = col_offset; a.tp = peers;
  return launch_rows<kModePartial>(dt, a, CueDev{}, st);
}

// N1 combine over the receive buffer: one thread per row waits (acquire) for
// every rank's partial of this call's tag, then merges as margin_combine.  The
// last CTA out publishes the tag as the completed epoch (the next call's tag
// is epoch + 1; buffers alternate by parity, so a rank one call ahead never
// overwrites a slot still being read) and re-arms the arrival counter.
__device__ __forceinline__ unsigned ld_acquire_sys(const float* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void margin_combine_p2p_kernel(TpPeers pe, long long n_rows, float c, float iota,
                                          float* __restrict__ margin, int* __restrict__ top1,
                                          int* __restrict__ top2, float* __restrict__ lse,
                                          uint8_t* __restrict__ status) {
  const unsigned tag = static_cast<unsigned>(*reinterpret_cast<const volatile int*>(pe.epoch)) + 1u;
  const float* buf = pe.recv[pe.rank] + static_cast<long long>(tag & 1u) * pe.world * pe.rows_cap * kPartWords;
  const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (r < n_rows) {
    Top2 t = top2_empty();
    int nan = 0;
    float v1[kMaxTpRanks], sr[kMaxTpRanks];
    for (int k = 0; k < pe.world; k++) {
      const float* p = buf + (static_cast<long long>(k) * pe.rows_cap + r) * kPartWords;
      while (ld_acquire_sys(p + 7) != tag) {
      }
      // plain loads after the acquire (ordered by it; L1 is not allocated for .cg)
      const float4 a4 = __ldcg(reinterpret_cast<const float4*>(p));
      const float2 b2 = __ldcg(reinterpret_cast<const float2*>(p + 4));
      t = top2_merge(t, Top2{a4.x, a4.y, __float_as_int(a4.z), __float_as_int(a4.w)});
      nan |= __float_as_int(b2.y);
      v1[k] = a4.x;
      sr[k] = b2.x;
    }
    int st = 0;
    if (nan || t.v1 == INFINITY) st = 1;
    else if (t.v1 == -INFINITY) st = 2;
    if (st) {
      margin[r] = qnan();
      if (top1) top1[r] = -1;
      if (top2) top2[r] = -1;
      if (lse) lse[r] = qnan();
      if (status) status[r] = static_cast<uint8_t>(st);
    } else {
      float S = 0.0f;
      for (int k = 0; k < pe.world; k++)
        if (sr[k] > 0.0f) S += sr[k] * ex2((v1[k] - t.v1) * c);
      margin[r] = (1.0f - ex2((t.v2 - t.v1) * c)) / S;
      if (top1) top1[r] = t.i1;
      if (top2) top2[r] = t.i2;
      if (lse) lse[r] = t.v1 * iota + logf(S);
      if (status) status[r] = 0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomic_add_acq_rel(pe.done, 1) == static_cast<int>(gridDim.x) - 1) {
      *pe.done = 0;
      *reinterpret_cast<volatile int*>(pe.epoch) = static_cast<int>(tag);
    }
  }
}

// H6 over peer memory (relay_stats_allreduce_p2p): p2p.cuh, one CTA.
__global__ void __launch_bounds__(256) stats_allreduce_p2p_kernel(TpPeers pe, unsigned long long* stats,
                                                                  long long words) {
  p2p_allreduce_block(pe, stats, words);
}

cudaError_t launch_stats_allreduce_p2p(const TpPeers& peers, unsigned long long* stats, long long words,
                                       cudaStream_t st) {
  stats_allreduce_p2p_kernel<<<1, 256, 0, st>>>(peers, stats, words);
  return cudaGetLastError();
}

cudaError_t launch_margin_combine_p2p(const TpPeers& peers, long long n_rows, float iota, float* margin, int* top1,
                                      int* top2, float* lse, uint8_t* status, cudaStream_t st) {
  const long long blocks = n_rows > 0 ? (n_rows + 127) / 128 : 1;
  margin_combine_p2p_kernel<<<static_cast<unsigned>(blocks), 128, 0, st>>>(peers, n_rows, iota * kLog2e, iota,
                                                                           margin, top1, top2, lse, status);
  return cudaGetLastError();
}

}  // namespace relay
