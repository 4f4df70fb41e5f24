// relay_device.cuh — device-side building blocks shared by the sm_100a kernels
// of librelay.so.  Nothing here is shared with oracle/ (which is plain C).
#pragma once

#include <cfloat>
#include <climits>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace relay {

constexpr unsigned kFull = 0xffffffffu;
// Lazy exp-reference slack in log2 units: a term is at most 2^16 before the
// reference is raised, so fp32 partial sums never overflow (K1).
constexpr float kSlack = 16.0f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float qnan() { return __int_as_float(0x7fffffff); }

// ---------------------------------------------------------------- top-2
// Order: value descending, then index ascending (P:141-146 + R3).  IEEE
// compares: -0 == +0; NaN never ranks (all comparisons with NaN are false).
__device__ __forceinline__ bool better(float a, int ia, float b, int ib) {
  return a > b || (a == b && ia < ib);
}

struct Top2 {
  float v1, v2;
  int i1, i2;
};

__device__ __forceinline__ Top2 top2_empty() { return Top2{-INFINITY, -INFINITY, INT_MAX, INT_MAX}; }

__device__ __forceinline__ void top2_push(Top2& t, float x, int j) {
  if (better(x, j, t.v1, t.i1)) {
    t.v2 = t.v1; t.i2 = t.i1; t.v1 = x; t.i1 = j;
  } else if (better(x, j, t.v2, t.i2)) {
    t.v2 = x; t.i2 = j;
  }
}

__device__ __forceinline__ Top2 top2_merge(const Top2& a, const Top2& b) {
  Top2 r;
  if (better(a.v1, a.i1, b.v1, b.i1)) {
    r.v1 = a.v1; r.i1 = a.i1;
    if (better(a.v2, a.i2, b.v1, b.i1)) { r.v2 = a.v2; r.i2 = a.i2; }
    else { r.v2 = b.v1; r.i2 = b.i1; }
  } else {
    r.v1 = b.v1; r.i1 = b.i1;
    if (better(a.v1, a.i1, b.v2, b.i2)) { r.v2 = a.v1; r.i2 = a.i1; }
    else { r.v2 = b.v2; r.i2 = b.i2; }
  }
  return r;
}

// ------------------------------------------------- softmax normaliser
// s = sum_j 2^(y_j - m), y = z * c (c = iota * log2 e), m a lazily raised
// reference (never above the row maximum).
struct Norm {
  float m, s;
};

__device__ __forceinline__ Norm norm_merge(const Norm& a, const Norm& b) {
  float m = fmaxf(a.m, b.m);
  return Norm{m, a.s * ex2(a.m - m) + b.s * ex2(b.m - m)};
}

// Row partial: everything a (row, range) pass produces.  flags bit 0 (huge):
// some exp reference reached |y| >= 2^28, where fp32 y = z*c can no longer
// resolve the distances that matter, so the row takes an exact second pass;
// bit 1: a NaN was seen (status 1).
struct Partial {
  Top2 t;
  Norm n;
  int flags;
};
constexpr int kFlagHuge = 1;
constexpr int kFlagNan = 2;

__device__ __forceinline__ Partial partial_merge(const Partial& a, const Partial& b) {
  return Partial{top2_merge(a.t, b.t), norm_merge(a.n, b.n), a.flags | b.flags};
}

__device__ __forceinline__ Partial shfl_xor_partial(const Partial& p, int off) {
  Partial o;
  o.t.v1 = __shfl_xor_sync(kFull, p.t.v1, off);
  o.t.v2 = __shfl_xor_sync(kFull, p.t.v2, off);
  o.t.i1 = __shfl_xor_sync(kFull, p.t.i1, off);
  o.t.i2 = __shfl_xor_sync(kFull, p.t.i2, off);
  o.n.m = __shfl_xor_sync(kFull, p.n.m, off);
  o.n.s = __shfl_xor_sync(kFull, p.n.s, off);
  o.flags = __shfl_xor_sync(kFull, p.flags, off);
  return o;
}

__device__ __forceinline__ Partial warp_reduce_partial(Partial p) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) p = partial_merge(p, shfl_xor_partial(p, off));
  return p;
}

// Order-preserving float <-> int key (for atomicMax on a shared threshold).
__device__ __forceinline__ int fkey(float f) {
  int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float unkey(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// Order-preserving key of a top-2 value with -0 folded onto +0 (better()
// ranks them equal; their tie then falls to the lower index).  Values are
// never NaN here (NaN never enters a top-2).
__device__ __forceinline__ int top_key(float v) {
  const int i = __float_as_int(v == 0.0f ? 0.0f : v);
  return i >= 0 ? i : i ^ 0x7fffffff;
}

// Warp-wide merge of 32 partials, the result on every lane, by redux.sync
// instead of a 5-round shuffle butterfly of partial_merge (35 shuffles and 10
// MUFU in a dependent chain: ~0.5 us of the decode step's tail).  Top-2:
// the best (value, index) is the max key, then the min index among lanes
// holding it; the 2nd best is the best of every lane's first entry with the
// winner's lane offering its second.  Normaliser: max exponent reference,
// each lane's sum rescaled to it, one sum.  Same results as partial_merge
// trees up to the rounding order of the normaliser sum.
__device__ __forceinline__ Partial warp_merge_all(const Partial& p) {
  const int k1 = top_key(p.t.v1);
  const int K1 = __reduce_max_sync(kFull, k1);
  const int I1 = static_cast<int>(
      __reduce_min_sync(kFull, k1 == K1 ? static_cast<unsigned>(p.t.i1) : 0xffffffffu));
  const bool hold = k1 == K1 && p.t.i1 == I1;
  const int k2 = top_key(hold ? p.t.v2 : p.t.v1);
  const int c2 = hold ? p.t.i2 : p.t.i1;
  const int K2 = __reduce_max_sync(kFull, k2);
  const int I2 = static_cast<int>(
      __reduce_min_sync(kFull, k2 == K2 ? static_cast<unsigned>(c2) : 0xffffffffu));
  const int KM = __reduce_max_sync(kFull, fkey(p.n.m));
  const float M = unkey(KM);
  float s = p.n.s * ex2(p.n.m - M);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  Partial r;
  r.t.v1 = unkey(K1);
  r.t.i1 = I1;
  r.t.v2 = unkey(K2);
  r.t.i2 = I2;
  r.n.m = M;
  r.n.s = s;
  r.flags = static_cast<int>(__reduce_or_sync(kFull, static_cast<unsigned>(p.flags)));
  return r;
}


// Finish a row: margin, lse, status (R4).  c = iota*log2e, iota = c/log2e.
// n.s sums 2^(fl(z_j c - m)) with fma, i.e. every term carries the same
// shift delta = exact(z1 c) - fl(z1 c) relative to the row maximum; it is
// removed exactly with fma(z1, c, -My) (the rounding error of a product is
// representable).  S_exact (when >= 0) replaces the normaliser (exact pass).
struct RowOut {
  float margin, lse;
  int i1, i2;
  int status;
};

__device__ __forceinline__ RowOut finish_row(const Partial& p, float c, float iota,
                                             bool exact = false, float S_exact = 0.0f) {
  RowOut o;
  if ((p.flags & kFlagNan) || isnan(exact ? S_exact : p.n.s) || p.t.v1 == INFINITY) {
    o.status = 1;
  } else if (p.t.v1 == -INFINITY) {
    o.status = 2;
  } else {
    o.status = 0;
  }
  if (o.status != 0) {
    o.margin = qnan(); o.lse = qnan(); o.i1 = -1; o.i2 = -1;
    return o;
  }
  float S, p2;
  if (exact) {                                    // exact pass: sum of 2^((z - z1) c)
    S = S_exact;
    p2 = ex2((p.t.v2 - p.t.v1) * c);
  } else {
    const float My = p.t.v1 * c;
    const float d1 = fmaf(p.t.v1, c, -My);        // exact(z1 c) - My
    S = p.n.s * ex2((p.n.m - My) - d1);           // S = sum_j exp((z_j - z1) iota)
    p2 = ex2(fmaf(p.t.v2, c, -My) - d1);          // exp((z2 - z1) iota), 0 for -inf
  }
  o.margin = (1.0f - p2) / S;
  o.lse = p.t.v1 * iota + logf(S);
  o.i1 = p.t.i1;
  o.i2 = p.t.i2;
  return o;
}

// ------------------------------------------------------------ loads
__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

struct U8x32 {
  uint32_t w[8];
};

__device__ __forceinline__ U8x32 ldg_stream32(const void* p) {
  U8x32 r;
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
        "=r"(r.w[6]), "=r"(r.w[7])
      : "l"(p));
  return r;
}

// Element formats.  unpack2 turns one 32-bit word into two fp32 values
// (exact for bf16/f16); pmax is the NaN-propagating packed max of two words
// (HMNMX2.NAN), used to reduce a whole stage before unpacking.
struct EBf16 {
  using T = uint16_t;
  static constexpr int SZ = 2;
  static constexpr bool kBf16 = true;
  __device__ static __forceinline__ void unpack2(uint32_t w, float& lo, float& hi) {
    lo = __uint_as_float(w << 16);
    hi = __uint_as_float(w & 0xffff0000u);
  }
  __device__ static __forceinline__ uint32_t pmax(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
  }
  __device__ static __forceinline__ float load1(const T* p) {
    return __uint_as_float(static_cast<uint32_t>(__ldg(reinterpret_cast<const unsigned short*>(p))) << 16);
  }
  __device__ static __forceinline__ uint4 neg_inf16() { return make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u); }
};

struct EF16 {
  using T = uint16_t;
  static constexpr int SZ = 2;
  static constexpr bool kBf16 = false;
  __device__ static __forceinline__ void unpack2(uint32_t w, float& lo, float& hi) {
    __half2 h = *reinterpret_cast<__half2*>(&w);
    float2 f = __half22float2(h);
    lo = f.x;
    hi = f.y;
  }
  __device__ static __forceinline__ uint32_t pmax(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.NaN.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
  }
  __device__ static __forceinline__ float load1(const T* p) {
    unsigned short b = __ldg(reinterpret_cast<const unsigned short*>(p));
    return __half2float(__ushort_as_half(b));
  }
  __device__ static __forceinline__ uint4 neg_inf16() { return make_uint4(0xfc00fc00u, 0xfc00fc00u, 0xfc00fc00u, 0xfc00fc00u); }
};

struct EF32 {
  using T = float;
  static constexpr int SZ = 4;
  static constexpr bool kBf16 = false;
  __device__ static __forceinline__ void unpack2(uint32_t, float&, float&) {}
  __device__ static __forceinline__ uint32_t pmax(uint32_t a, uint32_t) { return a; }
  __device__ static __forceinline__ float load1(const T* p) { return __ldg(p); }
  __device__ static __forceinline__ uint4 neg_inf16() { return make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u); }
};

// NaN-propagating maxima (FMNMX.NAN / FMNMX3.NAN).
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float max3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// --------------------------------------------- mbarrier + TMA bulk copy
// All helpers take 32-bit shared-window addresses computed once per kernel.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// The same address, opaque to the compiler: kept in a register instead of
// being re-derived from SR_CgaCtaId (an S2R) inside hot loops.
__device__ __forceinline__ uint32_t smem_u32_pinned(const void* p) {
  uint32_t r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

#ifndef RELAY_PRODUCER_SLEEP_NS
#define RELAY_PRODUCER_SLEEP_NS 256
#endif
// Producer-side wait: the thread is suspended (up to ~hint ns) instead of
// spinning on issue slots while the ring is full.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t done;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(20000u)
        : "memory");
    if (done) return;
    __nanosleep(RELAY_PRODUCER_SLEEP_NS);
  }
}

#ifndef RELAY_WAIT_HINT_NS
#define RELAY_WAIT_HINT_NS 0  // consumer try_wait suspend-time hint (0: none)
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#if RELAY_WAIT_HINT_NS > 0
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "n"(RELAY_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
#endif
}

// 1-D TMA: global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).  evict_first: logits are read once.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// L2 evict_last: the row stays in L2 for a second, L2-resident pass (N2).
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 16-byte global load with an L2 cache-eviction policy.
__device__ __forceinline__ uint4 ldg_hint(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ------------------------------------------ 16-byte vector helpers
template <class E>
__device__ __forceinline__ void unpack16(const uint4& r, float (&f)[16 / E::SZ]) {
  if constexpr (E::SZ == 4) {
    f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
    f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
  } else {
    E::unpack2(r.x, f[0], f[1]); E::unpack2(r.y, f[2], f[3]);
    E::unpack2(r.z, f[4], f[5]); E::unpack2(r.w, f[6], f[7]);
  }
}

// Maximum of one 16-byte vector (NaN-propagating).
template <class E>
__device__ __forceinline__ float vec_max(const uint4& r) {
  if constexpr (E::SZ == 2) {
    float lo, hi;
    E::unpack2(E::pmax(E::pmax(r.x, r.y), E::pmax(r.z, r.w)), lo, hi);
    return max_nan(lo, hi);
  } else {
    return max_nan(max_nan(__uint_as_float(r.x), __uint_as_float(r.y)),
                   max_nan(__uint_as_float(r.z), __uint_as_float(r.w)));
  }
}

// Element k (dynamic, < 16 / SZ) of a 16-byte vector, without local memory.
template <class E>
__device__ __forceinline__ float elem_at(const uint4& r, int k) {
  if constexpr (E::SZ == 2) {
    const uint32_t w = (k & 4) ? ((k & 2) ? r.w : r.z) : ((k & 2) ? r.y : r.x);
    float lo, hi;
    E::unpack2(w, lo, hi);
    return (k & 1) ? hi : lo;
  } else {
    return __uint_as_float((k & 2) ? ((k & 1) ? r.w : r.z) : ((k & 1) ? r.y : r.x));
  }
}

// Programmatic dependent launch (sm_90+): let the next kernel in the stream
// start its prologue / wait until the previous kernel has completed.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// Arrive on a named barrier without waiting (release: this thread's earlier
// accesses are performed for the threads that sync on it).
__device__ __forceinline__ void bar_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// bar_arrive that also pins the stage's loaded words: every load of raw[]
// completes before the arrive and every use of raw[] comes after it, so the
// ring slot is released as soon as it is read (the scheduler otherwise
// interleaves the loads with the math and releases late, shrinking the
// effective ring depth).
template <int UV>
__device__ __forceinline__ void bar_arrive_pinned(int id, int threads, uint4 (&raw)[UV]) {
#pragma unroll
  for (int u = 0; u < UV; u++)
    asm volatile("" : "+r"(raw[u].x), "+r"(raw[u].y), "+r"(raw[u].z), "+r"(raw[u].w));
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
#pragma unroll
  for (int u = 0; u < UV; u++)
    asm volatile("" : "+r"(raw[u].x), "+r"(raw[u].y), "+r"(raw[u].z), "+r"(raw[u].w));
}
// Order this thread's view of shared memory (generic proxy) before its
// subsequent async-proxy (TMA) operations on it.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------ thread-block clusters / DSMEM (K4)
// The shared::cluster address of the same variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_cluster(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// Arrive (release at cluster scope) on an mbarrier in another CTA of the cluster.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Wait (acquire at cluster scope) on a local mbarrier completed by remote arrivals.
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// The same 16 bytes through an opaque move (the compiler cannot reuse values
// derived from the input across it).
__device__ __forceinline__ uint4 opaque(uint4 v) {
  asm volatile("" : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w));
  return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr));
  return r;
}

}  // namespace relay
