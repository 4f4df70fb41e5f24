// sample_kernels.cu — K5, the second half of relay_step_sample (N2: the
// margin fused with the decode-side sampler).
//
// The paper samples every model at temperature 0.6 with top-p 0.95 (and top-k
// 20 for Qwen3).  K4 streams each row (margin, top-2, and a lower
// bound thk on the row's top_k-th largest logit) with L2 evict_last; K5
// re-reads each row, collects the logits >= thk (~100 per row), selects the
// exact top-k in (value desc, index asc) order, applies temperature and top-p,
// draws the token by inverse CDF with the caller's uniform (reading R20), and
// runs the decode-step switch (H8) on the drawn token.  The second read hits
// L2 only for small batches (B200's L2 holds ~60 MB per partition; configs[2]
// is 78 MB); DESIGN.md records the single-pass variants that measured slower.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "relay_device.cuh"
#include "relay_internal.h"
#include "draw.cuh"
#include "switch.cuh"

namespace relay {

constexpr int kSampleThreads = 512;

#ifdef RELAY_TRACE
// Tuning-only timeline of K5 (tools/k5_trace.py): %globaltimer stamps of the
// first row of each CTA, by thread 0.  1 candidates collected, 2 top list,
// 3 row mass, 4-12 nucleus phases, 15 row done.
__device__ unsigned long long g_trace5[1024][16];
__device__ __forceinline__ void stamp5(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_trace5[blockIdx.x][k] = t;
}
extern "C" int relay_debug_trace5_copy(unsigned long long* host, int n_ctas) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace5, sizeof(unsigned long long) * 16 * n_ctas));
}
#define TRACE5(k) stamp5(k)
#else
#define TRACE5(k) ((void)0)
#endif
constexpr int kCandCap = 1024;  // candidates held in shared memory; more -> exact global fallback
constexpr int kSlowCtas = 64;   // K6 grid: slow rows handled concurrently

__device__ __forceinline__ int atomic_add_acq_rel_i(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

struct SampleArgs {
  const void* logits;
  long long n_rows;
  int vocab;
  long long stride;
  const float* thk;         // [n_rows] K4's lower bound on the top_k-th largest logit
  const uint8_t* status;    // [n_rows] K4's row status (0 = sample)
  const float* margin;      // [n_rows] K4's margins (the switch's optional gate)
  float s_c;                // log2(e) / temperature
  int topk;                 // 1..kMaxTopK, <= vocab; 0 = no top-k (nucleus over the row)
  const float* zmax;        // [n_rows] K4's row maximum (nucleus mode)
  float topp;               // (0, 1]
  const float* uniform;     // [n_rows] in [0, 1)
  int* slow_cnt;            // [2] K6 list length, K6 CTAs done (zero between launches)
  int* slow_list;           // [n_rows] rows K5 handed to K6
  float* zsum;              // [n_rows] K5's row mass at the sampling temperature (listed rows)
  int k5_l2;                // tuning: 0 default policy, 1 evict_last, 2 evict_normal (RELAY_K5_L2)
  int* ready_q;             // [n_rows] rows in K4's completion order (row + 1; acquire; re-zeroed here)
  int* q_ctl;               // [4] queue head (K4), tail (this kernel's tickets), CTAs done
  int* sampled;             // [n_rows] out
  uint8_t* state;
  int* hist;
  int* small_run;
  float gate;
  int max_seg;
  uint8_t* flag;
  int16_t* cue_id;
};

// (v, i) ranks before (bv, bi): value descending, index ascending.
__device__ __forceinline__ bool ranks_before(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

__device__ __forceinline__ void warp_best(float& bv, int& bi) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_xor_sync(kFull, bv, off);
    const int oi = __shfl_xor_sync(kFull, bi, off);
    if (ranks_before(ov, oi, bv, bi)) { bv = ov; bi = oi; }
  }
}

// -inf entries are never candidates: their probability is 0, so they can
// neither be drawn nor move the top-p cut (R20).
__device__ __forceinline__ void push_candidate(float v, int j, float th, bool strict, float* s_cv,
                                               int* s_ci, int* s_cnt) {
  if ((strict ? v > th : v >= th) && v > -INFINITY) {  // false for NaN
    const int p = atomicAdd(s_cnt, 1);
    if (p < kCandCap) { s_cv[p] = v; s_ci[p] = j; }
  }
}

// Every finite logit >= th (> th when strict) of one row into the candidate
// list (block-wide).  MASS: also this thread's share of the row's mass at the
// sampling temperature, sum_j 2^(z_j s_c - z1 s_c) (packed FFMA2 / FADD2,
// MUFU.EX2; -inf entries give 2^-inf = 0).
template <class E, bool MASS>
__device__ float collect_candidates(const typename E::T* row, int vocab, float th, bool strict,
                                    float* s_cv, int* s_ci, int* s_cnt, float z1 = 0.0f,
                                    float s_c = 0.0f, int k5_l2 = 0) {
  constexpr int VEC = 16 / E::SZ;
  const float2 cc = make_float2(s_c, s_c);
  const float2 nm = make_float2(-z1 * s_c, -z1 * s_c);
  float2 acc = make_float2(0.0f, 0.0f);
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  auto scalar = [&](int j) {
    const float x = E::load1(row + j);
    push_candidate(x, j, th, strict, s_cv, s_ci, s_cnt);
    if constexpr (MASS) acc.x += ex2(fmaf(x, s_c, nm.x));
  };
  for (int j = threadIdx.x; j < head; j += blockDim.x) scalar(j);
  for (int j = tail + threadIdx.x; j < vocab; j += blockDim.x) scalar(j);
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  // top-k mode: the row's last use, leave L2; nucleus mode: a slow row is read again
  const uint64_t pol = k5_l2 == 1 ? policy_evict_last() : k5_l2 == 2 ? policy_evict_normal()
                       : MASS ? policy_evict_normal() : policy_evict_first();
  const volatile int* cnt_v = s_cnt;
  auto body = [&](const uint4& xv, int v) {
    if constexpr (MASS) {
      float f[VEC];
      unpack16<E>(xv, f);
#pragma unroll
      for (int k = 0; k < VEC; k += 2) {
        const float2 y = __ffma2_rn(make_float2(f[k], f[k + 1]), cc, nm);
        acc = __fadd2_rn(acc, make_float2(ex2(y.x), ex2(y.y)));
      }
    }
    // once the list overflowed only the fact matters (the caller resolves
    // the row exactly): a constant row would otherwise queue one atomic per
    // element on the counter
    if (vec_max<E>(xv) >= th && *cnt_v <= kCandCap) {
      float f[VEC];
      unpack16<E>(xv, f);
      unsigned m = 0;
#pragma unroll
      for (int k = 0; k < VEC; k++) m |= ((strict ? f[k] > th : f[k] >= th) && f[k] > -INFINITY) ? (1u << k) : 0u;
      if (m) {
        int p = atomicAdd(s_cnt, __popc(m));  // one slot reservation per vector
        while (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1;
          if (p < kCandCap) { s_cv[p] = f[k]; s_ci[p] = head + v * VEC + k; }
          p++;
        }
      }
    }
  };
  constexpr int U = 8;  // loads in flight per thread
  int v0 = threadIdx.x;
  for (; v0 + (U - 1) * static_cast<int>(blockDim.x) < nvec; v0 += U * blockDim.x) {  // full rounds
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; u++) x[u] = ldg_hint(vp + v0 + u * blockDim.x, pol);
#pragma unroll
    for (int u = 0; u < U; u++) body(x[u], v0 + u * blockDim.x);
  }
  for (int v = v0; v < nvec; v += blockDim.x) body(ldg_hint(vp + v, pol), v);  // the last round
  return acc.x + acc.y;
}

// The first `want` entries of the candidate list in (value desc, index asc)
// order into s_topv/s_topi: every thread ranks its candidates by counting
// the entries that rank before them (ranks are distinct: indices are).
// Returns how many exist (min(want, n)).
__device__ int rank_list(int want, int n, const float* s_cv, const int* s_ci, float* s_topv,
                         int* s_topi, int* s_k) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const float v = s_cv[e];
    const int i = s_ci[e];
    int rank = 0;
    int f = 0;
    // 4 independent compares per step (broadcast 16-byte shared loads): the
    // early exit is tested once per 4, so the loop is not latency-bound
    for (; f + 4 <= n && rank < want; f += 4) {
      const float4 va = *reinterpret_cast<const float4*>(s_cv + f);
      const int4 ia = *reinterpret_cast<const int4*>(s_ci + f);
      rank += ranks_before(va.x, ia.x, v, i) + ranks_before(va.y, ia.y, v, i) +
              ranks_before(va.z, ia.z, v, i) + ranks_before(va.w, ia.w, v, i);
    }
    for (; f < n && rank < want; f++) rank += ranks_before(s_cv[f], s_ci[f], v, i);
    if (rank < want) { s_topv[rank] = v; s_topi[rank] = i; }
  }
  if (threadIdx.x == 0) *s_k = n < want ? n : want;
  __syncthreads();
  return *s_k;
}

// The entries equal to v in index order: take(rank, index) for each of the
// first `limit` of them.  Chunks of 4 coalesced 16-byte vectors per thread
// (all loads in flight at once), ordered (vector slot, thread, element) =
// index order, with one block scan per chunk; stops after the chunk that
// reaches `limit`.  The unaligned head / tail scalars are taken by thread 0.
// Block-wide; s_scan holds >= 4 * (blockDim / 32) ints.
template <class E, class F>
__device__ void tie_scan(const typename E::T* row, int vocab, float v, int limit, int* s_scan, F take) {
  constexpr int VEC = 16 / E::SZ, U = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  __shared__ int s_base;
  if (threadIdx.x == 0) {
    int r = 0;
    for (int j = 0; j < head; j++)
      if (E::load1(row + j) == v) { if (r < limit) take(r, j); r++; }
    s_base = r;
  }
  __syncthreads();
  int base = s_base;
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  for (int c0 = 0; c0 < nvec && base < limit; c0 += U * blockDim.x) {  // block-uniform
    unsigned m[U];
    int cnt[U], incl[U];
    uint4 r[U];
#pragma unroll
    for (int q = 0; q < U; q++) {
      const int vi = c0 + q * blockDim.x + threadIdx.x;
      if (vi < nvec) r[q] = __ldg(vp + vi);
    }
#pragma unroll
    for (int q = 0; q < U; q++) {
      const int vi = c0 + q * blockDim.x + threadIdx.x;
      m[q] = 0;
      if (vi < nvec) {
        float f[VEC];
        unpack16<E>(r[q], f);
#pragma unroll
        for (int k = 0; k < VEC; k++) m[q] |= (f[k] == v) ? (1u << k) : 0u;
      }
      cnt[q] = __popc(m[q]);
      incl[q] = cnt[q];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(kFull, incl[q], off);
        if (lane >= off) incl[q] += t;
      }
    }
    __syncthreads();  // the previous chunk's reads of s_scan are done
    if (lane == 31) {
#pragma unroll
      for (int q = 0; q < U; q++) s_scan[q * nw + warp] = incl[q];
    }
    __syncthreads();
    int before_q = base;  // ties in earlier vector slots of this chunk
#pragma unroll
    for (int q = 0; q < U; q++) {
      int pre = 0, tot = 0;
      for (int w = 0; w < nw; w++) {
        const int x = s_scan[q * nw + w];
        if (w < warp) pre += x;
        tot += x;
      }
      int rk = before_q + pre + incl[q] - cnt[q];
      unsigned mm = m[q];
      const int vi = c0 + q * blockDim.x + threadIdx.x;
      while (mm && rk < limit) {
        const int k = __ffs(mm) - 1;
        mm &= mm - 1;
        take(rk++, head + vi * VEC + k);
      }
      before_q += tot;
    }
    base = before_q;
  }
  if (base < limit && threadIdx.x == 0) {
    int rk = base;
    for (int j = tail; j < vocab; j++)
      if (E::load1(row + j) == v) { if (rk < limit) take(rk, j); rk++; }
  }
  __syncthreads();
}

// The exact top-k of a row whose candidate list (entries >= thk) overflowed,
// e.g. a constant row.  theta = the k-th largest value in the (partial) list
// is a value of k real entries, so the row's k-th largest is >= theta; collect
// the entries > theta: on overflow raise theta again (strictly), else they are
// all of them and, if fewer than k, the rest of the top-k are the
// lowest-index entries equal to theta (collected in index order).
template <class E>
__device__ __noinline__ int refine_topk(const typename E::T* row, int vocab, int topk, float zmax, float* s_cv,
                                        int* s_ci, int* s_cnt, float* s_topv, int* s_topi, int* s_k,
                                        int* s_scan) {
  float theta;
  // at least topk entries of the (partial) list equal the row maximum: the
  // top-k are the lowest-index entries at the maximum (a constant row; no
  // ranking of the full list, which costs ~18 us when every value ties)
  int at_max = 0;  // entries of the list equal to the row maximum (block-uniform)
  for (int e0 = 0; e0 < kCandCap; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    at_max += __syncthreads_count(e < kCandCap && s_cv[e] == zmax);
  }
  if (at_max >= topk) {
    theta = zmax;
    if (threadIdx.x == 0) *s_cnt = 0;
    __syncthreads();
  } else {
  for (;;) {
    if (rank_list(topk, kCandCap, s_cv, s_ci, s_topv, s_topi, s_k) < topk) return *s_k;
    TRACE5(6);
    theta = s_topv[topk - 1];
    __syncthreads();
    if (threadIdx.x == 0) *s_cnt = 0;
    __syncthreads();
    // nothing exceeds the row maximum (K4's): a constant top needs no pass
    if (theta == zmax) break;
    collect_candidates<E, false>(row, vocab, theta, true, s_cv, s_ci, s_cnt);
    __syncthreads();
    if (*s_cnt <= kCandCap) break;
  }
  }
  const int c = *s_cnt;
  if (c >= topk) return rank_list(topk, c, s_cv, s_ci, s_topv, s_topi, s_k);
  // the lowest-index entries equal to theta, in index order
  const int need = topk - c;
  tie_scan<E>(row, vocab, theta, need, s_scan, [&](int r, int idx) {
    s_cv[c + r] = theta;
    s_ci[c + r] = idx;
  });
  TRACE5(7);
  return rank_list(topk, c + need, s_cv, s_ci, s_topv, s_topi, s_k);
}

// The drawn token (one warp) from the top-K list: draw.cuh.
__device__ __forceinline__ int draw_warp(const SampleArgs& a, float u, int K, const float* s_topv,
                                         const int* s_topi, float total_mass = -1.0f) {
  return draw_topk_warp(a.s_c, a.topp, u, K, s_topv, s_topi, total_mass);
}

// ---------------------------------------------------------------- nucleus
// No top-k (the R1-Distill setting): the kept set is the rank prefix
// whose higher-ranked mass is below top_p * Z, Z = the row's total mass at the
// sampling temperature, w(x) = 2^((x - z1) log2(e) / T).  When the top-64
// already hold top_p * Z the draw uses them; otherwise the row is resolved by
// mass-rank selection over value bins.

// f(x, j) for every element of the row (block-strided 16-byte vectors plus the
// unaligned head / tail), 4 vector loads in flight per thread.  Default L2
// policy: the slow paths read a row several times, the later passes hit L2.
template <class E, class F>
__device__ __forceinline__ void for_each_elem(const typename E::T* row, int vocab, F f) {
  constexpr int VEC = 16 / E::SZ;
  constexpr int U = 4;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  for (int j = threadIdx.x; j < head; j += blockDim.x) f(E::load1(row + j), j);
  for (int j = tail + threadIdx.x; j < vocab; j += blockDim.x) f(E::load1(row + j), j);
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  for (int v0 = threadIdx.x; v0 < nvec; v0 += U * blockDim.x) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int v = v0 + u * blockDim.x;
      if (v < nvec) r[u] = __ldg(vp + v);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int v = v0 + u * blockDim.x;
      if (v >= nvec) break;
      float x[VEC];
      unpack16<E>(r[u], x);
#pragma unroll
      for (int k = 0; k < VEC; k++) f(x[k], head + v * VEC + k);
    }
  }
}

__device__ __forceinline__ float block_sum(float v, float* s_red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  float t = 0.0f;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); w++) t += s_red[w];
  return t;
}

__device__ __forceinline__ float block_min(float v, float* s_red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fminf(v, __shfl_xor_sync(kFull, v, off));
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  float t = INFINITY;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); w++) t = fminf(t, s_red[w]);
  return t;
}

// Masses in fixed point, w_q(x) = rint(2^((x - z1) s_c) * 2^42) (uint64 sums:
// exact and order-free).  Shared-memory histograms accumulate them as three
// 14-bit digits with native 32-bit atomics (64-bit and float shared atomics
// are CAS loops on sm_100; under contention they serialise): every digit sum
// is < vocab * 2^14 < 2^32 for vocab < 2^18 (host-checked).
constexpr float kFix = 4398046511104.0f;  // 2^42

__device__ __forceinline__ unsigned long long wq(float x, float z1, float s_c) {
  return __float2ull_rn(ex2((x - z1) * s_c) * kFix);
}

struct NucleusSmem {
  unsigned d1[3][256];  // level 1: mass digits per bin (kept for the second selection)
  unsigned c1[256];     // level 1: count per bin
  unsigned d[3][256];   // deeper levels
  unsigned c[256];
  float red[kSampleThreads / 32];
  float redmin[kSampleThreads / 32];
  int sel_bin, sel_n;
  unsigned long long sel_before;
  int tok;                  // >= 0: the selected entry; -2: a tie block (tie_v, tie_j)
  unsigned long long incl;  // inclusive mass up to the selected entry
  float tie_v;
  int tie_j;
};

__device__ __forceinline__ unsigned long long digits_mass(const unsigned (*d)[256], int b) {
  return static_cast<unsigned long long>(d[0][b]) + (static_cast<unsigned long long>(d[1][b]) << 14) +
         (static_cast<unsigned long long>(d[2][b]) << 28);
}

// Warp-aggregated histogram update (bin b < 0: none); every lane calls it.
// When the whole warp hits one bin (constant rows, tie blocks) one set of
// atomics replaces 32.
__device__ __forceinline__ void hist_add(int b, unsigned long long w, unsigned (*d)[256], unsigned* c) {
  const int b0 = __shfl_sync(kFull, b, 0);
  int n = 1;
  if (__all_sync(kFull, b == b0)) {
    if (b0 < 0) return;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) w += __shfl_xor_sync(kFull, w, off);
    if ((threadIdx.x & 31) != 0) return;
    n = 32;
  }
  if (b < 0) return;
  const unsigned w0 = static_cast<unsigned>(w & 0x3fff), w1 = static_cast<unsigned>((w >> 14) & 0x3fff);
  const unsigned w2 = static_cast<unsigned>(w >> 28);  // < 2^14 per entry (w <= 2^42), or the warp's sum
  if (w0) atomicAdd(&d[0][b], w0);
  if (w1) atomicAdd(&d[1][b], w1);
  if (w2) atomicAdd(&d[2][b], w2);
  atomicAdd(&c[b], static_cast<unsigned>(n));
}

// f(x, j) for every element of the row with a block-uniform trip count (every
// lane of every warp calls f the same number of times; padding lanes get
// x = -inf, j = -1), so f may use warp collectives.
template <class E, class F>
__device__ __forceinline__ void for_each_elem_uniform(const typename E::T* row, int vocab, F f) {
  constexpr int VEC = 16 / E::SZ;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  {  // the unaligned head and tail: at most 2 * (VEC - 1) scalars, one round
    const int t = threadIdx.x;
    const int j = t < head ? t : (t - head < vocab - tail ? tail + (t - head) : -1);
    f(j >= 0 ? E::load1(row + j) : -INFINITY, j);
  }
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  constexpr int U = 4;
  for (int v0 = 0; v0 < nvec; v0 += U * blockDim.x) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int v = v0 + u * blockDim.x + threadIdx.x;
      r[u] = v < nvec ? __ldg(vp + v) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int v = v0 + u * blockDim.x + threadIdx.x;
      float x[VEC];
      unpack16<E>(r[u], x);
#pragma unroll
      for (int k = 0; k < VEC; k++) f(v < nvec ? x[k] : -INFINITY, v < nvec ? head + v * VEC + k : -1);
    }
  }
}

// The first entry in (value desc, index asc) order whose inclusive cumulative
// mass crosses `target` (> when strict, else >=), masses w_q (fixed point).
// Entries are binned by value, linearly over [lo, hi] (256 bins, largest
// values first: bin order is rank order, ties share a bin); the level-1 range
// is [z1 - 64 / s_c, z1] (below it an entry weighs < 2^-64 of the top one, so
// the excluded mass is < vocab * 2^-64 of Z).  The crossing bin's entries are
// ranked in the candidate list when they fit; otherwise the bin's exact value
// range [min, max] becomes the next level, until it holds one value — a tie
// block, whose entries rank by index: the crossing is the j-th of them (from
// the mass arithmetic), its index found later by tie_index (only the draw
// needs it).  Sets ns.tok / ns.tie_v / ns.tie_j and ns.incl (block-uniform).
// The level-1 histogram does not depend on the target: with l1_ready the one
// a previous call on the same row left in ns.d1 / ns.c1 is reused.
template <class E>
__device__ __noinline__ void select_by_mass(const typename E::T* row, int vocab, float z1, float s_c,
                                            double target, bool strict, bool l1_ready, NucleusSmem& ns,
                                            float* s_cv, int* s_ci, int* s_cnt, int* s_scan) {
  float hi = z1, lo = z1 - 64.0f / s_c;
  unsigned long long before = 0;  // mass of the entries ranked before [lo, hi]
  auto crosses = [&](unsigned long long c) {
    return strict ? static_cast<double>(c) > target : static_cast<double>(c) >= target;
  };
  for (int level = 0;; level++) {
    unsigned (*d)[256] = level == 0 ? ns.d1 : ns.d;
    unsigned* c = level == 0 ? ns.c1 : ns.c;
    const float scale = 256.0f / (hi - lo);  // hi > lo
    auto bin_of = [&](float x) -> int {      // -1: outside [lo, hi] (and NaN, -inf)
      if (!(x >= lo && x <= hi)) return -1;
      return min(255, static_cast<int>((hi - x) * scale));
    };
    if (level > 0 || !l1_ready) {
      for (int b = threadIdx.x; b < 256; b += blockDim.x) {
        d[0][b] = 0; d[1][b] = 0; d[2][b] = 0; c[b] = 0;
      }
      __syncthreads();
      for_each_elem_uniform<E>(row, vocab, [&](float x, int) {
        const int b = bin_of(x);
        hist_add(b, b >= 0 ? wq(x, z1, s_c) : 0ull, d, c);
      });
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long cum = before, bef = before;
      int bsel = -1;
      for (int b = 0; b < 256; b++) {
        if (!c[b]) continue;
        const unsigned long long next = cum + digits_mass(d, b);
        bsel = b;
        bef = cum;
        if (crosses(next)) break;
        cum = next;
      }
      ns.sel_bin = bsel;  // the crossing bin (or the last non-empty one: rounding)
      ns.sel_before = bef;
      ns.sel_n = bsel >= 0 ? static_cast<int>(c[bsel]) : 0;
    }
    __syncthreads();
    const int bsel = ns.sel_bin, n = ns.sel_n;
    before = ns.sel_before;
    if (n <= kCandCap) {
      if (threadIdx.x == 0) *s_cnt = 0;
      __syncthreads();
      for_each_elem<E>(row, vocab, [&](float x, int j) {
        if (bin_of(x) == bsel) {
          const int p = atomicAdd(s_cnt, 1);
          if (p < kCandCap) { s_cv[p] = x; s_ci[p] = j; }
        }
      });
      __syncthreads();
      // rank every entry (indices make ranks distinct), then scan in rank order
      for (int e = threadIdx.x; e < n; e += blockDim.x) {
        int rank = 0;
        for (int f = 0; f < n; f++) rank += ranks_before(s_cv[f], s_ci[f], s_cv[e], s_ci[e]);
        s_scan[rank] = e;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long cum = before, incl = before;
        int tok = n ? s_ci[s_scan[n - 1]] : -1;
        for (int k = 0; k < n; k++) {
          const int e = s_scan[k];
          cum += wq(s_cv[e], z1, s_c);
          incl = cum;
          if (crosses(cum)) { tok = s_ci[e]; break; }
        }
        ns.tok = tok;
        ns.incl = incl;
      }
      __syncthreads();
      return;
    }
    // too many entries: the bin's exact value range (one pass, no atomics)
    float mn = INFINITY, mx = -INFINITY;
    for_each_elem<E>(row, vocab, [&](float x, int) {
      if (bin_of(x) == bsel) { mn = fminf(mn, x); mx = fmaxf(mx, x); }
    });
    mn = block_min(mn, ns.redmin);
    mx = -block_min(-mx, ns.red);
    if (mn == mx) {
      // one value: the entries rank by index; the j-th tie (0-based) reaches
      // before + (j + 1) w
      const unsigned long long w = wq(mx, z1, s_c);
      const double q = (target - static_cast<double>(before)) / static_cast<double>(w);
      long long j = strict ? static_cast<long long>(floor(q)) : static_cast<long long>(ceil(q)) - 1;
      j = max(0LL, min(static_cast<long long>(n) - 1, j));
      __syncthreads();
      if (threadIdx.x == 0) {
        ns.tok = -2;
        ns.tie_v = mx;
        ns.tie_j = static_cast<int>(j);
        ns.incl = before + static_cast<unsigned long long>(j + 1) * w;
      }
      __syncthreads();
      return;
    }
    lo = mn;  // the bin's entries are exactly those in [mn, mx] (bins are monotone)
    hi = mx;
  }
}

// Index of the j-th (0-based, index order) entry equal to v.  One counting
// pass with every load of the row in flight (warp w counts the ties in its
// contiguous range of 16-byte vectors, coalesced), a scan over the warp
// ranges, then the index-ordered scan (tie_scan) of the one range that holds
// the j-th tie — instead of walking the row chunk by chunk from the start
// (a constant row's draw sits ~half-way: ~10 chunk latencies).
template <class E>
__device__ int tie_index(const typename E::T* row, int vocab, float v, int j, int* s_scan, int* s_found) {
  constexpr int VEC = 16 / E::SZ, U = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  const int per = (nvec + nw - 1) / nw;  // vectors per warp range
  const int lo = min(nvec, warp * per), hi = min(nvec, lo + per);
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  int cnt = 0;
  for (int i0 = lo; i0 < hi; i0 += 32 * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int i = i0 + u * 32 + lane;
      if (i < hi) r[u] = __ldg(vp + i);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int i = i0 + u * 32 + lane;
      if (i >= hi) continue;
      float f[VEC];
      unpack16<E>(r[u], f);
#pragma unroll
      for (int k = 0; k < VEC; k++) cnt += f[k] == v;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
  __shared__ int s_w, s_base;
  if (lane == 0) s_scan[warp] = cnt;
  if (threadIdx.x == 0) *s_found = -1;
  __syncthreads();
  if (threadIdx.x == 0) {
    // the head scalars come first in index order, then the warp ranges, then the tail
    int run = 0, w_sel = -1;
    for (int k = 0; k < head; k++)
      if (E::load1(row + k) == v) { if (run == j) *s_found = k; run++; }
    if (*s_found < 0) {
      for (int w = 0; w < nw; w++) {
        if (run + s_scan[w] > j) { w_sel = w; break; }
        run += s_scan[w];
      }
      if (w_sel < 0)
        for (int k = tail; k < vocab; k++)
          if (E::load1(row + k) == v) { if (run == j) *s_found = k; run++; }
    }
    s_w = w_sel;
    s_base = run;
  }
  __syncthreads();
  const int w_sel = s_w, base = s_base;
  if (w_sel >= 0) {  // block-uniform: the index-ordered scan of that warp's range
    const int wlo = min(nvec, w_sel * per), whi = min(nvec, wlo + per);
    const int off = head + wlo * VEC;
    tie_scan<E>(row + off, (whi - wlo) * VEC, v, j - base + 1, s_scan, [&](int r, int idx) {
      if (r == j - base) *s_found = off + idx;
    });
  }
  __syncthreads();
  return *s_found;
}

// Level 1 of the value-bin selection (independent of the target) and the
// row's total mass Z in fixed point (block-uniform).
template <class E>
__device__ __noinline__ unsigned long long build_level1(const typename E::T* row, int vocab, float z1,
                                                        float s_c, NucleusSmem& ns) {
  const float hi = z1, lo = z1 - 64.0f / s_c;
  const float scale = 256.0f / (hi - lo);
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    ns.d1[0][b] = 0; ns.d1[1][b] = 0; ns.d1[2][b] = 0; ns.c1[b] = 0;
  }
  __syncthreads();
  for_each_elem_uniform<E>(row, vocab, [&](float x, int) {
    const int b = (x >= lo && x <= hi) ? min(255, static_cast<int>((hi - x) * scale)) : -1;
    hist_add(b, b >= 0 ? wq(x, z1, s_c) : 0ull, ns.d1, ns.c1);
  });
  __syncthreads();
  unsigned long long z = 0;
  for (int b = 0; b < 256; b++) z += digits_mass(ns.d1, b);  // every thread (broadcast reads)
  __syncthreads();
  return z;
}

// ------------------------------------------------ nucleus, bf16 (exact keys)
// A bf16 row has few distinct values: within the mass-relevant range
// [z1 - 64 / s_c, z1] there are at most ~7,000 of them once magnitudes below
// 2^-24 are lumped onto 0 (their weights differ from w(0) by < 2^-19, T >=
// 0.05).  One pass counts entries per value (native 32-bit shared atomics);
// the mass of a value is count * w_q (exact, order-free); the cut and the
// draw are found on those counts, and only the drawn tie's index needs one
// more (early-exit) pass.  A crossing on the lump of non-zero tiny values, or
// a range of more than kNK values (T > ~100), takes the value-bin path.
constexpr int kNK = 8192;

struct Hist16 {
  unsigned c[kNK];  // count per key offset khi - key
  unsigned long long wsum[kSampleThreads / 32];
  int sel, last;
  unsigned long long before;
  unsigned long long tail;  // M_t: mass of the uncounted entries below t
  int lump_nonzero;
};

union NucleusShared {
  Hist16 h;
  NucleusSmem g;
};

// bf16 key of x, compacted: keys of magnitudes below 2^-24 (bf16 keys
// -13184 .. 13183: every tiny binade) collapse onto 0, the rest close the
// gap, so the keys of a mass-relevant range stay within kNK.
constexpr int kLumpHi = 13184;  // bf16 key of +2^-24 (0x3380)
__device__ __forceinline__ int lkey(float x) {
  const int k = fkey(x) >> 16;  // bf16: consecutive values, consecutive keys
  return k >= kLumpHi ? k - (kLumpHi - 1) : (k <= -kLumpHi - 1 ? k + kLumpHi : 0);
}

__device__ __forceinline__ float lval(int ck) {
  if (ck == 0) return 0.0f;
  const int k = ck > 0 ? ck + (kLumpHi - 1) : ck - kLumpHi;
  const unsigned h = k >= 0 ? static_cast<unsigned>(k) : ((static_cast<unsigned>(k) & 0xffffu) ^ 0x7fffu);
  return __uint_as_float(h << 16);
}

// The first key offset (rank order) whose inclusive mass reaches T (> T when
// strict): h.sel, h.before (block-uniform on return); returns the total mass.
// Each thread owns kNK / blockDim consecutive offsets; block scan.
__device__ unsigned long long find_key16(Hist16& h, int khi, float z1, float s_c, double T, bool strict) {
  constexpr int per = kNK / kSampleThreads;
  __syncthreads();  // earlier readers of h.sel / h.before / h.wsum are done
  const int o0 = threadIdx.x * per;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long mine = 0;
  int last = -1;
#pragma unroll 4
  for (int o = o0; o < o0 + per; o++) {
    const unsigned n = h.c[o];
    if (n) {
      mine += static_cast<unsigned long long>(n) * wq(lval(khi - o), z1, s_c);
      last = o;
    }
  }
  unsigned long long incl = mine;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long t = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) h.wsum[warp] = incl;
  if (threadIdx.x == 0) { h.sel = -1; h.last = -1; }
  __syncthreads();
  unsigned long long cum = incl - mine, total = 0;
  for (int w = 0; w < kSampleThreads / 32; w++) {
    if (w < warp) cum += h.wsum[w];
    total += h.wsum[w];
  }
  auto crosses = [&](unsigned long long c) {
    return strict ? static_cast<double>(c) > T : static_cast<double>(c) >= T;
  };
  if (last >= 0) atomicMax(&h.last, last);
  if (!crosses(cum) && crosses(cum + mine)) {  // the owner of the crossing
    for (int o = o0; o < o0 + per; o++) {
      const unsigned n = h.c[o];
      if (!n) continue;
      const unsigned long long m = static_cast<unsigned long long>(n) * wq(lval(khi - o), z1, s_c);
      if (crosses(cum + m)) { h.sel = o; h.before = cum; break; }
      cum += m;
    }
  }
  __syncthreads();
  const int sel = h.sel, lst = h.last;
  if (sel < 0 && lst >= 0) {  // block-uniform; rounding at the end: the last value
    __syncthreads();          // every thread has read h.sel
    if (threadIdx.x == 0) {
      h.sel = lst;
      h.before = total - static_cast<unsigned long long>(h.c[lst]) * wq(lval(khi - lst), z1, s_c);
    }
    __syncthreads();
  }
  return total;
}

// The nucleus draw of a bf16 row whose kept set reaches past the top
// kMaxTopK (R20): the cut = the first entry whose inclusive mass reaches
// top_p * Z, the draw = the first entry whose inclusive mass exceeds u * kept.
// Only values >= t are counted per value (shared atomics); the mass M_t of
// the entries below t is summed in registers.  Both crossings lie at or above
// t when M_t <= (1 - top_p) Z (else the cut entry and all after it, of mass >
// (1 - top_p) Z, would lie below t) and M_t < Z - u * kept (the draw and all
// after it carry at least that); t is chosen from the first pass's float Z so
// that this holds with a margin, checked exactly, and the pass is redone over
// the whole range [z1 - 64 / s_c, z1] when it does not.  Returns the drawn
// index, or -3 when the row needs the value-bin path (block-uniform).
template <class E>
__device__ __noinline__ int nucleus_draw_bf16(const typename E::T* row, int vocab, float z1, float s_c,
                                              float topp, float u, float Zf, Hist16& h, int* s_scan,
                                              int* s_found) {
  const int khi = lkey(z1);
  const int klo = lkey(z1 - 64.0f / s_c);
  if (khi - klo + 1 > kNK) return -3;
  const int lump = khi;  // offset of key 0 (when in range)
  // t: every entry below weighs < 2^((t - z1) s_c); vocab of them must stay
  // under a quarter of min(1 - top_p, 1 - u) of Z (Zf >= 1: relative to w(z1))
  float room = 1.0f - u;
  if (topp < 1.0f) room = fminf(room, 1.0f - topp);
  const float lt = log2f(fmaxf(room, 1e-30f) * fmaxf(Zf, 1.0f) * 0.25f / static_cast<float>(vocab));
  int kt = lkey(z1 + lt / s_c);
  if (kt < klo || !(lt < 0.0f)) kt = klo;
  for (int attempt = 0; attempt < 2; attempt++) {
    for (int o = threadIdx.x; o < kNK; o += blockDim.x) h.c[o] = 0;
    if (threadIdx.x == 0) { h.lump_nonzero = 0; h.tail = 0; }
    __syncthreads();
    unsigned long long tailm = 0;  // this thread's share of M_t (fixed point)
    {
      // one pass, 8 vectors in flight per thread; a warp whose 256 elements
      // share one key (constant rows, long tie blocks) adds them with one atomic
      constexpr int VEC = 8, U = 8;
      const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
      int head = static_cast<int>(((16 - (addr & 15)) & 15) / 2);
      if (head > vocab) head = vocab;
      const int nvec = (vocab - head) / VEC;
      const int tail = head + nvec * VEC;
      auto add = [&](float x, unsigned n) {
        if (!(x > -INFINITY)) return;
        const int k = lkey(x);
        if (k < kt) {
          tailm += static_cast<unsigned long long>(n) * wq(x, z1, s_c);
          return;
        }
        if (k == 0 && x != 0.0f) h.lump_nonzero = 1;
        atomicAdd(&h.c[khi - k], n);
      };
      for (int j = threadIdx.x; j < head; j += blockDim.x) add(E::load1(row + j), 1u);
      for (int j = tail + threadIdx.x; j < vocab; j += blockDim.x) add(E::load1(row + j), 1u);
      const uint4* vp = reinterpret_cast<const uint4*>(row + head);
      for (int v0 = 0; v0 < nvec; v0 += U * blockDim.x) {  // block-uniform trip count
        uint4 r[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
          const int v = v0 + q * blockDim.x + threadIdx.x;
          r[q] = v < nvec ? __ldg(vp + v) : make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
          const bool same = r[q].x == r[q].y && r[q].x == r[q].z && r[q].x == r[q].w &&
                            (r[q].x >> 16) == (r[q].x & 0xffffu);
          const unsigned w0 = __shfl_sync(kFull, r[q].x, 0);
          if (__all_sync(kFull, same && r[q].x == w0)) {
            if ((threadIdx.x & 31) == 0) add(__uint_as_float(w0 << 16), 256u);
            continue;
          }
          float f[VEC];
          unpack16<E>(r[q], f);
#pragma unroll
          for (int k = 0; k < VEC; k++) add(f[k], 1u);
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) tailm += __shfl_xor_sync(kFull, tailm, off);
    if ((threadIdx.x & 31) == 0 && tailm) atomicAdd(&h.tail, tailm);  // once per warp (a CAS loop: rare)
    TRACE5(4);
    const unsigned long long Mt = (__syncthreads(), h.tail);
    const unsigned long long Z = find_key16(h, khi, z1, s_c, 1e300, false) + Mt;
    TRACE5(5);
    // the cut
    unsigned long long kept = Z;
    bool ok = true;
    if (topp < 1.0f) {
      ok = static_cast<double>(Mt) <= (1.0 - static_cast<double>(topp)) * static_cast<double>(Z);
      if (ok) {
        const double Tc = static_cast<double>(topp) * static_cast<double>(Z);
        find_key16(h, khi, z1, s_c, Tc, false);
        const int o = h.sel;
        if (o < 0 || (o == lump && h.lump_nonzero)) return -3;
        const unsigned long long w = wq(lval(khi - o), z1, s_c);
        // ties at the cut value: the j-th (0-based) reaches before + (j + 1) w
        long long j = static_cast<long long>(ceil((Tc - static_cast<double>(h.before)) / static_cast<double>(w))) - 1;
        j = max(0LL, min(static_cast<long long>(h.c[o]) - 1, j));
        kept = h.before + static_cast<unsigned long long>(j + 1) * w;
      }
    }
    const double Td = static_cast<double>(u) * static_cast<double>(kept);
    ok = ok && static_cast<double>(Mt) < static_cast<double>(Z) - Td;
    if (!ok) {  // block-uniform: the bound was too tight, count the whole range
      if (kt == klo) return -3;
      kt = klo;
      __syncthreads();
      continue;
    }
    TRACE5(8);
    find_key16(h, khi, z1, s_c, Td, true);
    TRACE5(9);
    const int o = h.sel;
    if (o < 0 || (o == lump && h.lump_nonzero)) return -3;
    const unsigned long long w = wq(lval(khi - o), z1, s_c);
    long long j = static_cast<long long>(floor((Td - static_cast<double>(h.before)) / static_cast<double>(w)));
    j = max(0LL, min(static_cast<long long>(h.c[o]) - 1, j));
    const float v = lval(khi - o);
    __syncthreads();
    TRACE5(11);
    const int t = tie_index<E>(row, vocab, v, static_cast<int>(j), s_scan, s_found);
    TRACE5(12);
    return t;
  }
  return -3;
}

template <class E, bool NUC>
__global__ void __launch_bounds__(kSampleThreads, 2) sample_switch_kernel(SampleArgs a, CueDev cs) {
  using T = typename E::T;
  __shared__ __align__(16) float s_cv[kCandCap];
  __shared__ __align__(16) int s_ci[kCandCap];
  __shared__ float s_topv[kMaxTopK];
  __shared__ int s_topi[kMaxTopK];
  __shared__ int s_scan[kCandCap > kSampleThreads ? kCandCap : kSampleThreads];
  __shared__ float s_red[kSampleThreads / 32];
  __shared__ int s_cnt, s_k;
  __shared__ SmemCue sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TRACE5(13);
  if (warp == 0) load_smem_cue(cs, sc);  // immutable cue set: before the dependency wait
  if (threadIdx.x == 0) pdl_launch_dependents();
  // no grid-wide wait: K4 releases this kernel only after all its CTAs passed
  // their own dependency wait, and pushes each finished row (thk, status,
  // margin, top-2 written before) onto a queue with a release store; a CTA
  // takes a ticket and samples the ticket's row, so rows are sampled in the
  // order their margin passes finish (not in row order: K4's two-row SMs
  // finish last), overlapping K4's tail
  __shared__ long long s_row;
  for (;;) {
    if (threadIdx.x == 0) {
      s_cnt = 0;
      const int tk = atomicAdd(a.q_ctl + 1, 1);
      long long rr = -1;
      if (tk < a.n_rows) {
        int v;
        do {
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a.ready_q + tk) : "memory");
        } while (v == 0);
        a.ready_q[tk] = 0;   // read again only by the next step (after this grid)
        rr = v > 0 ? v - 1 : -2;  // -(r + 1): K4 drew the row itself (fused top-k draw)
      }
      s_row = rr;
    }
    __syncthreads();
    const long long r = s_row;
    if (r == -1) break;
    if (r == -2) {
      __syncthreads();  // s_row / s_cnt are rewritten by thread 0 next
      continue;
    }
    TRACE5(14);
    const T* row = static_cast<const T*>(a.logits) + r * a.stride;
    // warp 0's per-row inputs are fetched before the scan so that their
    // latency hides under it; the scan itself does not wait for the status
    SwitchIn in{};
    const float u = a.uniform[r];
    float m = 0.0f;
    if (warp == 0) {
      in = load_switch_in(a.hist, a.state, a.small_run, nullptr, r);
      m = a.margin[r];
    }
    constexpr bool nucleus = NUC;        // no top-k (a.topk == 0): top-p over the whole row
    const int kfast = nucleus ? kMaxTopK : a.topk;
    const float z1 = nucleus ? a.zmax[r] : 0.0f;
    TRACE5(0);
    const float zpart =
        collect_candidates<E, NUC>(row, a.vocab, a.thk[r], false, s_cv, s_ci, &s_cnt, z1, a.s_c, a.k5_l2);
    __syncthreads();
    TRACE5(1);
    const int st = a.status[r];   // uniform: every thread takes the same branches
    int K = 0;
    if (st == 0) {
      K = (s_cnt <= kCandCap)
              ? rank_list(kfast, s_cnt, s_cv, s_ci, s_topv, s_topi, &s_k)
              : refine_topk<E>(row, a.vocab, kfast, a.zmax[r], s_cv, s_ci, &s_cnt, s_topv, s_topi, &s_k, s_scan);
    }
    TRACE5(2);
    float Z = -1.0f;     // nucleus: the row's total mass (the top-p reference)
    bool slow = false;   // nucleus: the kept set reaches past the top kMaxTopK
    if (nucleus && st == 0) {
      Z = block_sum(zpart, s_red);
      float mk = 0.0f;  // mass of the top kMaxTopK
      for (int k = 0; k < K; k++) mk += ex2((s_topv[k] - z1) * a.s_c);
      slow = !(mk >= a.topp * Z);
      if (slow && threadIdx.x == 0) {
        // handed to the nucleus kernel (K6), which draws and switches it
        const int p = atomicAdd(a.slow_cnt, 1);
        a.slow_list[p] = static_cast<int>(r);
        a.zsum[r] = Z;
      }
    }
    TRACE5(3);
    if (warp == 0 && !slow) {
      int tok = -1;
      if (st == 0 && K > 0) tok = draw_warp(a, u, K, s_topv, s_topi, Z);
      if (lane == 0) a.sampled[r] = tok;
      switch_warp(cs, sc, tok, m, in, a.state + r, a.hist + r * kHist,
                  a.small_run ? a.small_run + r : nullptr, a.gate, a.max_seg, a.flag + r,
                  a.cue_id + r);
    }
    __syncthreads();
    TRACE5(15);
  }
  // the last CTA re-arms the queue for the next step (every row was pushed and taken)
  if (threadIdx.x == 0 && atomicAdd(a.q_ctl + 2, 1) == static_cast<int>(gridDim.x) - 1) {
    a.q_ctl[0] = 0;
    a.q_ctl[1] = 0;
    a.q_ctl[2] = 0;
  }
}

// K6: the rows K5 listed as slow (no top-k, a kept set reaching past the top
// kMaxTopK), one CTA per row: the exact nucleus draw, then the switch on the
// drawn token.  A kernel of its own so that K5 keeps its registers and shared
// memory lean; with nothing listed its CTAs exit at once.  The last CTA out
// re-arms the list (CUDA-graph replays need no reset).
template <class E>
__global__ void __launch_bounds__(kSampleThreads, 1) nucleus_slow_kernel(SampleArgs a, CueDev cs) {
  __shared__ __align__(16) float s_cv[kCandCap];
  __shared__ __align__(16) int s_ci[kCandCap];
  __shared__ int s_scan[kCandCap > kSampleThreads ? kCandCap : kSampleThreads];
  __shared__ NucleusShared hs;  // exact bf16 value counts, or value bins (f16 / f32 / rare bf16)
  __shared__ int s_cnt, s_k;
  __shared__ SmemCue sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) load_smem_cue(cs, sc);
  pdl_wait();  // K5's list and the rows' state
  const int n = *reinterpret_cast<volatile int*>(a.slow_cnt);
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int r = a.slow_list[i];
    const typename E::T* row = static_cast<const typename E::T*>(a.logits) + static_cast<long long>(r) * a.stride;
    const float z1 = a.zmax[r], Z = a.zsum[r], u = a.uniform[r];
    SwitchIn in{};
    float m = 0.0f;
    if (warp == 0) {
      in = load_switch_in(a.hist, a.state, a.small_run, nullptr, r);
      m = a.margin[r];
    }
    TRACE5(3);
    int tok = -3;
    if constexpr (E::kBf16) tok = nucleus_draw_bf16<E>(row, a.vocab, z1, a.s_c, a.topp, u, Z, hs.h, s_scan, &s_k);
    if (tok == -3) {  // block-uniform: value bins
      __syncthreads();
      NucleusSmem& ns = hs.g;
      const unsigned long long Zq = build_level1<E>(row, a.vocab, z1, a.s_c, ns);
      TRACE5(6);
      // the last kept entry: the first whose inclusive mass reaches top_p * Z
      unsigned long long kept = Zq;
      if (a.topp < 1.0f) {
        select_by_mass<E>(row, a.vocab, z1, a.s_c, static_cast<double>(a.topp) * static_cast<double>(Zq), false,
                          true, ns, s_cv, s_ci, &s_cnt, s_scan);
        kept = ns.incl;  // from the list or the tie arithmetic: no index needed
      }
      __syncthreads();
      TRACE5(7);
      // the draw: the first entry whose inclusive mass exceeds u * kept
      select_by_mass<E>(row, a.vocab, z1, a.s_c, static_cast<double>(u) * static_cast<double>(kept), true, true,
                        ns, s_cv, s_ci, &s_cnt, s_scan);
      tok = ns.tok;
      TRACE5(10);
      if (tok == -2)  // the tie_j-th entry of a tie block
        tok = tie_index<E>(row, a.vocab, ns.tie_v, ns.tie_j, s_scan, &s_k);
    }
    if (warp == 0) {
      if (lane == 0) a.sampled[r] = tok;
      switch_warp(cs, sc, tok, m, in, a.state + r, a.hist + r * kHist,
                  a.small_run ? a.small_run + r : nullptr, a.gate, a.max_seg, a.flag + r, a.cue_id + r);
    }
    __syncthreads();
    TRACE5(15);
  }
  if (threadIdx.x == 0) {
    // every CTA read n before arriving; the last arrival re-arms the list
    if (atomic_add_acq_rel_i(a.slow_cnt + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      a.slow_cnt[0] = 0;
      a.slow_cnt[1] = 0;
    }
  }
}

template <class E>
static cudaError_t launch_sample_t(const SampleArgs& a, const CueDev& cs, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long grid = a.n_rows;
  if (grid > 4LL * sms) grid = 4LL * sms;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kSampleThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = a.topk == 0 ? cudaLaunchKernelEx(&cfg, sample_switch_kernel<E, true>, a, cs)
                              : cudaLaunchKernelEx(&cfg, sample_switch_kernel<E, false>, a, cs);
  if (e != cudaSuccess || a.topk != 0) return e;
  // no top-k: the nucleus kernel for the rows K5 listed
  cfg.gridDim = dim3(static_cast<unsigned>(a.n_rows < kSlowCtas ? a.n_rows : kSlowCtas));
  return cudaLaunchKernelEx(&cfg, nucleus_slow_kernel<E>, a, cs);
}

cudaError_t launch_step_sample(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                               long long stride, float iota, float temperature, int topk, float topp,
                               const float* uniform, uint8_t* state, int* hist, int* small_run,
                               float gate, int max_seg, float* margin, int* top1, int* top2,
                               int* sampled, uint8_t* flag, int16_t* cue_id, const StepWs& ws,
                               cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  // no top-k: K4 bounds the top kMaxTopK (the fast path's list)
  // with a top-k K4 also draws each row (fused), K5 takes the rest
  const StepDraw draw{kLog2e / temperature, topp, uniform, sampled, flag, cue_id};
  cudaError_t e = launch_step_rows(cs, logits, dt, batch, vocab, stride, iota, state, hist, small_run,
                                   gate, max_seg, margin, top1, top2, ws,
                                   topk > 0 ? topk : min(kMaxTopK, vocab), st, topk > 0 ? &draw : nullptr);
  if (e != cudaSuccess) return e;
  SampleArgs a{};
  a.logits = logits; a.n_rows = batch; a.vocab = vocab; a.stride = stride;
  a.thk = ws.thk; a.status = ws.status; a.margin = margin; a.zmax = ws.zmax;
  a.s_c = kLog2e / temperature; a.topk = topk; a.topp = topp; a.uniform = uniform;
  a.sampled = sampled; a.state = state; a.hist = hist; a.small_run = small_run;
  a.gate = gate; a.max_seg = max_seg; a.flag = flag; a.cue_id = cue_id;
  a.slow_cnt = ws.work + 2; a.slow_list = ws.slow; a.zsum = ws.zsum;
  a.ready_q = ws.ready_q; a.q_ctl = ws.q_ctl;
  {
    const char* e = getenv("RELAY_K5_L2");
    a.k5_l2 = (e && !strcmp(e, "last")) ? 1 : (e && !strcmp(e, "normal")) ? 2 : 0;
  }
  switch (dt) {
    case 0: return launch_sample_t<EBf16>(a, cs, st);
    case 1: return launch_sample_t<EF16>(a, cs, st);
    default: return launch_sample_t<EF32>(a, cs, st);
  }
}

}  // namespace relay
