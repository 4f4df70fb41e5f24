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

#include "relay_device.cuh"
#include "relay_internal.h"
#include "switch.cuh"

namespace relay {

constexpr int kSampleThreads = 512;
constexpr int kCandCap = 1024;  // candidates held in shared memory; more -> exact global fallback

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
// list (block-wide).
template <class E>
__device__ float collect_candidates(const typename E::T* row, int vocab, float th, bool strict,
                                    float* s_cv, int* s_ci, int* s_cnt, float z1 = 0.0f,
                                    float s_c = 0.0f, bool want_mass = false) {
  float mass = 0.0f;  // this thread's share of sum_j 2^((z_j - z1) s_c) (want_mass)
  constexpr int VEC = 16 / E::SZ;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  for (int j = threadIdx.x; j < head; j += blockDim.x) {
    const float x = E::load1(row + j);
    push_candidate(x, j, th, strict, s_cv, s_ci, s_cnt);
    if (want_mass && x > -INFINITY) mass += ex2((x - z1) * s_c);
  }
  for (int j = tail + threadIdx.x; j < vocab; j += blockDim.x) {
    const float x = E::load1(row + j);
    push_candidate(x, j, th, strict, s_cv, s_ci, s_cnt);
    if (want_mass && x > -INFINITY) mass += ex2((x - z1) * s_c);
  }
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  const uint64_t pol = policy_evict_first();  // the row's last use: leave L2
  constexpr int U = 8;                        // loads in flight per thread
  for (int v0 = threadIdx.x; v0 < nvec; v0 += U * blockDim.x) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int v = v0 + u * blockDim.x;
      x[u] = v < nvec ? ldg_hint(vp + v, pol) : make_uint4(0xff800000u, 0xff800000u, 0xff800000u,
                                                            0xff800000u);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int v = v0 + u * blockDim.x;
      if (v >= nvec) continue;
      if (want_mass) {
        float f[VEC];
        unpack16<E>(x[u], f);
#pragma unroll
        for (int k = 0; k < VEC; k++) mass += (f[k] > -INFINITY) ? ex2((f[k] - z1) * s_c) : 0.0f;
      }
      if (vec_max<E>(x[u]) >= th) {
        float f[VEC];
        unpack16<E>(x[u], f);
#pragma unroll
        for (int k = 0; k < VEC; k++) push_candidate(f[k], head + v * VEC + k, th, strict, s_cv, s_ci, s_cnt);
      }
    }
  }
  return mass;
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
    for (int f = 0; f < n && rank < want; f++) rank += ranks_before(s_cv[f], s_ci[f], v, i);
    if (rank < want) { s_topv[rank] = v; s_topi[rank] = i; }
  }
  if (threadIdx.x == 0) *s_k = n < want ? n : want;
  __syncthreads();
  return *s_k;
}

// The exact top-k of a row whose candidate list (entries >= thk) overflowed,
// e.g. a constant row.  theta = the k-th largest value in the (partial) list
// is a value of k real entries, so the row's k-th largest is >= theta; collect
// the entries > theta: on overflow raise theta again (strictly), else they are
// all of them and, if fewer than k, the rest of the top-k are the
// lowest-index entries equal to theta (collected in index order).
template <class E>
__device__ int refine_topk(const typename E::T* row, int vocab, int topk, float* s_cv, int* s_ci,
                           int* s_cnt, float* s_topv, int* s_topi, int* s_k, int* s_scan) {
  float theta;
  for (;;) {
    if (rank_list(topk, kCandCap, s_cv, s_ci, s_topv, s_topi, s_k) < topk) return *s_k;
    theta = s_topv[topk - 1];
    __syncthreads();
    if (threadIdx.x == 0) *s_cnt = 0;
    __syncthreads();
    collect_candidates<E>(row, vocab, theta, true, s_cv, s_ci, s_cnt);
    __syncthreads();
    if (*s_cnt <= kCandCap) break;
  }
  const int c = *s_cnt;
  if (c >= topk) return rank_list(topk, c, s_cv, s_ci, s_topv, s_topi, s_k);
  // ties at theta in index order: thread t scans a contiguous range of
  // 16-byte vectors (plus the scalar head / tail, owned by threads 0 / last)
  constexpr int VEC = 16 / E::SZ;
  const int need = topk - c;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  const int per = (nvec + blockDim.x - 1) / blockDim.x;
  const int v0 = threadIdx.x * per, v1 = min(nvec, v0 + per);
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  const bool first = threadIdx.x == 0, last = threadIdx.x == blockDim.x - 1;
  int mine = 0;
  if (first)
    for (int j = 0; j < head; j++) mine += E::load1(row + j) == theta;
  for (int v = v0; v < v1; v++) {
    float f[VEC];
    unpack16<E>(vp[v], f);
#pragma unroll
    for (int k = 0; k < VEC; k++) mine += f[k] == theta;
  }
  if (last)
    for (int j = tail; j < vocab; j++) mine += E::load1(row + j) == theta;
  s_scan[threadIdx.x] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive prefix over the block (tiny)
    int run = 0;
    for (int t = 0; t < static_cast<int>(blockDim.x); t++) {
      const int m = s_scan[t];
      s_scan[t] = run;
      run += m;
    }
  }
  __syncthreads();
  int rank = s_scan[threadIdx.x];
  auto take = [&](float x, int j) {
    if (rank < need && x == theta) {
      s_cv[c + rank] = theta;
      s_ci[c + rank] = j;
      rank++;
    }
  };
  if (first)
    for (int j = 0; j < head; j++) take(E::load1(row + j), j);
  for (int v = v0; v < v1 && rank < need; v++) {
    float f[VEC];
    unpack16<E>(vp[v], f);
#pragma unroll
    for (int k = 0; k < VEC; k++) take(f[k], head + v * VEC + k);
  }
  if (last)
    for (int j = tail; j < vocab; j++) take(E::load1(row + j), j);
  __syncthreads();
  return rank_list(topk, c + need, s_cv, s_ci, s_topv, s_topi, s_k);
}

// The drawn token (one warp; every lane returns it) from the top-K list, R20:
// p_k = 2^((v_k - v_0) log2(e) / T); keep the first L (higher-ranked mass below
// top_p of the total, at least one); inverse CDF with the row's uniform.  Lane
// l holds ranks l and l + 32; prefix sums by warp scans, in rank order.
__device__ int draw_warp(const SampleArgs& a, float u, int K, const float* s_topv,
                         const int* s_topi, float total_mass = -1.0f) {
  const int lane = threadIdx.x & 31;
  const float v0 = s_topv[0];
  const float p0 = lane < K ? ex2((s_topv[lane] - v0) * a.s_c) : 0.0f;
  const float p1 = lane + 32 < K ? ex2((s_topv[lane + 32] - v0) * a.s_c) : 0.0f;
  float c0 = p0, c1 = p1;  // inclusive prefix sums within each half
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float t0 = __shfl_up_sync(kFull, c0, off);
    const float t1 = __shfl_up_sync(kFull, c1, off);
    if (lane >= off) { c0 += t0; c1 += t1; }
  }
  const float half0 = __shfl_sync(kFull, c0, 31);
  c1 += half0;                                   // ranks 32..63 continue the sum
  // the top-p reference mass: the top-K (R20), or the whole row (no top-k)
  const float total = total_mass >= 0.0f ? total_mass : __shfl_sync(kFull, c1, 31);
  // kept iff the mass of the higher ranks (exclusive prefix) is below top_p * total
  const float lim = a.topp * total;
  const unsigned keep0 = __ballot_sync(kFull, lane < K && (lane == 0 || c0 - p0 < lim));
  const unsigned keep1 = __ballot_sync(kFull, lane + 32 < K && c1 - p1 < lim);
  const int L = __popc(keep0) + __popc(keep1);   // kept ranks form a prefix
  const float kept = L <= 32 ? __shfl_sync(kFull, c0, L - 1) : __shfl_sync(kFull, c1, L - 33);
  const float target = u * kept;
  const unsigned hit0 = __ballot_sync(kFull, lane < L && c0 > target);
  const unsigned hit1 = __ballot_sync(kFull, lane + 32 < L && c1 > target);
  const int k = hit0 ? __ffs(hit0) - 1 : (hit1 ? 32 + __ffs(hit1) - 1 : L - 1);
  return s_topi[k];
}

// ---------------------------------------------------------------- nucleus
// No top-k (the R1-Distill setting): the kept set is the rank prefix
// whose higher-ranked mass is below top_p * Z, Z = the row's total mass at the
// sampling temperature, w(x) = 2^((x - z1) log2(e) / T).  When the top-64
// already hold top_p * Z the draw uses them; otherwise the row is resolved by
// mass-rank selection over value bins.

// f(x, j) for every element of the row (block-strided 16-byte vectors plus the
// unaligned head / tail).
template <class E, class F>
__device__ __forceinline__ void for_each_elem(const typename E::T* row, int vocab, F f) {
  constexpr int VEC = 16 / E::SZ;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row);
  int head = static_cast<int>(((16 - (addr & 15)) & 15) / E::SZ);
  if (head > vocab) head = vocab;
  const int nvec = (vocab - head) / VEC;
  const int tail = head + nvec * VEC;
  for (int j = threadIdx.x; j < head; j += blockDim.x) f(E::load1(row + j), j);
  for (int j = tail + threadIdx.x; j < vocab; j += blockDim.x) f(E::load1(row + j), j);
  const uint4* vp = reinterpret_cast<const uint4*>(row + head);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    float x[VEC];
    unpack16<E>(__ldcs(vp + v), x);
#pragma unroll
    for (int k = 0; k < VEC; k++) f(x[k], head + v * VEC + k);
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

struct NucleusSmem {
  float hm[256];   // mass per bin
  int hc[256];     // count per bin
  float red[kSampleThreads / 32];
  int sel_bin, sel_n;
  float sel_before;
  int tok;
  float incl;
};

// The first entry in (value desc, index asc) order whose inclusive cumulative
// mass crosses `target` (> when strict, else >=).  Entries are binned by their
// order-preserving key over [klo, khi] (256 bins, largest keys first); the
// crossing bin is refined the same way until its entries fit the list (ranked
// there) or share one key (one value: index order decides).  Keys below
// key(z1 - 160 T / log2 e) carry no fp32 mass and are left out.  Sets ns.tok
// and ns.incl (block-uniform).
template <class E>
__device__ void select_by_mass(const typename E::T* row, int vocab, float z1, float s_c, float target,
                               bool strict, NucleusSmem& ns, float* s_cv, int* s_ci, int* s_cnt,
                               int* s_scan) {
  long long klo = fkey(z1 - 160.0f / s_c), khi = fkey(z1);
  float before = 0.0f;  // mass of the entries ranked before the key range
  for (;;) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) { ns.hm[b] = 0.0f; ns.hc[b] = 0; }
    __syncthreads();
    const long long span = khi - klo + 1;
    auto bin_of = [&](float x) -> int {  // -1: outside [klo, khi]
      const long long k = fkey(x);
      if (!(x == x) || k < klo || k > khi) return -1;
      return static_cast<int>(((khi - k) * 256) / span);
    };
    for_each_elem<E>(row, vocab, [&](float x, int) {
      const int b = bin_of(x);
      if (b < 0) return;
      atomicAdd(&ns.hm[b], ex2((x - z1) * s_c));
      atomicAdd(&ns.hc[b], 1);
    });
    __syncthreads();
    if (threadIdx.x == 0) {
      float cum = before, bef = before;
      int bsel = -1;
      for (int b = 0; b < 256; b++) {
        if (!ns.hc[b]) continue;
        const float next = cum + ns.hm[b];
        bsel = b;
        bef = cum;
        if (strict ? next > target : next >= target) break;
        cum = next;
      }
      ns.sel_bin = bsel;  // the crossing bin (or the last non-empty one: rounding)
      ns.sel_before = bef;
      ns.sel_n = bsel >= 0 ? ns.hc[bsel] : 0;
    }
    __syncthreads();
    const int bsel = ns.sel_bin, n = ns.sel_n;
    before = ns.sel_before;
    // the selected bin's key range: keys k with ((khi - k) * 256) / span == bsel
    const long long bhi = khi - (static_cast<long long>(bsel) * span + 255) / 256;
    const long long blo = khi - ((static_cast<long long>(bsel) + 1) * span + 255) / 256 + 1;
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
        float cum = before;
        int tok = n ? s_ci[s_scan[n - 1]] : -1;
        float incl = cum;
        for (int k = 0; k < n; k++) {
          const int e = s_scan[k];
          cum += ex2((s_cv[e] - z1) * s_c);
          incl = cum;
          if (strict ? cum > target : cum >= target) { tok = s_ci[e]; break; }
        }
        ns.tok = tok;
        ns.incl = incl;
      }
      __syncthreads();
      return;
    }
    if (bhi == blo) {
      // one key, one value: the entries rank by index
      const float v = unkey(static_cast<int>(bhi));
      const float w = ex2((v - z1) * s_c);
      const float q = (target - before) / w;  // the j-th tie (0-based) reaches before + (j + 1) w
      int j = strict ? static_cast<int>(floorf(q)) : static_cast<int>(ceilf(q)) - 1;
      j = max(0, min(n - 1, j));
      const int per = (vocab + blockDim.x - 1) / blockDim.x;
      const int j0 = threadIdx.x * per, j1 = min(vocab, j0 + per);
      int mine = 0;
      for (int i = j0; i < j1; i++) mine += E::load1(row + i) == v;
      s_scan[threadIdx.x] = mine;
      __syncthreads();
      if (threadIdx.x == 0) {
        int run = 0;
        for (int t = 0; t < static_cast<int>(blockDim.x); t++) {
          const int m = s_scan[t];
          s_scan[t] = run;
          run += m;
        }
      }
      __syncthreads();
      int rank = s_scan[threadIdx.x];
      if (rank <= j && j < rank + mine) {
        for (int i = j0; i < j1; i++)
          if (E::load1(row + i) == v && rank++ == j) { ns.tok = i; ns.incl = before + (j + 1) * w; }
      }
      __syncthreads();
      return;
    }
    klo = blo;
    khi = bhi;
  }
}

template <class E>
__global__ void __launch_bounds__(kSampleThreads) sample_switch_kernel(SampleArgs a, CueDev cs) {
  using T = typename E::T;
  __shared__ float s_cv[kCandCap];
  __shared__ int s_ci[kCandCap];
  __shared__ float s_topv[kMaxTopK];
  __shared__ int s_topi[kMaxTopK];
  __shared__ int s_scan[kCandCap > kSampleThreads ? kCandCap : kSampleThreads];
  __shared__ NucleusSmem ns;
  __shared__ int s_cnt, s_k;
  __shared__ SmemCue sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) load_smem_cue(cs, sc);  // immutable cue set: before the dependency wait
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // K4's outputs (thk, status, margin) and the switch state
  for (long long r = blockIdx.x; r < a.n_rows; r += gridDim.x) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
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
    const bool nucleus = a.topk == 0;    // no top-k: top-p over the whole row
    const int kfast = nucleus ? kMaxTopK : a.topk;
    const float z1 = nucleus ? a.zmax[r] : 0.0f;
    const float zpart = collect_candidates<E>(row, a.vocab, a.thk[r], false, s_cv, s_ci, &s_cnt, z1,
                                              a.s_c, nucleus);
    __syncthreads();
    const int st = a.status[r];   // uniform: every thread takes the same branches
    int K = 0;
    if (st == 0) {
      K = (s_cnt <= kCandCap)
              ? rank_list(kfast, s_cnt, s_cv, s_ci, s_topv, s_topi, &s_k)
              : refine_topk<E>(row, a.vocab, kfast, s_cv, s_ci, &s_cnt, s_topv, s_topi, &s_k, s_scan);
    }
    float Z = -1.0f;     // nucleus: the row's total mass (the top-p reference)
    bool slow = false;   // nucleus: the kept set reaches past the top kMaxTopK
    if (nucleus && st == 0) {
      Z = block_sum(zpart, ns.red);
      float mk = 0.0f;  // mass of the top kMaxTopK
      for (int k = 0; k < K; k++) mk += ex2((s_topv[k] - z1) * a.s_c);
      slow = !(mk >= a.topp * Z);
      if (slow) {
        // the last kept entry: the first whose inclusive mass reaches top_p * Z
        float kept = Z;
        if (a.topp < 1.0f) {
          select_by_mass<E>(row, a.vocab, z1, a.s_c, a.topp * Z, false, ns, s_cv, s_ci, &s_cnt, s_scan);
          kept = ns.incl;
        }
        __syncthreads();
        // the draw: the first entry whose inclusive mass exceeds u * kept
        select_by_mass<E>(row, a.vocab, z1, a.s_c, u * kept, true, ns, s_cv, s_ci, &s_cnt, s_scan);
      }
    }
    if (warp == 0) {
      int tok = -1;
      if (st == 0 && slow) tok = ns.tok;
      else if (st == 0 && K > 0) tok = draw_warp(a, u, K, s_topv, s_topi, Z);
      if (lane == 0) a.sampled[r] = tok;
      switch_warp(cs, sc, tok, m, in, a.state + r, a.hist + r * kHist,
                  a.small_run ? a.small_run + r : nullptr, a.gate, a.max_seg, a.flag + r,
                  a.cue_id + r);
    }
    __syncthreads();
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
  return cudaLaunchKernelEx(&cfg, sample_switch_kernel<E>, a, cs);
}

cudaError_t launch_step_sample(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                               long long stride, float iota, float temperature, int topk, float topp,
                               const float* uniform, uint8_t* state, int* hist, int* small_run,
                               float gate, int max_seg, float* margin, int* top1, int* top2,
                               int* sampled, uint8_t* flag, int16_t* cue_id, const StepWs& ws,
                               cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  // no top-k: K4 bounds the top kMaxTopK (the fast path's list)
  cudaError_t e = launch_step_rows(cs, logits, dt, batch, vocab, stride, iota, state, hist, small_run,
                                   gate, max_seg, margin, top1, top2, ws,
                                   topk > 0 ? topk : min(kMaxTopK, vocab), st);
  if (e != cudaSuccess) return e;
  SampleArgs a{};
  a.logits = logits; a.n_rows = batch; a.vocab = vocab; a.stride = stride;
  a.thk = ws.thk; a.status = ws.status; a.margin = margin; a.zmax = ws.zmax;
  a.s_c = kLog2e / temperature; a.topk = topk; a.topp = topp; a.uniform = uniform;
  a.sampled = sampled; a.state = state; a.hist = hist; a.small_run = small_run;
  a.gate = gate; a.max_seg = max_seg; a.flag = flag; a.cue_id = cue_id;
  switch (dt) {
    case 0: return launch_sample_t<EBf16>(a, cs, st);
    case 1: return launch_sample_t<EF16>(a, cs, st);
    default: return launch_sample_t<EF32>(a, cs, st);
  }
}

}  // namespace relay
