// scan_kernels.cu — K2 relay_cue_scan and K3 relay_segment_reduce (sm_100a).
//
// K2: switch-cue occurrences by token matching + the
//     terminator bitmap.  One kernel: 512-position tiles staged in
//     shared memory with an 8-token halo; a forward decoupled look-back over
//     tile counts gives each tile its output offset, so occurrences come out
//     sorted by position (deterministic, no sort, no second pass).
// K3: post-sentence windows as a REVERSE segmented scan
//     keyed by segment tails (terminator or trajectory end): the aggregate at
//     s over [s, first tail >= s] is exactly the window of a cue at s.  One
//     kernel: tiles run right to left and take their carry from the tiles to
//     the right with a decoupled look-back (nearly every 2,048-token tile
//     holds a sentence end, so the look-back stops at the next tile), then
//     gather at occurrence starts and add per-cue integer moments (u64
//     atomics: order-free, so bit-identical across launch shapes and ranks).
// Both are tiny next to K1 (4 B per token vs ~300 KB per logit row).
#include <cfloat>

#include "p2p.cuh"
#include "relay_device.cuh"
#include "relay_internal.h"

namespace relay {

constexpr int kItems = kTile / kScanThreads;  // 8 consecutive positions per thread
static_assert(kItems == 8, "tile layout");

// Trajectory index of position t: offs[k] <= t < offs[k+1], or -1.
__device__ __forceinline__ int find_traj(const long long* offs, int n_traj, long long n_tok,
                                         long long t) {
  if (!offs) return (t >= 0 && t < n_tok) ? 0 : -1;
  int lo = 0, hi = n_traj + 1;  // upper_bound over offs[0..n_traj]
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (offs[mid] <= t) lo = mid + 1; else hi = mid;
  }
  int k = lo - 1;
  return (k >= 0 && k < n_traj) ? k : -1;
}

__device__ __forceinline__ long long traj_end(const long long* offs, long long n_tok, int k) {
  return offs ? offs[k + 1] : n_tok;
}

struct SmemPat {
  int tok[kMaxPat * kMaxLen];
  int len[kMaxPat];
  int cue[kMaxPat];
  int orig[kMaxPat];
};

__device__ __forceinline__ void load_patterns(const CueDev& cs, SmemPat& sp) {
  for (int i = threadIdx.x; i < cs.n_pat * kMaxLen; i += blockDim.x) sp.tok[i] = cs.pat_tok[i];
  for (int i = threadIdx.x; i < cs.n_pat; i += blockDim.x) {
    sp.len[i] = cs.pat_len[i];
    sp.cue[i] = cs.pat_cue[i];
    sp.orig[i] = cs.pat_orig[i];
  }
}

__device__ __forceinline__ bool match_at(const CueDev& cs, const SmemPat& sp, int p, const int* tk,
                                         long long room) {
  const int len = sp.len[p];
  if (len > room) return false;
  for (int k = 0; k < len; k++)
    if (!elem_ok(cs, tk[k], sp.tok[p * kMaxLen + k])) return false;
  return true;
}

// ------------------------------------------------------------------- K2
// Warp-ballot matching (north_star: "matches multi-token cue patterns over the
// generated token stream using warp ballots").  A CTA owns a tile of kTileB =
// 256 positions; warp w takes its group of 32 start positions.
// For a group at base b every lane holds tok[b + lane] and tok[b + 32 + lane]
// (the window the longest pattern can reach), and a pattern element e gives a
// 64-bit word  M_e = ballot(lo == e) | ballot(hi == e) << 32  (class elements
// (N4): ballot of a class-bitmap test).  Pattern p = (e_0 .. e_{L-1}) matches
// at start b + s iff bit s of  AND_k (M_{e_k} >> k)  and the trajectory has
// room (bit s of ballot(room >= L)).  LONGEST: patterns are visited longest
// first (lower caller index first among equal lengths) with a `claimed` mask,
// so each start keeps its longest match; ALL: one claim mask per cue.  The
// terminator word of the group is one ballot.  Compaction: per-warp counts,
// a block scan over the 8 warps, and a two-level decoupled look-back (32-tile
// blocks summed by their last arriving tile), so occurrences come out sorted
// by position in one pass; the look-back words carry a per-launch epoch tag
// (the last tile advances it), so no pass resets them.
constexpr int kTileB = kK2Tile;                 // positions per CTA (one 32-start group per warp)
constexpr int kGroupsB = kTileB / 32 / (kScanThreads / 32);  // groups per warp
constexpr int kK2Offs = 512;   // K2: trajectory offsets staged in shared memory up to this many

#ifdef RELAY_TRACE
// Tuning-only K2 timeline (tools/k2_trace.py): %globaltimer stamps by thread
// 0 of each tile: 0 entry, 1 patterns staged, 2 phase 1 done, 3 look-back
// done, 4 writes issued.
__device__ unsigned long long g_trace2[8192][16];
__device__ __forceinline__ void stamp2(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x < 8192) g_trace2[blockIdx.x][k] = t;
}
extern "C" int relay_debug_trace2_copy(unsigned long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace2, sizeof(unsigned long long) * 16 * n));
}
#define TRACE2(k) stamp2(k)
#else
#define TRACE2(k) ((void)0)
#endif

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i32(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Per group of 32 starts, one 64-bit ballot word per DISTINCT pattern element
// (W_d = ballot(lo == e_d) | ballot(hi == e_d) << 32; class elements (CLS, N4):
// ballots of a class-bitmap test), kept in the warp's shared-memory slot; a
// pattern is then AND_k funnelshift(W_{d_k}, k) — bit s set iff it matches
// at start b + s.  Per-length room masks likewise (bit s: >= L tokens left in
// the start's trajectory).
// Shared-memory accesses by 32-bit shared-window addresses computed once per
// CTA (generic pointers into the dynamic array made the compiler re-derive
// the window base from SR_CgaCtaId, an S2R, before every access of the
// pattern loop: ~450 cycles per pattern, 2.8 us of K2's 4 us match phase).
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint2 v) {
  asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

template <bool CLS>
__device__ __forceinline__ void group_words(const CueDev& cs, uint32_t dist_a, int nd, int lo, int hi, int room8,
                                            uint32_t w_a, uint32_t rm_a) {
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int d = 0; d < nd; d++) {
    const int e = static_cast<int>(lds32(dist_a + 4 * d));
    bool x, y;
    if constexpr (CLS) {
      x = elem_ok(cs, lo, e);
      y = elem_ok(cs, hi, e);
    } else {
      x = lo == e;
      y = hi == e;
    }
    const unsigned a = __ballot_sync(kFull, x);
    const unsigned b = __ballot_sync(kFull, y);
    if (lane == 0) sts64(w_a + 8 * d, make_uint2(a, b));
  }
#pragma unroll
  for (int L = 1; L <= kMaxLen; L++) {
    const unsigned r = __ballot_sync(kFull, room8 >= L);
    if (lane == 0) sts32(rm_a + 4 * L, r);
  }
  __syncwarp();
}

// Bit s: the pattern (its element word indices at pe_a, L of them) matches at
// start b + s with room.  Branch-free: all kMaxLen index loads, then all word
// loads, in flight together (entries past L read word 0 and are masked off).
__device__ __forceinline__ unsigned pattern_starts(uint32_t pe_a, int L, uint32_t w_a, uint32_t rm_a) {
  unsigned m = lds32(rm_a + 4 * L);
  uint32_t e[kMaxLen];
#pragma unroll
  for (int k = 0; k < kMaxLen; k++) e[k] = lds32(pe_a + 4 * k);
  uint2 v[kMaxLen];
#pragma unroll
  for (int k = 0; k < kMaxLen; k++) v[k] = lds64(w_a + 8 * (k < L ? e[k] : 0u));
#pragma unroll
  for (int k = 0; k < kMaxLen; k++) m &= k < L ? __funnelshift_r(v[k].x, v[k].y, k) : ~0u;
  return m;
}

template <bool CLS>
__global__ void __launch_bounds__(kScanThreads)
    cue_scan_kernel(CueDev cs, const int* __restrict__ tokens, long long n_tok,
                    const long long* __restrict__ offs, int n_traj, uint32_t* __restrict__ term_bits,
                    int* __restrict__ occ_pos, int* __restrict__ occ_pat, long long cap,
                    long long* __restrict__ n_occ, int* tile_flag, long long* tile_val, int* epoch) {
  __shared__ SmemPat sp;
  __shared__ int s_dist[kMaxPat * kMaxLen];
  __shared__ int s_eidx[kMaxPat * kMaxLen];
  extern __shared__ uint2 s_w_dyn[];   // per warp: the n_dist element words of its group
  __shared__ unsigned s_rm[kScanThreads / 32][kMaxLen + 1];     // per warp: room masks by length
  __shared__ int8_t s_best[kTileB];                 // LONGEST: sorted pattern index per start, -1 none
  __shared__ unsigned long long s_cues[kTileB];     // ALL: cue mask per start
  __shared__ int s_wcount[kScanThreads / 32];
  __shared__ long long s_prefix;
  const int tile = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long tile0 = static_cast<long long>(tile) * kTileB;
  TRACE2(0);
  // this launch's look-back tag (28 bits; 0 = never published)
  int ep = (*reinterpret_cast<const volatile int*>(epoch) + 1) & 0x0fffffff;
  if (ep == 0) ep = 1;
  static_assert(kGroupsB == 1, "one 32-start group per warp");
  // this warp's group: the token loads, the trajectory lookup and the
  // terminator test go first, so their latency overlaps the pattern staging
  const long long b = tile0 + static_cast<long long>(warp) * 32;
  const long long t = b + lane;
  const int lo = t < n_tok ? __ldg(tokens + t) : -1;
  const int hi = t + 32 < n_tok ? __ldg(tokens + t + 32) : -1;
  bool term = lo >= 0 && lo < cs.vocab && ((cs.term_tab[lo >> 5] >> (lo & 31)) & 1u);
  // the trajectory offsets in shared memory (one parallel load instead of a
  // chain of dependent global loads per binary search), when they fit
  __shared__ long long s_offs[kK2Offs];
  const bool offs_smem = offs && n_traj < kK2Offs;
  if (offs_smem)
    for (int i = threadIdx.x; i <= n_traj; i += blockDim.x) s_offs[i] = __ldg(offs + i);
  load_patterns(cs, sp);
  const int nd = cs.n_dist;
  for (int i = threadIdx.x; i < nd; i += blockDim.x) s_dist[i] = cs.dist_tok[i];
  for (int i = threadIdx.x; i < cs.n_pat * kMaxLen; i += blockDim.x) s_eidx[i] = cs.pat_eidx[i];
  __syncthreads();
  long long cur_beg = 0, cur_end = 0;
  if (t < n_tok) {
    const long long* of = offs_smem ? s_offs : offs;
    const int k = find_traj(of, n_traj, n_tok, t);
    cur_beg = (k < 0) ? t + 1 : (of ? of[k] : 0);
    cur_end = (k < 0) ? t + 1 : traj_end(of, n_tok, k);
    if (k < 0) cur_beg = cur_end;  // outside every trajectory: no room
  }
  const long long room = (t < n_tok && t >= cur_beg) ? cur_end - t : 0;
  TRACE2(1);
  const uint32_t ww = smem_u32_pinned(s_w_dyn) + static_cast<uint32_t>(8 * warp * nd);
  const uint32_t wrm = smem_u32_pinned(s_rm[warp]);
  const uint32_t dist_a = smem_u32_pinned(s_dist);
  const uint32_t eidx_a = smem_u32_pinned(s_eidx);
  // ---- phase 1: match, terminator words, per-warp counts
  int wcount = 0;
  if (b < n_tok) {
    // terminator bits (R19: a period between digit tokens of one trajectory is not an end)
    if (cs.dec_period >= 0) {
      int prev = __shfl_up_sync(kFull, lo, 1);
      if (lane == 0) prev = (t >= 1 && t - 1 < n_tok) ? __ldg(tokens + t - 1) : -1;
      const int nx = __shfl_down_sync(kFull, lo, 1);
      const int h0 = __shfl_sync(kFull, hi, 0);
      const int next = lane == 31 ? h0 : nx;
      if (term && room > 1 && t - 1 >= cur_beg && in_class(cs, cs.dec_period, lo) &&
          in_class(cs, cs.dec_dend, prev) && in_class(cs, cs.dec_dstart, next))
        term = false;
    }
    const unsigned tw = __ballot_sync(kFull, term);
    if (lane == 0) term_bits[b >> 5] = tw;
    __syncwarp();   // the previous group's words are read by every lane before they are overwritten
#ifdef RELAY_TRACE
    if (threadIdx.x == 0) stamp2(10);
#endif
    group_words<CLS>(cs, dist_a, nd, lo, hi, static_cast<int>(room < kMaxLen ? room : kMaxLen), ww, wrm);
#ifdef RELAY_TRACE
    if (threadIdx.x == 0) stamp2(11);
#endif
    if (cs.mode == 0) {
      unsigned claimed = 0;
      int best = -1;
#pragma unroll 4
      for (int p = 0; p < cs.n_pat; p++) {
        const int L = sp.len[p];
        // bit s: start b + s matches and has >= L tokens left in its trajectory
        const unsigned w = pattern_starts(eidx_a + 4 * p * kMaxLen, L, ww, wrm) & ~claimed;
        claimed |= w;
        if ((w >> lane) & 1u) best = p;
      }
      s_best[(b - tile0) + lane] = static_cast<int8_t>(best);
#ifdef RELAY_TRACE
      if (threadIdx.x == 0) stamp2(12);
#endif
      wcount += __popc(claimed);
    } else {
      unsigned long long cm = 0;   // this lane's cues
#pragma unroll 4
      for (int p = 0; p < cs.n_pat; p++) {
        const int L = sp.len[p];
        const unsigned w = pattern_starts(eidx_a + 4 * p * kMaxLen, L, ww, wrm);
        if ((w >> lane) & 1u) cm |= 1ull << sp.cue[p];
      }
      s_cues[(b - tile0) + lane] = cm;
      int c = __popcll(cm);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(kFull, c, off);
      wcount += c;
    }
  }
  if (lane == 0) s_wcount[warp] = wcount;
  __syncthreads();
  TRACE2(2);
  // ---- tile total, per-warp offsets, warp-parallel decoupled look-back (warp 0)
  if (warp == 0) {
    int wv = lane < kScanThreads / 32 ? s_wcount[lane] : 0;
    int incl = wv;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(kFull, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane < kScanThreads / 32) s_wcount[lane] = incl - wv;   // exclusive warp offsets
    const long long total = __shfl_sync(kFull, incl, 31);
    // Two-level look-back on one 64-bit word per tile, W[t] = tag << 36 |
    // count (a single-copy-atomic relaxed store: no fence, no acquire, no
    // second load for the value; the tag is this launch's epoch, so no pass
    // resets the words).  Tiles form blocks of 32: the block's last tile to
    // arrive (a counter in the workspace, re-zeroed by it) sums the block's
    // W into B[block]; a tile's prefix is the sum of B over earlier blocks
    // plus W over its earlier block mates.  Every tile reaching the scan at
    // once made a flat look-back read every predecessor's word (all tiles
    // polling the same lines: a ~3-6 us round trip at configs[1]).
    long long prefix = 0;
    {
      const unsigned long long tagw = static_cast<unsigned long long>(ep) << 36;
      const unsigned long long uep = static_cast<unsigned long long>(ep);
      constexpr unsigned long long kVal = (1ull << 34) - 1;
      unsigned long long* const words = reinterpret_cast<unsigned long long*>(tile_val);
      unsigned long long* const bsum = words + gridDim.x;   // (the workspace holds 2 words per tile)
      const int blk = tile >> 5, first = blk << 5;
      const int nb = min(32, static_cast<int>(gridDim.x) - first);
      if (lane == 0) st_relaxed_u64(words + tile, tagw | static_cast<unsigned long long>(total));
#ifdef RELAY_TRACE
      if (lane == 0) stamp2(8);
#endif
      int old = 0;
      if (lane == 0) old = atomicAdd(tile_flag + blk, 1);
      old = __shfl_sync(kFull, old, 0);
      const bool fin = old == nb - 1;          // the block's last arriver
      const int need = fin ? nb : tile - first;
      unsigned long long wv = lane < need ? ld_relaxed_u64(words + first + lane) : tagw;
      while (__any_sync(kFull, (wv >> 36) != uep))
        if ((wv >> 36) != uep) wv = ld_relaxed_u64(words + first + lane);
      long long mates = lane < tile - first ? static_cast<long long>(wv & kVal) : 0;
      long long whole = lane < nb ? static_cast<long long>(wv & kVal) : 0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        mates += __shfl_xor_sync(kFull, mates, off);
        whole += __shfl_xor_sync(kFull, whole, off);
      }
      if (fin && lane == 0) {
        st_relaxed_u64(bsum + blk, tagw | static_cast<unsigned long long>(whole));
        tile_flag[blk] = 0;                    // every tile of the block has counted
      }
      long long before = 0;                    // the earlier blocks
      for (int j0 = 0; j0 < blk; j0 += 32) {
        const int j = j0 + lane;
        unsigned long long bv = j < blk ? ld_relaxed_u64(bsum + j) : tagw;
        while (__any_sync(kFull, (bv >> 36) != uep))
          if ((bv >> 36) != uep) bv = ld_relaxed_u64(bsum + j);
        before += j < blk ? static_cast<long long>(bv & kVal) : 0;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) before += __shfl_xor_sync(kFull, before, off);
      prefix = before + mates;
    }
    if (lane == 0) {
      s_prefix = prefix;
      if (tile == gridDim.x - 1) {
        *n_occ = prefix + total;
        // every tile has published (this one's look-back saw them all), so
        // every CTA has read the epoch: the next launch takes the next one
        *epoch = ep;
      }
    }
  }
  __syncthreads();
  TRACE2(3);
  // ---- phase 2: ordered writes
  long long o = s_prefix + s_wcount[warp];
  if (b < n_tok) {
    if (cs.mode == 0) {
      const int best = s_best[(b - tile0) + lane];
      const unsigned has = __ballot_sync(kFull, best >= 0);
      if (best >= 0) {
        const long long q = o + __popc(has & ((1u << lane) - 1u));
        if (q < cap) { occ_pos[q] = static_cast<int>(t); occ_pat[q] = sp.orig[best]; }
      }
      o += __popc(has);
    } else {
      unsigned long long cm = s_cues[(b - tile0) + lane];
      const int c = __popcll(cm);
      int excl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(kFull, excl, off);
        if (lane >= off) excl += v;
      }
      const int tot = __shfl_sync(kFull, excl, 31);
      long long q = o + excl - c;
      if (cm) {
        // the tokens of the window again, for each cue's longest pattern
        int tk[kMaxLen];  // (room: this start's tokens left in its trajectory, from phase 1)
#pragma unroll
        for (int i = 0; i < kMaxLen; i++) tk[i] = (t + i < n_tok) ? __ldg(tokens + t + i) : -1;
        while (cm) {
          const int cue = __ffsll(cm) - 1;
          cm &= cm - 1;
          int best = -1;
          for (int p = 0; p < cs.n_pat && best < 0; p++)
            if (sp.cue[p] == cue && match_at(cs, sp, p, tk, room)) best = p;
          if (q < cap) { occ_pos[q] = static_cast<int>(t); occ_pat[q] = sp.orig[best]; }
          q++;
        }
      }
      o += tot;
    }
  }
  TRACE2(4);
}

// ------------------------------------------------------------------ K3
__device__ __forceinline__ Agg agg_identity() {
  Agg a;
  a.sumq = 0; a.low = 0; a.nan = 0; a.mn = INFINITY; a.end = -1; a.tail = 0; a.pad = 0;
  return a;
}

// L precedes R (L earlier positions).  The run starting at L's first
// position stops at its first tail.
__device__ __forceinline__ Agg agg_suffix(const Agg& L, const Agg& R) {
  if (L.tail) return L;
  Agg o;
  o.sumq = L.sumq + R.sumq;
  o.low = L.low + R.low;
  o.nan = L.nan + R.nan;
  o.mn = fminf(L.mn, R.mn);
  o.end = R.end;
  o.tail = R.tail;
  o.pad = 0;
  return o;
}

__device__ __forceinline__ Agg shfl_down_agg(const Agg& a, int off) {
  Agg o;
  o.sumq = __shfl_down_sync(kFull, a.sumq, off);
  o.low = __shfl_down_sync(kFull, a.low, off);
  o.nan = __shfl_down_sync(kFull, a.nan, off);
  o.mn = __shfl_down_sync(kFull, a.mn, off);
  o.end = __shfl_down_sync(kFull, a.end, off);
  o.tail = __shfl_down_sync(kFull, a.tail, off);
  o.pad = 0;
  return o;
}

// q = rint(m * 2^20) with m clamped to [0, 1] (NaN handled by the caller).
__device__ __forceinline__ unsigned long long q20(float m) {
  float c = fminf(fmaxf(m, 0.0f), 1.0f);
  return static_cast<unsigned long long>(__float2int_rn(c * 1048576.0f));
}

struct PosVal {
  Agg v;        // single-position aggregate
  int counted;  // counts in the global row
  int traj;     // trajectory index (-1 outside every trajectory)
};

// Per-position values for this thread's 8 consecutive positions.
__device__ __forceinline__ void load_positions(const float* __restrict__ margin,
                                               const uint32_t* __restrict__ term_bits,
                                               long long n_tok, const long long* offs, int n_traj,
                                               const long long* think_end, float tau,
                                               long long p0, PosVal (&pv)[kItems]) {
  int k = find_traj(offs, n_traj, n_tok, p0);
#pragma unroll
  for (int i = 0; i < kItems; i++) {
    const long long t = p0 + i;
    Agg a = agg_identity();
    int counted = 0;
    if (t < n_tok) {
      if (offs && (k < 0 || t >= offs[k + 1])) k = find_traj(offs, n_traj, n_tok, t);
      const float m = margin[t];
      const bool term = (term_bits[t >> 5] >> (t & 31)) & 1u;
      const bool in = k >= 0;
      const bool last = in && (t == traj_end(offs, n_tok, k) - 1);
      a.tail = (!in || term || last) ? 1 : 0;
      a.end = static_cast<int>(t);
      if (isnan(m)) {
        a.nan = 1;
      } else {
        a.sumq = q20(m);
        a.low = (m < tau) ? 1u : 0u;
        a.mn = m;
      }
      counted = in && (!think_end || t < think_end[k]);
    } else {
      a.tail = 1;
      a.end = static_cast<int>(t);
    }
    pv[i].v = a;
    pv[i].counted = counted;
    pv[i].traj = (t < n_tok) ? k : -1;
  }
}

// Is there a terminator in [a, b] (inclusive; a <= b)?  Word-wise scan.
__device__ __forceinline__ bool any_term(const uint32_t* __restrict__ term_bits, long long a,
                                         long long b) {
  long long w0 = a >> 5, w1 = b >> 5;
  for (long long w = w0; w <= w1; w++) {
    uint32_t m = term_bits[w];
    if (w == w0) m &= 0xffffffffu << (a & 31);
    if (w == w1 && (b & 31) != 31) m &= (2u << (b & 31)) - 1u;
    if (m) return true;
  }
  return false;
}

__device__ __forceinline__ int lower_bound_occ(const int* occ_pos, int n, long long key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (occ_pos[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// First index i in [0, n) with a[i] >= key (n if none), by one warp: each
// round samples 32 evenly spaced entries at once and keeps the bracket, so
// the search takes ceil(log32 n) + 1 round trips instead of log2 n dependent
// loads per thread.
__device__ __forceinline__ int warp_lower_bound(const int* __restrict__ a, int n, long long key) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n;  // the answer is in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const bool ge = idx >= hi || a[idx] >= key;
    const unsigned b = __ballot_sync(kFull, ge);
    const int f = b ? __ffs(b) - 1 : 32;
    const int nlo = f == 0 ? lo : lo + (f - 1) * step + 1;
    const int nhi = f == 32 ? hi : min(hi, lo + f * step);
    lo = nlo;
    hi = nhi;
  }
  const int idx = lo + lane;
  const bool ge = idx >= hi || a[idx] >= key;
  const unsigned b = __ballot_sync(kFull, ge);
  return b ? lo + __ffs(b) - 1 : hi;
}

#ifdef RELAY_TRACE
// Tuning-only K3 timeline (tools/k3_trace.py): stamps by thread 0 of each tile:
// 0 entry, 1 positions loaded, 2 moments added, 3 carry known, 4 occurrences
// gathered, 5 exit.
__device__ unsigned long long g_trace3[4096][8];
__device__ __forceinline__ void stamp3(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x < 4096) g_trace3[blockIdx.x][k] = t;
}
extern "C" int relay_debug_trace3_copy(unsigned long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace3, sizeof(unsigned long long) * 8 * n));
}
#define TRACE3(k) stamp3(k)
#else
#define TRACE3(k) ((void)0)
#endif
constexpr int kOccSmem = 1024;  // K3: a tile's occurrence positions staged in shared memory up to this many

// Published per-tile state for the reverse decoupled look-back.
constexpr int kTileHead = 1;   // value = aggregate from the tile start to its first tail
constexpr int kTileIncl = 2;   // value = aggregate from the tile start onwards (carry included)

// val[2t] holds the head, val[2t+1] the inclusive value; each is written once,
// before the flag that announces it, so a reader never sees a torn value.
__device__ __forceinline__ void publish(int* flag, Agg* val, const Agg& a, int state) {
  val->sumq = a.sumq; val->low = a.low; val->nan = a.nan; val->mn = a.mn;
  val->end = a.end; val->tail = a.tail; val->pad = 0;
  __threadfence();
  atomicExch(flag, state);
}

// K3: one pass per 2,048-position tile.  Tiles are processed right to left
// (tile = n_tiles-1-blockIdx.x), so a tile's carry comes from tiles that were
// dispatched earlier: the reverse segmented scan of (sum q, low, NaN, min, end)
// keyed by segment tails gives, at every position s, the aggregate over
// [s, first tail >= s] — the post-sentence window of a cue at s.  The same pass
// adds the global moments and every occurrence's window to the stats table.
__global__ void __launch_bounds__(kScanThreads)
    seg_fused_kernel(CueDev cs, const float* __restrict__ margin, const uint32_t* __restrict__ term_bits,
                     long long n_tok, const long long* __restrict__ offs, int n_traj,
                     const long long* __restrict__ think_end, float tau, const int* __restrict__ occ_pos,
                     const int* __restrict__ occ_pat, const long long* __restrict__ n_occ_p, long long cap,
                     int* __restrict__ seg_end, float* __restrict__ seg_mean, float* __restrict__ seg_min,
                     float* __restrict__ seg_lowfrac, unsigned long long* __restrict__ stats, int nf,
                     int rank, int per_traj, int* tile_flag, Agg* tile_val, int* done, TpPeers pe,
                     long long pe_words) {
  // per_traj: one table per trajectory ([n_traj][(n_cues+1)*nf]) instead of one
  // pe.world > 0 (relay_segment_reduce_p2p): the last CTA then all-reduces the
  // pe_words table words over peer memory (H6 fused into K3, p2p.cuh)
  const long long table_words = static_cast<long long>(cs.n_cues + 1) * nf;
  __shared__ Agg s_w[kScanThreads / 32];
  __shared__ Agg s_carry;
  __shared__ unsigned long long s_red[kScanThreads / 32][5];
  __shared__ float s_min[kScanThreads / 32];
  const int n_tiles = gridDim.x;
  const int tile = n_tiles - 1 - blockIdx.x;
  const long long base = static_cast<long long>(tile) * kTile;
  const long long p0 = base + threadIdx.x * kItems;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  PosVal pv[kItems];
  TRACE3(0);
  load_positions(margin, term_bits, n_tok, offs, n_traj, think_end, tau, p0, pv);
  TRACE3(1);
  // per-trajectory tables: a tile inside one trajectory reduces as a block;
  // a tile spanning trajectories adds each position on its own (rare)
  int tile_traj = 0;
  if (per_traj) {
    const long long last = (base + kTile < n_tok ? base + kTile : n_tok) - 1;
    const int k0 = find_traj(offs, n_traj, n_tok, base), k1 = find_traj(offs, n_traj, n_tok, last);
    tile_traj = (k0 == k1) ? k0 : -2;
  }
  if (tile_traj == -2) {
#pragma unroll
    for (int i = 0; i < kItems; i++) {
      if (!pv[i].counted) continue;
      unsigned long long* g = stats + pv[i].traj * table_words + static_cast<size_t>(cs.n_cues) * nf;
      pv[i].counted = 0;  // added here, not in the block reduce below
      if (pv[i].v.nan) {
        atomicAdd(g + 7, 1ull);
        continue;
      }
      const unsigned long long q = pv[i].v.sumq;
      atomicAdd(g + 0, 1ull); atomicAdd(g + 1, q); atomicAdd(g + 2, q * q); atomicAdd(g + 3, q);
      atomicAdd(g + 4, 1ull);
      if (pv[i].v.low) atomicAdd(g + 5, 1ull);
      atomicMin(g + kStatFields + rank,
                static_cast<unsigned long long>(__float_as_uint(fminf(fmaxf(pv[i].v.mn, 0.0f), 1.0f))));
    }
  }

  // ---- thread / warp / tile aggregates and global moments
  Agg h = pv[kItems - 1].v;
  unsigned long long gn = 0, gs = 0, gs2 = 0, glow = 0, gnan = 0;
  float gmin = INFINITY;
#pragma unroll
  for (int i = kItems - 1; i >= 0; i--) {
    if (i < kItems - 1) h = agg_suffix(pv[i].v, h);
    if (pv[i].counted) {
      if (pv[i].v.nan) {
        gnan++;
      } else {
        const unsigned long long q = pv[i].v.sumq;
        gn++; gs += q; gs2 += q * q; glow += pv[i].v.low;
        gmin = fminf(gmin, pv[i].v.mn);
      }
    }
  }
  Agg x = h;  // inclusive suffix over lanes (lane i: lanes i..31)
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Agg o = shfl_down_agg(x, off);
    if (lane + off < 32) x = agg_suffix(x, o);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    gn += __shfl_xor_sync(kFull, gn, off);
    gs += __shfl_xor_sync(kFull, gs, off);
    gs2 += __shfl_xor_sync(kFull, gs2, off);
    glow += __shfl_xor_sync(kFull, glow, off);
    gnan += __shfl_xor_sync(kFull, gnan, off);
    gmin = fminf(gmin, __shfl_xor_sync(kFull, gmin, off));
  }
  if (lane == 0) {
    s_w[warp] = x;
    s_red[warp][0] = gn; s_red[warp][1] = gs; s_red[warp][2] = gs2;
    s_red[warp][3] = glow; s_red[warp][4] = gnan;
    s_min[warp] = gmin;
  }
  __syncthreads();

  if (threadIdx.x == 0) {
    unsigned long long* grow = stats + (tile_traj > 0 ? tile_traj * table_words : 0) +
                               static_cast<size_t>(cs.n_cues) * nf;
    unsigned long long a[5] = {0, 0, 0, 0, 0};
    float mn = INFINITY;
    for (int w = 0; w < kScanThreads / 32; w++) {
      for (int f = 0; f < 5; f++) a[f] += s_red[w][f];
      mn = fminf(mn, s_min[w]);
    }
    if (a[0]) {
      atomicAdd(grow + 0, a[0]);   // n
      atomicAdd(grow + 1, a[1]);   // sum q
      atomicAdd(grow + 2, a[2]);   // sum q^2
      atomicAdd(grow + 3, a[1]);   // sum q (token-pooled)
      atomicAdd(grow + 4, a[0]);   // positions
      atomicAdd(grow + 5, a[3]);   // low
      atomicMin(grow + kStatFields + rank,
                static_cast<unsigned long long>(__float_as_uint(fminf(fmaxf(mn, 0.0f), 1.0f))));
    }
    if (a[4]) atomicAdd(grow + 7, a[4]);  // NaN positions
    TRACE3(2);

    // ---- tile head, publish, reverse look-back for the carry
    Agg head = s_w[kScanThreads / 32 - 1];
    for (int w = kScanThreads / 32 - 2; w >= 0; w--) head = agg_suffix(s_w[w], head);
    // A head holding a tail is already this tile's inclusive value.  Every
    // tile still needs its own carry (the run after its last tail), which the
    // look-back assembles from the heads of the tiles to the right: it stops
    // at the first head holding a tail or at an inclusive value.
    if (head.tail) {
      publish(tile_flag + tile, tile_val + 2 * tile + 1, head, kTileIncl);
    } else {
      publish(tile_flag + tile, tile_val + 2 * tile, head, kTileHead);
    }
    Agg carry = agg_identity();
    for (int j = tile + 1; j < n_tiles; j++) {
      int f;
      while ((f = *reinterpret_cast<volatile int*>(tile_flag + j)) == 0) {
      }
      __threadfence();
      const Agg* src = tile_val + 2 * j + (f == kTileIncl ? 1 : 0);
      Agg v;
      v.sumq = __ldcg(&src->sumq); v.low = __ldcg(&src->low);
      v.nan = __ldcg(&src->nan); v.mn = __ldcg(&src->mn);
      v.end = __ldcg(&src->end); v.tail = __ldcg(&src->tail); v.pad = 0;
      carry = agg_suffix(carry, v);
      if (f == kTileIncl || v.tail) break;
    }
    if (!head.tail) publish(tile_flag + tile, tile_val + 2 * tile + 1, agg_suffix(head, carry), kTileIncl);
    s_carry = carry;
  }
  __syncthreads();
  TRACE3(3);

  // ---- per-position suffix aggregates, gathered at the occurrences
  const long long nocc_ll = *n_occ_p < cap ? *n_occ_p : cap;
  const int nocc = static_cast<int>(nocc_ll);
  Agg wc = s_carry;
  for (int w = kScanThreads / 32 - 1; w > warp; w--) wc = agg_suffix(s_w[w], wc);
  Agg nx = shfl_down_agg(x, 1);  // lanes i+1..31
  const Agg cin = (lane < 31) ? agg_suffix(nx, wc) : wc;
  Agg sfx[kItems];
  Agg run = cin;
#pragma unroll
  for (int i = kItems - 1; i >= 0; i--) {
    run = agg_suffix(pv[i].v, run);
    sfx[i] = run;
  }
  // the tile's occurrences [olo, ohi): two warp searches, then (usually)
  // their positions in shared memory, so each thread finds its own without a
  // chain of dependent global loads
  __shared__ int s_orange[2];
  __shared__ int s_occ[kOccSmem];
  if (warp == 0) {
    const int olo = nocc > 0 ? warp_lower_bound(occ_pos, nocc, base) : 0;
    const int ohi = nocc > 0 ? warp_lower_bound(occ_pos, nocc, base + kTile) : 0;
    if (lane == 0) { s_orange[0] = olo; s_orange[1] = ohi; }
  }
  __syncthreads();
  const int olo = s_orange[0], ohi = s_orange[1];
  const bool occ_sm = ohi - olo <= kOccSmem;
  if (occ_sm)
    for (int o = olo + threadIdx.x; o < ohi; o += blockDim.x) s_occ[o - olo] = occ_pos[o];
  __syncthreads();
  if (ohi > olo && p0 < n_tok) {
    int lo;
    if (occ_sm) {   // first occurrence >= p0 among the tile's, in shared memory
      int a = 0, b = ohi - olo;
      while (a < b) {
        const int m = (a + b) >> 1;
        if (s_occ[m] < p0) a = m + 1; else b = m;
      }
      lo = olo + a;
    } else {
      lo = olo + lower_bound_occ(occ_pos + olo, ohi - olo, p0);
    }
    for (int o = lo; o < ohi; o++) {
      const long long s = occ_sm ? s_occ[o - olo] : occ_pos[o];
      if (s >= p0 + kItems) break;
      Agg a = sfx[0];
#pragma unroll
      for (int i = 1; i < kItems; i++)
        if (s == p0 + i) a = sfx[i];
      const int len = a.end - static_cast<int>(s) + 1;
      seg_end[o] = a.end;
      if (a.nan) {
        seg_mean[o] = qnan(); seg_min[o] = qnan(); seg_lowfrac[o] = qnan();
      } else {
        seg_mean[o] = static_cast<float>(static_cast<double>(a.sumq) / (1048576.0 * len));
        seg_min[o] = a.mn;
        seg_lowfrac[o] = static_cast<float>(static_cast<double>(a.low) / len);
      }
      // trigger (R13): no occurrence starts earlier in the same sentence,
      // i.e. the previous start is in another trajectory or a terminator lies
      // in [previous start, s - 1]
      int k = pv[0].traj;   // the position's trajectory, from load_positions
#pragma unroll
      for (int i = 1; i < kItems; i++)
        if (s == p0 + i) k = pv[i].traj;
      auto occ_at = [&](int j) -> long long { return occ_sm && j >= olo ? s_occ[j - olo] : occ_pos[j]; };
      int j = o - 1;
      while (j >= 0 && occ_at(j) == s) j--;
      bool trig = true;
      if (j >= 0) {
        const long long pp = occ_at(j);
        const long long ts = offs ? offs[k] : 0;
        trig = (pp < ts) || any_term(term_bits, pp, s - 1);
      }
      if (think_end && k >= 0 && s >= think_end[k]) continue;
      const int cue = cs.cue_of_orig[occ_pat[o]];
      unsigned long long* row = stats + (per_traj && k > 0 ? k * table_words : 0) +
                                static_cast<size_t>(cue) * nf;
      if (a.nan) {
        atomicAdd(row + 7, 1ull);
        continue;
      }
      const unsigned long long ln = static_cast<unsigned long long>(len);
      const unsigned long long sq = a.sumq;
      const unsigned long long mq = (2 * sq + ln) / (2 * ln);  // round half up
      atomicAdd(row + 0, 1ull);
      atomicAdd(row + 1, mq);
      atomicAdd(row + 2, mq * mq);
      atomicAdd(row + 3, sq);
      atomicAdd(row + 4, ln);
      atomicAdd(row + 5, static_cast<unsigned long long>(a.low));
      if (trig) atomicAdd(row + 6, 1ull);
      atomicMin(row + kStatFields + rank,
                static_cast<unsigned long long>(__float_as_uint(fminf(fmaxf(a.mn, 0.0f), 1.0f))));
    }
  }

  // ---- the last tile to finish resets the look-back flags for the next launch
  // (and, fused H6, all-reduces the finished table over peer memory)
  __shared__ int s_last;
  __syncthreads();
  TRACE3(4);
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1) == n_tiles - 1;
    if (s_last) {
      for (int j = 0; j < n_tiles; j++) tile_flag[j] = 0;
      __threadfence();
      *done = 0;
    }
  }
  __syncthreads();
  TRACE3(5);
  if (pe.world > 0 && s_last) p2p_allreduce_block(pe, stats, pe_words);
}

// ------------------------------------------------- N3 offload estimate
// Per trajectory {large, small_reasoning, answer} token counts of the runtime
// switching replayed offline with a selected cue set (R17).
__global__ void offload_init_kernel(long long n_tok, const long long* __restrict__ offs, int n_traj,
                                    const long long* __restrict__ think_end, long long* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_traj) return;
  const long long a = offs ? offs[k] : 0, b = offs ? offs[k + 1] : n_tok;
  long long te = think_end ? think_end[k] : b;
  te = te > b ? b : (te < a ? a : te);
  out[3 * k + 0] = te - a;
  out[3 * k + 1] = 0;
  out[3 * k + 2] = b - te;
}

__global__ void __launch_bounds__(256)
    offload_occ_kernel(CueDev cs, long long n_tok, const long long* __restrict__ offs, int n_traj,
                       const long long* __restrict__ think_end, const int* __restrict__ occ_pos,
                       const int* __restrict__ occ_pat, const long long* __restrict__ n_occ_p, long long cap,
                       const int* __restrict__ seg_end, const uint8_t* __restrict__ selected,
                       long long* __restrict__ out) {
  const long long nocc = *n_occ_p < cap ? *n_occ_p : cap;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nocc;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = occ_pat[i];
    if (!selected[cs.cue_of_orig[p]]) continue;
    const long long s = occ_pos[i];
    const int k = find_traj(offs, n_traj, n_tok, s);
    if (k < 0) continue;
    const long long a = offs ? offs[k] : 0, b = offs ? offs[k + 1] : n_tok;
    long long te = think_end ? think_end[k] : b;
    te = te > b ? b : (te < a ? a : te);
    const long long c = s + cs.len_of_orig[p] - 1;
    if (c >= te) continue;
    // first selected occurrence of its sentence, in list order
    const int e = seg_end[i];
    bool first = true;
    for (long long j = i - 1; j >= 0 && occ_pos[j] >= a && seg_end[j] == e; j--)
      if (selected[cs.cue_of_orig[occ_pat[j]]]) { first = false; break; }
    if (!first) continue;
    const long long last = e < te - 1 ? e : te - 1;
    if (last > c) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out + 3 * k + 1),
                static_cast<unsigned long long>(last - c));
      atomicAdd(reinterpret_cast<unsigned long long*>(out + 3 * k + 0),
                static_cast<unsigned long long>(-(last - c)));
    }
  }
}

cudaError_t launch_offload_estimate(const CueDev& cs, long long n_tok, const long long* offs, int n_traj,
                                    const long long* think_end, const int* occ_pos, const int* occ_pat,
                                    const long long* n_occ, long long cap, const int* seg_end,
                                    const uint8_t* cue_selected, long long* out, cudaStream_t st) {
  offload_init_kernel<<<(n_traj + 255) / 256, 256, 0, st>>>(n_tok, offs, n_traj, think_end, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || cap <= 0) return e;
  long long blocks = (cap + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  offload_occ_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(cs, n_tok, offs, n_traj, think_end, occ_pos,
                                                                     occ_pat, n_occ, cap, seg_end, cue_selected, out);
  return cudaGetLastError();
}

__global__ void stats_init_kernel(unsigned long long* stats, long long words, int nf, int rank) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < words) {
    const int f = i % nf;
    stats[i] = (f == kStatFields + rank) ? 0x7f800000ull : 0ull;
  }
}

// ------------------------------------------------------------ launchers
static inline int n_tiles_of(long long n_tok) {
  long long t = (n_tok + kTile - 1) / kTile;
  return static_cast<int>(t < 1 ? 1 : t);
}

cudaError_t launch_cue_scan(const CueDev& cs, const int* tokens, long long n_tok,
                            const long long* offs, int n_traj, uint32_t* term_bits, int* occ_pos,
                            int* occ_pat, long long cap, long long* n_occ, const ScanWs& ws,
                            cudaStream_t st) {
  long long nt = (n_tok + kTileB - 1) / kTileB;
  if (nt < 1) nt = 1;
  auto kern = cs.n_classes > 0 ? cue_scan_kernel<true> : cue_scan_kernel<false>;
  const size_t dyn = sizeof(uint2) * (kScanThreads / 32) * (cs.n_dist > 0 ? cs.n_dist : 1);
  kern<<<static_cast<unsigned>(nt), kScanThreads, dyn, st>>>(
      cs, tokens, n_tok, offs, n_traj, term_bits, occ_pos, occ_pat, cap, n_occ, ws.k2_flag, ws.k2_val,
      ws.k2_done);
  return cudaGetLastError();
}

cudaError_t launch_segment_reduce(const CueDev& cs, const float* margin, long long n_tok,
                                  const long long* offs, int n_traj, const long long* think_end,
                                  const uint32_t* term_bits, const int* occ_pos, const int* occ_pat,
                                  const long long* n_occ, long long cap, float tau, int* seg_end,
                                  float* seg_mean, float* seg_min, float* seg_lowfrac,
                                  unsigned long long* stats, int rank, int world, int per_traj,
                                  const ScanWs& ws, cudaStream_t st, const TpPeers* pe, long long pe_words) {
  if (n_tok <= 0) {  // nothing to reduce, but the collective still happens
    return pe ? launch_stats_allreduce_p2p(*pe, stats, pe_words, st) : cudaSuccess;
  }
  const int nt = n_tiles_of(n_tok);
  const int nf = kStatFields + world;
  TpPeers none{};
  seg_fused_kernel<<<nt, kScanThreads, 0, st>>>(cs, margin, term_bits, n_tok, offs, n_traj, think_end,
                                                tau, occ_pos, occ_pat, n_occ, cap, seg_end, seg_mean,
                                                seg_min, seg_lowfrac, stats, nf, rank, per_traj,
                                                ws.tile_flag, ws.tile_val, ws.done, pe ? *pe : none,
                                                pe_words);
  return cudaGetLastError();
}

cudaError_t launch_stats_init(unsigned long long* stats, int n_tables, int n_cues, int rank, int world,
                              cudaStream_t st) {
  const int nf = kStatFields + world;
  const long long n = static_cast<long long>(n_tables) * (n_cues + 1) * nf;
  stats_init_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(stats, n, nf, rank);
  return cudaGetLastError();
}

}  // namespace relay
