// draw.cuh — the decode-side draw of relay_step_sample (N2): the
// token from a row's top-K list at the sampling temperature with top-p, by
// inverse CDF with the caller's uniform (reading R20).  Used by K4's fused
// top-k draw (margin_kernels.cu) and by K5 (sample_kernels.cu).
#pragma once
#include "relay_device.cuh"

namespace relay {

// The drawn token (one warp; every lane returns it) from the top-K list, R20:
// p_k = 2^((v_k - v_0) log2(e) / T); keep the first L (higher-ranked mass below
// top_p of the total, at least one); inverse CDF with the row's uniform.  Lane
// l holds ranks l and l + 32; prefix sums by warp scans, in rank order.
__device__ __forceinline__ int draw_topk_warp(float s_c, float topp, float u, int K, const float* s_topv,
                                              const int* s_topi, float total_mass = -1.0f) {
  const int lane = threadIdx.x & 31;
  const float v0 = s_topv[0];
  const float p0 = lane < K ? ex2((s_topv[lane] - v0) * s_c) : 0.0f;
  const float p1 = lane + 32 < K ? ex2((s_topv[lane + 32] - v0) * s_c) : 0.0f;
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
  const float lim = topp * total;
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

}  // namespace relay
