// sample.cuh — the sampler's order and draw (N2, reading R20), shared by the
// inline sampler in K4 (relay_step_sample) and its fallback kernel K5.
#pragma once
#include "relay_device.cuh"

namespace relay {

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

// The drawn token (one warp; every lane returns it) from the top-K list, R20:
// p_k = 2^((v_k - v_0) log2(e) / T); keep the first L (higher-ranked mass below
// top_p of the total, at least one); inverse CDF with the row's uniform.  Lane
// l holds ranks l and l + 32; prefix sums by warp scans, in rank order.
__device__ __forceinline__ int draw_topk(float u, float s_c, float topp, int K, const float* s_topv,
                                         const int* s_topi) {
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
  const float total = __shfl_sync(kFull, c1, 31);
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
