// p2p.cuh — the peer-memory SUM all-reduce of uint64 words by one CTA per
// rank (H6 without NCCL), shared by the standalone kernel
// (relay_stats_allreduce_p2p) and K3's last CTA (relay_segment_reduce_p2p).
#pragma once

#include "relay_device.cuh"
#include "relay_internal.h"

namespace relay {

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const void* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Every thread of the CTA calls it.  This rank's words go into slot
// [parity][rank] of every rank's receive buffer (NVLink P2P stores), then one
// tag word per slot (st.release.sys after a system fence); once every rank's
// tag is in this rank's buffer (ld.acquire.sys) the world slices are summed
// in rank order into `words_p` — the same order on every rank.  The epoch
// advances by one (the tag of this call; parity buffers let a rank run one
// call ahead).  `words_p` may have been produced by atomics of other CTAs of
// the same grid: it is read through L2 (ld.cg).
__device__ __forceinline__ void p2p_allreduce_block(const TpPeers& pe, unsigned long long* words_p,
                                                    long long words) {
  const unsigned tag = static_cast<unsigned>(*reinterpret_cast<const volatile int*>(pe.epoch)) + 1u;
  const long long slot_words = pe.rows_cap * 4;  // uint64 words per slot (32-byte rows)
  const long long par = static_cast<long long>(tag & 1u) * pe.world;
  for (int k = 0; k < pe.world; k++) {
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(pe.recv[k]) + (par + pe.rank) * slot_words;
    for (long long w = threadIdx.x; w < words; w += blockDim.x) dst[w] = __ldcg(words_p + w);
  }
  __syncthreads();
  const unsigned long long* own = reinterpret_cast<const unsigned long long*>(pe.recv[pe.rank]);
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int k = 0; k < pe.world; k++) {
      unsigned* flag = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned long long*>(pe.recv[k]) +
                                                   (par + pe.rank) * slot_words + words);
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(tag) : "memory");
    }
    for (int k = 0; k < pe.world; k++)
      while (ld_acquire_sys_u32(own + (par + k) * slot_words + words) != tag) {
      }
  }
  __syncthreads();
  for (long long w = threadIdx.x; w < words; w += blockDim.x) {
    unsigned long long sum = 0;
    for (int k = 0; k < pe.world; k++) sum += __ldcg(own + (par + k) * slot_words + w);
    words_p[w] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile int*>(pe.epoch) = static_cast<int>(tag);
}

}  // namespace relay
