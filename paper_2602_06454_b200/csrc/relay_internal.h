// relay_internal.h — host/device structures and launcher declarations shared
// by relay_kernels.cu and relay_api.cu (not part of the public ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace relay {

constexpr int kMaxLen = 8;        // RELAY_MAX_CUE_LEN
constexpr int kMaxPat = 64;       // RELAY_MAX_PATTERNS
constexpr int kMaxCues = 64;      // RELAY_MAX_CUES
constexpr int kMaxClasses = 8;    // RELAY_MAX_CLASSES
constexpr int kMaxTopK = 64;      // RELAY_MAX_TOP_K
constexpr int kStatFields = 8;    // RELAY_STAT_FIELDS
constexpr int kTile = 2048;       // positions per CTA in K3
#ifndef RELAY_K2_TILE
#define RELAY_K2_TILE 256
#endif
constexpr int kK2Tile = RELAY_K2_TILE;  // positions per CTA in K2 (kScanThreads / 32 groups of 32 starts)
constexpr int kScanThreads = 256; // kTile / 8 consecutive positions per thread
constexpr int kHist = kMaxLen - 1;

// Device view of a cue set (all pointers device memory owned by the handle).
// Patterns are stored sorted by length descending (ties: original order), so
// the first match at a start / as a suffix is the longest.
struct CueDev {
  int n_pat, n_cues, mode, think_end;
  long long vocab;
  const int* pat_tok;      // [n_pat][kMaxLen], sorted
  const int* pat_len;      // [n_pat], sorted
  const int* pat_cue;      // [n_pat], sorted
  const int* pat_orig;     // [n_pat] sorted -> caller's pattern index
  const int* cue_of_orig;  // [n_pat] caller's pattern index -> cue
  const int* len_of_orig;  // [n_pat] caller's pattern index -> length
  const uint32_t* term_tab;  // [ceil(vocab/32)] terminator bitmap
  // N4 token classes: pattern element e < 0 matches any token of class -1-e
  int n_classes;
  const uint32_t* class_tab;  // [n_classes][ceil(vocab/32)]
  int dec_period, dec_dend, dec_dstart;  // decimal-number rule class ids (-1: off)
  // distinct pattern elements (K2's per-group ballot words) and, per sorted
  // pattern element, its index among them (-1 past the pattern's length)
  int n_dist;
  const int* dist_tok;   // [n_dist]
  const int* pat_eidx;   // [n_pat][kMaxLen]
};

// Token `tok` in class c (bit test; false outside [0, vocab)).
__device__ __forceinline__ bool in_class(const CueDev& cs, int c, int tok) {
  if (tok < 0 || tok >= cs.vocab) return false;
  const size_t words = static_cast<size_t>((cs.vocab + 31) >> 5);
  return (__ldg(cs.class_tab + c * words + (tok >> 5)) >> (tok & 31)) & 1u;
}

// Pattern element e against token tok: a token id, or a class (e < 0).
__device__ __forceinline__ bool elem_ok(const CueDev& cs, int tok, int e) {
  return e >= 0 ? tok == e : in_class(cs, -1 - e, tok);
}

// Aggregate of a run of positions for the reverse segmented scan (K3).
struct Agg {
  unsigned long long sumq;  // sum of q = rint(m 2^20)
  unsigned int low;         // #{m < tau}
  unsigned int nan;         // # NaN margins
  float mn;                 // min margin (+inf if none)
  int end;                  // index of the run's first segment tail (valid if tail)
  int tail;                 // 1 if the run contains a segment tail
  int pad;
};

// Workspace layouts (256-byte aligned pieces).  tile_flag and done must be
// zero before the first K3 launch (relay_workspace_init); K3 leaves them zero.
struct ScanWs {
  int* k2_flag;        // [n_tiles2] K2 32-tile block arrival counters (zero between launches)
  long long* k2_val;   // [n_tiles2][2] K2 look-back words: tile counts, then block sums (tag | count)
  int* k2_done;        // [1] K2 look-back epoch (the last launch's flag tag; any start value)
  int* tile_flag;      // [n_tiles] K3 look-back state (0 / head / inclusive)
  Agg* tile_val;       // [n_tiles][2] K3 published head / inclusive aggregate
  int* done;           // [1] K3 finished-tile counter
  size_t bytes;
};
ScanWs scan_ws_layout(void* base, long long n_tok, long long cap);

struct StepWs {
  int* counter;        // [batch] (zero between launches)
  float* part;         // [batch][nsplit][8] partial (v1, v2, i1, i2, m, s, huge, pad)
  int* work;           // [2] chunk counter, CTAs done (zero between launches)
  float* thk;          // [batch] relay_step_sample: K4's top-k bound per row
  uint8_t* status;     // [batch] relay_step_sample: K4's row status
  float* zmax;         // [batch] relay_step_sample: K4's row maximum
  int* slow;           // [batch] relay_step_sample: rows handed to the nucleus kernel
  int* ready_q;        // [batch] relay_step_sample: rows in the order K4 finished them (row + 1,
                       // release-stored; 0 = not yet), popped by K5 (which re-zeroes them)
  int* q_ctl;          // [4] relay_step_sample: queue head (K4), tail (K5), K5 CTAs done
  float* zsum;         // [batch] relay_step_sample: their mass at the sampling temperature
  size_t bytes;
};
constexpr int kMaxSplit = 32;
StepWs step_ws_layout(void* base, int batch);

// ---------------------------------------------------------------- launchers
cudaError_t launch_margin_rows(const void* logits, int dt, long long n_rows, int vocab,
                               long long stride, float iota, float* margin, int* top1, int* top2,
                               float* lse, uint8_t* status, cudaStream_t st);

cudaError_t launch_margin_partials(const void* logits, int dt, long long n_rows, int vocab,
                                  long long stride, long long col_offset, float iota, float* part,
                                  cudaStream_t st);
cudaError_t launch_margin_combine(const float* part, int n_shards, long long n_rows, float iota,
                                  float* margin, int* top1, int* top2, float* lse, uint8_t* status,
                                  cudaStream_t st);

// N1 fused with its exchange over peer memory (relay_margin_rows_tp): every
// rank's receive buffer is recv[2][world][rows_cap][8] floats (parity = the
// call's tag & 1); word 7 of a slot is the call's tag, stored with release
// semantics after the other seven.  epoch / done live on the owning device.
int num_sms();
cudaError_t launch_read_probe(const void* buf, long long bytes, unsigned* out, cudaStream_t st);
constexpr int kMaxTpRanks = 8;
struct TpPeers {
  float* recv[kMaxTpRanks];  // recv[k]: rank k's receive buffer (peer-mapped; own for k == rank)
  int world, rank;
  long long rows_cap;
  int* epoch;                // device: tag of the last completed call
  int* done;                 // device: combine CTAs finished (zero between calls)
};
cudaError_t launch_margin_partials_p2p(const void* logits, int dt, long long n_rows, int vocab, long long stride,
                                       long long col_offset, float iota, const TpPeers& peers, cudaStream_t st);
cudaError_t launch_stats_allreduce_p2p(const TpPeers& peers, unsigned long long* stats, long long words,
                                       cudaStream_t st);
cudaError_t launch_margin_combine_p2p(const TpPeers& peers, long long n_rows, float iota, float* margin, int* top1,
                                      int* top2, float* lse, uint8_t* status, cudaStream_t st);

cudaError_t launch_cue_scan(const CueDev& cs, const int* tokens, long long n_tok,
                            const long long* offs, int n_traj, uint32_t* term_bits, int* occ_pos,
                            int* occ_pat, long long cap, long long* n_occ, const ScanWs& ws,
                            cudaStream_t st);

struct TpPeers;
cudaError_t launch_segment_reduce(const CueDev& cs, const float* margin, long long n_tok,
                                  const long long* offs, int n_traj, const long long* think_end,
                                  const uint32_t* term_bits, const int* occ_pos, const int* occ_pat,
                                  const long long* n_occ, long long cap, float tau, int* seg_end,
                                  float* seg_mean, float* seg_min, float* seg_lowfrac,
                                  unsigned long long* stats, int rank, int world, int per_traj,
                                  const ScanWs& ws, cudaStream_t st, const TpPeers* pe = nullptr,
                                  long long pe_words = 0);

cudaError_t launch_offload_estimate(const CueDev& cs, long long n_tok, const long long* offs, int n_traj,
                                    const long long* think_end, const int* occ_pos, const int* occ_pat,
                                    const long long* n_occ, long long cap, const int* seg_end,
                                    const uint8_t* cue_selected, long long* out, cudaStream_t st);

cudaError_t launch_stats_init(unsigned long long* stats, int n_tables, int n_cues, int rank, int world,
                              cudaStream_t st);

cudaError_t launch_step_switch(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                               long long stride, float iota, const int* sampled, uint8_t* state,
                               int* hist, int* small_run, float gate, int max_seg, float* margin,
                               int* top1, int* top2, uint8_t* flag, int16_t* cue_id,
                               const StepWs& ws, cudaStream_t st);

// relay_step_sample: K4 margin pass (rows kept in L2, top-k bound per row) ...
// The sampler's parameters when K4 draws the token itself (relay_step_sample
// with a top-k): log2(e) / temperature, top-p, the uniforms, the output.
struct StepDraw {
  float s_c;
  float topp;
  const float* uniform;
  int* sampled;
  uint8_t* flag;     // the switch's outputs (K4 runs it on the drawn token)
  int16_t* cue_id;
};
cudaError_t launch_step_rows(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                             long long stride, float iota, uint8_t* state, int* hist, int* small_run,
                             float gate, int max_seg, float* margin, int* top1, int* top2,
                             const StepWs& ws, int topk, cudaStream_t st, const StepDraw* draw = nullptr);
// ... then K5: exact top-k from L2, temperature / top-p, inverse-CDF draw, switch
cudaError_t launch_step_sample(const CueDev& cs, const void* logits, int dt, int batch, int vocab,
                               long long stride, float iota, float temperature, int topk, float topp,
                               const float* uniform, uint8_t* state, int* hist, int* small_run,
                               float gate, int max_seg, float* margin, int* top1, int* top2,
                               int* sampled, uint8_t* flag, int16_t* cue_id, const StepWs& ws,
                               cudaStream_t st);

}  // namespace relay

// The opaque relay_tp_exchange_t of include/relay.h (relay_comm.cu owns it;
// relay_api.cu reads the peer table for relay_segment_reduce_p2p).
struct relay_tp_exchange_s {
  relay::TpPeers pe{};
  float* own = nullptr;     // this rank's receive buffer (cudaMalloc)
  int* counters = nullptr;  // [2]: epoch, done
  bool opened[relay::kMaxTpRanks] = {};
  int device = 0;
};
