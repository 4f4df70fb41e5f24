// switch.cuh — the decode-step switch (H8) shared by K4 (relay_step_switch)
// and K5 (relay_step_sample): the runtime state machine of P:307-314 (§4.3,
// fig:mechanism P:209-216) for one sequence, run by one warp.
#pragma once
#include "relay_device.cuh"
#include "relay_internal.h"

namespace relay {

struct SmemCue {
  int tok[kMaxPat * kMaxLen];
  int len[kMaxPat];
  int cue[kMaxPat];
};

// Runtime switching (§4.3, fig:mechanism P:209-216) for one
// sequence, by one warp: lanes test the (length-sorted) patterns as suffixes of
// hist ++ tok in parallel; the lowest matching lane is the longest pattern.
// The per-sequence switch inputs, loaded by the epilogue warp before it waits
// for the item (so the loads are off the critical path): lane i < 7 holds
// hist[i]; every lane holds state, small_run and the sampled token.
struct SwitchIn {
  int hist_lane;
  int state;
  int small_run;
  int sampled;
};

__device__ __forceinline__ SwitchIn load_switch_in(const int* hist, const uint8_t* state,
                                                   const int* small_run, const int* sampled,
                                                   long long r) {
  const int lane = threadIdx.x & 31;
  SwitchIn in;
  in.hist_lane = lane < kHist ? hist[r * kHist + lane] : -1;
  in.state = state[r];
  in.small_run = small_run ? small_run[r] : 0;
  in.sampled = sampled ? sampled[r] : -1;
  return in;
}

// Stage the cue set's patterns in shared memory (one warp).
__device__ __forceinline__ void load_smem_cue(const CueDev& cs, SmemCue& sc) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < cs.n_pat * kMaxLen; i += 32) sc.tok[i] = cs.pat_tok[i];
  for (int i = lane; i < cs.n_pat; i += 32) {
    sc.len[i] = cs.pat_len[i];
    sc.cue[i] = cs.pat_cue[i];
  }
  __syncwarp();
}

// The longest pattern that is a suffix of hist ++ tok (-1: none), or -1
// without a test when tok cannot trigger a switch.  Warp-uniform.
__device__ __forceinline__ int switch_match(const CueDev& cs, const SmemCue& sc, int tok, const SwitchIn& in) {
  const int lane = threadIdx.x & 31;
  const uint8_t state = static_cast<uint8_t>(in.state);
  const bool valid = tok >= 0 && tok < cs.vocab && !(state & 2);
  // seq[0..6] = hist (oldest first), seq[7] = tok; lane i < 8 holds seq[i]
  int mine = in.hist_lane;
  if (lane == kHist) mine = tok;
  int best = -1;
  if (valid && tok != cs.think_end && (state & 1) == 0) {
    for (int base = 0; base < cs.n_pat; base += 32) {
      const int p = base + lane;
      bool ok = p < cs.n_pat;
      const int len = ok ? sc.len[p] : 0;
#pragma unroll
      for (int i = 0; i < kMaxLen; i++) {
        const int v = __shfl_sync(kFull, mine, i);
        const int k = i - (kMaxLen - len);  // pattern position of seq[i]
        if (ok && k >= 0 && !elem_ok(cs, v, sc.tok[p * kMaxLen + k])) ok = false;
      }
      const unsigned b = __ballot_sync(kFull, ok);
      if (b) { best = base + __ffs(b) - 1; break; }
    }
  }
  return best;
}

// The state machine step for one sequence.  best: switch_match's result for
// tok when the caller computed it already (a sampled token is known before
// the row's margin, so K4 matches it while the consumers stream), else -2.
static __device__ void switch_warp(const CueDev& cs, const SmemCue& sc, int tok, float m, const SwitchIn& in,
                            uint8_t* state_p, int* hist, int* small_run_p, float gate, int max_seg,
                            uint8_t* flag_out, int16_t* cue_out, int best = -2) {
  const int lane = threadIdx.x & 31;
  const uint8_t state = static_cast<uint8_t>(in.state);
  const bool valid = tok >= 0 && tok < cs.vocab && !(state & 2);
  if (best == -2) best = switch_match(cs, sc, tok, in);
  // The decision is warp-uniform (every input is); the history shift comes
  // from the registers loaded before the item (lane k writes hist[k] = old
  // hist[k + 1]), so no lane reloads hist from global memory, and the stores
  // fire from lane 0.
  const int nxt = __shfl_down_sync(kFull, in.hist_lane, 1);
  const int sr = in.small_run;
  int cue = -1, flag = 0;
  uint8_t st = state;
  bool shift = false, clear = false, inc = false;
  if (valid) {
    if (tok == cs.think_end) {
      flag = 3; st = 3; clear = true;
    } else if ((state & 1) == 0) {
      if (best >= 0 && !(gate >= 0.0f && m < gate)) {
        flag = 1; cue = sc.cue[best]; st = 1; clear = true;
      } else {
        shift = true;
      }
    } else {
      const bool term = (cs.term_tab[tok >> 5] >> (tok & 31)) & 1u;
      if (term) {
        flag = 2; st = 0; clear = true;
      } else if (max_seg > 0 && sr + 1 >= max_seg) {
        flag = 4; st = 0; clear = true;
      } else {
        inc = true;
      }
    }
  }
  if (lane < kHist && (shift || clear)) hist[lane] = clear ? -1 : (lane == kHist - 1 ? tok : nxt);
  if (lane == 0) {
    if (valid) {
      if (small_run_p && (clear || inc)) *small_run_p = clear ? 0 : sr + 1;
      *state_p = st;
    }
    *flag_out = static_cast<uint8_t>(flag);
    *cue_out = static_cast<int16_t>(cue);
  }
}


}  // namespace relay
