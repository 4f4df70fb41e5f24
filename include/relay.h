/*
 * relay.h — C ABI of librelay.so: the B200 (sm_100a) hot path of RelayGen
 * (arXiv 2602.06454): per-token probability margins from logits, switch-cue
 * scanning, post-sentence segment statistics and the decode-step switch flag.
 *
 * Citations: "P:n" = PAPER.md line n (§ / equation / table named alongside),
 * "S:n" = SPEC.md line n.  DESIGN.md "Readings" R1..R19 records every reading
 * of a silent or ambiguous passage that an entry point below depends on.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless marked [host].  The caller owns every
 *    buffer, the stream and the workspace; the library allocates device memory
 *    only inside relay_cueset_create[_ex] (the cue set's own copy: < 20 KB,
 *    plus vocab/8 bytes per token class).
 *  - Hot calls (margin_rows, cue_scan, segment_reduce, stats_init,
 *    step_switch) are asynchronous on `stream`: they never synchronise, never
 *    allocate and never read device memory from the host, so they can be
 *    captured in a CUDA graph.  `stream` is a cudaStream_t (NULL = legacy).
 *  - Host-side argument validation returns an error with NO device work.
 *    Launch failures return RELAY_ERR_CUDA.  relay_last_error() gives a
 *    thread-local message for the last non-OK return.
 *  - Per-row data errors are not return codes: see row_status.
 */
#ifndef RELAY_H_
#define RELAY_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RELAY_VERSION 1
#define RELAY_MAX_CUE_LEN 8     /* tokens per pattern; the configs need 1..6 */
#define RELAY_MAX_PATTERNS 64
#define RELAY_MAX_CUES 64
#define RELAY_MAX_CLASSES 8     /* token classes per cue set (N4) */
#define RELAY_STAT_FIELDS 8     /* + world_size min slots per stats row */

/* stats row layout: row c < n_cues is cue c, row n_cues is the global row. */
enum {
  RELAY_F_N = 0,        /* cue: valid occurrences counted; global: positions counted   */
  RELAY_F_SUM_MQ = 1,   /* cue: sum of window means in Q20; global: sum of q           */
  RELAY_F_SUM_MQ2 = 2,  /* cue: sum of squared window means (Q40); global: sum of q^2  */
  RELAY_F_SUM_WQ = 3,   /* cue: sum of window sums of q; global: sum of q             */
  RELAY_F_SUM_LEN = 4,  /* cue: sum of window lengths; global: positions counted      */
  RELAY_F_SUM_LOW = 5,  /* #{m < tau} inside windows (global: over positions)          */
  RELAY_F_TRIG = 6,     /* cue: occurrences first in their sentence; global: 0         */
  RELAY_F_INVALID = 7,  /* windows (global: positions) holding a NaN margin, excluded  */
  RELAY_F_MIN0 = 8      /* + rank: float bits of this rank's minimum margin            */
};
/* q = rint(m * 2^20) (Q20 fixed point, round-half-even); a window mean is
 * floor((2*sum_q + len) / (2*len)).  Integer fields make the table exact and
 * order-free, so 1 GPU and N GPUs (after the sum all-reduce) agree bit for bit. */

typedef enum {
  RELAY_OK = 0,
  RELAY_ERR_INVALID = 1,      /* bad argument (see each call)                      */
  RELAY_ERR_CUDA = 2,         /* a CUDA launch / runtime call failed               */
  RELAY_ERR_NCCL = 3,         /* NCCL not loadable or an NCCL call failed          */
  RELAY_ERR_ALLOC = 4,        /* cue-set device allocation failed                  */
  RELAY_ERR_UNSUPPORTED = 5,  /* e.g. no sm_100 device                             */
  RELAY_ERR_WORKSPACE = 7     /* ws NULL or smaller than relay_workspace_bytes()   */
} relay_status_t;

typedef enum { RELAY_DT_BF16 = 0, RELAY_DT_F16 = 1, RELAY_DT_F32 = 2 } relay_dtype_t;

typedef enum {
  RELAY_FLAG_NONE = 0,
  RELAY_FLAG_L2S = 1,         /* a switch cue completed on the large model  */
  RELAY_FLAG_S2L = 2,         /* sentence end on the small model            */
  RELAY_FLAG_TO_ANSWER = 3,   /* </think>: the small model owns the answer  */
  RELAY_FLAG_S2L_BUDGET = 4   /* optional small-segment budget hit (off by default) */
} relay_flag_t;

typedef struct CUstream_st* relay_stream_t;   /* == cudaStream_t */
typedef struct relay_cueset_s* relay_cueset_t; /* immutable after create; shareable */

int relay_version(void);

/* Measurement utility (not a step of the method): a read-only stream over
 * `bytes` of device memory at `buf` (16-byte aligned, bytes % 16 == 0),
 * XOR-folded into out[relay_read_probe_words()] (device, uint32, caller-owned;
 * folded into, so zero it first if the value matters).  bench.py times it as
 * the read-only HBM ceiling quoted next to K1's fraction of the copy peak.
 * Errors: NULL pointers, misaligned buf, bad size. */
int32_t relay_read_probe_words(void);
relay_status_t relay_read_probe(const void* buf, int64_t bytes, uint32_t* out, relay_stream_t stream);
const char* relay_status_string(relay_status_t s);
const char* relay_last_error(void);

/* ------------------------------------------------------------------ H1 --
 * relay_margin_rows — probability margin per logit row.
 * Defines (§3.2): p_t = softmax(z_t), m_t = p_t,(1) - p_t,(2).
 * Computed as i1 = argmax z, i2 = argmax over j != i1 (ties: lowest index,
 * IEEE equality, R3), M = z[i1]*iota, S = sum_j exp(z_j*iota - M),
 * margin = (1 - exp(z[i2]*iota - M)) / S, lse = M + ln S.  Probabilities are
 * never materialised.  Indices use the unscaled values.
 *   logits      [n_rows][row_stride] elements of `dt`, row-major; any alignment
 *               of the element type; columns [vocab, row_stride) are never read.
 *   vocab       >= 2 entries per row that participate (R2: all of them).
 *   inv_temperature  iota > 0; 1.0f is the paper (R1).
 *   margin      float[n_rows] (required).
 *   top1, top2  int32[n_rows] (nullable).   lse  float[n_rows] (nullable).
 *   row_status  uint8[n_rows] (nullable): 0 ok; 1 the row holds NaN or +inf
 *               (margin/lse NaN, indices -1); 2 no finite entry (same) (R4).
 * Errors: RELAY_ERR_INVALID if vocab < 2, row_stride < vocab, n_rows < 0,
 * inv_temperature <= 0 or not finite, logits/margin NULL while n_rows > 0, or
 * dt unknown.  n_rows == 0 is a no-op. */
relay_status_t relay_margin_rows(const void* logits, relay_dtype_t dt, int64_t n_rows,
                                 int64_t vocab, int64_t row_stride, float inv_temperature,
                                 float* margin, int32_t* top1, int32_t* top2, float* lse,
                                 uint8_t* row_status, relay_stream_t stream);

/* ------------------------------------------------------ H1 across TP ranks --
 * the margin when the LM head is tensor-parallel and each
 * rank holds a column shard [col_offset, col_offset + shard_vocab) of every
 * logit row.  relay_margin_partials reduces the shard (same streaming kernel
 * as relay_margin_rows) to RELAY_PARTIAL_WORDS floats per row:
 *   [0] v1 = shard max, [1] v2, [2] i1, [3] i2 (int32 bits, GLOBAL indices;
 *   INT32_MAX when absent), [4] S_rel = sum over the shard of
 *   exp((z_j - v1) iota), [5] NaN flag (int32 bits), [6..7] 0.
 * The caller gathers the partials of all shards ([n_shards][n_rows][8], e.g.
 * one NCCL all-gather of 32 B per row per rank) and relay_margin_combine
 * merges them: top-2 by (value desc, global index asc), S = sum_k S_k
 * exp((v1_k - M) iota), margin = (1 - exp((v2 - M) iota)) / S — the same
 * definition as relay_margin_rows on the full row.
 * Errors: as relay_margin_rows (shard_vocab >= 1 allowed), n_shards < 1,
 * col_offset < 0 or col_offset + shard_vocab >= 2^31. */
#define RELAY_PARTIAL_WORDS 8
relay_status_t relay_margin_partials(const void* logits, relay_dtype_t dt, int64_t n_rows,
                                     int64_t shard_vocab, int64_t row_stride, int64_t col_offset,
                                     float inv_temperature, float* partials, relay_stream_t stream);
relay_status_t relay_margin_combine(const float* partials, int32_t n_shards, int64_t n_rows,
                                    float inv_temperature, float* margin, int32_t* top1,
                                    int32_t* top2, float* lse, uint8_t* row_status,
                                    relay_stream_t stream);

/* relay_margin_rows_tp — N1 with the exchange fused into the streaming
 * kernel over peer memory (NVLink P2P through CUDA IPC, no NCCL): each row's
 * 32-byte partial is stored by the kernel's epilogue straight into every
 * rank's receive buffer as soon as the row is reduced (the tag word last,
 * st.release.sys), so the transfer overlaps the stream; a combine kernel on
 * each rank waits (ld.acquire.sys) for all ranks' partials of the call and
 * writes the full-row margin / top1 / top2 / lse / status exactly as
 * relay_margin_combine would.  Every rank of the group calls it once per
 * batch with the same n_rows (collective; stream-ordered, no host sync).
 * Set-up (collective): relay_tp_exchange_create allocates this rank's
 * receive buffer (2 x world x rows_cap x 32 B, device memory owned by the
 * handle) and returns its CUDA IPC handle (RELAY_IPC_HANDLE_BYTES, [host]);
 * the caller gathers the handles of all ranks in rank order (e.g. a
 * torch.distributed all_gather_object) and passes them to
 * relay_tp_exchange_connect, which maps the peers' buffers.  Calls are tagged
 * from a device-side epoch (CUDA-graph safe); buffers alternate by call
 * parity, so a rank one call ahead never overwrites a slot still being read.
 * Errors: world_size not in [1, 8], rank out of range, rows_cap < 1,
 * n_rows > rows_cap, an unconnected rank, and as relay_margin_partials. */
#define RELAY_IPC_HANDLE_BYTES 64
typedef struct relay_tp_exchange_s* relay_tp_exchange_t;
relay_status_t relay_tp_exchange_create(int32_t rank, int32_t world_size, int64_t rows_cap,
                                        uint8_t* ipc_handle_out, relay_tp_exchange_t* out);
relay_status_t relay_tp_exchange_connect(relay_tp_exchange_t x, const uint8_t* ipc_handles);
relay_status_t relay_tp_exchange_destroy(relay_tp_exchange_t x);
relay_status_t relay_margin_rows_tp(relay_tp_exchange_t x, const void* logits_shard, relay_dtype_t dt,
                                    int64_t n_rows, int64_t shard_vocab, int64_t row_stride,
                                    int64_t col_offset, float inv_temperature, float* margin,
                                    int32_t* top1, int32_t* top2, float* lse, uint8_t* row_status,
                                    relay_stream_t stream);

/* relay_stats_allreduce_p2p — H6 without NCCL: the SUM all-reduce of the
 * statistics table(s) over peer memory through a relay_tp_exchange_t created
 * for the same group (its own handle: the call shares the exchange's epoch).
 * One CTA per rank stores the table into every rank's slot (NVLink P2P), tags
 * it (st.release.sys after a system fence), waits for every rank's tag
 * (ld.acquire.sys) and sums the world slices in rank order into `stats`:
 * bit-identical to relay_stats_allreduce.  Collective, stream-ordered.
 * Size the exchange with rows_cap >= (table bytes + 8) / 32.
 * Errors: as relay_stats_allreduce; world_size differing from the
 * exchange's; a table that does not fit a slot (RELAY_ERR_INVALID). */
relay_status_t relay_stats_allreduce_p2p(relay_tp_exchange_t x, uint64_t* stats, int32_t n_tables,
                                         int32_t n_cues, int32_t world_size, relay_stream_t stream);

/* relay_segment_reduce_p2p — relay_segment_reduce (H3-H5) with H6 fused into
 * the same kernel: the CTA that finishes the table last all-reduces it (all
 * n_tables tables) over peer memory exactly as relay_stats_allreduce_p2p
 * does, so the table leaves K3 already summed over the group (compute and
 * collective in one kernel; no NCCL).  Collective over the exchange's group:
 * every rank calls it once per pass (n_tok may be 0 on a rank).  Arguments
 * as relay_segment_reduce plus the exchange (rank / world_size must be the
 * exchange's; slots sized for the tables, e.g. via a StatsExchange).
 * Errors: as relay_segment_reduce and relay_stats_allreduce_p2p. */
relay_status_t relay_segment_reduce_p2p(relay_tp_exchange_t x, relay_cueset_t cs, const float* margin,
                                        int64_t n_tok, const int64_t* traj_offsets, int32_t n_traj,
                                        const int64_t* think_end_pos, const uint32_t* term_bits,
                                        const int32_t* occ_pos, const int32_t* occ_pat, const int64_t* n_occ,
                                        int64_t occ_capacity, float tau, int32_t* seg_end, float* seg_mean,
                                        float* seg_min, float* seg_lowfrac, uint64_t* stats, int32_t rank,
                                        int32_t world_size, uint32_t flags, void* ws, size_t ws_bytes,
                                        relay_stream_t stream);

/* ------------------------------------------------------------- cue set --
 * A model pair's switch-cue set (tab:switch_cue_sets) as token-ID
 * patterns (R5: the caller tokenises every surface variant) plus the sentence
 * terminator set ("sentence-ending punctuation", R8) and </think>.
 *   pat_tokens  [host] int32 CSR tokens; pat_offsets [host] int32[n_patterns+1].
 *   pat_cue     [host] int32[n_patterns] -> cue id in [0, n_cues).
 *   terminator  [host] uint8[vocab], nonzero = sentence-ending token.
 *   think_end_token  the </think> id, or -1.
 *   match_mode  0 LONGEST (one occurrence per start, the longest pattern, R7),
 *               1 ALL (one occurrence per (start, cue), that cue's longest).
 * Errors: RELAY_ERR_INVALID for n_patterns outside [1, 64], n_cues outside
 * [1, 64], an empty or >8-token pattern, a token outside [0, vocab), a cue id
 * outside [0, n_cues), two identical patterns, vocab < 2, match_mode > 1.
 * RELAY_ERR_ALLOC / RELAY_ERR_CUDA on device allocation/copy failure.
 * Ownership: the handle owns its device copies; destroy frees them (call it
 * after the last stream using the handle has been synchronised). */
relay_status_t relay_cueset_create(const int32_t* pat_tokens, const int32_t* pat_offsets,
                                   int32_t n_patterns, const int32_t* pat_cue, int32_t n_cues,
                                   const uint8_t* terminator, int64_t vocab,
                                   int32_t think_end_token, uint32_t match_mode,
                                   relay_cueset_t* out);
/* N4 (text-faithful cues): the same, with token classes.  A pattern element
 * e < 0 matches any token of class c = -1 - e, so one pattern covers a
 * surface form whose tokenisation varies with the next token, e.g. "So "
 * (tab:switch_cue_sets) = {So, <any space-initial token>} [R18].
 *   classes       [host] uint8[n_classes][vocab], nonzero = member; n_classes
 *                 in [0, RELAY_MAX_CLASSES].
 *   decimal_rule  [host] int32[3] = {period, digit_end, digit_start} class ids,
 *                 or NULL: relay_cue_scan then does not end a sentence at a
 *                 terminator that is a period token between a digit-ending
 *                 and a digit-starting token of the same trajectory (S:168-172
 *                 "not inside a decimal number") [R19].  Offline only:
 *                 relay_step_switch decides S->L on the sampled token alone
 *                 (the next token is not known yet).
 * Equal-length patterns that both match at a start: the lower pattern index
 * wins (in both match modes and in relay_step_switch) [R18].
 * Errors: as relay_cueset_create; a negative element that is not a class id;
 * n_classes out of range; classes NULL with n_classes > 0; a decimal_rule
 * entry that is not a class id. */
relay_status_t relay_cueset_create_ex(const int32_t* pat_tokens, const int32_t* pat_offsets,
                                      int32_t n_patterns, const int32_t* pat_cue, int32_t n_cues,
                                      const uint8_t* terminator, int64_t vocab, int32_t think_end_token,
                                      uint32_t match_mode, const uint8_t* classes, int32_t n_classes,
                                      const int32_t* decimal_rule, relay_cueset_t* out);
relay_status_t relay_cueset_destroy(relay_cueset_t cs);
int32_t relay_cueset_n_cues(relay_cueset_t cs);

/* Workspace (caller-owned device memory) for cue_scan + segment_reduce (up to
 * n_tok positions) and step_switch / step_sample (up to batch rows): a scan
 * region followed by a step region, so one workspace may serve both.
 * relay_workspace_bytes gives the bytes for these capacities.
 * relay_workspace_init zeroes the whole workspace (stream-ordered) and
 * registers its capacities with the library (host-side, per process): every
 * later call lays out its counters and flags by the registered capacities,
 * not by its own n_tok / batch, so a workspace reused for smaller problems
 * finds every persistent zero where the previous call left it (the kernels
 * leave them zero again, so CUDA-graph replays need no reset).  Calls with a
 * workspace that was not initialised, with a different ws_bytes, or with
 * n_tok / batch above the capacities return RELAY_ERR_WORKSPACE.  Re-init
 * re-registers (new capacities); relay_workspace_release forgets a workspace
 * (call it before freeing the memory if the address may be reused).  One
 * workspace must not be used by two calls running concurrently.
 * Errors (init): RELAY_ERR_INVALID (NULL ws, negative capacities, n_tok >=
 * 2^31); RELAY_ERR_WORKSPACE (ws_bytes below relay_workspace_bytes). */
size_t relay_workspace_bytes(int64_t n_tok, int64_t occ_capacity, int32_t batch);
relay_status_t relay_workspace_init(void* ws, size_t ws_bytes, int64_t n_tok, int64_t occ_capacity,
                                    int32_t batch, relay_stream_t stream);
relay_status_t relay_workspace_release(void* ws);

/* ------------------------------------------------------------------ H2 --
 * relay_cue_scan — switch-cue occurrences by "simple token matching"
 * ("each occurrence of a discourse-level cue").
 * For each start s of each trajectory [a, b): in LONGEST mode the longest
 * pattern with s + len <= b and tokens[s..s+len) == pattern; patterns never
 * cross a trajectory end.  Occurrences are written in ascending s (ALL mode:
 * then ascending cue id).  term_bits bit t = terminator[tokens[t]] (bit t%32
 * of word t/32; bits past n_tok are 0).
 *   tokens       int32[n_tok], ids in [0, vocab) (other ids never match and
 *                are not terminators).
 *   traj_offsets int64[n_traj+1] nondecreasing, 0 <= offsets <= n_tok; NULL =>
 *                one trajectory [0, n_tok).  Positions outside every
 *                trajectory never start an occurrence.
 *   term_bits    uint32[ceil(n_tok/32)] out.
 *   occ_pos, occ_pat  int32[occ_capacity] out: start and pattern index.
 *   n_occ        int64 device scalar out: the TRUE count even when it
 *                exceeds occ_capacity (then only the first occ_capacity are
 *                written; the caller checks after synchronising).
 * Errors: RELAY_ERR_INVALID (NULL cs/tokens/term_bits/n_occ, n_tok < 0 or
 * >= 2^31, n_tok x cues >= 2^34 with match_mode 1 ALL (K2's look-back counts;
 * never reached in LONGEST), n_traj < 1 with offsets, occ_capacity < 0, occ_pos/occ_pat NULL
 * with occ_capacity > 0); RELAY_ERR_WORKSPACE. */
relay_status_t relay_cue_scan(relay_cueset_t cs, const int32_t* tokens, int64_t n_tok,
                              const int64_t* traj_offsets, int32_t n_traj, uint32_t* term_bits,
                              int32_t* occ_pos, int32_t* occ_pat, int64_t occ_capacity,
                              int64_t* n_occ, void* ws, size_t ws_bytes, relay_stream_t stream);

/* ------------------------------------------------------------ H3 - H5 --
 * relay_segment_reduce — post-sentence windows and the statistics table.
 * Window ("the remainder of the sentence in which the cue appears",
 * P:246 "from the cue position to the next sentence boundary", "from
 * that token until the end of the sentence"): [s, e] inclusive (R9), e = the
 * first t >= s in s's trajectory with a terminator, else the trajectory's
 * last token (R10).  Per occurrence: seg_end = e, seg_mean = mean margin,
 * seg_min, seg_lowfrac = #{m < tau}/len (R11); NaN in the window -> NaN
 * outputs and the occurrence is counted in RELAY_F_INVALID instead.
 * ACCUMULATES (+=) into `stats` ((n_cues+1) rows x (8+world_size) uint64):
 * per cue c: n, sum mean_q, sum mean_q^2, sum window
 * q, sum len, sum low, n_triggers (first occurrence in its sentence, R13),
 * invalid, min into slot 8+rank; global row ("all token positions"):
 * n, sum q, sum q^2, low count, NaN count, min.  With think_end_pos
 * (int64[n_traj], nullable), occurrences at s >= think_end_pos[k] are left out
 * of the cue rows and positions t >= think_end_pos[k] out of the global row
 * (R14); seg_* are still written for them.
 *   margin      float[n_tok] in [0, 1] (relay_margin_rows output; values
 *               outside are clamped to [0,1] for the table only).
 *   term_bits, occ_pos, occ_pat, n_occ: relay_cue_scan outputs (same
 *               traj_offsets); the first min(*n_occ, occ_capacity) are used.
 *   seg_end int32, seg_mean/seg_min/seg_lowfrac float [occ_capacity] out.
 *   stats must have been set by relay_stats_init for (n_cues, rank, world_size).
 *   flags: 0, or RELAY_SEG_PER_TRAJECTORY: `stats` is then n_traj tables, one
 *          per trajectory ([n_traj][(n_cues+1)*(8+world_size)], set by
 *          relay_stats_init_tables), and each occurrence / position adds to
 *          its own trajectory's table.  The tables sum (min for the min slots,
 *          relay_stats_merge) to the single table, so calibration can be
 *          re-run on any subset of trajectories without another pass (the
 *          calibration-size study, Table 5).
 * Bound: the u64 sum of squared Q20 margins is exact for < 2^24 summands, so
 * one call takes n_tok < 2^24 and a table (accumulated over calls and ranks)
 * must stay below 2^24 positions per row (relay_stats_finalize checks).
 * Errors: RELAY_ERR_INVALID (NULLs, n_tok outside [0, 2^24), rank outside
 * [0,world_size), world_size < 1, !(tau finite), unknown flags);
 * RELAY_ERR_WORKSPACE. */
#define RELAY_SEG_PER_TRAJECTORY 1u
relay_status_t relay_segment_reduce(relay_cueset_t cs, const float* margin, int64_t n_tok,
                                    const int64_t* traj_offsets, int32_t n_traj,
                                    const int64_t* think_end_pos, const uint32_t* term_bits,
                                    const int32_t* occ_pos, const int32_t* occ_pat,
                                    const int64_t* n_occ, int64_t occ_capacity, float tau,
                                    int32_t* seg_end, float* seg_mean, float* seg_min,
                                    float* seg_lowfrac, uint64_t* stats, int32_t rank,
                                    int32_t world_size, uint32_t flags, void* ws, size_t ws_bytes,
                                    relay_stream_t stream);

/* Zero the table, then set this rank's min slots to +inf bits (0x7f800000)
 * and every other slot to 0, so that after a SUM all-reduce slot r holds rank
 * r's minimum (H6: one sum-only collective). */
relay_status_t relay_stats_init(uint64_t* stats, int32_t n_cues, int32_t rank, int32_t world_size,
                                relay_stream_t stream);
/* The same for n_tables consecutive tables (RELAY_SEG_PER_TRAJECTORY). */
relay_status_t relay_stats_init_tables(uint64_t* stats, int32_t n_tables, int32_t n_cues, int32_t rank,
                                       int32_t world_size, relay_stream_t stream);
/* Words in one table: (n_cues+1) * (8+world_size); 0 for bad arguments. */
size_t relay_stats_words(int32_t n_cues, int32_t world_size);
/* [host] Merge tables (host memory, n_tables consecutive tables) into one.
 * rank in [0, world_size): tables of that rank (before the all-reduce):
 * fields 0-7 and the other ranks' min slots add (they hold 0 on this rank),
 * the rank's own min slot takes the minimum (float bit patterns of values in
 * [0,1] / +inf order like the integers); with nothing merged the own slot is
 * +inf and the others 0, exactly as relay_stats_init leaves a table.
 * rank = -1: tables already all-reduced: every min slot takes the minimum.
 * Hence summing the per-rank merges equals merging (rank -1) the summed
 * tables.  mask (uint8 [n_tables], nullable = all) picks the tables.  out may
 * not alias tables.
 * Errors: RELAY_ERR_INVALID (NULLs, n_tables < 0, n_cues range, rank outside
 * [-1, world_size)). */
relay_status_t relay_stats_merge(const uint64_t* tables, int32_t n_tables, const uint8_t* mask,
                                 int32_t n_cues, int32_t rank, int32_t world_size, uint64_t* out);

/* ------------------------------------------------------------------ H6 --
 * relay_stats_allreduce — the path's one cross-GPU exchange: an in-place SUM
 * all-reduce (ncclAllReduce, uint64) of n_tables consecutive stats tables on
 * `stream`.  Trajectories are sharded across ranks (data parallel over the
 * calibration traces), each rank reduces its shard into its own
 * table (relay_stats_init with its rank), and after this call every rank
 * holds the table of the whole corpus: integer fields add exactly and slot
 * 8+r holds rank r's minimum (the other ranks contribute 0 there).
 *   nccl_comm  an ncclComm_t over world_size ranks, this process's device
 *              current — from relay_nccl_comm_init, or one torch created
 *              (ProcessGroupNCCL._comm_ptr()); not owned by the call.
 * NCCL is resolved at run time (dlopen "libnccl.so.2"; the copy torch loaded
 * when torch is in the process).
 * Errors: RELAY_ERR_INVALID (NULLs, n_tables < 1, n_cues / world_size range);
 * RELAY_ERR_NCCL (NCCL missing or the call failed). */
#define RELAY_NCCL_ID_BYTES 128
relay_status_t relay_stats_allreduce(void* nccl_comm, uint64_t* stats, int32_t n_tables, int32_t n_cues,
                                     int32_t world_size, relay_stream_t stream);
/* [host] Library-owned communicators: rank 0 calls relay_nccl_unique_id and
 * sends the RELAY_NCCL_ID_BYTES bytes to every rank (e.g. a
 * torch.distributed broadcast); every rank then calls relay_nccl_comm_init
 * with its CUDA device current (collective: blocks until all ranks join).
 * relay_nccl_comm_destroy(NULL) is a no-op. */
/* The NCCL this library resolved at run time (dlopen "libnccl.so.2"):
 * ncclGetVersion's code (e.g. 22809 for 2.28.9) and, when path is non-NULL,
 * the file it was loaded from (path_len bytes, NUL-terminated).  A
 * communicator created by another NCCL copy (e.g. torch's) may be passed to
 * relay_stats_allreduce only if this is the same library (same version and
 * file): the binding checks both and otherwise builds its own communicator.
 * Errors: RELAY_ERR_INVALID (NULL version); RELAY_ERR_NCCL (not loadable). */
relay_status_t relay_nccl_version(int32_t* version, char* path, int32_t path_len);
relay_status_t relay_nccl_unique_id(uint8_t* id_out);
relay_status_t relay_nccl_comm_init(const uint8_t* id, int32_t world_size, int32_t rank, void** comm);
relay_status_t relay_nccl_comm_destroy(void* comm);

/* ------------------------------------------------------------------ H7 --
 * relay_stats_finalize [host] — per-cue and global summaries and the switch-
 * cue selection (§4.2: "selected as a switch cue if its post-
 * sentence margin is higher than the global average by at least one standard
 * error").  host_stats is the (all-reduced) table copied to the host.
 *   mean  = sum_mq / (n 2^20); std = population std from exact 128-bit
 *   integer moments; se = std / sqrt(n); token_mean = sum_wq/(sum_len 2^20);
 *   min = min over the world_size slots; low_frac = sum_low / sum_len.
 *   rule 0: mean_c >= mu + SE_global (R15, default); 1: mean_c >= mu + se_c;
 *   2: mean_c > mu (App. B); 3: every candidate (the "all candidates"
 *   ablation, tab:cue_selection_ablation P:427-445).  Always n_c >= min_count.  With
 *   fewer than 2 global positions std/se are NaN and nothing is selected.
 *   out [host] relay_cue_summary_t[n_cues+1]; out[n_cues] is the global row.
 * Errors: RELAY_ERR_INVALID for NULLs, n_cues/world_size out of range, rule>3,
 * or a row with n >= 2^24 (its sum of squares may have wrapped). */
typedef struct {
  int64_t n;
  double mean, std, se, token_mean, min, low_frac;
  int64_t n_triggers;
  int64_t n_invalid;
  int32_t selected;
} relay_cue_summary_t;
relay_status_t relay_stats_finalize(const uint64_t* host_stats, int32_t n_cues, int32_t world_size,
                                    int64_t min_count, int32_t rule, relay_cue_summary_t* out);

/* ------------------------------------------------------------------ N3 --
 * relay_offload_estimate — the runtime switching (§4.3) replayed
 * offline on a trace with a selected cue set, giving the large-model
 * utilization of tab:speedup per trajectory (R17):
 * reasoning = [a, te) with te = think_end_pos[k] (b when NULL), the answer
 * [te, b) is the small model's; in each sentence (same window end) the first
 * occurrence, in list order, of a selected cue completing at c < te hands
 * positions c+1 .. min(e, te-1) to the small model.
 *   occ_pos/occ_pat/n_occ: relay_cue_scan outputs; seg_end: relay_segment_reduce's.
 *   cue_selected  uint8[n_cues] (device), e.g. from relay_stats_finalize.
 *   out  int64[n_traj][3] = {large, small_reasoning, answer} token counts.
 * Errors: RELAY_ERR_INVALID for NULLs / ranges as relay_segment_reduce. */
relay_status_t relay_offload_estimate(relay_cueset_t cs, int64_t n_tok, const int64_t* traj_offsets,
                                      int32_t n_traj, const int64_t* think_end_pos,
                                      const int32_t* occ_pos, const int32_t* occ_pat,
                                      const int64_t* n_occ, int64_t occ_capacity,
                                      const int32_t* seg_end, const uint8_t* cue_selected,
                                      int64_t* out, relay_stream_t stream);

/* ------------------------------------------------------------------ H8 --
 * relay_step_switch — one decode step for `batch` live sequences: the H1
 * margin of each row, then RelayGen's runtime switch (§4.3,
 * fig:mechanism P:209-216) as an on-device flag, priority </think> > cue >
 * terminator > budget (R16):
 *   answer stage -> NONE;  tok == think_end -> TO_ANSWER, state = answer|small;
 *   large: the longest pattern that is a suffix of hist ++ tok -> L2S + cue id
 *          (suppressed when margin_gate >= 0 and the row margin < margin_gate;
 *          the paper has no gate: pass -1);
 *   small: terminator[tok] -> S2L; else max_small_segment > 0 and
 *          small_run + 1 >= max_small_segment -> S2L_BUDGET (paper: 0 = off);
 *   otherwise NONE, large appends tok to hist, small increments small_run.
 *   Every switch clears hist and small_run.  Cues on the small model are
 *   ignored.  tok = sampled[b], or top1 when sampled == NULL; an
 *   invalid tok (row status != 0 and no sample) gives NONE with no update.
 *   logits [batch][row_stride] of dt; state uint8[batch] in/out (bit0 active
 *   model 0 large / 1 small, bit1 answer stage); hist int32[batch][7] in/out,
 *   oldest first, right-aligned, -1 padded; small_run int32[batch] in/out
 *   (nullable when max_small_segment == 0); outputs margin float, top1/top2
 *   int32 (nullable), flag uint8, cue_id int16 (-1 unless L2S) [batch].
 *   ws: relay_workspace_bytes(0, 0, batch) bytes, zeroed once by
 *   relay_workspace_init.
 * Errors: as relay_margin_rows, plus batch < 0, NULL state/hist/flag/cue_id,
 * RELAY_ERR_WORKSPACE. */
relay_status_t relay_step_switch(relay_cueset_t cs, const void* logits, relay_dtype_t dt,
                                 int32_t batch, int64_t vocab, int64_t row_stride,
                                 float inv_temperature, const int32_t* sampled, uint8_t* state,
                                 int32_t* hist, int32_t* small_run, float margin_gate,
                                 int32_t max_small_segment, float* margin, int32_t* top1,
                                 int32_t* top2, uint8_t* flag, int16_t* cue_id, void* ws,
                                 size_t ws_bytes, relay_stream_t stream);

/* ------------------------------------------------------------------ N2 --
 * relay_step_sample — the decode step with the sampler fused in: the same
 * margin and switch as relay_step_switch, with the token DRAWN from the row
 * instead of passed in.  The paper samples at temperature 0.6, top-p 0.95
 * and (Qwen3) top-k 20; R20 fixes the order of the operations:
 * the top_k entries by (value desc, index asc), p_k = exp((z_k - z_(1)) /
 * temperature) over them, the first L kept with L the smallest count whose
 * mass reaches top_p of the top-k mass (at least one), then the first k with
 * p_0 + ... + p_k > uniform[b] * (kept mass).  The row is read from HBM once:
 * the margin pass keeps it in L2 and bounds its top_k-th largest logit; a
 * second kernel re-reads it from L2, keeps the logits above the bound, selects
 * the exact top-k and draws (an exact fallback covers pathological rows,
 * e.g. a constant row).  Rows with status != 0 draw -1 (no switch update).
 *   temperature > 0; top_k in [1, RELAY_MAX_TOP_K] (clamped to vocab), or 0
 *   for no top-k (the R1-Distill setting: top_p over the whole row, p_k
 *   normalised by the row's total mass; rows whose kept set reaches past the
 *   top 64 are resolved by mass-rank selection: bf16 rows by one counting
 *   pass over their distinct values plus an early-exit pass for the drawn
 *   tie's index, f16/f32 rows over value bins, several extra passes;
 *   masses are fixed point, so the selection is deterministic; needs
 *   vocab < 2^18, else RELAY_ERR_UNSUPPORTED);
 *   top_p in (0, 1]; uniform float[batch] in [0, 1) (device; the caller's
 *   random numbers); sampled int32[batch] out; other arguments, outputs and
 *   workspace as relay_step_switch (rows are streamed whole per CTA).
 * Errors: as relay_step_switch, plus top_k / top_p / temperature out of
 * range, NULL uniform or sampled. */
#define RELAY_MAX_TOP_K 64
relay_status_t relay_step_sample(relay_cueset_t cs, const void* logits, relay_dtype_t dt,
                                 int32_t batch, int64_t vocab, int64_t row_stride,
                                 float inv_temperature, float temperature, int32_t top_k,
                                 float top_p, const float* uniform, uint8_t* state, int32_t* hist,
                                 int32_t* small_run, float margin_gate, int32_t max_small_segment,
                                 float* margin, int32_t* top1, int32_t* top2, int32_t* sampled,
                                 uint8_t* flag, int16_t* cue_id, void* ws, size_t ws_bytes,
                                 relay_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* RELAY_H_ */
