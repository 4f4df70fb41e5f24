// relay_api.cu — the C ABI of librelay.so (include/relay.h): argument
// validation, the cue-set handle, workspace layout, launches and the host-side
// finalize (H7).  Every hot call is stream-ordered and allocation-free.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <unordered_map>
#include <vector>

#include "../../include/relay.h"
#include "relay_internal.h"

using namespace relay;

struct relay_cueset_s {
  CueDev dev;
  void* block;  // one device allocation holding every array
};

namespace relay {

thread_local char g_err[512] = "";

// shared with relay_comm.cu
relay_status_t fail(relay_status_t s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

}  // namespace relay

namespace {

relay_status_t cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RELAY_OK;
  return fail(RELAY_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

long long tiles_of(long long n_tok) {
  long long t = (n_tok + kTile - 1) / kTile;
  return t < 1 ? 1 : t;
}

bool valid_dtype(relay_dtype_t dt) { return dt == RELAY_DT_BF16 || dt == RELAY_DT_F16 || dt == RELAY_DT_F32; }

relay_status_t check_offsets_args(const int64_t* offs, int32_t n_traj) {
  if (offs && n_traj < 1) return fail(RELAY_ERR_INVALID, "n_traj must be >= 1 with traj_offsets");
  return RELAY_OK;
}

}  // namespace

namespace relay {

ScanWs scan_ws_layout(void* base, long long n_tok, long long cap) {
  ScanWs w{};
  const long long nt = tiles_of(n_tok);
  if (cap < 0) cap = 0;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align256(bytes);
    return q;
  };
  const long long nt2 = (n_tok + kK2Tile - 1) / kK2Tile + 1;  // K2 tiles
  w.k2_flag = reinterpret_cast<int*>(take(sizeof(int) * nt2));
  w.k2_val = reinterpret_cast<long long*>(take(2 * sizeof(long long) * nt2));
  w.k2_done = reinterpret_cast<int*>(take(sizeof(int)));
  w.tile_flag = reinterpret_cast<int*>(take(sizeof(int) * nt));
  w.tile_val = reinterpret_cast<Agg*>(take(2 * sizeof(Agg) * nt));
  w.done = reinterpret_cast<int*>(take(sizeof(int)));
  (void)cap;
  w.bytes = off;
  return w;
}

StepWs step_ws_layout(void* base, int batch) {
  StepWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align256(bytes);
    return q;
  };
  if (batch < 0) batch = 0;
  w.counter = reinterpret_cast<int*>(take(sizeof(int) * (batch + 1)));
  w.part = reinterpret_cast<float*>(take(sizeof(float) * 8 * kMaxSplit * (static_cast<size_t>(batch) + 1)));  // kPartWords = 8
  w.work = reinterpret_cast<int*>(take(sizeof(int) * 4));
  w.thk = reinterpret_cast<float*>(take(sizeof(float) * (static_cast<size_t>(batch) + 1)));
  w.status = reinterpret_cast<uint8_t*>(take(static_cast<size_t>(batch) + 1));
  w.zmax = reinterpret_cast<float*>(take(sizeof(float) * (static_cast<size_t>(batch) + 1)));
  w.slow = reinterpret_cast<int*>(take(sizeof(int) * (static_cast<size_t>(batch) + 1)));
  w.ready_q = reinterpret_cast<int*>(take(sizeof(int) * (static_cast<size_t>(batch) + 1)));
  w.q_ctl = reinterpret_cast<int*>(take(sizeof(int) * 4));
  w.zsum = reinterpret_cast<float*>(take(sizeof(float) * (static_cast<size_t>(batch) + 1)));
  w.bytes = off;
  return w;
}

// Workspace registry (host side): every call lays its counters and flags out
// by the capacities the workspace was initialised with, never by the call's
// own n_tok / batch, so a workspace reused with a smaller problem finds every
// persistent zero where it was left (a size-dependent layout would put them
// on stale data of another array).
namespace {
struct WsCaps {
  size_t bytes;
  long long n_tok, occ;
  int batch;
};
std::mutex g_ws_mu;
std::unordered_map<const void*, WsCaps> g_ws;
}  // namespace

void ws_register(const void* ws, size_t bytes, long long n_tok, long long occ, int batch) {
  std::lock_guard<std::mutex> g(g_ws_mu);
  g_ws[ws] = WsCaps{bytes, n_tok, occ, batch};
}

void ws_unregister(const void* ws) {
  std::lock_guard<std::mutex> g(g_ws_mu);
  g_ws.erase(ws);
}

// The scan layout of a registered workspace, checked against this call's n_tok.
relay_status_t ws_scan(void* ws, size_t ws_bytes, long long n_tok, ScanWs* out) {
  if (!ws) return fail(RELAY_ERR_WORKSPACE, "ws is NULL");
  WsCaps c;
  {
    std::lock_guard<std::mutex> g(g_ws_mu);
    auto it = g_ws.find(ws);
    if (it == g_ws.end()) return fail(RELAY_ERR_WORKSPACE, "ws was not initialised by relay_workspace_init");
    c = it->second;
  }
  if (ws_bytes != c.bytes) return fail(RELAY_ERR_WORKSPACE, "ws_bytes %zu differs from the %zu it was initialised with",
                                       ws_bytes, c.bytes);
  if (n_tok > c.n_tok) return fail(RELAY_ERR_WORKSPACE, "n_tok %lld exceeds the workspace's %lld", n_tok, c.n_tok);
  *out = scan_ws_layout(ws, c.n_tok, c.occ);
  return RELAY_OK;
}

// The step layout (after the scan region) of a registered workspace.
relay_status_t ws_step(void* ws, size_t ws_bytes, int batch, StepWs* out) {
  if (!ws) return fail(RELAY_ERR_WORKSPACE, "ws is NULL");
  WsCaps c;
  {
    std::lock_guard<std::mutex> g(g_ws_mu);
    auto it = g_ws.find(ws);
    if (it == g_ws.end()) return fail(RELAY_ERR_WORKSPACE, "ws was not initialised by relay_workspace_init");
    c = it->second;
  }
  if (ws_bytes != c.bytes) return fail(RELAY_ERR_WORKSPACE, "ws_bytes %zu differs from the %zu it was initialised with",
                                       ws_bytes, c.bytes);
  if (batch > c.batch) return fail(RELAY_ERR_WORKSPACE, "batch %d exceeds the workspace's %d", batch, c.batch);
  const size_t off = scan_ws_layout(nullptr, c.n_tok, c.occ).bytes;
  *out = step_ws_layout(static_cast<char*>(ws) + off, c.batch);
  return RELAY_OK;
}

}  // namespace relay

extern "C" {

int relay_version(void) { return RELAY_VERSION; }

int32_t relay_read_probe_words(void) { return 2 * relay::num_sms(); }

relay_status_t relay_read_probe(const void* buf, int64_t bytes, uint32_t* out, relay_stream_t stream) {
  if (!buf || !out) return fail(RELAY_ERR_INVALID, "buf and out are required");
  if (bytes < 16 || (bytes & 15) || (reinterpret_cast<uintptr_t>(buf) & 15))
    return fail(RELAY_ERR_INVALID, "bytes must be a positive multiple of 16 and buf 16-byte aligned");
  return cuda_status(relay::launch_read_probe(buf, bytes, out, reinterpret_cast<cudaStream_t>(stream)),
                     "relay_read_probe launch");
}

const char* relay_status_string(relay_status_t s) {
  switch (s) {
    case RELAY_OK: return "ok";
    case RELAY_ERR_INVALID: return "invalid argument";
    case RELAY_ERR_CUDA: return "CUDA error";
    case RELAY_ERR_ALLOC: return "allocation failed";
    case RELAY_ERR_UNSUPPORTED: return "unsupported";
    case RELAY_ERR_NCCL: return "NCCL error";
    case RELAY_ERR_WORKSPACE: return "workspace missing or too small";
  }
  return "unknown status";
}

const char* relay_last_error(void) { return g_err; }

relay_status_t relay_margin_rows(const void* logits, relay_dtype_t dt, int64_t n_rows, int64_t vocab,
                                 int64_t row_stride, float inv_temperature, float* margin,
                                 int32_t* top1, int32_t* top2, float* lse, uint8_t* row_status,
                                 relay_stream_t stream) {
  if (!valid_dtype(dt)) return fail(RELAY_ERR_INVALID, "unknown dtype %d", static_cast<int>(dt));
  if (vocab < 2) return fail(RELAY_ERR_INVALID, "vocab must be >= 2 (got %lld)", static_cast<long long>(vocab));
  if (vocab > 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "vocab must be < 2^31");
  if (row_stride < vocab) return fail(RELAY_ERR_INVALID, "row_stride < vocab");
  if (vocab * (dt == RELAY_DT_F32 ? 4 : 2) >= 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "row bytes must be < 2^31");
  if (n_rows < 0) return fail(RELAY_ERR_INVALID, "n_rows < 0");
  if (!(inv_temperature > 0.0f) || !std::isfinite(inv_temperature))
    return fail(RELAY_ERR_INVALID, "inv_temperature must be finite and > 0");
  if (n_rows == 0) return RELAY_OK;
  if (!logits || !margin) return fail(RELAY_ERR_INVALID, "logits and margin are required");
  return cuda_status(launch_margin_rows(logits, static_cast<int>(dt), n_rows, static_cast<int>(vocab),
                                        row_stride, inv_temperature, margin, top1, top2, lse,
                                        row_status, reinterpret_cast<cudaStream_t>(stream)),
                     "relay_margin_rows launch");
}

relay_status_t relay_margin_partials(const void* logits, relay_dtype_t dt, int64_t n_rows,
                                     int64_t shard_vocab, int64_t row_stride, int64_t col_offset,
                                     float inv_temperature, float* partials, relay_stream_t stream) {
  if (!valid_dtype(dt)) return fail(RELAY_ERR_INVALID, "unknown dtype %d", static_cast<int>(dt));
  if (shard_vocab < 1) return fail(RELAY_ERR_INVALID, "shard_vocab must be >= 1");
  if (col_offset < 0 || col_offset + shard_vocab >= 0x7fffffffLL)
    return fail(RELAY_ERR_INVALID, "col_offset out of range");
  if (shard_vocab * (dt == RELAY_DT_F32 ? 4 : 2) >= 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "row bytes must be < 2^31");
  if (row_stride < shard_vocab) return fail(RELAY_ERR_INVALID, "row_stride < shard_vocab");
  if (n_rows < 0) return fail(RELAY_ERR_INVALID, "n_rows < 0");
  if (!(inv_temperature > 0.0f) || !std::isfinite(inv_temperature))
    return fail(RELAY_ERR_INVALID, "inv_temperature must be finite and > 0");
  if (n_rows == 0) return RELAY_OK;
  if (!logits || !partials) return fail(RELAY_ERR_INVALID, "logits and partials are required");
  return cuda_status(launch_margin_partials(logits, static_cast<int>(dt), n_rows, static_cast<int>(shard_vocab),
                                            row_stride, col_offset, inv_temperature, partials,
                                            reinterpret_cast<cudaStream_t>(stream)),
                     "relay_margin_partials launch");
}

relay_status_t relay_margin_combine(const float* partials, int32_t n_shards, int64_t n_rows,
                                    float inv_temperature, float* margin, int32_t* top1, int32_t* top2,
                                    float* lse, uint8_t* row_status, relay_stream_t stream) {
  if (n_shards < 1) return fail(RELAY_ERR_INVALID, "n_shards must be >= 1");
  if (n_rows < 0) return fail(RELAY_ERR_INVALID, "n_rows < 0");
  if (!(inv_temperature > 0.0f) || !std::isfinite(inv_temperature))
    return fail(RELAY_ERR_INVALID, "inv_temperature must be finite and > 0");
  if (n_rows == 0) return RELAY_OK;
  if (!partials || !margin) return fail(RELAY_ERR_INVALID, "partials and margin are required");
  return cuda_status(launch_margin_combine(partials, n_shards, n_rows, inv_temperature, margin, top1, top2,
                                           lse, row_status, reinterpret_cast<cudaStream_t>(stream)),
                     "relay_margin_combine launch");
}

relay_status_t relay_cueset_create_ex(const int32_t* pat_tokens, const int32_t* pat_offsets,
                                      int32_t n_patterns, const int32_t* pat_cue, int32_t n_cues,
                                      const uint8_t* terminator, int64_t vocab, int32_t think_end_token,
                                      uint32_t match_mode, const uint8_t* classes, int32_t n_classes,
                                      const int32_t* decimal_rule, relay_cueset_t* out) {
  if (!out) return fail(RELAY_ERR_INVALID, "out is NULL");
  if (n_classes < 0 || n_classes > kMaxClasses)
    return fail(RELAY_ERR_INVALID, "n_classes must be in [0, %d]", kMaxClasses);
  if (n_classes > 0 && !classes) return fail(RELAY_ERR_INVALID, "classes is NULL");
  if (decimal_rule) {
    for (int i = 0; i < 3; i++)
      if (decimal_rule[i] < 0 || decimal_rule[i] >= n_classes)
        return fail(RELAY_ERR_INVALID, "decimal_rule[%d] is not a class id", i);
  }
  *out = nullptr;
  if (!pat_tokens || !pat_offsets || !pat_cue || !terminator)
    return fail(RELAY_ERR_INVALID, "pattern arrays and terminator are required");
  if (n_patterns < 1 || n_patterns > kMaxPat) return fail(RELAY_ERR_INVALID, "n_patterns must be in [1, %d]", kMaxPat);
  if (n_cues < 1 || n_cues > kMaxCues) return fail(RELAY_ERR_INVALID, "n_cues must be in [1, %d]", kMaxCues);
  if (vocab < 2 || vocab > 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "vocab out of range");
  if (match_mode > 1) return fail(RELAY_ERR_INVALID, "match_mode must be 0 or 1");
  if (pat_offsets[0] != 0) return fail(RELAY_ERR_INVALID, "pat_offsets[0] must be 0");
  std::vector<int> len(n_patterns);
  for (int p = 0; p < n_patterns; p++) {
    len[p] = pat_offsets[p + 1] - pat_offsets[p];
    if (len[p] < 1 || len[p] > kMaxLen) return fail(RELAY_ERR_INVALID, "pattern %d has length %d (1..%d)", p, len[p], kMaxLen);
    if (pat_cue[p] < 0 || pat_cue[p] >= n_cues) return fail(RELAY_ERR_INVALID, "pattern %d cue id out of range", p);
    for (int k = 0; k < len[p]; k++) {
      int t = pat_tokens[pat_offsets[p] + k];
      if (t < 0 && -1 - t < n_classes) continue;  // class element
      if (t < 0 || t >= vocab)
        return fail(RELAY_ERR_INVALID, "pattern %d element %d is neither a token in [0, vocab) nor a class", p, t);
    }
  }
  for (int p = 0; p < n_patterns; p++)
    for (int q = p + 1; q < n_patterns; q++)
      if (len[p] == len[q] &&
          std::memcmp(pat_tokens + pat_offsets[p], pat_tokens + pat_offsets[q], sizeof(int32_t) * len[p]) == 0)
        return fail(RELAY_ERR_INVALID, "patterns %d and %d are identical", p, q);
  // sort by length descending, stable in the caller's order
  std::vector<int> order(n_patterns);
  for (int p = 0; p < n_patterns; p++) order[p] = p;
  for (int a = 1; a < n_patterns; a++)
    for (int b = a; b > 0 && len[order[b]] > len[order[b - 1]]; b--) std::swap(order[b], order[b - 1]);
  std::vector<int> h_tok(static_cast<size_t>(n_patterns) * kMaxLen, -1), h_len(n_patterns), h_cue(n_patterns),
      h_orig(n_patterns), h_cue_orig(n_patterns);
  for (int i = 0; i < n_patterns; i++) {
    const int p = order[i];
    h_len[i] = len[p];
    h_cue[i] = pat_cue[p];
    h_orig[i] = p;
    for (int k = 0; k < len[p]; k++) h_tok[static_cast<size_t>(i) * kMaxLen + k] = pat_tokens[pat_offsets[p] + k];
  }
  for (int p = 0; p < n_patterns; p++) h_cue_orig[p] = pat_cue[p];
  // distinct pattern elements (K2 computes one ballot word per element per
  // 32-start group and evaluates every pattern from them)
  std::vector<int> h_dist, h_eidx(static_cast<size_t>(n_patterns) * kMaxLen, -1);
  for (int i = 0; i < n_patterns; i++)
    for (int k = 0; k < h_len[i]; k++) {
      const int e = h_tok[static_cast<size_t>(i) * kMaxLen + k];
      int d = 0;
      while (d < static_cast<int>(h_dist.size()) && h_dist[d] != e) d++;
      if (d == static_cast<int>(h_dist.size())) h_dist.push_back(e);
      h_eidx[static_cast<size_t>(i) * kMaxLen + k] = d;
    }
  const size_t words = static_cast<size_t>((vocab + 31) / 32);
  std::vector<uint32_t> h_term(words, 0u);
  for (int64_t v = 0; v < vocab; v++)
    if (terminator[v]) h_term[v >> 5] |= 1u << (v & 31);
  std::vector<uint32_t> h_cls(words * static_cast<size_t>(n_classes), 0u);
  for (int c = 0; c < n_classes; c++)
    for (int64_t v = 0; v < vocab; v++)
      if (classes[static_cast<size_t>(c) * vocab + v]) h_cls[c * words + (v >> 5)] |= 1u << (v & 31);
  size_t off_tok = 0, off_len = align256(h_tok.size() * 4), off_cue = off_len + align256(n_patterns * 4),
         off_orig = off_cue + align256(n_patterns * 4), off_co = off_orig + align256(n_patterns * 4),
         off_lo = off_co + align256(n_patterns * 4), off_term = off_lo + align256(n_patterns * 4),
         off_cls = off_term + align256(words * 4), off_dist = off_cls + align256(h_cls.size() * 4 + 4),
         off_eidx = off_dist + align256(h_dist.size() * 4), total = off_eidx + align256(h_eidx.size() * 4);
  std::vector<char> host(total, 0);
  std::memcpy(host.data() + off_tok, h_tok.data(), h_tok.size() * 4);
  std::memcpy(host.data() + off_len, h_len.data(), n_patterns * 4);
  std::memcpy(host.data() + off_cue, h_cue.data(), n_patterns * 4);
  std::memcpy(host.data() + off_orig, h_orig.data(), n_patterns * 4);
  std::memcpy(host.data() + off_co, h_cue_orig.data(), n_patterns * 4);
  std::memcpy(host.data() + off_lo, len.data(), n_patterns * 4);
  std::memcpy(host.data() + off_term, h_term.data(), words * 4);
  if (!h_cls.empty()) std::memcpy(host.data() + off_cls, h_cls.data(), h_cls.size() * 4);
  std::memcpy(host.data() + off_dist, h_dist.data(), h_dist.size() * 4);
  std::memcpy(host.data() + off_eidx, h_eidx.data(), h_eidx.size() * 4);
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, total);
  if (e != cudaSuccess) return fail(RELAY_ERR_ALLOC, "cudaMalloc(%zu): %s", total, cudaGetErrorString(e));
  e = cudaMemcpy(d, host.data(), total, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d);
    return cuda_status(e, "cue set upload");
  }
  relay_cueset_s* cs = new (std::nothrow) relay_cueset_s;
  if (!cs) {
    cudaFree(d);
    return fail(RELAY_ERR_ALLOC, "host allocation failed");
  }
  char* b = static_cast<char*>(d);
  cs->block = d;
  cs->dev.n_pat = n_patterns;
  cs->dev.n_cues = n_cues;
  cs->dev.mode = static_cast<int>(match_mode);
  cs->dev.think_end = think_end_token;
  cs->dev.vocab = vocab;
  cs->dev.pat_tok = reinterpret_cast<const int*>(b + off_tok);
  cs->dev.pat_len = reinterpret_cast<const int*>(b + off_len);
  cs->dev.pat_cue = reinterpret_cast<const int*>(b + off_cue);
  cs->dev.pat_orig = reinterpret_cast<const int*>(b + off_orig);
  cs->dev.cue_of_orig = reinterpret_cast<const int*>(b + off_co);
  cs->dev.len_of_orig = reinterpret_cast<const int*>(b + off_lo);
  cs->dev.term_tab = reinterpret_cast<const uint32_t*>(b + off_term);
  cs->dev.n_classes = n_classes;
  cs->dev.class_tab = reinterpret_cast<const uint32_t*>(b + off_cls);
  cs->dev.n_dist = static_cast<int>(h_dist.size());
  cs->dev.dist_tok = reinterpret_cast<const int*>(b + off_dist);
  cs->dev.pat_eidx = reinterpret_cast<const int*>(b + off_eidx);
  cs->dev.dec_period = decimal_rule ? decimal_rule[0] : -1;
  cs->dev.dec_dend = decimal_rule ? decimal_rule[1] : -1;
  cs->dev.dec_dstart = decimal_rule ? decimal_rule[2] : -1;
  *out = cs;
  return RELAY_OK;
}

relay_status_t relay_cueset_create(const int32_t* pat_tokens, const int32_t* pat_offsets,
                                   int32_t n_patterns, const int32_t* pat_cue, int32_t n_cues,
                                   const uint8_t* terminator, int64_t vocab, int32_t think_end_token,
                                   uint32_t match_mode, relay_cueset_t* out) {
  return relay_cueset_create_ex(pat_tokens, pat_offsets, n_patterns, pat_cue, n_cues, terminator, vocab,
                                think_end_token, match_mode, nullptr, 0, nullptr, out);
}

relay_status_t relay_cueset_destroy(relay_cueset_t cs) {
  if (!cs) return RELAY_OK;
  cudaError_t e = cudaFree(cs->block);
  delete cs;
  return cuda_status(e, "cue set free");
}

int32_t relay_cueset_n_cues(relay_cueset_t cs) { return cs ? cs->dev.n_cues : -1; }

size_t relay_workspace_bytes(int64_t n_tok, int64_t occ_capacity, int32_t batch) {
  size_t a = scan_ws_layout(nullptr, n_tok < 0 ? 0 : n_tok, occ_capacity).bytes;
  size_t b = step_ws_layout(nullptr, batch < 0 ? 0 : batch).bytes;
  return a + b;  // the step region follows the scan region: one workspace may serve both
}

relay_status_t relay_workspace_init(void* ws, size_t ws_bytes, int64_t n_tok, int64_t occ_capacity, int32_t batch,
                                    relay_stream_t stream) {
  if (!ws) return fail(RELAY_ERR_INVALID, "ws is NULL");
  if (n_tok < 0 || n_tok >= 0x7fffffffLL || occ_capacity < 0 || batch < 0)
    return fail(RELAY_ERR_INVALID, "capacities out of range");
  const size_t need = relay_workspace_bytes(n_tok, occ_capacity, batch);
  if (ws_bytes < need) return fail(RELAY_ERR_WORKSPACE, "need %zu workspace bytes for these capacities", need);
  relay_status_t s = cuda_status(cudaMemsetAsync(ws, 0, ws_bytes, reinterpret_cast<cudaStream_t>(stream)),
                                 "workspace init");
  if (s == RELAY_OK) relay::ws_register(ws, ws_bytes, n_tok, occ_capacity, batch);
  return s;
}

relay_status_t relay_workspace_release(void* ws) {
  relay::ws_unregister(ws);
  return RELAY_OK;
}

relay_status_t relay_cue_scan(relay_cueset_t cs, const int32_t* tokens, int64_t n_tok,
                              const int64_t* traj_offsets, int32_t n_traj, uint32_t* term_bits,
                              int32_t* occ_pos, int32_t* occ_pat, int64_t occ_capacity, int64_t* n_occ,
                              void* ws, size_t ws_bytes, relay_stream_t stream) {
  if (!cs || !n_occ) return fail(RELAY_ERR_INVALID, "cs and n_occ are required");
  if (n_tok < 0 || n_tok >= 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "n_tok must be in [0, 2^31)");
  if (n_tok > 0 && (!tokens || !term_bits)) return fail(RELAY_ERR_INVALID, "tokens and term_bits are required");
  if (occ_capacity < 0) return fail(RELAY_ERR_INVALID, "occ_capacity < 0");
  if (occ_capacity > 0 && (!occ_pos || !occ_pat)) return fail(RELAY_ERR_INVALID, "occ_pos/occ_pat are required");
  relay_status_t s = check_offsets_args(traj_offsets, n_traj);
  if (s != RELAY_OK) return s;
  ScanWs w;
  s = ws_scan(ws, ws_bytes, n_tok, &w);
  if (s != RELAY_OK) return s;
  // K2's look-back words hold occurrence counts below 2^34 (at most one per
  // start in LONGEST mode, one per start and cue in ALL mode)
  if (n_tok * (cs->dev.mode == 0 ? 1LL : static_cast<long long>(cs->dev.n_cues)) >= (1LL << 34))
    return fail(RELAY_ERR_INVALID, "n_tok x cues must stay below 2^34 (K2's look-back counts)");
  return cuda_status(launch_cue_scan(cs->dev, tokens, n_tok, reinterpret_cast<const long long*>(traj_offsets),
                                     traj_offsets ? n_traj : 1, term_bits, occ_pos, occ_pat, occ_capacity,
                                     reinterpret_cast<long long*>(n_occ), w,
                                     reinterpret_cast<cudaStream_t>(stream)),
                     "relay_cue_scan launch");
}

size_t relay_stats_words(int32_t n_cues, int32_t world_size) {
  if (n_cues < 0 || world_size < 1) return 0;
  return static_cast<size_t>(n_cues + 1) * (kStatFields + world_size);
}

relay_status_t relay_stats_init_tables(uint64_t* stats, int32_t n_tables, int32_t n_cues, int32_t rank,
                                       int32_t world_size, relay_stream_t stream) {
  if (!stats) return fail(RELAY_ERR_INVALID, "stats is NULL");
  if (n_tables < 1) return fail(RELAY_ERR_INVALID, "n_tables < 1");
  if (n_cues < 1 || n_cues > kMaxCues) return fail(RELAY_ERR_INVALID, "n_cues out of range");
  if (world_size < 1 || rank < 0 || rank >= world_size) return fail(RELAY_ERR_INVALID, "bad rank/world_size");
  return cuda_status(launch_stats_init(reinterpret_cast<unsigned long long*>(stats), n_tables, n_cues, rank,
                                       world_size, reinterpret_cast<cudaStream_t>(stream)),
                     "relay_stats_init launch");
}

relay_status_t relay_stats_init(uint64_t* stats, int32_t n_cues, int32_t rank, int32_t world_size,
                                relay_stream_t stream) {
  return relay_stats_init_tables(stats, 1, n_cues, rank, world_size, stream);
}

relay_status_t relay_stats_merge(const uint64_t* tables, int32_t n_tables, const uint8_t* mask,
                                 int32_t n_cues, int32_t rank, int32_t world_size, uint64_t* out) {
  if (!out || (n_tables > 0 && !tables)) return fail(RELAY_ERR_INVALID, "tables and out are required");
  if (n_tables < 0) return fail(RELAY_ERR_INVALID, "n_tables < 0");
  if (n_cues < 1 || n_cues > kMaxCues) return fail(RELAY_ERR_INVALID, "n_cues out of range");
  if (world_size < 1 || rank < -1 || rank >= world_size) return fail(RELAY_ERR_INVALID, "bad rank/world_size");
  const int nf = kStatFields + world_size;
  // a min slot takes the minimum if it is this rank's (or every slot, rank -1:
  // tables already all-reduced); the other slots hold 0 on this rank and add
  auto is_min = [&](size_t i) {
    const int f = static_cast<int>(i % nf);
    return f >= kStatFields && (rank < 0 || f == kStatFields + rank);
  };
  const size_t words = static_cast<size_t>(n_cues + 1) * nf;
  for (size_t i = 0; i < words; i++) out[i] = is_min(i) ? 0x7f800000ull : 0ull;
  for (int32_t t = 0; t < n_tables; t++) {
    if (mask && !mask[t]) continue;
    const uint64_t* tab = tables + static_cast<size_t>(t) * words;
    for (size_t i = 0; i < words; i++) {
      if (!is_min(i)) out[i] += tab[i];
      else if (tab[i] < out[i]) out[i] = tab[i];
    }
  }
  return RELAY_OK;
}

static relay_status_t segment_reduce_impl(relay_tp_exchange_t x, relay_cueset_t cs, const float* margin, int64_t n_tok,
                                    const int64_t* traj_offsets, int32_t n_traj, const int64_t* think_end_pos,
                                    const uint32_t* term_bits, const int32_t* occ_pos, const int32_t* occ_pat,
                                    const int64_t* n_occ, int64_t occ_capacity, float tau, int32_t* seg_end,
                                    float* seg_mean, float* seg_min, float* seg_lowfrac, uint64_t* stats,
                                    int32_t rank, int32_t world_size, uint32_t flags, void* ws,
                                    size_t ws_bytes, relay_stream_t stream) {
  if (!cs || !stats || !n_occ) return fail(RELAY_ERR_INVALID, "cs, stats and n_occ are required");
  if (flags & ~RELAY_SEG_PER_TRAJECTORY) return fail(RELAY_ERR_INVALID, "unknown flags 0x%x", flags);
  if (n_tok < 0 || n_tok >= (1LL << 24))
    return fail(RELAY_ERR_INVALID, "n_tok must be in [0, 2^24): the table's u64 sum of squares of Q20 margins");
  if (n_tok > 0 && (!margin || !term_bits)) return fail(RELAY_ERR_INVALID, "margin and term_bits are required");
  if (occ_capacity < 0) return fail(RELAY_ERR_INVALID, "occ_capacity < 0");
  if (occ_capacity > 0 && (!occ_pos || !occ_pat || !seg_end || !seg_mean || !seg_min || !seg_lowfrac))
    return fail(RELAY_ERR_INVALID, "occurrence and seg_* arrays are required");
  if (world_size < 1 || rank < 0 || rank >= world_size) return fail(RELAY_ERR_INVALID, "bad rank/world_size");
  if (!std::isfinite(tau)) return fail(RELAY_ERR_INVALID, "tau must be finite");
  if (think_end_pos && !traj_offsets) return fail(RELAY_ERR_INVALID, "think_end_pos needs traj_offsets");
  relay_status_t s = check_offsets_args(traj_offsets, n_traj);
  if (s != RELAY_OK) return s;
  const long long n_tables = (flags & RELAY_SEG_PER_TRAJECTORY) ? (traj_offsets ? n_traj : 1) : 1;
  const long long words = static_cast<long long>(relay_stats_words(relay_cueset_n_cues(cs), world_size)) * n_tables;
  if (x) {
    if (x->pe.world != world_size || x->pe.rank != rank)
      return fail(RELAY_ERR_INVALID, "rank/world_size differ from the exchange's");
    for (int k = 0; k < x->pe.world; k++)
      if (!x->pe.recv[k]) return fail(RELAY_ERR_INVALID, "exchange not connected (rank %d)", k);
    if (words * 8 + 8 > x->pe.rows_cap * 32)
      return fail(RELAY_ERR_INVALID, "exchange slots hold %lld B, the table(s) need %lld B + 8",
                  x->pe.rows_cap * 32, words * 8);
  }
  ScanWs w;
  s = ws_scan(ws, ws_bytes, n_tok, &w);
  if (s != RELAY_OK) return s;
  return cuda_status(
      launch_segment_reduce(cs->dev, margin, n_tok, reinterpret_cast<const long long*>(traj_offsets),
                            traj_offsets ? n_traj : 1, reinterpret_cast<const long long*>(think_end_pos),
                            term_bits, occ_pos, occ_pat, reinterpret_cast<const long long*>(n_occ),
                            occ_capacity, tau, seg_end, seg_mean, seg_min, seg_lowfrac,
                            reinterpret_cast<unsigned long long*>(stats), rank, world_size,
                            (flags & RELAY_SEG_PER_TRAJECTORY) ? 1 : 0, w,
                            reinterpret_cast<cudaStream_t>(stream), x ? &x->pe : nullptr, words),
      "relay_segment_reduce launch");
}

relay_status_t relay_segment_reduce(relay_cueset_t cs, const float* margin, int64_t n_tok,
                                    const int64_t* traj_offsets, int32_t n_traj, const int64_t* think_end_pos,
                                    const uint32_t* term_bits, const int32_t* occ_pos, const int32_t* occ_pat,
                                    const int64_t* n_occ, int64_t occ_capacity, float tau, int32_t* seg_end,
                                    float* seg_mean, float* seg_min, float* seg_lowfrac, uint64_t* stats,
                                    int32_t rank, int32_t world_size, uint32_t flags, void* ws,
                                    size_t ws_bytes, relay_stream_t stream) {
  return segment_reduce_impl(nullptr, cs, margin, n_tok, traj_offsets, n_traj, think_end_pos, term_bits, occ_pos,
                             occ_pat, n_occ, occ_capacity, tau, seg_end, seg_mean, seg_min, seg_lowfrac, stats,
                             rank, world_size, flags, ws, ws_bytes, stream);
}

relay_status_t relay_segment_reduce_p2p(relay_tp_exchange_t x, relay_cueset_t cs, const float* margin, int64_t n_tok,
                                        const int64_t* traj_offsets, int32_t n_traj, const int64_t* think_end_pos,
                                        const uint32_t* term_bits, const int32_t* occ_pos, const int32_t* occ_pat,
                                        const int64_t* n_occ, int64_t occ_capacity, float tau, int32_t* seg_end,
                                        float* seg_mean, float* seg_min, float* seg_lowfrac, uint64_t* stats,
                                        int32_t rank, int32_t world_size, uint32_t flags, void* ws,
                                        size_t ws_bytes, relay_stream_t stream) {
  if (!x) return fail(RELAY_ERR_INVALID, "x is NULL");
  return segment_reduce_impl(x, cs, margin, n_tok, traj_offsets, n_traj, think_end_pos, term_bits, occ_pos,
                             occ_pat, n_occ, occ_capacity, tau, seg_end, seg_mean, seg_min, seg_lowfrac, stats,
                             rank, world_size, flags, ws, ws_bytes, stream);
}

relay_status_t relay_offload_estimate(relay_cueset_t cs, int64_t n_tok, const int64_t* traj_offsets,
                                      int32_t n_traj, const int64_t* think_end_pos, const int32_t* occ_pos,
                                      const int32_t* occ_pat, const int64_t* n_occ, int64_t occ_capacity,
                                      const int32_t* seg_end, const uint8_t* cue_selected, int64_t* out,
                                      relay_stream_t stream) {
  if (!cs || !n_occ || !cue_selected || !out) return fail(RELAY_ERR_INVALID, "cs, n_occ, cue_selected and out are required");
  if (n_tok < 0 || n_tok >= 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "n_tok must be in [0, 2^31)");
  if (occ_capacity < 0) return fail(RELAY_ERR_INVALID, "occ_capacity < 0");
  if (occ_capacity > 0 && (!occ_pos || !occ_pat || !seg_end)) return fail(RELAY_ERR_INVALID, "occurrence arrays are required");
  if (think_end_pos && !traj_offsets) return fail(RELAY_ERR_INVALID, "think_end_pos needs traj_offsets");
  relay_status_t s = check_offsets_args(traj_offsets, n_traj);
  if (s != RELAY_OK) return s;
  return cuda_status(launch_offload_estimate(cs->dev, n_tok, reinterpret_cast<const long long*>(traj_offsets),
                                             traj_offsets ? n_traj : 1,
                                             reinterpret_cast<const long long*>(think_end_pos), occ_pos, occ_pat,
                                             reinterpret_cast<const long long*>(n_occ), occ_capacity, seg_end,
                                             cue_selected, reinterpret_cast<long long*>(out),
                                             reinterpret_cast<cudaStream_t>(stream)),
                     "relay_offload_estimate launch");
}

relay_status_t relay_stats_finalize(const uint64_t* host_stats, int32_t n_cues, int32_t world_size,
                                    int64_t min_count, int32_t rule, relay_cue_summary_t* out) {
  if (!host_stats || !out) return fail(RELAY_ERR_INVALID, "host_stats and out are required");
  if (n_cues < 1 || n_cues > kMaxCues) return fail(RELAY_ERR_INVALID, "n_cues out of range");
  if (world_size < 1) return fail(RELAY_ERR_INVALID, "world_size < 1");
  if (rule < 0 || rule > 3) return fail(RELAY_ERR_INVALID, "rule must be 0, 1, 2 or 3");
  const int nf = kStatFields + world_size;
  const double Q = 1048576.0;
  // sum q^2 (q <= 2^20) is exact in u64 only below 2^24 summands per row
  for (int r = 0; r <= n_cues; r++)
    if (host_stats[static_cast<size_t>(r) * nf + RELAY_F_N] >= (1ull << 24))
      return fail(RELAY_ERR_INVALID, "table row %d holds >= 2^24 positions/occurrences: its u64 sum of squares "
                  "may have wrapped (split the corpus into tables of < 2^24 positions)", r);
  for (int r = 0; r <= n_cues; r++) {
    const uint64_t* row = host_stats + static_cast<size_t>(r) * nf;
    relay_cue_summary_t& o = out[r];
    const uint64_t n = row[RELAY_F_N];
    const uint64_t s1 = row[RELAY_F_SUM_MQ], s2 = row[RELAY_F_SUM_MQ2];
    o.n = static_cast<int64_t>(n);
    o.n_triggers = static_cast<int64_t>(row[RELAY_F_TRIG]);
    o.n_invalid = static_cast<int64_t>(row[RELAY_F_INVALID]);
    o.selected = 0;
    float mn = INFINITY;
    for (int k = 0; k < world_size; k++) {
      uint32_t bits = static_cast<uint32_t>(row[RELAY_F_MIN0 + k]);
      float f;
      std::memcpy(&f, &bits, sizeof f);
      mn = std::fmin(mn, f);
    }
    if (n == 0) {
      o.mean = o.std = o.se = o.token_mean = o.min = o.low_frac = NAN;
      continue;
    }
    o.mean = static_cast<double>(s1) / (static_cast<double>(n) * Q);
    // n^2 var = n s2 - s1^2, exact in 128-bit integers
    const unsigned __int128 a = static_cast<unsigned __int128>(n) * s2;
    const unsigned __int128 b = static_cast<unsigned __int128>(s1) * s1;
    const unsigned __int128 d = a > b ? a - b : 0;
    const double var = static_cast<double>(d) / (static_cast<double>(n) * static_cast<double>(n) * Q * Q);
    o.std = std::sqrt(var);
    o.se = o.std / std::sqrt(static_cast<double>(n));
    const uint64_t lens = row[RELAY_F_SUM_LEN];
    o.token_mean = lens ? static_cast<double>(row[RELAY_F_SUM_WQ]) / (static_cast<double>(lens) * Q) : NAN;
    o.low_frac = lens ? static_cast<double>(row[RELAY_F_SUM_LOW]) / static_cast<double>(lens) : NAN;
    o.min = mn;
  }
  relay_cue_summary_t& g = out[n_cues];
  if (g.n < 2) {
    g.std = g.se = NAN;
    return RELAY_OK;
  }
  for (int c = 0; c < n_cues; c++) {
    relay_cue_summary_t& o = out[c];
    if (o.n < 1 || o.n < min_count) continue;
    if (rule == 0) o.selected = o.mean >= g.mean + g.se;
    else if (rule == 1) o.selected = o.mean >= g.mean + o.se;
    else if (rule == 2) o.selected = o.mean > g.mean;
    else o.selected = 1;  // rule 3: every candidate with n >= min_count
  }
  return RELAY_OK;
}

relay_status_t relay_step_switch(relay_cueset_t cs, const void* logits, relay_dtype_t dt, int32_t batch,
                                 int64_t vocab, int64_t row_stride, float inv_temperature,
                                 const int32_t* sampled, uint8_t* state, int32_t* hist, int32_t* small_run,
                                 float margin_gate, int32_t max_small_segment, float* margin, int32_t* top1,
                                 int32_t* top2, uint8_t* flag, int16_t* cue_id, void* ws, size_t ws_bytes,
                                 relay_stream_t stream) {
  if (!cs) return fail(RELAY_ERR_INVALID, "cs is NULL");
  if (!valid_dtype(dt)) return fail(RELAY_ERR_INVALID, "unknown dtype");
  if (vocab < 2 || vocab > 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "vocab out of range");
  if (vocab != cs->dev.vocab) return fail(RELAY_ERR_INVALID, "vocab differs from the cue set's");
  if (row_stride < vocab) return fail(RELAY_ERR_INVALID, "row_stride < vocab");
  if (batch < 0) return fail(RELAY_ERR_INVALID, "batch < 0");
  if (static_cast<long long>(batch) * vocab >= (1LL << 51)) return fail(RELAY_ERR_INVALID, "batch * vocab must be < 2^51");
  if (!(inv_temperature > 0.0f) || !std::isfinite(inv_temperature))
    return fail(RELAY_ERR_INVALID, "inv_temperature must be finite and > 0");
  if (max_small_segment < 0) return fail(RELAY_ERR_INVALID, "max_small_segment < 0");
  if (max_small_segment > 0 && !small_run) return fail(RELAY_ERR_INVALID, "small_run required with a budget");
  if (batch == 0) return RELAY_OK;
  if (!logits || !state || !hist || !margin || !flag || !cue_id)
    return fail(RELAY_ERR_INVALID, "logits/state/hist/margin/flag/cue_id are required");
  StepWs w;
  const relay_status_t ws_s = ws_step(ws, ws_bytes, batch, &w);
  if (ws_s != RELAY_OK) return ws_s;
  return cuda_status(launch_step_switch(cs->dev, logits, static_cast<int>(dt), batch, static_cast<int>(vocab),
                                        row_stride, inv_temperature, sampled, state, hist, small_run, margin_gate,
                                        max_small_segment, margin, top1, top2, flag, cue_id, w,
                                        reinterpret_cast<cudaStream_t>(stream)),
                     "relay_step_switch launch");
}

relay_status_t relay_step_sample(relay_cueset_t cs, const void* logits, relay_dtype_t dt, int32_t batch,
                                 int64_t vocab, int64_t row_stride, float inv_temperature, float temperature,
                                 int32_t top_k, float top_p, const float* uniform, uint8_t* state,
                                 int32_t* hist, int32_t* small_run, float margin_gate, int32_t max_small_segment,
                                 float* margin, int32_t* top1, int32_t* top2, int32_t* sampled, uint8_t* flag,
                                 int16_t* cue_id, void* ws, size_t ws_bytes, relay_stream_t stream) {
  if (!cs) return fail(RELAY_ERR_INVALID, "cs is NULL");
  if (!valid_dtype(dt)) return fail(RELAY_ERR_INVALID, "unknown dtype");
  if (vocab < 2 || vocab > 0x7fffffffLL) return fail(RELAY_ERR_INVALID, "vocab out of range");
  if (vocab != cs->dev.vocab) return fail(RELAY_ERR_INVALID, "vocab differs from the cue set's");
  if (row_stride < vocab) return fail(RELAY_ERR_INVALID, "row_stride < vocab");
  if (batch < 0) return fail(RELAY_ERR_INVALID, "batch < 0");
  if (static_cast<long long>(batch) * vocab >= (1LL << 51)) return fail(RELAY_ERR_INVALID, "batch * vocab must be < 2^51");
  if (!(inv_temperature > 0.0f) || !std::isfinite(inv_temperature))
    return fail(RELAY_ERR_INVALID, "inv_temperature must be finite and > 0");
  if (!(temperature > 0.0f) || !std::isfinite(temperature))
    return fail(RELAY_ERR_INVALID, "temperature must be finite and > 0");
  if (top_k < 0 || top_k > kMaxTopK) return fail(RELAY_ERR_INVALID, "top_k must be in [0, %d]", kMaxTopK);
  if (!(top_p > 0.0f && top_p <= 1.0f)) return fail(RELAY_ERR_INVALID, "top_p must be in (0, 1]");
  // no top-k: fixed-point masses are summed in 14-bit digits, each sum < vocab * 2^14 < 2^32
  if (top_k == 0 && vocab >= (1LL << 18)) return fail(RELAY_ERR_UNSUPPORTED, "top_k = 0 needs vocab < 2^18");
  if (max_small_segment < 0) return fail(RELAY_ERR_INVALID, "max_small_segment < 0");
  if (max_small_segment > 0 && !small_run) return fail(RELAY_ERR_INVALID, "small_run required with a budget");
  if (batch == 0) return RELAY_OK;
  if (!logits || !state || !hist || !margin || !flag || !cue_id || !uniform || !sampled)
    return fail(RELAY_ERR_INVALID, "logits/state/hist/margin/flag/cue_id/uniform/sampled are required");
  StepWs w;
  const relay_status_t ws_s = ws_step(ws, ws_bytes, batch, &w);
  if (ws_s != RELAY_OK) return ws_s;
  const int k = static_cast<int>(top_k < vocab ? top_k : vocab);  // 0: no top-k
  return cuda_status(launch_step_sample(cs->dev, logits, static_cast<int>(dt), batch, static_cast<int>(vocab),
                                        row_stride, inv_temperature, temperature, k, top_p, uniform, state,
                                        hist, small_run, margin_gate, max_small_segment, margin, top1, top2,
                                        sampled, flag, cue_id, w, reinterpret_cast<cudaStream_t>(stream)),
                     "relay_step_sample launch");
}

}  // extern "C"
