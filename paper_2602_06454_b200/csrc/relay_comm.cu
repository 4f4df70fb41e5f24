// relay_comm.cu — H6: the one cross-GPU exchange of the path, a SUM
// all-reduce of the integer statistics table(s) over NCCL (NVLink / NVSwitch;
// NVLS in-switch reduction when NCCL picks it).  The path shards by
// trajectory (P:377-378 calibration traces are independent), so nothing else
// is exchanged.  NCCL is resolved at run time (dlopen "libnccl.so.2"): in a
// process that already loaded torch's NCCL the soname matches that library,
// so a communicator torch created (ProcessGroupNCCL._comm_ptr) is usable here.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "../../include/relay.h"
#include "relay_internal.h"

namespace relay {
relay_status_t fail(relay_status_t s, const char* fmt, ...);
}

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(dlsym(h, "ncclGetVersion"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.error_string;
  });
  return api;
}

relay_status_t nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return RELAY_OK;
  return relay::fail(RELAY_ERR_NCCL, "%s: %s", what, nccl().error_string(r));
}

}  // namespace

extern "C" {

relay_status_t relay_nccl_version(int32_t* version, char* path, int32_t path_len) {
  if (!version) return relay::fail(RELAY_ERR_INVALID, "version is NULL");
  const NcclApi& a = nccl();
  if (!a.ok || !a.get_version) return relay::fail(RELAY_ERR_NCCL, "libnccl.so.2 not loadable");
  int v = 0;
  relay_status_t s = nccl_status(a.get_version(&v), "ncclGetVersion");
  if (s != RELAY_OK) return s;
  *version = v;
  if (path && path_len > 0) {
    Dl_info info{};
    path[0] = 0;
    if (dladdr(reinterpret_cast<void*>(a.all_reduce), &info) && info.dli_fname) {
      std::strncpy(path, info.dli_fname, static_cast<size_t>(path_len) - 1);
      path[path_len - 1] = 0;
    }
  }
  return RELAY_OK;
}

relay_status_t relay_nccl_unique_id(uint8_t* id_out) {
  if (!id_out) return relay::fail(RELAY_ERR_INVALID, "id_out is NULL");
  const NcclApi& a = nccl();
  if (!a.ok) return relay::fail(RELAY_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  relay_status_t s = nccl_status(a.get_unique_id(&id), "ncclGetUniqueId");
  if (s == RELAY_OK) std::memcpy(id_out, id.internal, RELAY_NCCL_ID_BYTES);
  return s;
}

relay_status_t relay_nccl_comm_init(const uint8_t* id, int32_t world_size, int32_t rank, void** comm) {
  if (!id || !comm) return relay::fail(RELAY_ERR_INVALID, "id and comm are required");
  if (world_size < 1 || rank < 0 || rank >= world_size)
    return relay::fail(RELAY_ERR_INVALID, "bad rank/world_size");
  const NcclApi& a = nccl();
  if (!a.ok) return relay::fail(RELAY_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, RELAY_NCCL_ID_BYTES);
  ncclComm_t c = nullptr;
  relay_status_t s = nccl_status(a.comm_init_rank(&c, world_size, uid, rank), "ncclCommInitRank");
  *comm = (s == RELAY_OK) ? static_cast<void*>(c) : nullptr;
  return s;
}

relay_status_t relay_nccl_comm_destroy(void* comm) {
  if (!comm) return RELAY_OK;
  const NcclApi& a = nccl();
  if (!a.ok) return relay::fail(RELAY_ERR_NCCL, "libnccl.so.2 not loadable");
  return nccl_status(a.comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

relay_status_t relay_stats_allreduce(void* nccl_comm, uint64_t* stats, int32_t n_tables, int32_t n_cues,
                                     int32_t world_size, relay_stream_t stream) {
  if (!nccl_comm || !stats) return relay::fail(RELAY_ERR_INVALID, "nccl_comm and stats are required");
  if (n_tables < 1) return relay::fail(RELAY_ERR_INVALID, "n_tables < 1");
  const size_t words = relay_stats_words(n_cues, world_size);
  if (words == 0 || n_cues < 1) return relay::fail(RELAY_ERR_INVALID, "bad n_cues/world_size");
  const NcclApi& a = nccl();
  if (!a.ok) return relay::fail(RELAY_ERR_NCCL, "libnccl.so.2 not loadable");
  // in place; uint64 addition (every bound in relay.h keeps the true sums < 2^64)
  return nccl_status(a.all_reduce(stats, stats, words * static_cast<size_t>(n_tables), ncclUint64, ncclSum,
                                  static_cast<ncclComm_t>(nccl_comm), reinterpret_cast<cudaStream_t>(stream)),
                     "ncclAllReduce");
}

// ------------------------------------------- N1 fused over peer memory

relay_status_t relay_tp_exchange_create(int32_t rank, int32_t world_size, int64_t rows_cap, uint8_t* ipc_handle_out,
                                        relay_tp_exchange_t* out) {
  if (!out || !ipc_handle_out) return relay::fail(RELAY_ERR_INVALID, "out and ipc_handle_out are required");
  *out = nullptr;
  if (world_size < 1 || world_size > relay::kMaxTpRanks || rank < 0 || rank >= world_size)
    return relay::fail(RELAY_ERR_INVALID, "world_size must be in [1, %d] and rank in [0, world_size)",
                       relay::kMaxTpRanks);
  if (rows_cap < 1 || rows_cap > (1LL << 31)) return relay::fail(RELAY_ERR_INVALID, "rows_cap must be in [1, 2^31]");
  auto* x = new relay_tp_exchange_s();
  cudaGetDevice(&x->device);
  const size_t bytes = sizeof(float) * 8 * 2 * static_cast<size_t>(world_size) * static_cast<size_t>(rows_cap);
  cudaError_t e = cudaMalloc(&x->own, bytes);
  if (e == cudaSuccess) e = cudaMemset(x->own, 0, bytes);  // tag 0 never matches a call's tag (>= 1)
  if (e == cudaSuccess) e = cudaMalloc(&x->counters, 2 * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(x->counters, 0, 2 * sizeof(int));
  cudaIpcMemHandle_t h{};
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, x->own);
  if (e != cudaSuccess) {
    if (x->own) cudaFree(x->own);
    if (x->counters) cudaFree(x->counters);
    delete x;
    return relay::fail(e == cudaErrorMemoryAllocation ? RELAY_ERR_ALLOC : RELAY_ERR_CUDA,
                       "relay_tp_exchange_create: %s", cudaGetErrorString(e));
  }
  std::memcpy(ipc_handle_out, &h, RELAY_IPC_HANDLE_BYTES);
  x->pe.world = world_size;
  x->pe.rank = rank;
  x->pe.rows_cap = rows_cap;
  x->pe.epoch = x->counters;
  x->pe.done = x->counters + 1;
  x->pe.recv[rank] = x->own;
  *out = x;
  return RELAY_OK;
}

relay_status_t relay_tp_exchange_connect(relay_tp_exchange_t x, const uint8_t* ipc_handles) {
  if (!x || !ipc_handles) return relay::fail(RELAY_ERR_INVALID, "x and ipc_handles are required");
  for (int k = 0; k < x->pe.world; k++) {
    if (k == x->pe.rank || x->opened[k]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handles + static_cast<size_t>(k) * RELAY_IPC_HANDLE_BYTES, RELAY_IPC_HANDLE_BYTES);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return relay::fail(RELAY_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", k, cudaGetErrorString(e));
    x->pe.recv[k] = static_cast<float*>(p);
    x->opened[k] = true;
  }
  return RELAY_OK;
}

relay_status_t relay_tp_exchange_destroy(relay_tp_exchange_t x) {
  if (!x) return RELAY_OK;
  for (int k = 0; k < x->pe.world; k++)
    if (x->opened[k]) cudaIpcCloseMemHandle(x->pe.recv[k]);
  cudaFree(x->own);
  cudaFree(x->counters);
  delete x;
  return RELAY_OK;
}

relay_status_t relay_margin_rows_tp(relay_tp_exchange_t x, const void* logits, relay_dtype_t dt, int64_t n_rows,
                                    int64_t shard_vocab, int64_t row_stride, int64_t col_offset,
                                    float inv_temperature, float* margin, int32_t* top1, int32_t* top2, float* lse,
                                    uint8_t* row_status, relay_stream_t stream) {
  if (!x) return relay::fail(RELAY_ERR_INVALID, "x is NULL");
  for (int k = 0; k < x->pe.world; k++)
    if (!x->pe.recv[k]) return relay::fail(RELAY_ERR_INVALID, "exchange not connected (rank %d)", k);
  if (dt != RELAY_DT_BF16 && dt != RELAY_DT_F16 && dt != RELAY_DT_F32)
    return relay::fail(RELAY_ERR_INVALID, "unknown dtype %d", static_cast<int>(dt));
  if (shard_vocab < 1) return relay::fail(RELAY_ERR_INVALID, "shard_vocab must be >= 1");
  if (col_offset < 0 || col_offset + shard_vocab >= 0x7fffffffLL)
    return relay::fail(RELAY_ERR_INVALID, "col_offset out of range");
  if (shard_vocab * (dt == RELAY_DT_F32 ? 4 : 2) >= 0x7fffffffLL)
    return relay::fail(RELAY_ERR_INVALID, "row bytes must be < 2^31");
  if (row_stride < shard_vocab) return relay::fail(RELAY_ERR_INVALID, "row_stride < shard_vocab");
  if (n_rows < 0 || n_rows > x->pe.rows_cap) return relay::fail(RELAY_ERR_INVALID, "n_rows must be in [0, rows_cap]");
  if (!(inv_temperature > 0.0f) || !(inv_temperature < INFINITY))
    return relay::fail(RELAY_ERR_INVALID, "inv_temperature must be finite and > 0");
  if (n_rows > 0 && (!logits || !margin)) return relay::fail(RELAY_ERR_INVALID, "logits and margin are required");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = relay::launch_margin_partials_p2p(logits, static_cast<int>(dt), n_rows, static_cast<int>(shard_vocab),
                                                    row_stride, col_offset, inv_temperature, x->pe, st);
  if (e == cudaSuccess)
    e = relay::launch_margin_combine_p2p(x->pe, n_rows, inv_temperature, margin, top1, top2, lse, row_status, st);
  if (e != cudaSuccess) return relay::fail(RELAY_ERR_CUDA, "relay_margin_rows_tp launch: %s", cudaGetErrorString(e));
  return RELAY_OK;
}

relay_status_t relay_stats_allreduce_p2p(relay_tp_exchange_t x, uint64_t* stats, int32_t n_tables, int32_t n_cues,
                                         int32_t world_size, relay_stream_t stream) {
  if (!x || !stats) return relay::fail(RELAY_ERR_INVALID, "x and stats are required");
  if (n_tables < 1) return relay::fail(RELAY_ERR_INVALID, "n_tables < 1");
  if (world_size != x->pe.world) return relay::fail(RELAY_ERR_INVALID, "world_size differs from the exchange's");
  const size_t words = relay_stats_words(n_cues, world_size) * static_cast<size_t>(n_tables);
  if (words == 0 || n_cues < 1) return relay::fail(RELAY_ERR_INVALID, "bad n_cues/world_size");
  // a slot is rows_cap x 32 B: the table plus one tag word must fit
  if (static_cast<long long>(words) * 8 + 8 > x->pe.rows_cap * 32)
    return relay::fail(RELAY_ERR_INVALID, "exchange slots hold %lld B, the table needs %zu B + 8",
                       x->pe.rows_cap * 32, words * 8);
  for (int k = 0; k < x->pe.world; k++)
    if (!x->pe.recv[k]) return relay::fail(RELAY_ERR_INVALID, "exchange not connected (rank %d)", k);
  const cudaError_t e = relay::launch_stats_allreduce_p2p(x->pe, reinterpret_cast<unsigned long long*>(stats),
                                                          static_cast<long long>(words),
                                                          reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return relay::fail(RELAY_ERR_CUDA, "relay_stats_allreduce_p2p launch: %s", cudaGetErrorString(e));
  return RELAY_OK;
}

}  // extern "C"
