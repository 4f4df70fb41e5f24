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

}  // extern "C"
