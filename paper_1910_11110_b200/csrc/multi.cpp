// Multi-GPU plumbing of the trace path: traces are independent
// (SPEC.md:158-159, 543 -- "independent runs may execute concurrently with no shared
// state"), so each device owns a contiguous trace-id shard and the only exchange is ONE
// sum-allreduce of the COH_N_COUNTERS uint64 counter vector over NVLink/NVSwitch.
//
// NCCL is bound at run time (dlopen of libnccl.so.2, preferring a copy already mapped into
// the process, e.g. by torch) so that the library loads on hosts without NCCL; every NCCL
// failure comes back as COH_E_NCCL with the NCCL error string in coh_last_error.
//
//   coh_comm_unique_id / coh_comm_init_rank : one process per GPU (the bench's torchrun
//                                             ranks), ncclCommInitRank
//   coh_comm_init_all                       : one process driving n devices, ncclCommInitAll
//   coh_comm_allreduce_counters             : the exchange (ncclUint64, ncclSum), stream-ordered
//   coh_eval_traces_multi                   : per-device counted evaluation + the grouped
//                                             allreduce, all enqueued on the callers' streams
//   coh_shard_split / coh_counters_host     : host-side shard arithmetic and the counter vector
//                                             of a host result batch (no GPU needed)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"

namespace {

struct NcclApi {
  void* so = nullptr;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& nccl_state() {
  static NcclApi api;
  return api;
}

const NcclApi* nccl() {
  NcclApi& api = nccl_state();
  static std::once_flag once;
  std::call_once(once, [&api] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {  // an already-mapped copy first (same library as torch's)
      if ((api.so = dlopen(n, RTLD_NOW | RTLD_NOLOAD))) break;
    }
    if (!api.so)
      for (const char* n : names)
        if ((api.so = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    if (!api.so) {
      api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&api](const char* s) { return dlsym(api.so, s); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommInitAll || !api.CommDestroy || !api.AllReduce ||
        !api.GroupStart || !api.GroupEnd || !api.GetErrorString) {
      api.why = "libnccl.so.2 lacks a required symbol";
      api.so = nullptr;
    }
  });
  return api.so ? &api : nullptr;
}

std::string nccl_why() {
  nccl();
  return nccl_state().why;
}

}  // namespace

struct coh_comm {
  coh_ctx* ctx = nullptr;  // the device context this rank evaluates on
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
  std::string err;
};

namespace {

int nccl_fail(coh_ctx* ctx, const char* what, ncclResult_t r) {
  const NcclApi* api = nccl();
  if (ctx) ctx->err = std::string(what) + ": " + (api ? api->GetErrorString(r) : "NCCL unavailable");
  return COH_E_NCCL;
}

int no_nccl(coh_ctx* ctx) {
  if (ctx) ctx->err = "NCCL unavailable: " + nccl_why();
  return COH_E_NCCL;
}

}  // namespace

extern "C" {

int coh_nccl_version(int* version) {
  const NcclApi* api = nccl();
  if (!api || !version) return COH_E_NCCL;
  if (!api->GetVersion) return COH_E_NCCL;
  return api->GetVersion(version) == ncclSuccess ? COH_OK : COH_E_NCCL;
}

int coh_comm_unique_id(uint8_t id[COH_COMM_ID_BYTES]) {
  const NcclApi* api = nccl();
  if (!id) return COH_E_ARG;
  if (!api) return COH_E_NCCL;
  ncclUniqueId u;
  if (api->GetUniqueId(&u) != ncclSuccess) return COH_E_NCCL;
  static_assert(sizeof u == COH_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof u);
  return COH_OK;
}

int coh_comm_init_rank(coh_ctx* ctx, const uint8_t id[COH_COMM_ID_BYTES], int world, int rank, coh_comm** out) {
  if (!ctx || !id || !out || world < 1 || rank < 0 || rank >= world) return COH_E_ARG;
  *out = nullptr;
  const NcclApi* api = nccl();
  if (!api) return no_nccl(ctx);
  if (cudaSetDevice(ctx->device) != cudaSuccess) {
    ctx->err = "cudaSetDevice failed";
    return COH_E_CUDA;
  }
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  coh_comm* c = new coh_comm();
  c->ctx = ctx;
  c->world = world;
  c->rank = rank;
  ncclResult_t r = api->CommInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(ctx, "ncclCommInitRank", r);
  }
  *out = c;
  return COH_OK;
}

int coh_comm_init_all(coh_ctx* const* ctxs, int n_dev, coh_comm** comms) {
  if (!ctxs || !comms || n_dev < 1) return COH_E_ARG;
  for (int d = 0; d < n_dev; ++d) {
    if (!ctxs[d]) return COH_E_ARG;
    comms[d] = nullptr;
  }
  const NcclApi* api = nccl();
  if (!api) return no_nccl(ctxs[0]);
  std::vector<int> devs(n_dev);
  for (int d = 0; d < n_dev; ++d) devs[d] = ctxs[d]->device;
  std::vector<ncclComm_t> raw(n_dev, nullptr);
  ncclResult_t r = api->CommInitAll(raw.data(), n_dev, devs.data());
  if (r != ncclSuccess) return nccl_fail(ctxs[0], "ncclCommInitAll", r);
  for (int d = 0; d < n_dev; ++d) {
    comms[d] = new coh_comm();
    comms[d]->ctx = ctxs[d];
    comms[d]->comm = raw[d];
    comms[d]->world = n_dev;
    comms[d]->rank = d;
  }
  return COH_OK;
}

void coh_comm_destroy(coh_comm* c) {
  if (!c) return;
  const NcclApi* api = nccl();
  if (api && c->comm) api->CommDestroy(c->comm);
  delete c;
}

int coh_comm_allreduce_counters(coh_comm* c, uint64_t* d_counters, void* stream) {
  if (!c || !d_counters) return COH_E_ARG;
  const NcclApi* api = nccl();
  if (!api) return no_nccl(c->ctx);
  ncclResult_t r = api->AllReduce(d_counters, d_counters, COH_N_COUNTERS, ncclUint64, ncclSum, c->comm,
                                  static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? COH_OK : nccl_fail(c->ctx, "ncclAllReduce", r);
}

int coh_eval_traces_multi(coh_comm* const* comms, int n_dev, const coh_trace_batch* shards,
                          coh_trace_result* const* d_results, uint32_t* const* d_boundary,
                          uint64_t* const* d_counters, void* const* streams) {
  if (!comms || n_dev < 1 || !shards || !d_results || !d_counters || !streams) return COH_E_ARG;
  for (int d = 0; d < n_dev; ++d)
    if (!comms[d] || !comms[d]->ctx || !d_counters[d]) return COH_E_ARG;
  const NcclApi* api = nccl();
  if (!api) return no_nccl(comms[0]->ctx);
  // 1) every shard's counted evaluation, each on its own device and stream
  for (int d = 0; d < n_dev; ++d) {
    coh_ctx* ctx = comms[d]->ctx;
    if (cudaSetDevice(ctx->device) != cudaSuccess) {
      ctx->err = "cudaSetDevice failed";
      return COH_E_CUDA;
    }
    const int rc = coh_eval_traces_counted(ctx, &shards[d], d_results[d], d_boundary ? d_boundary[d] : nullptr,
                                           d_counters[d], streams[d]);
    if (rc) return rc;
  }
  // 2) the one exchange: a grouped allreduce (one process, n communicators)
  ncclResult_t r = api->GroupStart();
  if (r != ncclSuccess) return nccl_fail(comms[0]->ctx, "ncclGroupStart", r);
  for (int d = 0; d < n_dev; ++d) {
    r = api->AllReduce(d_counters[d], d_counters[d], COH_N_COUNTERS, ncclUint64, ncclSum, comms[d]->comm,
                       static_cast<cudaStream_t>(streams[d]));
    if (r != ncclSuccess) {
      api->GroupEnd();
      return nccl_fail(comms[d]->ctx, "ncclAllReduce", r);
    }
  }
  r = api->GroupEnd();
  return r == ncclSuccess ? COH_OK : nccl_fail(comms[0]->ctx, "ncclGroupEnd", r);
}

int coh_shard_split(uint32_t rank, uint32_t world, uint64_t total, uint64_t* first, uint64_t* count) {
  if (!first || !count || world == 0 || rank >= world) return COH_E_ARG;
  const uint64_t base = total / world, extra = total % world;
  *first = rank * base + (rank < extra ? rank : extra);
  *count = base + (rank < extra ? 1u : 0u);
  return COH_OK;
}

int coh_counters_host(const coh_trace_result* results, uint64_t n_traces, uint64_t* counters) {
  if (!counters || (n_traces && !results)) return COH_E_ARG;
  std::memset(counters, 0, sizeof(uint64_t) * COH_N_COUNTERS);
  for (uint64_t t = 0; t < n_traces; ++t) {
    const coh_trace_result& r = results[t];
    counters[0] += r.status == COH_RUN_STUCK;
    counters[1] += r.status == COH_RUN_FUEL_EXHAUSTED;
    counters[2] += r.violations > 0;
    counters[3] += r.status == COH_RUN_DEFECT;
    counters[4] += r.steps;
    counters[5] += r.transfers;
    counters[6] += r.transfer_bytes;
    counters[7] += r.violations;
    counters[8] += r.calls_done;
    counters[9] += 1;
    counters[10] += (r.stuck_flags & COH_FLAG_UNSAFE) != 0;
  }
  return COH_OK;
}

}  // extern "C"
