// C ABI of the trace evaluator: context, validation, launch geometry, host-buffer
// pipeline.  The reference equivalent is the by-value C++ API of namespace cohere
// (semantics.hpp:253 run, modes.hpp:105 run_annotated); errors that the reference
// throws come back here as status codes + coh_last_error.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gen_common.h"
#include "internal.hpp"

namespace {

int cuda_fail(coh_ctx* ctx, cudaError_t e, const char* what) {
  if (ctx) ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
  return COH_E_CUDA;
}
#define COH_CUDA(ctx, call)                                   \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

int arg_fail(coh_ctx* ctx, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return COH_E_ARG;
}

int validate(coh_ctx* ctx, const coh_trace_batch* b) {
  if (!ctx) return COH_E_ARG;
  if (!b) return arg_fail(ctx, "batch is NULL");
  if (b->n_arrays < 1 || b->n_arrays > COH_MAX_ARRAYS)
    return arg_fail(ctx, "n_arrays must be in [1, 64], got " + std::to_string(b->n_arrays));
  if (b->n_traces && b->n_calls && !b->records) return arg_fail(ctx, "records is NULL");
  if (b->flags & ~(COH_BATCH_BLOCKS | COH_BATCH_PACKED12 | COH_BATCH_OVERLAP)) return arg_fail(ctx, "unknown batch flags");
  if ((b->flags & COH_BATCH_BLOCKS) && (b->flags & COH_BATCH_PACKED12))
    return arg_fail(ctx, "COH_BATCH_PACKED12 records cannot carry COH_REC_CONT");
  return COH_OK;
}

// Uniform element sizes let the kernel fold bytes = transfers * size; otherwise it sums
// the per-array transfer counters (26-bit) times the per-array sizes.
int bytes_mode(coh_ctx* ctx, const coh_trace_batch* b, bool* uniform, uint64_t* ub) {
  *uniform = true;
  *ub = 1;
  if (!b->array_bytes) return COH_OK;
  *ub = b->array_bytes[0];
  for (uint32_t a = 1; a < b->n_arrays; ++a)
    if (b->array_bytes[a] != *ub) *uniform = false;
  if (!*uniform && (uint64_t)b->n_calls * 2u >= (1u << 26))
    return arg_fail(ctx, "non-uniform array_bytes supports n_calls < 2^25");
  return COH_OK;
}

int eval_device(coh_ctx* ctx, const coh_trace_batch* b, const uint16_t* d_records,
                uint64_t n_traces, coh_trace_result* d_results, uint32_t* d_boundary,
                cudaStream_t s, uint64_t* d_counters = nullptr) {
  bool uniform;
  uint64_t ub;
  int rc = bytes_mode(ctx, b, &uniform, &ub);
  if (rc) return rc;
  if (n_traces == 0) return COH_OK;
  // non-uniform sizes: a stream-ordered copy private to this launch (launches of one
  // context on different streams may run concurrently, so no per-context buffer)
  uint64_t* d_bytes = nullptr;
  if (!uniform) {
    COH_CUDA(ctx, cudaMallocAsync(reinterpret_cast<void**>(&d_bytes), sizeof(uint64_t) * COH_MAX_ARRAYS, s));
    COH_CUDA(ctx, cudaMemcpyAsync(d_bytes, b->array_bytes, sizeof(uint64_t) * b->n_arrays,
                                  cudaMemcpyHostToDevice, s));
  }
  cohb::TraceLaunch L;
  L.records = d_records;
  L.n_traces = n_traces;
  L.n_calls = b->n_calls;
  L.n_arrays = b->n_arrays;
  L.fuel = b->fuel;
  // fuel >= 6 steps x n_calls can never run out (max 6 steps per block): drop the check
  L.check_fuel = (int64_t)b->fuel < 6 * (int64_t)b->n_calls;
  L.uniform_bytes = uniform;
  L.bytes_uniform = ub;
  L.d_array_bytes = d_bytes;
  L.d_lut = ctx->d_lut;
  L.d_slow = ctx->d_slow;
  L.results = d_results;
  L.boundary = d_boundary;
  L.counters = d_counters;
  L.sms = ctx->sms;  // the launcher sizes a persistent grid for the chosen variant
  // the launch's ticket and counter sums: the next slot of the context's ring, private
  // to this launch (launches of one context on different streams may run concurrently);
  // long launches (more than five rounds of traces per thread) hand out trace batches
  L.slot = ctx->d_slots + (ctx->slot_next.fetch_add(1u, std::memory_order_relaxed) % cohb::kLaunchSlots);
  L.dynamic = n_traces > 5ull * 1024ull * (uint64_t)ctx->sms;
  L.overlap = (b->flags & COH_BATCH_OVERLAP) && uniform;
  L.flags = b->flags;
  std::string err;
  rc = (b->flags & COH_BATCH_BLOCKS) ? cohb::launch_trace_blocks(L, s, &err) : cohb::launch_trace_eval(L, s, &err);
  if (d_bytes) cudaFreeAsync(d_bytes, s);
  if (rc) {
    ctx->err = err;
    return rc;
  }
  ctx->launches++;
  return COH_OK;
}

}  // namespace

extern "C" {

const char* coh_version(void) { return "cohere-b200 0.1 (sm_100a)"; }

int coh_ctx_create(int device, coh_ctx** out) {
  if (!out) return COH_E_ARG;
  *out = nullptr;
  coh_ctx* ctx = new coh_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return COH_E_CUDA;
  }
  static cohb::CallTable table;  // pure function of the rules; rebuilt per ctx
  cohb::build_call_table(&table);
  int rc = COH_OK;
  do {
    if ((e = cudaMalloc(&ctx->d_lut, sizeof table.lut)) != cudaSuccess) break;
    if ((e = cudaMalloc(&ctx->d_slow, sizeof table.slow)) != cudaSuccess) break;
    if ((e = cudaMemcpy(ctx->d_lut, table.lut, sizeof table.lut, cudaMemcpyHostToDevice)) != cudaSuccess) break;
    if ((e = cudaMemcpy(ctx->d_slow, table.slow, sizeof table.slow, cudaMemcpyHostToDevice)) != cudaSuccess) break;
    if ((e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) break;
    if ((e = cudaMalloc(&ctx->d_slots, sizeof(cohb::LaunchSlot) * cohb::kLaunchSlots)) != cudaSuccess) break;
    if ((e = cudaMemset(ctx->d_slots, 0, sizeof(cohb::LaunchSlot) * cohb::kLaunchSlots)) != cudaSuccess) break;
    {  // stream-ordered scratch (cudaMallocAsync) stays in the pool instead of being unmapped at every sync
      cudaMemPool_t pool;
      uint64_t keep = ~0ull;
      if ((e = cudaDeviceGetDefaultMemPool(&pool, device)) != cudaSuccess) break;
      if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) break;
    }
    if ((e = cohb::runs_ctx_init(ctx->sms, &ctx->runs_grid)) != cudaSuccess) break;
    if ((e = cohb::elem_ctx_init()) != cudaSuccess) break;
    int tpb = 0;
    std::string err;
    rc = cohb::trace_eval_occupancy(&ctx->blocks_per_sm, &tpb, 256, &err);
  } while (0);
  if (e != cudaSuccess || rc != COH_OK) {
    coh_ctx_destroy(ctx);
    return COH_E_CUDA;
  }
  *out = ctx;
  return COH_OK;
}

void coh_ctx_destroy(coh_ctx* ctx) {
  if (!ctx) return;
  cudaFree(ctx->d_lut);
  cudaFree(ctx->d_slow);
  cudaFree(ctx->d_slots);
  for (int k = 0; k < 2; ++k) {
    cudaFree(ctx->d_pk[k]);
    cudaFree(ctx->d_rec[k]);
    cudaFree(ctx->d_res[k]);
    cudaFree(ctx->d_bnd[k]);
    if (ctx->hs[k]) cudaStreamDestroy(ctx->hs[k]);
  }
  delete ctx;
}

const char* coh_last_error(const coh_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

uint64_t coh_launch_count(const coh_ctx* ctx) { return ctx ? ctx->launches : 0; }

void* coh_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}
void coh_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int coh_gen_records(coh_ctx* ctx, uint64_t seed, uint64_t trace0, uint64_t n_traces,
                    uint32_t n_calls, uint32_t n_arrays, uint32_t adv_per1024,
                    uint16_t* d_records, void* stream) {
  if (!ctx) return COH_E_ARG;
  if (n_arrays < 1 || n_arrays > COH_MAX_ARRAYS) return arg_fail(ctx, "n_arrays must be in [1, 64]");
  if (!d_records && n_traces && n_calls) return arg_fail(ctx, "d_records is NULL");
  std::string err;
  int rc = cohb::launch_gen_records(seed, trace0, n_traces, n_calls, n_arrays, adv_per1024,
                                    d_records, stream, &err);
  if (rc) ctx->err = err;
  else ctx->launches++;
  return rc;
}

int coh_gen_records_blocks(coh_ctx* ctx, uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                           uint32_t n_arrays, uint32_t adv_per1024, uint32_t cont_per1024, uint16_t* d_records,
                           void* stream) {
  int rc = coh_gen_records(ctx, seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, d_records, stream);
  if (rc) return rc;
  std::string err;
  rc = cohb::launch_gen_blocks(seed, trace0, n_traces, n_calls, cont_per1024, d_records, stream, &err);
  if (rc) ctx->err = err;
  else if (cont_per1024 && n_traces && n_calls) ctx->launches++;
  return rc;
}

int coh_gen_records_blocks_host(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                                uint32_t n_arrays, uint32_t adv_per1024, uint32_t cont_per1024, uint16_t* h_records) {
  const int rc = coh_gen_records_host(seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, h_records);
  if (rc || !cont_per1024) return rc;
  for (uint64_t t = 0; t < n_traces; ++t) {
    uint64_t in_block = 0;
    for (uint32_t i = 0; i < n_calls; ++i) {
      uint16_t& r = h_records[((uint64_t)(i / 8u) * n_traces + t) * 8u + i % 8u];
      const uint64_t bit = 1ull << COH_REC_ARRAY(r);
      if (i > 0 && !(in_block & bit) && coh_gen_cont(seed, trace0 + t, i, cont_per1024)) {
        r = (uint16_t)(r | COH_REC_CONT);
        in_block |= bit;
      } else {
        in_block = bit;
      }
    }
  }
  return COH_OK;
}

int coh_pack_records12(const uint16_t* records, uint64_t n_traces, uint32_t n_calls, uint8_t* out) {
  if ((n_traces && n_calls) && (!records || !out)) return COH_E_ARG;
  const uint64_t chunks = (uint64_t)((n_calls + 7u) / 8u) * n_traces;
  for (uint64_t q = 0; q < chunks; ++q) {
    uint32_t w[3] = {0u, 0u, 0u};
    for (uint32_t k = 0; k < 8; ++k) {
      const uint16_t r = records[q * 8u + k];
      const uint64_t v = ((uint64_t)COH_REC_ARRAY(r) << 6) | COH_REC_TYPE(r);
      const uint32_t bit = 12u * k;
      w[bit >> 5] |= (uint32_t)(v << (bit & 31u));
      if ((bit & 31u) > 20u) w[(bit >> 5) + 1] |= (uint32_t)(v >> (32u - (bit & 31u)));
    }
    std::memcpy(out + q * 12u, w, 12);
  }
  return COH_OK;
}

int coh_gen_records_host(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                         uint32_t n_arrays, uint32_t adv_per1024, uint16_t* h_records) {
  if (n_arrays < 1 || n_arrays > COH_MAX_ARRAYS) return COH_E_ARG;
  if (!h_records && n_traces && n_calls) return COH_E_ARG;
  const uint32_t n_chunks = (n_calls + 7u) / 8u;
  for (uint32_t c = 0; c < n_chunks; ++c)
    for (uint64_t t = 0; t < n_traces; ++t)
      for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t i = c * 8u + k;
        h_records[((uint64_t)c * n_traces + t) * 8u + k] =
            i < n_calls ? coh_gen_record(seed, trace0 + t, i, n_arrays, adv_per1024) : 0;
      }
  return COH_OK;
}

int coh_eval_traces(coh_ctx* ctx, const coh_trace_batch* batch, coh_trace_result* d_results,
                    uint32_t* d_boundary, void* stream) {
  int rc = validate(ctx, batch);
  if (rc) return rc;
  if (batch->flags & COH_BATCH_PACKED12) return arg_fail(ctx, "COH_BATCH_PACKED12 is for coh_eval_traces_host");
  if (batch->n_traces && !d_results) return arg_fail(ctx, "d_results is NULL");
  return eval_device(ctx, batch, batch->records, batch->n_traces, d_results, d_boundary,
                     static_cast<cudaStream_t>(stream));
}

int coh_eval_traces_counted(coh_ctx* ctx, const coh_trace_batch* batch, coh_trace_result* d_results,
                            uint32_t* d_boundary, uint64_t* d_counters, void* stream) {
  int rc = validate(ctx, batch);
  if (rc) return rc;
  if (batch->flags & COH_BATCH_PACKED12) return arg_fail(ctx, "COH_BATCH_PACKED12 is for coh_eval_traces_host");
  if (batch->n_traces && !d_results) return arg_fail(ctx, "d_results is NULL");
  if (!d_counters) return arg_fail(ctx, "d_counters is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (batch->n_traces == 0) {
    COH_CUDA(ctx, cudaMemsetAsync(d_counters, 0, sizeof(uint64_t) * COH_N_COUNTERS, s));
    return COH_OK;
  }
  return eval_device(ctx, batch, batch->records, batch->n_traces, d_results, d_boundary, s, d_counters);
}

int coh_eval_traces_host(coh_ctx* ctx, const coh_trace_batch* batch, coh_trace_result* h_results,
                         uint32_t* h_boundary) {
  int rc = validate(ctx, batch);
  if (rc) return rc;
  const uint64_t n = batch->n_traces;
  if (n == 0) return COH_OK;
  if (!h_results) return arg_fail(ctx, "h_results is NULL");
  const uint32_t n_chunks = (batch->n_calls + 7u) / 8u;
  const uint32_t n_words = coh_boundary_words(batch->n_calls);
  const bool packed = batch->flags & COH_BATCH_PACKED12;
  coh_trace_batch dev_batch = *batch;  // what the device sees after unpacking
  // (no COH_BATCH_OVERLAP here: a slice's kernel reads what the copy / unpack before it wrote)
  dev_batch.flags &= ~(COH_BATCH_PACKED12 | COH_BATCH_OVERLAP);
  // Slices of S traces: H2D of slice k+1 overlaps the kernel and D2H of slice k.
  static const uint64_t slice = [] {  // COH_HOST_SLICE: traces per slice (A/B timing)
    const char* v = std::getenv("COH_HOST_SLICE");
    const unsigned long long x = v ? std::strtoull(v, nullptr, 10) : 0ull;
    return x >= 1024ull ? (uint64_t)x : (uint64_t)(1ull << 16);  // 64K: measured 7.63 vs 7.70 ms (128K) per 1M
  }();
  uint64_t S = std::min<uint64_t>(n, slice);
  const size_t rec_b = (size_t)n_chunks * 16u * S, res_b = sizeof(coh_trace_result) * S,
               bnd_b = (size_t)n_words * 4u * S, pk_b = (size_t)n_chunks * 12u * S;
  for (int k = 0; k < 2; ++k) {
    if (!ctx->hs[k]) COH_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->hs[k], cudaStreamNonBlocking));
    if (ctx->rec_cap < rec_b) {
      cudaFree(ctx->d_rec[k]);
      COH_CUDA(ctx, cudaMalloc(&ctx->d_rec[k], std::max<size_t>(rec_b, 16)));
    }
    if (packed && ctx->pk_cap < pk_b) {
      cudaFree(ctx->d_pk[k]);
      COH_CUDA(ctx, cudaMalloc(&ctx->d_pk[k], std::max<size_t>(pk_b, 16)));
    }
    if (ctx->res_cap < res_b) {
      cudaFree(ctx->d_res[k]);
      COH_CUDA(ctx, cudaMalloc(&ctx->d_res[k], res_b));
    }
    if (ctx->bnd_cap < bnd_b) {
      cudaFree(ctx->d_bnd[k]);
      COH_CUDA(ctx, cudaMalloc(&ctx->d_bnd[k], std::max<size_t>(bnd_b, 4)));
    }
  }
  ctx->rec_cap = std::max(ctx->rec_cap, rec_b);
  ctx->res_cap = std::max(ctx->res_cap, res_b);
  ctx->bnd_cap = std::max(ctx->bnd_cap, bnd_b);
  if (packed) ctx->pk_cap = std::max(ctx->pk_cap, pk_b);
  int k = 0;
  for (uint64_t t0 = 0; t0 < n; t0 += S, k ^= 1) {
    const uint64_t m = std::min<uint64_t>(S, n - t0);
    cudaStream_t s = ctx->hs[k];
    if (n_chunks && packed) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(batch->records) + t0 * 12u;
      COH_CUDA(ctx, cudaMemcpy2DAsync(ctx->d_pk[k], m * 12u, src, n * 12u, m * 12u, n_chunks,
                                      cudaMemcpyHostToDevice, s));
      std::string err;
      rc = cohb::launch_unpack12(static_cast<const uint8_t*>(ctx->d_pk[k]), ctx->d_rec[k], m, n_chunks, s, &err);
      if (rc) {
        ctx->err = err;
        return rc;
      }
      ctx->launches++;
    } else if (n_chunks) {
      COH_CUDA(ctx, cudaMemcpy2DAsync(ctx->d_rec[k], m * 16u, batch->records + t0 * 8u, n * 16u,
                                      m * 16u, n_chunks, cudaMemcpyHostToDevice, s));
    }
    rc = eval_device(ctx, &dev_batch, ctx->d_rec[k], m, ctx->d_res[k], h_boundary ? ctx->d_bnd[k] : nullptr, s);
    if (rc) return rc;
    COH_CUDA(ctx, cudaMemcpyAsync(h_results + t0, ctx->d_res[k], sizeof(coh_trace_result) * m,
                                  cudaMemcpyDeviceToHost, s));
    if (h_boundary && n_words)
      COH_CUDA(ctx, cudaMemcpy2DAsync(h_boundary + t0, n * 4u, ctx->d_bnd[k], m * 4u, m * 4u,
                                      n_words, cudaMemcpyDeviceToHost, s));
  }
  COH_CUDA(ctx, cudaStreamSynchronize(ctx->hs[0]));
  COH_CUDA(ctx, cudaStreamSynchronize(ctx->hs[1]));
  return COH_OK;
}

int coh_measure_link(coh_ctx* ctx, size_t bytes, int reps, double* h2d_gbs, double* d2h_gbs) {
  if (!ctx || !h2d_gbs || !d2h_gbs || bytes == 0) return COH_E_ARG;
  void *h = nullptr, *d = nullptr;
  COH_CUDA(ctx, cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
  if (cudaMalloc(&d, bytes) != cudaSuccess) {
    cudaFreeHost(h);
    ctx->err = "coh_measure_link: device allocation";
    return COH_E_CUDA;
  }
  cudaStream_t s;
  cudaEvent_t e0, e1;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best[2] = {0, 0};
  for (int dir = 0; dir < 2; ++dir)
    for (int r = 0; r < std::max(1, reps); ++r) {
      cudaEventRecord(e0, s);
      if (dir == 0) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
      else cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      best[dir] = std::max(best[dir], (double)bytes / (ms / 1e3) / 1e9);
    }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  cudaFree(d);
  cudaFreeHost(h);
  *h2d_gbs = best[0];
  *d2h_gbs = best[1];
  return COH_OK;
}

int coh_reduce_counters(coh_ctx* ctx, const coh_trace_result* d_results, uint64_t n_traces,
                        uint64_t* d_counters, void* stream) {
  if (!ctx) return COH_E_ARG;
  if (!d_counters) return arg_fail(ctx, "d_counters is NULL");
  std::string err;
  int rc = cohb::launch_reduce_counters(d_results, n_traces, d_counters, stream, &err);
  if (rc) ctx->err = err;
  else if (n_traces) ctx->launches++;
  return rc;
}

}  // extern "C"

// ---- declarations ----------------------------------------------------------------------
struct coh_decls {
  std::vector<uint64_t> bytes;                          // arrays
  std::vector<uint32_t> cells;                          // buffers
  std::vector<std::vector<uint32_t>> vlo, vhi;          // views per buffer
  std::string err;
};

extern "C" {

int coh_decls_create(coh_decls** out) {
  if (!out) return COH_E_ARG;
  *out = new coh_decls();
  return COH_OK;
}

void coh_decls_destroy(coh_decls* d) { delete d; }

const char* coh_decls_error(const coh_decls* d) { return d ? d->err.c_str() : "no declarations"; }

int coh_decls_array(coh_decls* d, uint64_t bytes, uint32_t* id) {
  if (!d || !id) return COH_E_ARG;
  if (d->bytes.size() >= COH_MAX_ARRAYS) {
    d->err = "more than 64 whole-array variables";
    return COH_E_CONSTRUCTION;
  }
  *id = (uint32_t)d->bytes.size();
  d->bytes.push_back(bytes);
  return COH_OK;
}

int coh_decls_buffer(coh_decls* d, uint32_t n_cells, uint32_t* id) {
  if (!d || !id) return COH_E_ARG;
  if (n_cells == 0) {  // program.hpp:57-63: a buffer has at least one element
    d->err = "buffer size must be positive";
    return COH_E_CONSTRUCTION;
  }
  *id = (uint32_t)d->cells.size();
  d->cells.push_back(n_cells);
  d->vlo.emplace_back();
  d->vhi.emplace_back();
  return COH_OK;
}

int coh_decls_view(coh_decls* d, uint32_t buffer, uint32_t lo, uint32_t hi, uint32_t* view_index) {
  if (!d || !view_index || buffer >= d->cells.size()) return COH_E_ARG;
  if (lo > hi || hi >= d->cells[buffer]) {  // program.hpp:65-68
    d->err = "view range does not fit its buffer";
    return COH_E_CONSTRUCTION;
  }
  if (d->vlo[buffer].size() >= COH_MAX_VIEWS) {
    d->err = "more than 16 views on one buffer";
    return COH_E_CONSTRUCTION;
  }
  *view_index = (uint32_t)d->vlo[buffer].size();
  d->vlo[buffer].push_back(lo);
  d->vhi[buffer].push_back(hi);
  return COH_OK;
}

int coh_decls_trace_batch(const coh_decls* d, coh_trace_batch* b) {
  if (!d || !b || d->bytes.empty()) return COH_E_ARG;
  b->n_arrays = (uint32_t)d->bytes.size();
  b->array_bytes = d->bytes.data();
  return COH_OK;
}

int coh_decls_elem_program(const coh_decls* d, uint32_t buffer, coh_elem_program* p) {
  if (!d || !p || buffer >= d->cells.size()) return COH_E_ARG;
  p->n_cells = d->cells[buffer];
  p->n_views = (uint32_t)d->vlo[buffer].size();
  p->view_lo = d->vlo[buffer].data();
  p->view_hi = d->vhi[buffer].data();
  return COH_OK;
}

}  // extern "C"
