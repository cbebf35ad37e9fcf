/*
 * cohere_b200.h — C ABI of the B200-native batched evaluator for the access-mode
 * calculus of arXiv 1910.11110 (reference: /root/reference/proj, namespace cohere).
 *
 * The reference has no FFI layer; its boundary is the header-only C++ API in
 * namespace cohere (proj/include/cohere/cohere.hpp:5-14).  Every entry point below
 * names the reference function(s) it replaces.  Plain pointers and sizes only; no
 * exception crosses this ABI: failures are int status codes plus coh_last_error().
 *
 * Ordinals mirror the reference enums exactly:
 *   coh_effect     <- cohere::EffectKind  (validity.hpp:35)   Push, Pull, Read, Write, Noop
 *   coh_site       <- cohere::Site        (ast.hpp:22)         Local, Remote
 *   coh_mode_kind  <- AccessMode::Kind    (program.hpp:188)    R, W, RW
 *   coh_run_status <- cohere::RunStatus   (semantics.hpp:220)  Done, Stuck, FuelExhausted
 *                     (+ COH_RUN_DEFECT: a malformed record; the reference would throw)
 *
 * Threading: thread-compatible (one host thread per ctx), stream-ordered; results are
 * deterministic and independent of launch geometry and GPU count.
 */
#ifndef COHERE_B200_H
#define COHERE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------ */
enum {
  COH_OK = 0,
  COH_E_CONSTRUCTION = 1,     /* <= cohere::ConstructionError (program.hpp:16-18)       */
  COH_E_DEFECT = 2,           /* <= std::logic_error (program.hpp:147-151, semantics.hpp:156) */
  COH_E_OVERLAP_CONFLICT = 3, /* <= cohere::OverlapInferenceError (overlap.hpp:24-30)   */
  COH_E_CUDA = 4,
  COH_E_NCCL = 5,
  COH_E_ARG = 6
};

enum { COH_PUSH = 0, COH_PULL = 1, COH_READ = 2, COH_WRITE = 3, COH_NOOP = 4 };
enum { COH_LOCAL = 0, COH_REMOTE = 1 };
enum { COH_R = 0, COH_W = 1, COH_RW = 2 };
enum { COH_RUN_DONE = 0, COH_RUN_STUCK = 1, COH_RUN_FUEL_EXHAUSTED = 2, COH_RUN_DEFECT = 3 };
enum { COH_KEY_CONCRETE = 0, COH_KEY_ABSTRACT = 1 }; /* VarKey::Kind Scalar / Abstract */

/* ---- whole-array component-call records ------------------------------------------
 * One uint16 per component call (one DeclBlock with a single AccessMode on one array,
 * program.hpp:212-235), SURVEY §8(d):
 *   bit 0      COH_REC_CONT: the call continues the previous call's block (multi-mode
 *              DeclBlocks, program.hpp:212-235), honoured only in batches flagged
 *              COH_BATCH_BLOCKS (ignored otherwise)
 *   bit 1      reserved (zero; ignored)
 *   bits 2-7   call type = mode kind R/W/RW (bits 2-3; 3 is malformed -> COH_RUN_DEFECT)
 *              | site << 2 (bit 4: 0 CPU/Local, 1 GPU/Remote)
 *              | body variant << 3 (bits 5-7: 0 = canonical well-declared body, 1..7
 *                adversarial; see DESIGN.md §3 / coh_calltable_program)
 *   bits 8-13  array id (the scalar "a<id>" of the reference harness; an id >= n_arrays
 *              is a missing key -> COH_RUN_DEFECT)
 *   bits 14-15 reserved (zero; ignored)
 * The two fields sit in separate bytes so the device turns a record into a store-slot
 * address and a call-table address with one masked logic op each.
 * Device layout, "call-major interleaved": rec(t, i) = records[((i/8)*n_traces + t)*8 + i%8]
 * so one 128-bit load brings 8 calls of one trace and a warp's loads are contiguous.
 * Padding records (i >= n_calls) are ignored.
 */
#define COH_REC_TYPE(r) (((r) >> 2) & 63u)
#define COH_REC_ARRAY(r) (((r) >> 8) & 63u)
#define COH_REC_KIND(r) (((r) >> 2) & 3u)
#define COH_REC_SITE(r) (((r) >> 4) & 1u)
#define COH_REC_VARIANT(r) (((r) >> 5) & 7u)
#define COH_MAKE_REC(arr, kind, site, var) \
  ((uint16_t)((((arr) & 63u) << 8) | (((kind) & 3u) << 2) | (((site) & 1u) << 4) | (((var) & 7u) << 5)))
#define COH_MAX_ARRAYS 64
#define COH_N_VARIANTS 8
#define COH_REC_CONT 0x1u

/* Per-array 4-bit state nibble: bit0 concrete local valid, bit1 concrete remote valid,
 * bit2 abstract local valid, bit3 abstract remote valid.  initial_store (program.hpp:
 * 174-184) puts every key at (V,I): nibble 0x5. */
#define COH_STATE_INITIAL 0x5u

/* Per-trace result: 64 bytes.  Replaces AnnotatedRun{status, store, stuck, boundary_ok,
 * steps, ...} (modes.hpp:95-103) plus the transfer accounting the reference lacks
 * (SURVEY §8(d) "transfer accounting rule").  state: the final store, one nibble per
 * array a at state[a / 8] >> (4 * (a % 8)): bit0 store.at(scalar(a)).local == V,
 * bit1 .remote == V, bit2 store.at(abstract(a)).local == V, bit3 .remote == V. */
typedef struct coh_trace_result {
  uint32_t state[8];        /* nibble-packed final store (arrays >= n_arrays: 0)      */
  uint64_t transfer_bytes;  /* sum over executed concrete push/pull of array_bytes[a] */
  uint32_t steps;           /* AnnotatedRun::steps                                    */
  uint32_t transfers;       /* executed concrete Push/Pull steps                      */
  uint32_t calls_done;      /* completed blocks == boundary_ok.size()                 */
  uint32_t violations;      /* completed blocks whose boundary check failed           */
  uint32_t stuck_call;      /* block index of the Stuck / FuelExhausted / defect call  */
  uint8_t status;           /* COH_RUN_*                                              */
  uint8_t stuck_array;      /* StuckInfo::key (array id)                              */
  uint8_t stuck_effect;     /* StuckInfo::effect (COH_PUSH..)                         */
  uint8_t stuck_flags;      /* bit0 StuckInfo::site, bit1 key kind (COH_KEY_*),
                               bits2-3 StuckInfo::actual (bit2 local V, bit3 remote V),
                               bit4 COH_FLAG_UNSAFE: is_unsafe (program.hpp:166-170) of
                               the final store, some key (I,I) -- unreachable by Property 2 */
} coh_trace_result;
#define COH_FLAG_UNSAFE 0x10u

static inline uint32_t coh_result_nibble(const coh_trace_result* r, uint32_t a) {
  return (r->state[a >> 3] >> (4u * (a & 7u))) & 15u;
}

typedef struct coh_trace_batch {
  const uint16_t* records;     /* device, layout above                                 */
  uint64_t n_traces;
  uint32_t n_calls;            /* blocks per trace (>= 1)                              */
  uint32_t n_arrays;           /* 1..64                                                */
  int32_t fuel;                /* shared across blocks, as run_annotated (modes.hpp:110) */
  uint32_t flags;              /* COH_BATCH_*                                          */
  const uint64_t* array_bytes; /* host, n_arrays entries (NULL => 1 byte each)         */
} coh_trace_batch;

/* COH_BATCH_BLOCKS: records carry COH_REC_CONT, so a block (one DeclBlock) is a record
 * without the bit followed by the records with it: its modes in record order (arrays
 * distinct, else the block is a construction defect), translated as translate_block does
 * (modes.hpp:53-59): every mode's guard in order, then every record's body in order.
 * Per-block outputs (calls_done, violations, stuck_call, boundary bits) then count and
 * index blocks, not records. */
#define COH_BATCH_BLOCKS 0x1u
/* COH_BATCH_PACKED12 (coh_eval_traces_host only): the host records are packed 12 bits per
 * call, the record's two fields without the free bits -- (array << 6) | call type -- so
 * the host->device link carries 12 bytes per 8 calls instead of 16.  Chunk c (8 calls)
 * of trace t is the 12 bytes at ((c * n_traces + t) * 12), call k of the chunk the bits
 * [12k, 12k + 12) of those 96 little-endian bits.  Unpacked on the device per pipeline
 * slice.  Not combinable with COH_BATCH_BLOCKS (no room for COH_REC_CONT). */
#define COH_BATCH_PACKED12 0x2u
/* COH_BATCH_OVERLAP (coh_eval_traces / _counted, whole-array batches; ignored by
 * coh_eval_traces_host, whose kernels read what its own copies wrote): the launch may begin
 * before the previous kernel on the same stream has finished (programmatic dependent
 * launch: its blocks take the SMs the previous launch's last blocks free, so a stream of
 * batches does not drain the GPU between launches).  The caller guarantees that the
 * previous kernel on the stream writes nothing this batch reads, and reads or writes none
 * of this batch's outputs (results, boundary words, counters) -- e.g. consecutive batches
 * with their own output buffers.  Without the flag a launch is ordered as usual. */
#define COH_BATCH_OVERLAP 0x4u
/* Pack call-major 16-bit records (layout above) into the COH_BATCH_PACKED12 form;
 * out holds ((n_calls + 7) / 8) * n_traces * 12 bytes. */
int coh_pack_records12(const uint16_t* records, uint64_t n_traces, uint32_t n_calls, uint8_t* out);

/* boundary_ok bitmaps: word-major, boundary[(i/32)*n_traces + t] bit (i%32) is
 * boundary_ok[i] of trace t; bits for calls >= calls_done are 0. */
static inline uint32_t coh_boundary_words(uint32_t n_calls) { return (n_calls + 31u) / 32u; }

/* ---- context -------------------------------------------------------------------- */
typedef struct coh_ctx coh_ctx;
int coh_ctx_create(int device, coh_ctx** out);
void coh_ctx_destroy(coh_ctx* ctx);
const char* coh_last_error(const coh_ctx* ctx);
const char* coh_version(void);

/* ---- host call-table compiler (no GPU needed) -------------------------------------
 * Replaces translate_mode / translate_block (modes.hpp:31-59) + effect_signature /
 * apply_signature (validity.hpp:79-120) + the swap rule of apply_effect_at
 * (semantics.hpp:109-130), compiled into a (call type x 16 states) table.
 * call type = record bits 2..7 (kind | site<<2 | variant<<3), 64 types.
 * coh_calltable_describe fills, for one (type, state), what the reference run of that
 * block from that store produces.  Returns COH_OK or COH_E_ARG. */
typedef struct coh_call_outcome {
  uint8_t status;        /* COH_RUN_DONE / COH_RUN_STUCK / COH_RUN_DEFECT         */
  uint8_t state_after;   /* nibble after the block (store as left when stuck)     */
  uint8_t steps;         /* completed reduction steps                              */
  uint8_t transfers;     /* executed concrete Push/Pull                            */
  uint8_t viol_before;   /* !leq(abstract, concrete) before (modes.hpp:71-75)      */
  uint8_t viol_after;
  uint8_t stuck_effect, stuck_flags; /* as coh_trace_result                        */
} coh_call_outcome;
int coh_calltable_describe(uint32_t call_type, uint32_t state, coh_call_outcome* out);
/* Micro-op listing of one call type's translated block (guards then body). ops[k]:
 * bits0-1 op (0 end,1 if-valid(x^) skip2,2 if-gvalid(x^) skip2,3 effect),
 * bits2-4 effect, bit5 site, bit6 target abstract.  Returns op count. */
int coh_calltable_program(uint32_t call_type, uint8_t ops[8]);

/* ---- synthetic record generator -------------------------------------
 * h = splitmix64(seed ^ (trace_id << 20) ^ call_idx)
 *   array   = ((h & 0xffffffff) * n_arrays) >> 32
 *   kind    = (((h >> 32) & 0xffff) * 3) >> 16
 *   site    = (h >> 48) & 1
 *   variant = ((h >> 49) & 0x3ff) < adv_per1024 ? 1 + ((((h >> 59) & 0x1f) * 7) >> 5) : 0
 * Identical on host and device.  trace ids [trace0, trace0 + n_traces). */
int coh_gen_records(coh_ctx* ctx, uint64_t seed, uint64_t trace0, uint64_t n_traces,
                    uint32_t n_calls, uint32_t n_arrays, uint32_t adv_per1024,
                    uint16_t* d_records, void* stream);
int coh_gen_records_host(uint64_t seed, uint64_t trace0, uint64_t n_traces,
                         uint32_t n_calls, uint32_t n_arrays, uint32_t adv_per1024,
                         uint16_t* h_records);
/* The same records with COH_REC_CONT marks for COH_BATCH_BLOCKS: call i > 0 continues the
 * current block with probability cont_per1024/1024 when its array is not yet in the block
 *   cont(t, i) = (splitmix64(seed ^ 0x5851F42D4C957F2D ^ (trace_id << 20) ^ i) & 0x3ff) < cont_per1024
 * (each trace walked in call order).  Identical on host and device. */
int coh_gen_records_blocks(coh_ctx* ctx, uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                           uint32_t n_arrays, uint32_t adv_per1024, uint32_t cont_per1024, uint16_t* d_records,
                           void* stream);
int coh_gen_records_blocks_host(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                                uint32_t n_arrays, uint32_t adv_per1024, uint32_t cont_per1024, uint16_t* h_records);
static inline size_t coh_records_elems(uint64_t n_traces, uint32_t n_calls) {
  return (size_t)((n_calls + 7u) / 8u) * (size_t)n_traces * 8u;
}

/* ---- the hot path: batched trace evaluation ---------------------------------------
 * Replaces, per trace, cohere::run_annotated (modes.hpp:105-125) over a program whose
 * blocks are the trace's calls: translate_block (modes.hpp:53) -> run (semantics.hpp:
 * 253-287, fuel shared, Done checked before fuel, Stuck consumes no step) ->
 * abstraction_correct (modes.hpp:79-90) after each completed block.
 * d_results: device, n_traces entries.  d_boundary: device, coh_boundary_words(n_calls)
 * * n_traces words (may be NULL).  stream: cudaStream_t (NULL = legacy default). */
int coh_eval_traces(coh_ctx* ctx, const coh_trace_batch* batch, coh_trace_result* d_results,
                    uint32_t* d_boundary, void* stream);

/* coh_eval_traces + the counter reduction below fused into the same kernel (zeroes
 * d_counters first): the form the multi-GPU step uses before its allreduce. */
int coh_eval_traces_counted(coh_ctx* ctx, const coh_trace_batch* batch, coh_trace_result* d_results,
                            uint32_t* d_boundary, uint64_t* d_counters, void* stream);

/* Same, from HOST buffers (records/results/boundary in host memory, ideally pinned):
 * chunked H2D -> kernel -> D2H pipelined over two streams inside the call; returns
 * after the results are on the host.  batch->records is a host pointer here. */
int coh_eval_traces_host(coh_ctx* ctx, const coh_trace_batch* batch,
                         coh_trace_result* h_results, uint32_t* h_boundary);

/* Sum of per-trace counters into COH_N_COUNTERS uint64 (device):
 * [0] traces stuck, [1] traces fuel-exhausted, [2] traces with >=1 boundary violation,
 * [3] defect traces, [4] steps, [5] transfers, [6] transfer_bytes, [7] violating blocks,
 * [8] completed blocks (sum of calls_done), [9] traces, [10] unsafe traces (is_unsafe).
 * Evaluated calls = [8] + [0] + [1] + [3].  This vector is what the multi-GPU path
 * allreduces; integer sums make it exact and order-independent. */
#define COH_N_COUNTERS 11
int coh_reduce_counters(coh_ctx* ctx, const coh_trace_result* d_results, uint64_t n_traces,
                        uint64_t* d_counters, void* stream);

/* ---- multi-GPU (config C4) ---------------------------------------------
 * Traces are independent units ("independent runs may execute
 * concurrently with no shared state"; the reference itself is single-threaded), so device
 * d owns a contiguous trace-id shard and the ONLY exchange is one NCCL sum-allreduce of
 * the COH_N_COUNTERS uint64 counters.  New in this build (the reference has no collective).
 * NCCL is bound at run time (libnccl.so.2); any NCCL failure returns COH_E_NCCL. */
#define COH_COMM_ID_BYTES 128
typedef struct coh_comm coh_comm;
int coh_nccl_version(int* version);
/* One process per GPU: rank 0 makes the id, every rank receives it out of band. */
int coh_comm_unique_id(uint8_t id[COH_COMM_ID_BYTES]);
int coh_comm_init_rank(coh_ctx* ctx, const uint8_t id[COH_COMM_ID_BYTES], int world, int rank,
                       coh_comm** out);
/* One process driving n_dev devices (ncclCommInitAll): comms[d] belongs to ctxs[d]. */
int coh_comm_init_all(coh_ctx* const* ctxs, int n_dev, coh_comm** comms);
void coh_comm_destroy(coh_comm* comm);
/* Sum d_counters (device, COH_N_COUNTERS) over all ranks, in place, on `stream`. */
int coh_comm_allreduce_counters(coh_comm* comm, uint64_t* d_counters, void* stream);
/* Single-process multi-device step: coh_eval_traces_counted of shards[d] on comms[d]'s
 * device and streams[d], then one grouped allreduce of every d_counters[d]; afterwards
 * each d_counters[d] holds the whole job's counters.  d_boundary may be NULL. */
int coh_eval_traces_multi(coh_comm* const* comms, int n_dev, const coh_trace_batch* shards,
                          coh_trace_result* const* d_results, uint32_t* const* d_boundary,
                          uint64_t* const* d_counters, void* const* streams);
/* Host helpers (no GPU): rank's contiguous share of `total` traces (sizes differ by at
 * most one), and the counter vector of a host result batch (what the kernel computes). */
int coh_shard_split(uint32_t rank, uint32_t world, uint64_t total, uint64_t* first, uint64_t* count);
int coh_counters_host(const coh_trace_result* results, uint64_t n_traces, uint64_t* counters);

/* TraceMode::Full for one trace (semantics.hpp:231-235, 279-280): every reduction step of
 * run_annotated over the trace's blocks (records in plain call order, one trace; flags
 * as coh_trace_batch.flags), run on the device.  Per step: the record it belongs to, the
 * rule (cohere::StepRule ordinal: 0 effect, 1 remote-effect, 4 if-true, 5 if-false), the
 * head statement and the key it changed.  *status = the run's COH_RUN_*.  Returns COH_OK,
 * or -(steps) - 1 when cap was too small (the first cap steps are written). */
typedef struct coh_trace_step {
  uint32_t call;   /* record index                                                      */
  uint8_t rule;    /* StepRule                                                          */
  uint8_t array;   /* the array of the head statement                                   */
  uint8_t head;    /* effect | site << 3 | abstract target << 4; if-steps 0x80 | gvalid  */
  uint8_t delta;   /* bit 4: a key changed; bit 2 it is the abstract key; bits 0-1 its pair */
} coh_trace_step;
int coh_trace_steps(coh_ctx* ctx, const uint16_t* records, uint32_t n_calls, uint32_t n_arrays, int32_t fuel,
                    uint32_t flags, coh_trace_step* steps, uint32_t cap, uint32_t* n_steps, uint32_t* status);

/* Kernels launched by this ctx since creation (the bench's gpu_launches claim). */
uint64_t coh_launch_count(const coh_ctx* ctx);

/* Best-of-reps pinned cudaMemcpyAsync bandwidth (GB/s) in each direction: the host-device
 * link roofline of the container path (config C5). */
int coh_measure_link(coh_ctx* ctx, size_t bytes, int reps, double* h2d_gbs, double* d2h_gbs);

/* Pinned host memory for the host-buffer entry points. */
void* coh_host_alloc(size_t bytes);
void coh_host_free(void* p);

/* ==== element-granular path (overlapping sub-array views) ========
 * One element program = one buffer of n_cells cells, up to COH_MAX_VIEWS views (absolute
 * inclusive ranges, program.hpp:31-46), and a sequence of component calls, each one
 * declared mode on one view plus a body of up to two element range effects
 * (`w x[i]` / `r x[i]` for every i in [lo, hi], view-relative, program.hpp:94-101).
 * Before running, every call's modes are closed over view overlaps exactly as
 * rewrite_program / infer_overlap_closure do (overlap.hpp:182-242).
 * Store layout on the device: two bit planes per buffer, L (local valid) and R (remote
 * valid), bit i of word i/32; initial_store puts every cell at (V,I): L = 1, R = 0.   */
#define COH_MAX_VIEWS 16
#define COH_ELEM_MAX_CALLS 65535 /* calls per element program (larger: COH_E_CONSTRUCTION) */
typedef struct coh_elem_op {
  uint8_t effect;   /* COH_READ or COH_WRITE */
  uint8_t site;     /* COH_LOCAL / COH_REMOTE */
  uint16_t pad;
  uint32_t lo, hi;  /* view-relative, inclusive */
} coh_elem_op;
typedef struct coh_elem_call {
  uint32_t view;      /* declared view index */
  uint8_t kind;       /* COH_R / COH_W / COH_RW */
  uint8_t site;
  uint8_t n_body;     /* 0..2 */
  uint8_t pad;
  coh_elem_op body[2];
} coh_elem_call;
typedef struct coh_elem_program {
  uint32_t n_cells;
  uint32_t n_views;
  const uint32_t* view_lo;   /* absolute, inclusive */
  const uint32_t* view_hi;
  uint32_t n_calls;
  int32_t fuel;
  const coh_elem_call* calls;
  /* Pre-fragmented start (rho = 2^-frag_log2; 0 = none): cell i starts
   * coherent, at (V,V), instead of initial_store's (V,I) iff bit i%32 of
   * coh_frag_mask(frag_seed, frag_log2, i/32) is set -- as if those cells had already been
   * synchronised.  Every view stays abstraction-correct ((V,I) <= (V,V), modes.hpp:71-75);
   * a sync's delta then skips the coherent cells, so its transfer ranges fragment with
   * density rho.  The prelude takes no steps; the run is run_annotated from that store. */
  uint64_t frag_seed;
  uint32_t frag_log2;        /* 0..32 */
  uint32_t pad;
} coh_elem_program;

/* Word w of the fragmentation mask (each cell set with probability 2^-frag_log2).  Draw 0
 * is a murmur3 finalizer of the seed and the word index.  frag_log2 <= 5: the AND of
 * frag_log2 draws (draw j+1 = a xorshift32 step of draw j), cells independent.
 * frag_log2 > 5: at most one cell per word -- cell (x & 31) iff the top frag_log2 - 5 bits
 * of draw 0 are all ones (probability 2^-(frag_log2-5) per word, 2^-frag_log2 per cell). */
static inline uint32_t coh_frag_mask(uint64_t frag_seed, uint32_t frag_log2, uint32_t w) {
  if (frag_log2 == 0) return 0u;
  uint32_t x = ((uint32_t)frag_seed ^ (w * 0x9E3779B9u)) + (uint32_t)(frag_seed >> 32);
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  if (frag_log2 > 5) {
    const uint32_t t = frag_log2 - 5;  /* 1..27 */
    return (x >> (32u - t)) == ((1u << t) - 1u) ? 1u << (x & 31u) : 0u;
  }
  uint32_t m = x;
  for (uint32_t j = 1; j < frag_log2; ++j) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    m &= x;
  }
  return m;
}

/* Per-program outcome.  stuck key: element b[stuck_index] (key kind concrete) or the
 * abstract key of view stuck_index (key kind abstract).  Transfers are the executed
 * concrete whole-view syncs; their transfer ranges are the maximal runs of changed
 * cells of each sync's delta (semantics.hpp:125-128, 155-166). */
typedef struct coh_elem_result {
  uint8_t status, stuck_effect, stuck_flags, pad;  /* stuck_flags as coh_trace_result */
  uint32_t stuck_call;
  uint32_t stuck_index;
  uint32_t calls_done;
  uint32_t violations;
  uint32_t transfers;
  uint64_t steps;
  uint64_t transfer_cells;   /* sum of run lengths ("minimal" transfer, in cells)    */
  uint64_t n_runs;
  uint64_t vpu_cells;        /* VectorPU-faithful: whole view range per sync */
} coh_elem_result;

typedef struct coh_elem_stats {
  double device_ms;        /* init + all stages, CUDA events on the evaluation stream     */
  uint64_t alg_bytes;      /* algorithmic bytes: sync 3m/8 + 8 per run,
                              read m/8, write m/4, view check m/8 or m/4                  */
  uint64_t launches;
  uint64_t tiles;
  uint32_t stages;
  uint32_t pad;
} coh_elem_stats;

/* Evaluate n element programs (one buffer each) on the device; host inputs and outputs.
 * Replaces, per program, rewrite_program + run_annotated over views (overlap.hpp:234,
 * modes.hpp:105) with element bodies, and extracts the transfer ranges of every
 * whole-view sync.  Optional outputs (NULL to skip):
 *   planes_out    [n][2][plane_words] final L and R planes (bit i of word i/32)
 *   view_abs_out  [n][COH_MAX_VIEWS] final abstract pair of every view (bit0 L, bit1 R)
 *   boundary_out  [n][boundary_words] boundary_ok bit per completed call
 *   runs_out      [n][runs_cap][2] transfer ranges (first, last cell), ascending per sync
 * Returns COH_E_CONSTRUCTION for malformed programs (program.hpp:57-110 analogues). */
int coh_elem_eval(coh_ctx* ctx, const coh_elem_program* progs, uint32_t n_progs,
                  coh_elem_result* results, uint32_t* planes_out, uint32_t plane_words,
                  uint8_t* view_abs_out, uint32_t* boundary_out, uint32_t boundary_words,
                  uint32_t* runs_out, uint64_t runs_cap, coh_elem_stats* stats);

/* Synthetic element program (views + calls) for program id `prog_id`; see DESIGN.md §3b.
 * view_lo/view_hi: n_views entries; calls: n_calls entries. */
int coh_elem_gen(uint64_t seed, uint64_t prog_id, uint32_t n_cells, uint32_t n_views,
                 uint32_t n_calls, uint32_t adv_per1024, uint32_t* view_lo, uint32_t* view_hi,
                 coh_elem_call* calls);

/* ---- declarations (Declarations, program.hpp:141-226) ------------------------------
 * A declarations object: whole-array variables (arrays, with their byte sizes) and
 * buffers with views, numbered in declaration order; it fills the declaration part of
 * a trace batch or an element program.  Construction defects (more than 64 arrays or 16
 * views, a view outside its buffer, an empty buffer) are COH_E_CONSTRUCTION
 * (ConstructionError).  Pointers it hands out live as long as the object. */
typedef struct coh_decls coh_decls;
int coh_decls_create(coh_decls** out);
void coh_decls_destroy(coh_decls* d);
const char* coh_decls_error(const coh_decls* d);
int coh_decls_array(coh_decls* d, uint64_t bytes, uint32_t* id);
int coh_decls_buffer(coh_decls* d, uint32_t n_cells, uint32_t* id);
int coh_decls_view(coh_decls* d, uint32_t buffer, uint32_t lo, uint32_t hi, uint32_t* view_index);
/* n_arrays and array_bytes of *b (records, n_traces, n_calls and fuel are the caller's) */
int coh_decls_trace_batch(const coh_decls* d, coh_trace_batch* b);
/* n_cells, n_views, view_lo, view_hi of *p for one buffer (calls and fuel are the caller's) */
int coh_decls_elem_program(const coh_decls* d, uint32_t buffer, coh_elem_program* p);

/* ==== coherent container runtime (config C5) ======================
 * VectorPU's coherence control on the calculus: each vector is one
 * whole-array variable with pinned host + device copies and its calculus state (concrete
 * and abstract pairs, starting at (V,I)/(V,I), program.hpp:174-184).  A component call
 * executes the translated block (modes.hpp:31-59): guards on the abstract flags issue
 * cudaMemcpyAsync (push = H2D for a GPU component, pull = D2H for a CPU component) on the
 * runtime stream, then the component runs, then its body effects.  Stuck steps return
 * COH_E_DEFECT (StuckInfo text in coh_last_error).  The bytes moved equal the
 * evaluator's prediction for the same call sequence (transfers x vector bytes).       */
typedef struct coh_rt coh_rt;
typedef struct coh_rt_arg {
  uint32_t vec;
  uint32_t kind;       /* COH_R / COH_W / COH_RW */
} coh_rt_arg;
/* GPU components receive the component stream and must launch on it; CPU components get
 * NULL and run on the calling thread once their own arguments' copies have landed
 * (uploads and downloads run on side streams, ordered per vector by events). */
typedef void (*coh_rt_fn)(void* user, void* stream);
typedef struct coh_rt_stats {
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t h2d_copies, d2h_copies;
  uint64_t calls, syncs_elided, stuck_calls;
  double copy_ms;  /* device time of the copies (CUDA events around each cudaMemcpyAsync; counted
                      once the runtime has synchronised past them: CPU calls, coh_rt_sync) */
} coh_rt_stats;
int coh_rt_create(coh_ctx* ctx, coh_rt** out);
void coh_rt_destroy(coh_rt* rt);
int coh_rt_vector(coh_rt* rt, size_t bytes, uint32_t* id);
void* coh_rt_host_ptr(coh_rt* rt, uint32_t id);
void* coh_rt_device_ptr(coh_rt* rt, uint32_t id);
void* coh_rt_stream(coh_rt* rt);
int coh_rt_state(coh_rt* rt, uint32_t id, uint8_t* nibble);  /* cl | cr<<1 | al<<2 | ar<<3 */
int coh_rt_call(coh_rt* rt, uint32_t site, const coh_rt_arg* args, uint32_t n_args, coh_rt_fn fn, void* user);
int coh_rt_sync(coh_rt* rt);
/* Asynchronous CPU components (on != 0): a CPU component is enqueued as a stream-ordered
 * host function (cudaLaunchHostFunc) after its arguments' copies, and coh_rt_call returns
 * at once, so the copies of later calls overlap it.  Such a component must not call CUDA;
 * its user data must stay valid and its effects become visible at coh_rt_sync. */
int coh_rt_set_async(coh_rt* rt, int on);
int coh_rt_get_stats(const coh_rt* rt, coh_rt_stats* out);
/* Built-in trivial components over float vectors: W -> x = 1, RW -> x = 0.5x + 1,
 * R -> checksum.  user points to a coh_rt_touch. */
typedef struct coh_rt_touch {
  coh_rt* rt;
  uint32_t n;
  uint32_t vec[8];
  uint32_t kind[8];
  uint64_t bytes[8];
  double checksum;
} coh_rt_touch;
void coh_rt_touch_cpu(void* user, void* stream);
void coh_rt_touch_gpu(void* user, void* stream);

/* ---- views: VectorPU's pvector<T>(mother, lo, hi) ----------------
 * A buffer is a mother vector of n_cells elements (pinned host + device copies) whose
 * validity is element-granular: planes L (CPU valid) and R (GPU valid), bit i of word
 * i/32, starting at L = 1, R = 0 (program.hpp:174-184).  Views are inclusive cell ranges
 * of one buffer, in declaration order, each with its abstract pair (starting (V,I)).
 * coh_rt_call_view runs one component call on the buffer's views exactly as the element
 * evaluator (coh_elem_eval) runs the same coh_elem_call: the overlap closure (W/RW on
 * view x adds a same-site RW on every overlapping view, overlap.hpp:182-230), the guards
 * (a whole-view sync when the abstract flag is not valid at the component's site: stuck
 * at the first cell whose source bit is 0, otherwise every maximal run of cells whose
 * destination bit is 0 is copied with one cudaMemcpyAsync, semantics.hpp:155-166), the
 * abstract writes, then the body ops in order (READ needs the site's bit on its range,
 * WRITE sets it and clears the other; partial effects persist when a READ gets stuck),
 * and the component (run only when the block completes).  Copies: pull = D2H before a
 * CPU component, push = H2D before a GPU component, on the runtime stream.  Stuck returns
 * COH_E_DEFECT.  Every copy is logged (coh_rt_copy_log) so tests can compare it with the
 * evaluator's transfer ranges.                                                         */
typedef struct coh_rt_copy {
  uint32_t buffer;
  uint32_t first, last;  /* cells, inclusive */
  uint32_t h2d;          /* 1 = push (host -> device), 0 = pull */
} coh_rt_copy;
int coh_rt_buffer(coh_rt* rt, uint32_t n_cells, uint32_t elem_bytes, uint32_t* id);
int coh_rt_view(coh_rt* rt, uint32_t buffer, uint32_t lo, uint32_t hi, uint32_t* view_index);
int coh_rt_call_view(coh_rt* rt, uint32_t buffer, const coh_elem_call* call, coh_rt_fn fn, void* user);
int coh_rt_view_state(coh_rt* rt, uint32_t buffer, uint32_t view_index, uint8_t* abs_pair);
/* planes_out: 2 x ceil(n_cells / 32) words (L then R); synchronises the runtime stream */
int coh_rt_buffer_planes(coh_rt* rt, uint32_t buffer, uint32_t* planes_out);
void* coh_rt_buffer_host_ptr(coh_rt* rt, uint32_t buffer);
void* coh_rt_buffer_device_ptr(coh_rt* rt, uint32_t buffer);
/* copies issued so far, in order: *n = total; up to cap entries are written */
int coh_rt_copy_log(const coh_rt* rt, coh_rt_copy* out, uint64_t cap, uint64_t* n);

/* ==== general block programs and schedule sweeps ================
 * Programs in the full calculus (scalars + one buffer with overlapping views, several
 * modes per block, element bodies, opaque/validity if and while), generated natively by
 * a restatement of the test kit's gen_well_declared (testkit.hpp:364-447, mt19937_64
 * draw order) and closed over overlaps (overlap.hpp:182-230).  coh_sweep runs every
 * schedule of length <= max_decisions exactly as all_schedules_run (testkit.hpp:465-517)
 * does — run_annotated per prefix, a run that exhausted its prefix branches into the two
 * one-longer prefixes — with every run a GPU thread (one frontier level per launch). */
typedef struct coh_gen_limits {   /* GenLimits, testkit.hpp:279-287 (same order/defaults) */
  uint32_t max_blocks, max_body_depth, max_vars, max_buffer_len, max_loop_unroll;
  uint32_t allow_arrays, allow_overlaps, pad;
} coh_gen_limits;
/* The generated program in the reference's canonical pretty() form (pretty.hpp:120-139).
 * Returns COH_OK / COH_E_OVERLAP_CONFLICT, or -(needed size) if cap is too small. */
int coh_gen_program_text(uint64_t seed, const coh_gen_limits* limits, char* buf, size_t cap);
typedef struct coh_sweep_leaf {
  uint64_t seed;
  uint32_t schedule;          /* answers, bit k = k-th opaque decision                    */
  uint8_t sched_len;
  uint8_t status;             /* COH_RUN_*                                                */
  uint8_t blocks_done;        /* boundary_ok.size()                                       */
  uint8_t boundary_ok;        /* bit b = boundary_ok[b]                                    */
  uint32_t steps;
  uint8_t consumed, overflowed;
  uint8_t stuck_key;          /* key index (s_i = i, s_i^ = S+i, v_j^ = 2S+j, b0[c] = 2S+V+c) */
  uint8_t stuck_info;         /* effect | site << 3 | abstract key << 4 | actual << 5       */
  uint64_t store;             /* 2 bits per key: bit0 local V, bit1 remote V               */
} coh_sweep_leaf;
typedef struct coh_sweep_stats {
  uint64_t programs, runs, done, stuck, fuel_exhausted, runs_with_violation, nodes, conflicts;
  double device_ms;
  uint64_t launches;
} coh_sweep_stats;
int coh_sweep(coh_ctx* ctx, uint64_t seed0, uint32_t n_seeds, const coh_gen_limits* limits,
              uint32_t max_decisions, int32_t fuel, coh_sweep_leaf* leaves, uint64_t leaves_cap,
              coh_sweep_stats* stats);
/* Acceptance criterion 1 (tests/acceptance.cpp:107-138): every straight-line raw program of
 * length <= max_len (<= 8) over the ten effect forms on one scalar (enumerate_raw_programs,
 * testkit.hpp:241-268, in its order), run on the GPU block interpreter from initial_store;
 * outcome counts and the number of programs that ever leave a key (I,I). statuses[i]
 * (optional) = COH_RUN_* of program i. */
typedef struct coh_enum_stats {
  uint64_t programs, done, stuck, fuel_exhausted, unsafe, steps;
} coh_enum_stats;
int coh_enum_straight_line(coh_ctx* ctx, uint32_t max_len, int32_t fuel, coh_enum_stats* stats, uint8_t* statuses,
                           uint64_t statuses_cap);

/* ---- DSL front end and CLI reporting ----------------------
 * The reference command line (tools/cohere_main.cpp:80-230) over program text.
 * command: "check" | "run" | "trace" | "infer" | "translate" (cmd_check / cmd_run /
 * cmd_infer / cmd_translate); opts mirror its flags (--raw, --json, --no-overlap, --fuel,
 * --schedule, --trace).  Writes what the CLI prints to stdout / stderr (NUL-terminated) and its
 * exit code (0 ok, 1 diagnostics / overlap conflict, 2 usage / parse / construction
 * error, 3 stuck, 4 fuel exhausted).  Parsing (parse.hpp), overlap closure (overlap.hpp),
 * the static checker (checker.hpp) and the printers (pretty.hpp) are host passes; "run"
 * executes the translated program on the GPU (the general block interpreter of
 * coh_sweep: at most 32 store keys, schedules of at most 64 answers), which records one
 * (instruction, rule, store) entry per step for "trace" / --trace (at most 4M steps).
 * ctx may be NULL except for "run" / "trace".  Returns COH_OK (the CLI outcome is in *exit_code), a negative value
 * -(needed bytes) when out/err were too small (the texts are truncated), or COH_E_*. */
typedef struct coh_cli_opts {
  int raw, json, no_overlap;
  int32_t fuel;              /* --fuel (default 10000; must be >= 1)  */
  const char* schedule;      /* --schedule "0101" or NULL             */
  int trace;                 /* run --trace                           */
} coh_cli_opts;
int coh_cli(coh_ctx* ctx, const char* command, const char* src, const coh_cli_opts* opts,
            char* out, size_t out_cap, char* err, size_t err_cap, int* exit_code);
/* Batched host passes: "check", "infer" or "translate" over n program
 * texts on n_threads host threads (<= 0: all).  Program i's stdout is out[out_off[i] ..
 * out_off[i+1]), its stderr err[err_off[i] .. err_off[i+1]) (offsets: n + 1 entries; the
 * texts are not NUL-terminated), its exit code exit_codes[i] -- each exactly what coh_cli
 * gives for it.  Returns COH_OK, COH_E_ARG, or -(needed bytes) - 1 if a buffer is short. */
int coh_cli_batch(const char* command, const char* const* srcs, uint32_t n, const coh_cli_opts* opts,
                  int n_threads, char* out, size_t out_cap, uint64_t* out_off, char* err, size_t err_cap,
                  uint64_t* err_off, int* exit_codes);

/* ---- batched overlap registry and mode closure -----------------
 * OverlapRegistry (overlap.hpp:33-175) and infer_overlap_closure (overlap.hpp:177-230)
 * for many views and many blocks at once.  A view: its buffer id, inclusive absolute
 * range, and name_rank = the position of its name in std::string order (the reference's
 * query results and `needed` map are name-sorted; the rank decides which view an
 * OverlapInferenceError names); its declaration order is its index.  A mode: var = view
 * index (flags bit0 set) or scalar id, kind COH_R/W/RW, site, flags bit1 = shadow.
 * All pointers are device memory; calls are stream-ordered. */
typedef struct coh_view { uint32_t buffer; int32_t lo, hi; uint32_t name_rank; } coh_view;
typedef struct coh_mode { uint32_t var; uint8_t kind, site, flags, pad; } coh_mode;
typedef struct coh_registry coh_registry;
/* build_registry (overlap.hpp:232-239) for n_views views (ranges must fit their buffers) */
int coh_registry_build(coh_ctx* ctx, const coh_view* d_views, uint32_t n_views, coh_registry** out, void* stream);
void coh_registry_destroy(coh_registry* r);
/* query(view) (overlap.hpp:86-108) for each probe view: up to hits_stride hits written
 * name-sorted at d_hits[q * hits_stride], the total count in d_hit_count[q]. */
int coh_registry_query(coh_ctx* ctx, const coh_registry* r, const uint32_t* d_probes, uint32_t n_probes,
                       uint32_t* d_hits, uint32_t hits_stride, uint32_t* d_hit_count, void* stream);
/* infer_overlap_closure for each block b (modes d_modes[d_block_off[b] .. d_block_off[b+1])):
 * the closed list at d_out[b * out_stride], its length in d_out_count[b], d_status[b] = -1,
 * or d_status[b] = y for OverlapInferenceError(y), or -2 when the block exceeds the
 * per-block limits (64 declared modes, 64 inferred views, out_stride). */
int coh_overlap_closure(coh_ctx* ctx, const coh_registry* r, const coh_mode* d_modes, const uint32_t* d_block_off,
                        uint32_t n_blocks, coh_mode* d_out, uint32_t out_stride, uint32_t* d_out_count,
                        int32_t* d_status, void* stream);

/* ---- bit-plane primitives ---------------------------------------
 * A plane is a run of 32-bit words in device memory (d_words 16-byte aligned); cell i of
 * the plane starting at word `word_off` is bit i%32 of word word_off + i/32.  A range is
 * the cells [lo, hi] (inclusive; lo > hi = empty) of one plane.  Batched over ranges, one
 * persistent launch per call, stream-ordered.  Semantics:
 *   range_set / range_clear  bits [lo, hi] := 1 / 0 (element writes w x[i] on a range;
 *                            ranges may share edge words)
 *   first_zero               d_first[k] = the first cell of range k whose bit is 0 (the
 *                            stuck cell of a whole-view sync, semantics.hpp:155-166), or
 *                            0xFFFFFFFF
 *   extract_zero_runs        maximal runs of 0 bits in each range, ascending (the transfer
 *                            ranges of a whole-view sync): run j of range k is
 *                            [d_run_start[g], d_run_end[g]] with g = d_run_off[k] + j;
 *                            d_run_off has n + 1 entries (its last = the total; runs beyond
 *                            `cap` are counted but not written)
 *   view_check               d_ok[k] = abstraction_correct of one view (modes.hpp:84-88)
 *                            with abstract pair d_abs_pair[k] (bit0 local V, bit1 remote V)
 *                            against planes L (local valid) and R (remote valid) */
typedef struct coh_bitmap_range { uint64_t word_off; uint32_t lo, hi; } coh_bitmap_range;
int coh_bitmap_range_set(coh_ctx* ctx, uint32_t* d_words, const coh_bitmap_range* d_ranges, uint32_t n, void* stream);
int coh_bitmap_range_clear(coh_ctx* ctx, uint32_t* d_words, const coh_bitmap_range* d_ranges, uint32_t n, void* stream);
int coh_bitmap_first_zero(coh_ctx* ctx, const uint32_t* d_words, const coh_bitmap_range* d_ranges, uint32_t n,
                          uint32_t* d_first, void* stream);
int coh_bitmap_extract_zero_runs(coh_ctx* ctx, const uint32_t* d_words, const coh_bitmap_range* d_ranges, uint32_t n,
                                 uint32_t* d_run_start, uint32_t* d_run_end, uint64_t cap, uint64_t* d_run_off,
                                 void* stream);
int coh_bitmap_view_check(coh_ctx* ctx, const uint32_t* d_L, const uint32_t* d_R, const coh_bitmap_range* d_ranges,
                          const uint8_t* d_abs_pair, uint32_t n, uint8_t* d_ok, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COHERE_B200_H */
