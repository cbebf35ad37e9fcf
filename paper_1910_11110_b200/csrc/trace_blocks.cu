// k_trace_blocks — traces whose blocks carry several access modes (COH_BATCH_BLOCKS: a
// record with COH_REC_CONT continues the previous record's DeclBlock, program.hpp:
// 212-235).  One thread per trace.  A block is first checked as the DeclBlock
// constructor would (a declared, well-formed mode per record, every array at most once)
// and then run as translate_block lays it out (modes.hpp:53-59): every mode's guard in
// record order -- `if (valid(x^)) {} else {pull x; pull x^}` (gvalid / push for GPU
// modes, Local-site syncs) and `w x^` for W / RW -- then every record's body in record
// order; run (semantics.hpp:253-287) with the trace's shared fuel, Done checked before
// fuel, Stuck taking no step; abstraction_correct (modes.hpp:79-90) after each completed
// block.  Single-mode traces are the fast path's business (trace_eval.cu); with no
// COH_REC_CONT bit this kernel gives field-for-field the same results.
//
// State: one byte per (array, thread) in shared memory (nibble cl | cr << 1 | al << 2 |
// ar << 3; 0xFF = not declared), a running count of arrays whose abstraction is violated
// (updated on every write), records read straight from the call-major layout.
#include <cuda_runtime.h>

#include "internal.hpp"

namespace cohb {
namespace {

constexpr int kBT = 128;  // traces per block

__device__ __forceinline__ uint32_t swap_pair(uint32_t p) { return ((p & 1u) << 1) | ((p >> 1) & 1u); }

__device__ __forceinline__ uint32_t violating(uint32_t nib) {  // !leq(abstract, concrete)
  const uint32_t c = nib & 3u, a = (nib >> 2) & 3u;
  return !(a == c || (c == 3u && (a == 1u || a == 2u)));
}

struct BlocksParams {
  uint64_t prog[kCallTypes];  // per call type: its translated block as micro-ops (calltable.cpp
                              // block_ops, one byte each: guard ops first, then the body)
  const uint16_t* rec;
  uint64_t n_traces;
  uint32_t n_calls, n_arrays;
  int32_t fuel;
  bool uniform;
  uint64_t bytes_uniform;
  const uint64_t* array_bytes;  // device (non-uniform sizes)
  coh_trace_result* res;
  uint32_t* bnd;
  unsigned long long* counters;
};

__global__ void __launch_bounds__(kBT) k_trace_blocks(const BlocksParams p) {
  __shared__ uint8_t st[COH_MAX_ARRAYS][kBT];
  const uint32_t tid = threadIdx.x;
  const uint64_t t = (uint64_t)blockIdx.x * kBT + tid;
  if (t >= p.n_traces) return;
  const uint64_t n = p.n_traces;
  for (uint32_t a = 0; a < COH_MAX_ARRAYS; ++a) st[a][tid] = a < p.n_arrays ? COH_STATE_INITIAL : 0xFFu;
  auto rec = [&](uint32_t i) -> uint32_t { return __ldg(p.rec + ((uint64_t)(i >> 3) * n + t) * 8u + (i & 7u)); };
  auto bytes_of = [&](uint32_t a) -> uint64_t { return p.uniform ? p.bytes_uniform : p.array_bytes[a]; };

  uint32_t steps = 0, xfers = 0, blocks_done = 0, viol_blocks = 0, viol = 0;
  uint64_t tbytes = 0;
  uint32_t status = COH_RUN_DONE, stuck_call = 0, stuck_arr = 0, stuck_eff = 0, stuck_flags = 0;
  uint32_t word = 0;  // boundary_ok bits of the current 32-block group
  const uint32_t n_words = (p.n_calls + 31u) / 32u;
  // A flat state machine: every iteration executes at most one micro-op for every lane,
  // so lanes on different blocks, phases and records run the same instruction stream
  // (nested per-block / per-record loops diverged: ~4 of 32 lanes active per instruction).
  // Cursor: block [b0, b1), phase (0 guards, 1 bodies), record i, op k of its program.
  uint32_t b0 = 0, b1 = 0, i = 0, k = 0, phase = 2;  // phase 2: open the next block
  uint32_t r = 0;
  uint64_t prog = 0;
  bool live = p.n_calls > 0;
  while (live) {
    if (phase == 2) {  // the next block: b0 and the COH_REC_CONT records after it
      b0 = b1;
      if (b0 >= p.n_calls) break;
      b1 = b0 + 1;
      while (b1 < p.n_calls && (rec(b1) & COH_REC_CONT)) ++b1;
      // DeclBlock construction (program.hpp:212-235): declared arrays, valid modes, each
      // array once; a failure is a construction defect at this block, before any step
      unsigned long long seen = 0ull;
      bool defect = false;
      for (uint32_t j = b0; j < b1 && !defect; ++j) {
        const uint32_t rj = rec(j), a = COH_REC_ARRAY(rj);
        if (a >= p.n_arrays || COH_REC_KIND(rj) == 3u || ((seen >> a) & 1ull)) {
          defect = true;
          stuck_arr = a;
        }
        seen |= 1ull << a;
      }
      if (defect) {
        status = COH_RUN_DEFECT;
        break;
      }
      phase = 0, i = b0, k = 0;
      r = rec(i);
      prog = p.prog[COH_REC_TYPE(r)];
    }
    // the op range of record i in this phase: guard ops first, then the body
    const uint32_t kind = COH_REC_KIND(r);
    const uint32_t n_guard = kind == COH_R ? 3u : kind == COH_W ? 1u : 4u;
    const uint32_t n_all = (uint32_t)(64 - __clzll((long long)prog) + 7) >> 3;  // ops are non-zero bytes
    if (k < (phase ? n_guard : 0u)) k = n_guard;
    if (k < (phase ? n_all : n_guard)) {
      if ((int32_t)steps >= p.fuel) {  // an op remains: Done was not reached
        status = COH_RUN_FUEL_EXHAUSTED;
        stuck_arr = COH_REC_ARRAY(rec(b0));
        break;
      }
      const uint32_t a = COH_REC_ARRAY(r);
      const uint32_t nib = st[a][tid];
      const uint32_t op = (uint32_t)(prog >> (8u * k)) & 0xFFu, kop = op & 3u;
      if (kop != OP_EFFECT) {  // if (valid(x^)) / if (gvalid(x^)): one step; valid skips the two syncs
        ++steps;
        k += ((nib >> (1u + kop)) & 1u) ? 3u : 1u;
        continue;
      }
      const uint32_t eff = (op >> 2) & 7u, esite = (op >> 5) & 1u, abstract = (op >> 6) & 1u;
      const uint32_t pair = abstract ? (nib >> 2) & 3u : nib & 3u;
      // validity.hpp:79-120 with the remote swap (semantics.hpp:109-130), branch-free
      const uint32_t q = esite ? swap_pair(pair) : pair;
      const bool sync = eff == COH_PUSH || eff == COH_PULL;
      const uint32_t ok = eff == COH_PUSH ? (q & 1u) : eff == COH_PULL ? (q >> 1) : eff == COH_READ ? (q & 1u) : 1u;
      if (!ok) {
        status = COH_RUN_STUCK;
        stuck_arr = a;
        stuck_eff = eff;
        stuck_flags = esite | (abstract << 1) | (pair << 2);
        break;
      }
      const uint32_t rq = sync ? 3u : eff == COH_READ ? q : eff == COH_WRITE ? 1u : q;
      const uint32_t after = esite ? swap_pair(rq) : rq;
      const uint32_t nn = abstract ? ((nib & 3u) | (after << 2)) : ((nib & 12u) | after);
      viol += violating(nn) - violating(nib);
      st[a][tid] = (uint8_t)nn;
      ++steps;
      if (!abstract && sync) {
        ++xfers;
        tbytes += bytes_of(a);
      }
      ++k;
      continue;
    }
    // record i's ops of this phase are done: the next record, phase or block
    if (++i < b1) {
      k = 0;
    } else if (phase == 0) {
      phase = 1, i = b0, k = 0;
    } else {
      // abstraction_correct after the completed block
      if (viol) ++viol_blocks;
      else word |= 1u << (blocks_done & 31u);
      ++blocks_done;
      if ((blocks_done & 31u) == 0u) {
        if (p.bnd) p.bnd[(uint64_t)(blocks_done / 32u - 1u) * n + t] = word;
        word = 0u;
      }
      phase = 2;
      continue;
    }
    r = rec(i);
    prog = p.prog[COH_REC_TYPE(r)];
  }
  if (status != COH_RUN_DONE) stuck_call = blocks_done;
  if (p.bnd) {
    uint32_t w = blocks_done / 32u;
    if (blocks_done & 31u) p.bnd[(uint64_t)w++ * n + t] = word;
    for (; w < n_words; ++w) p.bnd[(uint64_t)w * n + t] = 0u;
  }
  // the final store, nibble-packed; is_unsafe (program.hpp:166-170)
  uint32_t sw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool unsafe = false;
  for (uint32_t a = 0; a < p.n_arrays; ++a) {
    const uint32_t nib = st[a][tid];
    sw[a >> 3] |= nib << (4u * (a & 7u));
    unsafe |= !(nib & 3u) || !(nib & 12u);
  }
  if (unsafe) stuck_flags |= COH_FLAG_UNSAFE;
  uint4* out = reinterpret_cast<uint4*>(p.res + t);
  out[0] = make_uint4(sw[0], sw[1], sw[2], sw[3]);
  out[1] = make_uint4(sw[4], sw[5], sw[6], sw[7]);
  out[2] = make_uint4((uint32_t)tbytes, (uint32_t)(tbytes >> 32), steps, xfers);
  out[3] = make_uint4(blocks_done, viol_blocks, stuck_call,
                      status | (stuck_arr << 8) | (stuck_eff << 16) | (stuck_flags << 24));
  if (p.counters) {
    const unsigned long long v[COH_N_COUNTERS] = {
        status == COH_RUN_STUCK, status == COH_RUN_FUEL_EXHAUSTED, viol_blocks != 0u, status == COH_RUN_DEFECT,
        steps, xfers, tbytes, viol_blocks, blocks_done, 1u, unsafe ? 1u : 0u};
#pragma unroll
    for (int k = 0; k < COH_N_COUNTERS; ++k)
      if (v[k]) atomicAdd(p.counters + k, v[k]);
  }
}

}  // namespace

int launch_trace_blocks(const TraceLaunch& L, void* stream, std::string* err) {
  BlocksParams p;
  for (uint32_t t = 0; t < (uint32_t)kCallTypes; ++t) {  // the host call-table compiler's programs
    uint8_t ops[8];
    const int n = coh_calltable_program(t, ops);
    p.prog[t] = 0;
    for (int k = 0; k < n && k < 8; ++k) p.prog[t] |= (uint64_t)ops[k] << (8 * k);
  }
  p.rec = L.records;
  p.n_traces = L.n_traces;
  p.n_calls = L.n_calls;
  p.n_arrays = L.n_arrays;
  p.fuel = L.fuel;
  p.uniform = L.uniform_bytes;
  p.bytes_uniform = L.bytes_uniform;
  p.array_bytes = L.d_array_bytes;
  p.res = L.results;
  p.bnd = L.boundary;
  p.counters = reinterpret_cast<unsigned long long*>(L.counters);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (L.counters) {
    const cudaError_t e = cudaMemsetAsync(L.counters, 0, sizeof(uint64_t) * COH_N_COUNTERS, s);
    if (e != cudaSuccess) {
      *err = std::string("trace_blocks counters: ") + cudaGetErrorString(e);
      return COH_E_CUDA;
    }
  }
  const uint64_t grid = (L.n_traces + kBT - 1) / kBT;
  if (grid > 0x7FFFFFFFull) {
    *err = "trace_blocks: too many traces";
    return COH_E_ARG;
  }
  k_trace_blocks<<<(uint32_t)grid, kBT, 0, s>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("trace_blocks launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

}  // namespace cohb
