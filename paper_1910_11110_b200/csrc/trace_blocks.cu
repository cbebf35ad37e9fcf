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
  const uint32_t* lut;        // the fast path's call table (internal.hpp: lut_word, entry layout)
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

struct Lane {  // one trace's running outcome
  uint32_t steps = 0, xfers = 0, viol = 0;
  uint64_t tbytes = 0;
  uint32_t status = COH_RUN_DONE, stuck_arr = 0, stuck_eff = 0, stuck_flags = 0;
};

// The exact semantics of one block [b0, b1) from the current store, op by op: every
// mode's guard in record order, then every body (translate_block, modes.hpp:53-59); run
// with the trace's fuel (semantics.hpp:253-287).  Taken at most once per trace -- for the
// block in which the trace gets stuck or runs out of fuel.  Returns true if it completed.
__device__ bool run_block_exact(const BlocksParams& p, uint8_t (*st)[kBT], uint32_t tid, uint64_t t, uint32_t b0,
                                uint32_t b1, Lane& L) {
  const uint64_t n = p.n_traces;
  for (uint32_t phase = 0; phase < 2; ++phase)
    for (uint32_t i = b0; i < b1; ++i) {
      const uint32_t r = __ldg(p.rec + ((uint64_t)(i >> 3) * n + t) * 8u + (i & 7u));
      const uint32_t a = COH_REC_ARRAY(r), kind = COH_REC_KIND(r);
      const uint64_t prog = p.prog[COH_REC_TYPE(r)];
      const uint32_t n_guard = kind == COH_R ? 3u : kind == COH_W ? 1u : 4u;
      const uint32_t n_all = (uint32_t)(64 - __clzll((long long)prog) + 7) >> 3;  // ops are non-zero bytes
      uint32_t nib = st[a][tid];
      for (uint32_t k = phase ? n_guard : 0u; k < (phase ? n_all : n_guard);) {
        if ((int32_t)L.steps >= p.fuel) {  // an op remains: Done was not reached
          st[a][tid] = (uint8_t)nib;
          L.status = COH_RUN_FUEL_EXHAUSTED;
          L.stuck_arr = COH_REC_ARRAY(__ldg(p.rec + ((uint64_t)(b0 >> 3) * n + t) * 8u + (b0 & 7u)));
          return false;
        }
        const uint32_t op = (uint32_t)(prog >> (8u * k)) & 0xFFu, kop = op & 3u;
        if (kop != OP_EFFECT) {  // if (valid(x^)) / if (gvalid(x^)): one step; valid skips the two syncs
          ++L.steps;
          k += ((nib >> (1u + kop)) & 1u) ? 3u : 1u;
          continue;
        }
        const uint32_t eff = (op >> 2) & 7u, esite = (op >> 5) & 1u, abstract = (op >> 6) & 1u;
        const uint32_t pair = abstract ? (nib >> 2) & 3u : nib & 3u;
        const uint32_t q = esite ? swap_pair(pair) : pair;  // validity.hpp:79-120, remote = swapped
        const bool sync = eff == COH_PUSH || eff == COH_PULL;
        const uint32_t ok = eff == COH_PUSH ? (q & 1u) : eff == COH_PULL ? (q >> 1) : eff == COH_READ ? (q & 1u) : 1u;
        if (!ok) {
          st[a][tid] = (uint8_t)nib;
          L.status = COH_RUN_STUCK;
          L.stuck_arr = a;
          L.stuck_eff = eff;
          L.stuck_flags = esite | (abstract << 1) | (pair << 2);
          return false;
        }
        const uint32_t rq = sync ? 3u : eff == COH_READ ? q : eff == COH_WRITE ? 1u : q;
        const uint32_t after = esite ? swap_pair(rq) : rq;
        const uint32_t nn = abstract ? ((nib & 3u) | (after << 2)) : ((nib & 12u) | after);
        L.viol += violating(nn) - violating(nib);
        nib = nn;
        ++L.steps;
        if (!abstract && sync) {
          ++L.xfers;
          L.tbytes += p.uniform ? p.bytes_uniform : p.array_bytes[a];
        }
        ++k;
      }
      st[a][tid] = (uint8_t)nib;
    }
  return true;
}

// The fast path runs the records of all lanes in lockstep (record i for every lane per
// iteration, so the warp stays converged): each record is one lookup in the host-compiled
// call table (new state, steps, transfers, change of the violated-array count), applied at
// once with the old state kept for undo.  For a block without a stuck record whose steps
// fit the fuel, the outcome equals the translate_block order's (its modes touch distinct
// arrays, so the order of their effects does not matter and the counts add up), and the
// block commits at its end (boundary bit from the violated count).  Otherwise the block is
// undone and re-run exactly (run_block_exact): it is where the trace stops.
// UNIFORM: one element size (bytes = transfers x size, folded in at the end); FUEL: the fuel
// can run out within the batch (else the commit needs no fuel test).
template <bool UNIFORM, bool FUEL>
__global__ void __launch_bounds__(kBT) k_trace_blocks(const BlocksParams p) {
  __shared__ uint8_t st[COH_MAX_ARRAYS][kBT];
  __shared__ uint8_t undo[COH_MAX_ARRAYS][kBT];
  __shared__ uint32_t s_lut[kLutEntries];
  __shared__ unsigned long long s_cnt[COH_N_COUNTERS];
  const uint32_t tid = threadIdx.x;
  for (uint32_t k = tid; k < (uint32_t)kLutEntries; k += kBT) s_lut[k] = __ldg(p.lut + k);
  if (tid < COH_N_COUNTERS) s_cnt[tid] = 0ull;
  __syncthreads();
  const uint64_t t = (uint64_t)blockIdx.x * kBT + tid;
  unsigned long long cv[COH_N_COUNTERS] = {};  // this thread's counter contributions
  if (t < p.n_traces) {
  const uint64_t n = p.n_traces;
  for (uint32_t a = 0; a < COH_MAX_ARRAYS; ++a) st[a][tid] = a < p.n_arrays ? COH_STATE_INITIAL : 0xFFu;

  Lane L;
  uint32_t blocks_done = 0, viol_blocks = 0;
  uint32_t word = 0;  // boundary_ok bits of the current 32-block group
  const uint32_t n_words = (p.n_calls + 31u) / 32u;
  // the open block
  uint32_t b0 = 0, bsteps = 0, bxfers = 0, defect_arr = 0;
  uint64_t bbytes = 0, seen = 0;  // seen: arrays named by the block (undo holds their states before it)
  int bdv = 0;
  bool slow = false, defect = false, stopped = false;

  auto close_block = [&](uint32_t b1) {
    if (!slow && !defect && (!FUEL || (int64_t)L.steps + bsteps <= (int64_t)p.fuel)) {  // commit
      L.steps += bsteps;
      L.xfers += bxfers;
      if (!UNIFORM) L.tbytes += bbytes;
      L.viol += (uint32_t)bdv;
      if (L.viol) ++viol_blocks;
      else word |= 1u << (blocks_done & 31u);
      ++blocks_done;
      if ((blocks_done & 31u) == 0u) {
        if (p.bnd) p.bnd[(uint64_t)(blocks_done / 32u - 1u) * n + t] = word;
        word = 0u;
      }
    } else {  // undo, then the block's exact outcome (the trace stops in it)
      for (uint64_t m = seen; m; m &= m - 1) {
        const uint32_t a = (uint32_t)__ffsll((long long)m) - 1u;
        st[a][tid] = undo[a][tid];
      }
      if (defect) {  // DeclBlock construction fails before any step
        L.status = COH_RUN_DEFECT;
        L.stuck_arr = defect_arr;
      } else if (run_block_exact(p, st, tid, t, b0, b1, L)) {  // (not reached: slow or over the fuel)
        L.status = COH_RUN_DEFECT;
      }
      stopped = true;
    }
    bsteps = bxfers = 0;
    if (!UNIFORM) bbytes = 0;
    bdv = 0;
    seen = 0;
    slow = defect = false;
  };

  // 8 records of this trace per 128-bit load, the next chunk in flight while one is used
  const uint4* const rec4 = reinterpret_cast<const uint4*>(p.rec) + t;
  const uint32_t n_chunks = (p.n_calls + 7u) / 8u;
  uint4 chunk = make_uint4(0u, 0u, 0u, 0u), next = n_chunks ? __ldcs(rec4) : chunk;
  for (uint32_t i = 0; i < p.n_calls && !stopped; ++i) {
    if ((i & 7u) == 0u) {
      chunk = next;
      if ((i >> 3) + 1u < n_chunks) next = __ldcs(rec4 + (uint64_t)((i >> 3) + 1u) * n);
    }
    const uint32_t wsel = (i & 4u) ? ((i & 2u) ? chunk.w : chunk.z) : ((i & 2u) ? chunk.y : chunk.x);
    const uint32_t r = (wsel >> (16u * (i & 1u))) & 0xFFFFu;
    if (i > 0 && !(r & COH_REC_CONT)) {
      close_block(i);
      if (stopped) break;
      b0 = i;
    }
    const uint32_t a = COH_REC_ARRAY(r), type = COH_REC_TYPE(r);
    if (a >= p.n_arrays || COH_REC_KIND(r) == 3u || ((seen >> a) & 1ull)) {  // DeclBlock defect (first wins)
      if (!defect) defect_arr = a;
      defect = true;
      continue;
    }
    seen |= 1ull << a;
    const uint32_t s0 = st[a][tid];
    undo[a][tid] = (uint8_t)s0;
    const uint32_t e = s_lut[s0 * 64u + (type ^ ((s0 * 9u) & 63u))];  // internal.hpp lut_word
    if ((int32_t)e < 0) {  // stuck (whatever the order of the block's modes)
      slow = true;
      continue;
    }
    st[a][tid] = (uint8_t)((e >> 8) & 15u);
    const uint32_t x = (e >> 23) & 0x3Fu;
    bsteps += (e >> 16) & 0x7Fu;
    bxfers += x;
    if (!UNIFORM && x) bbytes += (uint64_t)x * p.array_bytes[a];
    bdv += (int)((e >> 29) & 7u) - 1;
  }
  if (!stopped && p.n_calls) close_block(p.n_calls);
  const uint32_t stuck_call = L.status != COH_RUN_DONE ? blocks_done : 0u;
  if (p.bnd) {
    uint32_t w = blocks_done / 32u;
    if (blocks_done & 31u) p.bnd[(uint64_t)w++ * n + t] = word;
    for (; w < n_words; ++w) p.bnd[(uint64_t)w * n + t] = 0u;
  }
  // the final store, nibble-packed; is_unsafe (program.hpp:166-170)
  uint32_t sw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool unsafe = false;
#pragma unroll
  for (uint32_t a = 0; a < COH_MAX_ARRAYS; ++a) {
    if (a >= p.n_arrays) break;
    const uint32_t nib = st[a][tid];
    sw[a >> 3] |= nib << (4u * (a & 7u));
    unsafe |= !(nib & 3u) || !(nib & 12u);
  }
  if (UNIFORM) L.tbytes = (uint64_t)L.xfers * p.bytes_uniform;
  uint32_t stuck_flags = L.stuck_flags;
  if (unsafe) stuck_flags |= COH_FLAG_UNSAFE;
  uint4* out = reinterpret_cast<uint4*>(p.res + t);
  out[0] = make_uint4(sw[0], sw[1], sw[2], sw[3]);
  out[1] = make_uint4(sw[4], sw[5], sw[6], sw[7]);
  out[2] = make_uint4((uint32_t)L.tbytes, (uint32_t)(L.tbytes >> 32), L.steps, L.xfers);
  out[3] = make_uint4(blocks_done, viol_blocks, stuck_call,
                      L.status | (L.stuck_arr << 8) | (L.stuck_eff << 16) | (stuck_flags << 24));
  const unsigned long long v[COH_N_COUNTERS] = {
      L.status == COH_RUN_STUCK, L.status == COH_RUN_FUEL_EXHAUSTED, viol_blocks != 0u, L.status == COH_RUN_DEFECT,
      L.steps, L.xfers, L.tbytes, viol_blocks, blocks_done, 1u, unsafe ? 1u : 0u};
#pragma unroll
  for (int k = 0; k < COH_N_COUNTERS; ++k) cv[k] = v[k];
  }  // t < n_traces
  if (p.counters) {  // warp sums, one shared atomic per warp, one global atomic per block
    const uint32_t lane = tid & 31u;
#pragma unroll
    for (int k = 0; k < COH_N_COUNTERS; ++k) {
      unsigned long long x = cv[k];
#pragma unroll
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
      if (lane == 0 && x) atomicAdd(&s_cnt[k], x);
    }
    __syncthreads();
    if (tid < COH_N_COUNTERS && s_cnt[tid]) atomicAdd(p.counters + tid, s_cnt[tid]);
  }
}

}  // namespace

int launch_trace_blocks(const TraceLaunch& L, void* stream, std::string* err) {
  BlocksParams p;
  p.lut = L.d_lut;
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
  const bool fuel = L.check_fuel;
  if (p.uniform && !fuel) k_trace_blocks<true, false><<<(uint32_t)grid, kBT, 0, s>>>(p);
  else if (p.uniform) k_trace_blocks<true, true><<<(uint32_t)grid, kBT, 0, s>>>(p);
  else if (!fuel) k_trace_blocks<false, false><<<(uint32_t)grid, kBT, 0, s>>>(p);
  else k_trace_blocks<false, true><<<(uint32_t)grid, kBT, 0, s>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("trace_blocks launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

}  // namespace cohb
