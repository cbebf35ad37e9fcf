// trace_eval — one thread steps one whole-array component-call trace through the
// access-mode calculus.  Replaces, per trace, cohere::run_annotated (modes.hpp:105-125):
// for each block, translate_block (modes.hpp:53-59) + run (semantics.hpp:253-287) with
// shared fuel + abstraction_correct (modes.hpp:79-90).
//
// Layout:
//   * per-thread store: one u16 word per array in shared memory, column-interleaved
//     s_st[a][tid] (bank = tid mod 32 -> conflict-free for any array ids in a warp);
//     bits 0-3 = state nibble (cl, cr, al, ar), bits 4-15 = per-array transfer count.
//   * call table: 64 call types x 16 states of uint64 in shared memory (8 KB), compiled
//     on the host by calltable.cpp from the restated rules.
//   * records: call-major interleaved, 128-bit streaming loads of 8 calls, 32 calls
//     (4 loads) prefetched one group ahead.
//   * accumulator register: steps (bits 0-7, flushed every 32 calls), count of arrays
//     whose abstraction is currently violated (bits 8-15; boundary_ok <=> zero),
//     transfers (bits 16-22, flushed every 32 calls).
//   * stuck / fuel / malformed calls leave the fast path and replay the call's micro-ops
//     exactly (slow_call), which yields StuckInfo and the partial state.
#include <cuda_runtime.h>

#include "internal.hpp"

namespace cohb {

constexpr int kNT = 128;  // threads (traces in flight) per block

struct KParams {
  const uint4* rec;
  uint64_t n_traces;
  uint32_t n_calls;
  uint32_t n_arrays;
  int32_t fuel;
  uint32_t pad;
  uint64_t bytes_uniform;
  const uint64_t* array_bytes;
  const uint64_t* lut;
  const uint64_t* prog;
  coh_trace_result* res;
  uint32_t* bnd;
};

struct SlowOut {
  uint32_t status, word, steps, transfers, effect, flags;
};

// Exact replay of one block's micro-ops from `state` with `rem` fuel left
// (semantics.hpp:253-287: Done before fuel; Stuck consumes no step).
__device__ __noinline__ void slow_call(uint64_t prog, uint32_t old_word, int rem, SlowOut* o) {
  uint32_t s = old_word & 15u;
  uint32_t steps = 0, tr = 0, status = COH_RUN_DONE, eff_out = 0, flags = 0;
  int k = 0;
  while (true) {
    const uint32_t op = (uint32_t)(prog >> (8 * k)) & 0xFFu;
    if (k >= 8 || op == OP_END) break;
    if (op == OP_DEFECT) { status = COH_RUN_DEFECT; break; }  // construction defect first
    if ((int)steps >= rem) { status = COH_RUN_FUEL_EXHAUSTED; break; }
    const uint32_t kop = op & 3u;
    if (kop == OP_IF_VALID || kop == OP_IF_GVALID) {
      const uint32_t taken = kop == OP_IF_VALID ? (s >> 2) & 1u : (s >> 3) & 1u;
      ++steps;
      k += taken ? 3 : 1;
      continue;
    }
    const uint32_t eff = (op >> 2) & 7u, site = (op >> 5) & 1u, abs_t = (op >> 6) & 1u;
    const uint32_t sh = abs_t ? 2u : 0u;
    const uint32_t before = (s >> sh) & 3u;
    uint32_t q = site ? (((before & 1u) << 1) | (before >> 1)) : before;  // swap if remote
    int after;
    switch (eff) {
      case COH_PUSH: after = (q & 1u) ? 3 : -1; break;
      case COH_PULL: after = (q & 2u) ? 3 : -1; break;
      case COH_READ: after = (q & 1u) ? (int)q : -1; break;
      case COH_WRITE: after = 1; break;
      default: after = (int)q; break;
    }
    if (after < 0) {
      status = COH_RUN_STUCK;
      eff_out = eff;
      flags = site | (abs_t << 1) | (before << 2);
      break;
    }
    q = (uint32_t)after;
    if (site) q = ((q & 1u) << 1) | (q >> 1);
    s = (s & ~(3u << sh)) | (q << sh);
    ++steps;
    if (!abs_t && (eff == COH_PUSH || eff == COH_PULL)) ++tr;
    ++k;
  }
  o->status = status;
  o->word = (old_word & ~15u) + (tr << 4) + s;
  o->steps = steps;
  o->transfers = tr;
  o->effect = eff_out;
  o->flags = flags;
}

// FLAGS: kFuel = fuel may run out (fuel < 6 x n_calls), kBytes = non-uniform array
// sizes (per-array transfer counters), kArr = n_arrays < 64 (range-check array ids).
enum : int { kFuel = 1, kBytes = 2, kArr = 4 };

template <int FLAGS>
__global__ void __launch_bounds__(kNT) k_trace_eval(const KParams p) {
  constexpr bool CHECK_FUEL = FLAGS & kFuel;
  constexpr bool UNIFORM = !(FLAGS & kBytes);
  constexpr bool CHECK_ARR = FLAGS & kArr;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* s_lut = reinterpret_cast<uint64_t*>(smem);   // 1024 entries
  uint64_t* s_bytes = s_lut + kLutEntries;                // 64 entries
  uint16_t* s_st = reinterpret_cast<uint16_t*>(s_bytes + COH_MAX_ARRAYS);
  const int tid = threadIdx.x;
  for (int i = tid; i < kLutEntries; i += kNT) s_lut[i] = p.lut[i];
  if (!UNIFORM)
    for (int i = tid; i < COH_MAX_ARRAYS; i += kNT)
      s_bytes[i] = i < (int)p.n_arrays ? p.array_bytes[i] : 0ull;
  uint16_t* col = s_st + tid;  // this thread's column: col[a * kNT], all 64 arrays
  for (uint32_t a = 0; a < COH_MAX_ARRAYS; ++a) col[a * kNT] = (uint16_t)COH_STATE_INITIAL;
  __syncthreads();  // the only block barrier: afterwards each thread owns its column

  const uint64_t n = p.n_traces;
  const uint32_t n_calls = p.n_calls;
  const uint32_t n_chunks = (n_calls + 7u) / 8u;
  const uint32_t n_groups = n_calls / 32u;
  const uint32_t n_words = (n_calls + 31u) / 32u;
  const uint64_t stride = (uint64_t)gridDim.x * kNT;

  for (uint64_t base = (uint64_t)blockIdx.x * kNT; base < n; base += stride) {
    const uint64_t t = base + tid;
    if (t < n) {
      const uint4* rp = p.rec + t;
      uint32_t acc = 0, bnd = 0, steps = 0, transfers = 0, viol_blocks = 0;
      uint32_t status = COH_RUN_DONE, stuck_call = 0, stuck_arr = 0, stuck_eff = 0, stuck_flags = 0;
      uint32_t calls_done = n_calls;
      int fuel_left = p.fuel;
      uint32_t g = 0;

      // One call.  i = call index (compile-time within the unrolled group).
#define COH_CALL(REC, I)                                                                  \
  {                                                                                       \
    const uint32_t r_ = (REC);                                                            \
    uint16_t* sp_ = col + (r_ & 63u) * kNT;                                               \
    const uint32_t old_ = *sp_;                                                           \
    const uint64_t e_ = s_lut[((r_ >> 2) & 0x3F0u) | (old_ & 15u)];                       \
    const uint32_t lo_ = (uint32_t)e_, hi_ = (uint32_t)(e_ >> 32);                        \
    bool slow_ = (int)lo_ < 0;                                                            \
    if (CHECK_FUEL) slow_ |= (int)((acc + hi_) & 0xFFu) > fuel_left;                      \
    if (CHECK_ARR) slow_ |= (r_ & 63u) >= p.n_arrays;                                     \
    if (slow_) {                                                                          \
      SlowOut so_;                                                                        \
      if (CHECK_ARR && (r_ & 63u) >= p.n_arrays)                                          \
        so_ = SlowOut{COH_RUN_DEFECT, old_, 0u, 0u, 0u, 0u};                              \
      else                                                                                \
        slow_call(p.prog[(r_ >> 6) & 63u], old_, p.fuel - (int)steps - (int)(acc & 0xFFu), &so_); \
      *sp_ = (uint16_t)so_.word;                                                          \
      steps += (acc & 0xFFu) + so_.steps;                                                 \
      transfers += ((acc >> 16) & 0x7Fu) + so_.transfers;                                 \
      acc &= 0xFF00u;                                                                     \
      status = so_.status;                                                                \
      stuck_call = (I);                                                                   \
      stuck_arr = r_ & 63u;                                                               \
      stuck_eff = so_.effect;                                                             \
      stuck_flags = so_.flags;                                                            \
      calls_done = (I);                                                                   \
      goto terminated;                                                                    \
    }                                                                                     \
    *sp_ = (uint16_t)(old_ + lo_);                                                        \
    acc += hi_;                                                                           \
    bnd |= ((acc & 0xFF00u) == 0u) ? (1u << ((I) & 31u)) : 0u;                            \
  }

      {
        uint4 nxt[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if ((uint32_t)j < n_chunks) nxt[j] = __ldcs(rp + (uint64_t)j * n);
        for (g = 0; g < n_groups; ++g) {
          uint4 cur[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) cur[j] = nxt[j];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t c = 4u * (g + 1u) + (uint32_t)j;
            if (c < n_chunks) nxt[j] = __ldcs(rp + (uint64_t)c * n);
          }
          const uint32_t i0 = g * 32u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            COH_CALL(cur[j].x & 0xFFFFu, i0 + 8 * j + 0);
            COH_CALL(cur[j].x >> 16, i0 + 8 * j + 1);
            COH_CALL(cur[j].y & 0xFFFFu, i0 + 8 * j + 2);
            COH_CALL(cur[j].y >> 16, i0 + 8 * j + 3);
            COH_CALL(cur[j].z & 0xFFFFu, i0 + 8 * j + 4);
            COH_CALL(cur[j].z >> 16, i0 + 8 * j + 5);
            COH_CALL(cur[j].w & 0xFFFFu, i0 + 8 * j + 6);
            COH_CALL(cur[j].w >> 16, i0 + 8 * j + 7);
          }
          if (p.bnd) p.bnd[(uint64_t)g * n + t] = bnd;
          viol_blocks += 32u - __popc(bnd);
          bnd = 0;
          steps += acc & 0xFFu;
          transfers += (acc >> 16) & 0x7Fu;
          acc &= 0xFF00u;
          if (CHECK_FUEL) fuel_left = p.fuel - (int)steps;
        }
        // tail: n_calls % 32 calls, chunks already prefetched into nxt
        const uint32_t tail = n_calls - n_groups * 32u;
        if (tail) {
          const uint32_t i0 = n_groups * 32u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t w[4] = {nxt[j].x, nxt[j].y, nxt[j].z, nxt[j].w};
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              const uint32_t i = i0 + 8u * j + h;
              if (i < n_calls) COH_CALL((w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu, i);
            }
          }
          viol_blocks += tail - __popc(bnd);
          steps += acc & 0xFFu;
          transfers += (acc >> 16) & 0x7Fu;
          acc &= 0xFF00u;
          if (p.bnd) p.bnd[(uint64_t)n_groups * n + t] = bnd;
        }
        goto finished;
      }
#undef COH_CALL

    terminated : {
      // completed calls of the current group are bits [0, calls_done % 32)
      const uint32_t done_in_group = calls_done & 31u;
      g = calls_done / 32u;
      viol_blocks += done_in_group - __popc(bnd);
      if (p.bnd) {
        p.bnd[(uint64_t)g * n + t] = bnd;
        for (uint32_t w = g + 1; w < n_words; ++w) p.bnd[(uint64_t)w * n + t] = 0u;
      }
    }
    finished : {
      uint64_t cl = 0, cr = 0, al = 0, ar = 0, tbytes = 0;
#pragma unroll
      for (int a = 0; a < COH_MAX_ARRAYS; ++a) {
        if ((uint32_t)a < p.n_arrays) {
          const uint32_t w = col[a * kNT];
          cl |= (uint64_t)(w & 1u) << a;
          cr |= (uint64_t)((w >> 1) & 1u) << a;
          al |= (uint64_t)((w >> 2) & 1u) << a;
          ar |= (uint64_t)((w >> 3) & 1u) << a;
          if (!UNIFORM) tbytes += (uint64_t)(w >> 4) * s_bytes[a];
        }
      }
      if (UNIFORM) tbytes = (uint64_t)transfers * p.bytes_uniform;
      // reset this thread's column for its next trace (phantom arrays >= n_arrays
      // are never written: a call naming one stops the trace as a defect first)
      for (uint32_t a = 0; a < p.n_arrays; ++a) col[a * kNT] = (uint16_t)COH_STATE_INITIAL;
      uint4* out = reinterpret_cast<uint4*>(p.res + t);
      __stcs(out + 0, make_uint4((uint32_t)cl, (uint32_t)(cl >> 32), (uint32_t)cr, (uint32_t)(cr >> 32)));
      __stcs(out + 1, make_uint4((uint32_t)al, (uint32_t)(al >> 32), (uint32_t)ar, (uint32_t)(ar >> 32)));
      __stcs(out + 2, make_uint4((uint32_t)tbytes, (uint32_t)(tbytes >> 32), steps, transfers));
      __stcs(out + 3, make_uint4(calls_done, viol_blocks, stuck_call,
                                 status | (stuck_arr << 8) | (stuck_eff << 16) | (stuck_flags << 24)));
    }
    }
  }
}

static size_t trace_smem_bytes(uint32_t) {
  return sizeof(uint64_t) * (kLutEntries + COH_MAX_ARRAYS) + sizeof(uint16_t) * kNT * COH_MAX_ARRAYS;
}

template <int F>
static int launch_one(const TraceLaunch& L, const KParams& kp, cudaStream_t s, std::string* err) {
  const size_t smem = trace_smem_bytes(L.n_arrays);
  k_trace_eval<F><<<L.grid, kNT, smem, s>>>(kp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("trace_eval launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

int trace_eval_occupancy(int* blocks_per_sm, int* threads_per_block, uint32_t n_arrays,
                         std::string* err) {
  int b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b, k_trace_eval<0>, kNT, trace_smem_bytes(n_arrays));
  if (e != cudaSuccess) {
    *err = std::string("occupancy: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  *blocks_per_sm = b;
  *threads_per_block = kNT;
  return COH_OK;
}

int launch_trace_eval(const TraceLaunch& L, void* stream, std::string* err) {
  if (L.n_traces == 0) return COH_OK;
  KParams kp;
  kp.rec = reinterpret_cast<const uint4*>(L.records);
  kp.n_traces = L.n_traces;
  kp.n_calls = L.n_calls;
  kp.n_arrays = L.n_arrays;
  kp.fuel = L.fuel;
  kp.pad = 0;
  kp.bytes_uniform = L.bytes_uniform;
  kp.array_bytes = L.d_array_bytes;
  kp.lut = L.d_lut;
  kp.prog = L.d_prog;
  kp.res = L.results;
  kp.bnd = L.boundary;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int f = (L.check_fuel ? kFuel : 0) | (L.uniform_bytes ? 0 : kBytes) |
                (L.n_arrays < COH_MAX_ARRAYS ? kArr : 0);
  switch (f) {
    case 0: return launch_one<0>(L, kp, s, err);
    case 1: return launch_one<1>(L, kp, s, err);
    case 2: return launch_one<2>(L, kp, s, err);
    case 3: return launch_one<3>(L, kp, s, err);
    case 4: return launch_one<4>(L, kp, s, err);
    case 5: return launch_one<5>(L, kp, s, err);
    case 6: return launch_one<6>(L, kp, s, err);
    default: return launch_one<7>(L, kp, s, err);
  }
}

void trace_eval_set_smem_attr() {
  const int mx = (int)trace_smem_bytes(COH_MAX_ARRAYS);
  cudaFuncSetAttribute(k_trace_eval<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_trace_eval<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_trace_eval<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_trace_eval<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_trace_eval<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_trace_eval<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_trace_eval<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_trace_eval<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

}  // namespace cohb
