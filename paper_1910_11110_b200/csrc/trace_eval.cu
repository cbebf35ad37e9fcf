// trace_eval — one thread steps one whole-array component-call trace through the
// access-mode calculus.  Replaces, per trace, cohere::run_annotated (modes.hpp:105-125):
// for each block, translate_block (modes.hpp:53-59) + run (semantics.hpp:253-287) with
// shared fuel + abstraction_correct (modes.hpp:79-90).
//
// Layout:
//   * per-thread store: one u32 word per array in shared memory, column-interleaved
//     s_st[a][tid] (bank = tid mod 32: conflict-free whatever arrays a warp touches);
//     bits 2-5 = state nibble (cl, cr, al, ar), bits 6-31 = per-array transfer count.
//   * call table (calltable.cpp): 64 call types x 16 states of u32, XOR-swizzled
//     (slot = type*16 + (state ^ (type & 15))) so the common (type, state) pairs of a
//     warp land in distinct banks; lo16 = accumulator addend, hi16 = signed delta of
//     the state word.
//   * records: call-major interleaved, 128-bit streaming loads of 8 calls, a ring of
//     4 loads (32 calls) in flight per thread.
//   * accumulator: bits 0-7 steps since the last flush (flushed every 32 calls),
//     bits 8-15 number of arrays whose abstraction is currently violated (boundary_ok
//     <=> zero), bit 15 poisoned by slow entries (stuck / defect).
//   * slow calls (stuck, fuel, malformed) replay the call's micro-ops exactly
//     (slow_call) after leaving the unrolled loop; they yield StuckInfo + partial state.
#include <cuda_runtime.h>

#include "internal.hpp"

namespace cohb {

constexpr int kNT = 128;  // traces (threads) per block

// One static shared block so every access is [register + compile-time symbol offset]:
//   words [0, 1024)            call table (4 KB)
//   words [1024, 1024 + 64*NT) per-trace stores, s_st[a][tid] (32 KB)
//   then 64 x u64              per-array sizes (non-uniform bytes only)
constexpr int kStOff = kLutEntries;
__shared__ __align__(16) uint32_t s_mem[kLutEntries + COH_MAX_ARRAYS * kNT + 2 * COH_MAX_ARRAYS];
#define s_lut (s_mem)
#define s_st (s_mem + kStOff)
#define s_bytes (reinterpret_cast<uint64_t*>(s_mem + kStOff + COH_MAX_ARRAYS * kNT))

struct KParams {
  const uint4* rec;
  uint64_t n_traces;
  uint32_t n_calls;
  uint32_t n_arrays;
  int32_t fuel;
  uint32_t pad;
  uint64_t bytes_uniform;
  const uint64_t* array_bytes;
  const uint32_t* lut;
  const uint64_t* prog;
  coh_trace_result* res;
  uint32_t* bnd;
};

struct SlowOut {
  uint32_t status, word, steps, effect, flags;
};

// Exact replay of one block's micro-ops from the state word `old_word` with `rem` fuel
// left (semantics.hpp:253-287: Done before fuel; Stuck consumes no step, store kept).
__device__ __noinline__ void slow_call(uint64_t prog, uint32_t old_word, int rem, SlowOut* o) {
  uint32_t s = (old_word >> kStateShift) & 15u;
  uint32_t steps = 0, tr = 0, status = COH_RUN_DONE, eff_out = 0, flags = 0;
  for (int k = 0; k < 8;) {
    const uint32_t op = (uint32_t)(prog >> (8 * k)) & 0xFFu;
    if (op == OP_END) break;
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
    uint32_t q = site ? (((before & 1u) << 1) | (before >> 1)) : before;  // swapped(before)
    int after;
    switch (eff) {
      case COH_PUSH: after = (q & 1u) ? 3 : -1; break;   // (V,X) -> (V,V)
      case COH_PULL: after = (q & 2u) ? 3 : -1; break;   // (X,V) -> (V,V)
      case COH_READ: after = (q & 1u) ? (int)q : -1; break;
      case COH_WRITE: after = 1; break;                  // (X,Y) -> (V,I)
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
  o->word = (old_word & ~(15u << kStateShift)) + (tr << kCountShift) + (s << kStateShift);
  o->steps = steps;
  o->effect = eff_out;
  o->flags = flags;
}

__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// bnd = 2*bnd + (acc & 0xFF00 != 0): the carry of (x + 0xFFFFFFFF) is (x != 0).
__device__ __forceinline__ uint32_t shift_in_violation(uint32_t bnd, uint32_t acc) {
  uint32_t out;
  asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, 0xFFFFFFFF;\n\taddc.u32 %0, %2, %2;\n\t}"
      : "=r"(out)
      : "r"(acc & 0xFF00u), "r"(bnd));
  return out;
}

// FLAGS: kFuel = fuel may run out (fuel < 6 x n_calls), kBytes = non-uniform array
// sizes, kArr = n_arrays < 64 (range-check array ids).
enum : int { kFuel = 1, kBytes = 2, kArr = 4 };

template <int FLAGS>
__global__ void __launch_bounds__(kNT) k_trace_eval(const KParams p) {
  constexpr bool CHECK_FUEL = FLAGS & kFuel;
  constexpr bool UNIFORM = !(FLAGS & kBytes);
  constexpr bool CHECK_ARR = FLAGS & kArr;
  const int tid = threadIdx.x;
  for (int i = tid; i < kLutEntries; i += kNT) s_lut[i] = p.lut[i];
  if (!UNIFORM)
    for (int i = tid; i < COH_MAX_ARRAYS; i += kNT)
      s_bytes[i] = i < (int)p.n_arrays ? p.array_bytes[i] : 0ull;
  constexpr uint32_t kInit = COH_STATE_INITIAL << kStateShift;
#pragma unroll 8
  for (int a = 0; a < COH_MAX_ARRAYS; ++a) s_st[a * kNT + tid] = kInit;
  __syncthreads();  // the only block barrier: afterwards each thread owns its column

  const uint32_t col = (uint32_t)__cvta_generic_to_shared(s_st) + 4u * tid;
  const uint32_t lut = (uint32_t)__cvta_generic_to_shared(s_lut);
  char* const stc = reinterpret_cast<char*>(s_st) + 4 * tid;  // this thread's column
  const uint64_t n = p.n_traces;
  const uint32_t n_calls = p.n_calls, n_arrays = p.n_arrays;
  const uint32_t n_chunks = (n_calls + 7u) / 8u;
  const uint32_t n_groups = n_calls / 32u;
  const uint32_t n_words = (n_calls + 31u) / 32u;
  const uint64_t stride = (uint64_t)gridDim.x * kNT;

  for (uint64_t base = (uint64_t)blockIdx.x * kNT; base < n; base += stride) {
    const uint64_t t = base + tid;
    if (t >= n) continue;
    const uint4* rp = p.rec + t;
    uint32_t acc = 0, steps = 0, viol_blocks = 0;
    // bnd: shift register of boundary-VIOLATION bits of the current 32-call group,
    // seeded with a sentinel 1: after k calls the sentinel sits at bit k (call 0's bit
    // at k-1); the stored boundary_ok word is its reversed complement.
    uint32_t bnd = 1u, i0 = 0;
    uint32_t status = COH_RUN_DONE, stuck_call = 0, stuck_arr = 0, stuck_eff = 0, stuck_flags = 0;
    uint32_t calls_done = n_calls;
    int fuel_left = p.fuel;

    // One call; R = 16-bit record (bits above 15 may hold garbage).  Nothing per call
    // site survives into the slow path (it re-derives the call from the sentinel), so
    // the fast path carries no bookkeeping moves.
#define COH_CALL(R)                                                                         \
  {                                                                                         \
    const uint32_t r_ = (R);                                                                \
    uint32_t* sp_ = reinterpret_cast<uint32_t*>(stc + (r_ & 63u) * 512u); /* s_st[a][tid] */ \
    const uint32_t old_ = *sp_;                                                             \
    const uint32_t e_ = *reinterpret_cast<const uint32_t*>(                                 \
        reinterpret_cast<const char*>(s_lut) + ((r_ & 0xFC0u) | (((r_ >> 4) ^ old_) & 0x3Cu))); \
    acc += e_;                                                                              \
    bool stop_ = false;                                                                     \
    if (CHECK_FUEL) stop_ |= (int)(acc & 0xFFu) > fuel_left;                                \
    if (CHECK_ARR) stop_ |= (r_ & 63u) >= n_arrays;                                         \
    if (!stop_) *sp_ = old_ + (uint32_t)((int32_t)e_ >> 16); /* slow entries: +0 */         \
    if (__builtin_expect(stop_ || (acc & 0x8000u) != 0u, 0)) goto slow_path;               \
    bnd = shift_in_violation(bnd, acc);                                                     \
  }
#define COH_CHUNK(W)            \
  COH_CALL((W).x)               \
  COH_CALL((W).x >> 16)         \
  COH_CALL((W).y)               \
  COH_CALL((W).y >> 16)         \
  COH_CALL((W).z)               \
  COH_CALL((W).z >> 16)         \
  COH_CALL((W).w)               \
  COH_CALL((W).w >> 16)

    {
      uint4 ring[4];  // fully (re)initialised per trace so nothing stays live across traces
#pragma unroll
      for (int j = 0; j < 4; ++j)
        ring[j] = (uint32_t)j < n_chunks ? __ldcs(rp + (uint64_t)j * n) : make_uint4(0u, 0u, 0u, 0u);
      for (uint32_t g = 0; g < n_groups; ++g) {
        i0 = g * 32u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 cur = ring[j];
          const uint32_t cn = 4u * (g + 1u) + (uint32_t)j;
          if (cn < n_chunks) ring[j] = __ldcs(rp + (uint64_t)cn * n);
          COH_CHUNK(cur)
        }
        // 32 calls done: the sentinel was shifted out, call 0's violation bit is bit 31
        bnd = ~__brev(bnd);
        if (p.bnd) p.bnd[(uint64_t)g * n + t] = bnd;
        viol_blocks += 32u - __popc(bnd);
        bnd = 1u;
        steps += acc & 0xFFu;
        acc &= 0xFF00u;
        if (CHECK_FUEL) fuel_left = p.fuel - (int)steps;
      }
      const uint32_t tail = n_calls - n_groups * 32u;
      if (tail) {
        i0 = n_groups * 32u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t w4[4] = {ring[j].x, ring[j].y, ring[j].z, ring[j].w};
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            if (8u * j + h < tail) COH_CALL(w4[h >> 1] >> (16 * (h & 1)))
          }
        }
        const uint32_t word = (~__brev(bnd ^ (1u << tail))) >> (32u - tail);
        viol_blocks += tail - __popc(word);
        steps += acc & 0xFFu;
        acc &= 0xFF00u;
        if (p.bnd) p.bnd[(uint64_t)n_groups * n + t] = word;
      }
      goto finished;
    }
#undef COH_CHUNK
#undef COH_CALL

  slow_path : {
    // which call: k calls of this group completed (sentinel position)
    const uint32_t k = 31u - __clz(bnd);
    const uint32_t i = i0 + k;
    const uint4 chunk = __ldcs(rp + (uint64_t)(i / 8u) * n);
    const uint32_t w4[4] = {chunk.x, chunk.y, chunk.z, chunk.w};
    const uint32_t r = (w4[(i & 7u) >> 1] >> (16u * (i & 1u))) & 0xFFFFu;
    const uint32_t a = r & 63u;
    const uint32_t old = lds(col + (a << 9));  // untouched: the fast path did not store
    const uint32_t e = lds(lut + ((r & 0xFC0u) | (((r >> 4) ^ old) & 0x3Cu)));
    acc -= e;  // undo the accumulate (low 16 bits exact)
    SlowOut so;
    if (CHECK_ARR && a >= n_arrays) {
      so = SlowOut{COH_RUN_DEFECT, old, 0u, 0u, 0u};
    } else {
      slow_call(p.prog[(r >> 6) & 63u], old, p.fuel - (int)steps - (int)(acc & 0xFFu), &so);
    }
    sts(col + (a << 9), so.word);
    steps += (acc & 0xFFu) + so.steps;
    status = so.status;
    stuck_call = i;
    stuck_arr = a;
    stuck_eff = so.effect;
    stuck_flags = so.flags;
    calls_done = i;
    const uint32_t word = k ? ((~__brev(bnd ^ (1u << k))) >> (32u - k)) : 0u;
    viol_blocks += k - __popc(word);
    if (p.bnd) {
      const uint32_t g = i / 32u;
      p.bnd[(uint64_t)g * n + t] = word;
      for (uint32_t w = g + 1; w < n_words; ++w) p.bnd[(uint64_t)w * n + t] = 0u;
    }
  }
  finished : {
    uint32_t sw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t transfers = 0;
    uint64_t tbytes = 0;
#pragma unroll
    for (int a = 0; a < COH_MAX_ARRAYS; ++a) {
      if (a < (int)n_arrays) {
        const uint32_t w = lds(col + (a << 9));
        sts(col + (a << 9), kInit);  // reset for this thread's next trace
        const int sh = 4 * (a & 7) - (int)kStateShift;
        sw[a >> 3] |= (sh >= 0 ? (w << sh) : (w >> -sh)) & (15u << (4 * (a & 7)));
        transfers += w >> kCountShift;
        if (!UNIFORM) tbytes += (uint64_t)(w >> kCountShift) * s_bytes[a];
      }
    }
    if (UNIFORM) tbytes = (uint64_t)transfers * p.bytes_uniform;
    uint4* out = reinterpret_cast<uint4*>(p.res + t);
    __stcs(out + 0, make_uint4(sw[0], sw[1], sw[2], sw[3]));
    __stcs(out + 1, make_uint4(sw[4], sw[5], sw[6], sw[7]));
    __stcs(out + 2, make_uint4((uint32_t)tbytes, (uint32_t)(tbytes >> 32), steps, transfers));
    __stcs(out + 3, make_uint4(calls_done, viol_blocks, stuck_call,
                               status | (stuck_arr << 8) | (stuck_eff << 16) | (stuck_flags << 24)));
  }
  }
}

template <int F>
static int launch_one(const TraceLaunch& L, const KParams& kp, cudaStream_t s, std::string* err) {
  k_trace_eval<F><<<L.grid, kNT, 0, s>>>(kp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("trace_eval launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

int trace_eval_occupancy(int* blocks_per_sm, int* threads_per_block, uint32_t, std::string* err) {
  int b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_trace_eval<0>, kNT, 0);
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

void trace_eval_set_smem_attr() {}

}  // namespace cohb
