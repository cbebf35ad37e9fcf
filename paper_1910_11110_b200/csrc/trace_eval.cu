// trace_eval — one thread steps one whole-array component-call trace through the
// access-mode calculus.  Replaces, per trace, cohere::run_annotated (modes.hpp:105-125):
// for each block, translate_block (modes.hpp:53-59) + run (semantics.hpp:253-287) with
// shared fuel + abstraction_correct (modes.hpp:79-90).
//
// Layout:
//   * per-thread store: one word per array in shared memory (u16, or u32 for traces
//     longer than 511 calls), bank-interleaved so a warp's lanes never conflict whatever
//     arrays they touch; bits 2-5 = state nibble (cl, cr, al, ar), bits 6+ = per-array
//     transfer count.
//   * call table (calltable.cpp): 64 call types x 16 states of u32, XOR-swizzled
//     (slot = type*16 + (state ^ (type & 15))) so the common (type, state) pairs of a
//     warp land in distinct banks; lo16 = signed delta of the store word, hi16 = signed
//     accumulator addend.
//   * records: call-major interleaved, 128-bit streaming loads of 8 calls, a ring of
//     4 loads (32 calls) in flight per thread.
//   * accumulator (clean 32-bit): bits 0-7 steps since the last flush (every 32 calls),
//     bits 8-14 number of arrays whose abstraction is currently violated (boundary_ok
//     <=> acc < 0x100), bit 15 set by slow entries (stuck / defect).
//   * slow calls (stuck, fuel, malformed) leave the unrolled loop; the call is
//     re-derived from a sentinel in the boundary shift register and its exact outcome
//     (StuckInfo, partial state and steps) read from a host-compiled table indexed by
//     (type, state, remaining fuel).
#include <cuda_runtime.h>

#include <type_traits>

#include "internal.hpp"

namespace cohb {

constexpr int kNT = 128;  // traces (threads) per block

// Per-trace store word: u16 (kNarrow, 128 B per trace, n_calls <= 511 so the 10-bit
// per-array transfer counter cannot overflow) or u32 (wide, 256 B per trace).
// Narrow slots are lane-interleaved so that a warp's 32 lanes always hit 32 distinct
// banks whatever arrays they touch:
//   u16 index = a*kNT + (warp>>1)*64 + 2*lane + (warp&1)  ->  bank = lane.
// Shared block (per instantiation): [call table 4 KB][stores][64 x u64 array sizes].
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
  const uint32_t* slow;
  coh_trace_result* res;
  uint32_t* bnd;
  unsigned long long* counters;  // optional fused COH_N_COUNTERS reduction (zeroed by the launcher)
};

// bnd = 2*bnd + (acc >= 0x100): the accumulator is clean (steps | viol << 8), so the
// carry of acc + 0xFFFFFF00 is exactly "some array's abstraction is violated".
__device__ __forceinline__ uint32_t shift_in_violation(uint32_t bnd, uint32_t acc) {
  uint32_t out;
  asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, 0xFFFFFF00;\n\taddc.u32 %0, %2, %2;\n\t}"
      : "=r"(out)
      : "r"(acc), "r"(bnd));
  return out;
}

// FLAGS: kFuel = fuel may run out (fuel < 6 x n_calls), kBytes = non-uniform array
// sizes, kArr = n_arrays < 64 (range-check array ids), kWide = u32 store words.
enum : int { kFuel = 1, kBytes = 2, kArr = 4, kWide = 8 };

template <int FLAGS>
__global__ void __launch_bounds__(kNT, (FLAGS & kWide) ? 6 : 10) k_trace_eval(const KParams p) {
  constexpr bool CHECK_FUEL = FLAGS & kFuel;
  constexpr bool UNIFORM = !(FLAGS & kBytes);
  constexpr bool CHECK_ARR = FLAGS & kArr;
  constexpr bool WIDE = FLAGS & kWide;
  using Word = typename std::conditional<WIDE, uint32_t, uint16_t>::type;
  constexpr uint32_t kStride = sizeof(Word) * kNT;  // bytes between arrays of one column
  constexpr int kStWords = COH_MAX_ARRAYS * kNT * (int)sizeof(Word) / 4;
  __shared__ __align__(16) uint32_t s_mem[kLutEntries + kStWords + 2 * COH_MAX_ARRAYS];
  __shared__ unsigned long long s_cnt[COH_N_COUNTERS];
  uint32_t* const s_lut = s_mem;
  char* const s_stb = reinterpret_cast<char*>(s_mem + kLutEntries);
  uint64_t* const s_bytes = reinterpret_cast<uint64_t*>(s_mem + kLutEntries + kStWords);

  const int tid = threadIdx.x;
  for (int i = tid; i < kLutEntries; i += kNT) s_lut[i] = p.lut[i];
  if (!UNIFORM)
    for (int i = tid; i < COH_MAX_ARRAYS; i += kNT)
      s_bytes[i] = i < (int)p.n_arrays ? p.array_bytes[i] : 0ull;
  constexpr uint32_t kInit = COH_STATE_INITIAL << kStateShift;
  constexpr uint32_t kInitWord = WIDE ? kInit : (kInit | (kInit << 16));
  for (int i = tid; i < kStWords; i += kNT) s_mem[kLutEntries + i] = kInitWord;
  if (tid < COH_N_COUNTERS) s_cnt[tid] = 0ull;
  __syncthreads();  // the only block barrier: afterwards each thread owns its column

  const uint32_t warp = tid >> 5, lane = tid & 31;
  const uint32_t thread_off = WIDE ? 4u * tid : (warp >> 1) * 128u + 4u * lane + 2u * (warp & 1u);
  char* const stc = s_stb + thread_off;  // this thread's column: stc + a * kStride
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
    Word* sp_ = reinterpret_cast<Word*>(stc + (r_ & 63u) * kStride);   /* store[a][tid] */ \
    const uint32_t old_ = *sp_;                                                             \
    const uint32_t e_ = *reinterpret_cast<const uint32_t*>(                                 \
        reinterpret_cast<const char*>(s_lut) + ((r_ & 0xFC0u) | (((r_ >> 4) ^ old_) & 0x3Cu))); \
    acc += (uint32_t)((int32_t)e_ >> 16);                                                   \
    bool stop_ = false;                                                                     \
    if (CHECK_FUEL) stop_ |= (int)(acc & 0xFFu) > fuel_left;                                \
    if (CHECK_ARR) stop_ |= (r_ & 63u) >= n_arrays;                                         \
    if (!stop_) *sp_ = (Word)(old_ + (WIDE ? (uint32_t)(int32_t)(int16_t)e_ : e_));         \
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
    Word* const sp = reinterpret_cast<Word*>(stc + a * kStride);
    const uint32_t old = *sp;  // untouched: the fast path did not store
    const uint32_t e = *reinterpret_cast<const uint32_t*>(
        reinterpret_cast<const char*>(s_lut) + ((r & 0xFC0u) | (((r >> 4) ^ old) & 0x3Cu)));
    acc -= (uint32_t)((int32_t)e >> 16);  // undo the accumulate
    // exact outcome from the host-compiled slow table (type, state, remaining fuel)
    const int rem_i = p.fuel - (int)steps - (int)(acc & 0xFFu);
    const uint32_t rem = rem_i <= 0 ? 0u : (rem_i >= 7 ? 7u : (uint32_t)rem_i);
    const uint32_t s0 = (old >> kStateShift) & 15u;
    const uint32_t info = (CHECK_ARR && a >= n_arrays)
                              ? (uint32_t)COH_RUN_DEFECT | (s0 << 7)
                              : __ldg(p.slow + slow_index((r >> 6) & 63u, s0, rem));
    struct {
      uint32_t status, word, steps, effect, flags;
    } so;
    so.status = info & 3u;
    so.steps = (info >> 2) & 7u;
    so.word = (old & ~(15u << kStateShift)) + (((info >> 5) & 3u) << kCountShift) +
              (((info >> 7) & 15u) << kStateShift);
    so.effect = (info >> 11) & 7u;
    so.flags = (info >> 14) & 15u;
    *sp = (Word)so.word;
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
        Word* const wp = reinterpret_cast<Word*>(stc + a * kStride);
        const uint32_t w = *wp;
        *wp = (Word)kInit;  // reset for this thread's next trace
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
    if (p.counters) {  // fused counter reduction: warp redux, one shared atomic per warp
      const uint32_t m = __activemask();
      const bool leader = (lane == (uint32_t)(__ffs(m) - 1));
      uint32_t v[9] = {status == COH_RUN_STUCK, status == COH_RUN_FUEL_EXHAUSTED, viol_blocks != 0u,
                       status == COH_RUN_DEFECT, steps, transfers, viol_blocks, calls_done, 1u};
      const int slot[9] = {0, 1, 2, 3, 4, 5, 7, 8, 9};
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        v[k] = __reduce_add_sync(m, v[k]);
        if (leader && v[k]) atomicAdd(&s_cnt[slot[k]], (unsigned long long)v[k]);
      }
      if (UNIFORM) {  // bytes = transfers x size: one multiply by the leader
        if (leader && v[5]) atomicAdd(&s_cnt[6], (unsigned long long)v[5] * p.bytes_uniform);
      } else if (tbytes) {  // non-uniform sizes: per-lane shared atomic
        atomicAdd(&s_cnt[6], (unsigned long long)tbytes);
      }
    }
  }
  }
  if (p.counters) {
    __syncthreads();
    if (tid < COH_N_COUNTERS && s_cnt[tid]) atomicAdd(p.counters + tid, s_cnt[tid]);
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

int trace_eval_occupancy(int* blocks_per_sm, int* threads_per_block, uint32_t n_calls, std::string* err) {
  int b = 0;
  cudaError_t e = trace_eval_wide(n_calls)
                      ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_trace_eval<kWide>, kNT, 0)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_trace_eval<0>, kNT, 0);
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
  kp.slow = L.d_slow;
  kp.res = L.results;
  kp.bnd = L.boundary;
  kp.counters = reinterpret_cast<unsigned long long*>(L.counters);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (L.counters) {
    cudaError_t e = cudaMemsetAsync(L.counters, 0, sizeof(uint64_t) * COH_N_COUNTERS, s);
    if (e != cudaSuccess) {
      *err = std::string("counter memset: ") + cudaGetErrorString(e);
      return COH_E_CUDA;
    }
  }
  const int f = (L.check_fuel ? kFuel : 0) | (L.uniform_bytes ? 0 : kBytes) |
                (L.n_arrays < COH_MAX_ARRAYS ? kArr : 0) | (trace_eval_wide(L.n_calls) ? kWide : 0);
  switch (f) {
#define COH_CASE(F) \
  case F: return launch_one<F>(L, kp, s, err);
    COH_CASE(0) COH_CASE(1) COH_CASE(2) COH_CASE(3) COH_CASE(4) COH_CASE(5) COH_CASE(6) COH_CASE(7)
    COH_CASE(8) COH_CASE(9) COH_CASE(10) COH_CASE(11) COH_CASE(12) COH_CASE(13) COH_CASE(14)
    COH_CASE(15)
#undef COH_CASE
  }
  return COH_E_ARG;
}

void trace_eval_set_smem_attr() {}

}  // namespace cohb
