// trace_eval — one thread steps one whole-array component-call trace through the
// access-mode calculus.  Replaces, per trace, cohere::run_annotated (modes.hpp:105-125):
// for each block, translate_block (modes.hpp:53-59) + run (semantics.hpp:253-287) with
// shared fuel + abstraction_correct (modes.hpp:79-90).
//
// Layout:
//   * per-thread store: one clean u16 slot per array in shared memory (internal.hpp
//     slot_word: state nibble at bits 2-5 and 8-11), lane-interleaved so a warp's lanes
//     never conflict whatever arrays they touch:
//       byte offset = (warp>>2)*16K + a*256 + ((warp>>1)&1)*128 + 4*lane + 2*(warp&1)
//       ->  bank = lane (each 128 threads of a 256-thread block own a 16 KB region).
//     Slots of arrays >= n_arrays hold the poison word (a missing key).
//   * call table: 17 rows x 64 u32, addressed by (record & 0xFC) ^ slot (internal.hpp
//     lut_word); lo16 = the slot word after the call, hi16 = signed accumulator addend.
//   * records: the record's array byte (bits 8-13) is the slot offset, its type byte
//     (bits 2-7) XOR the slot is the table offset: per call one masked logic op each,
//     plus one IMAD.HI per pair to bring the odd call down.  128-bit streaming loads of
//     8 calls, two register rings of 4 loads (32 calls each) alternating, continued
//     across traces; addresses advance by byte increments.
//   * accumulator (32-bit register): bits 0-6 steps and 7-12 transfers since the last
//     flush (every 16 calls), 13-19 number of arrays whose abstraction is violated
//     (boundary_ok <=> acc < 0x2000); a slow entry (stuck / defect / poison) adds -32768,
//     so "acc < 0" is the stop predicate.  Once it is set the accumulator, the store and
//     the boundary shift register freeze (predicated updates), and the branch to the slow
//     path is taken once per 8 calls.
//   * slow calls: the call index is recovered from a sentinel in the boundary shift
//     register and its exact outcome (StuckInfo, partial state and steps) read from a
//     host-compiled table indexed by (type, state, remaining fuel) — no interpreter on the
//     device.
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.hpp"

namespace cohb {

#ifndef COH_TE_NT
#define COH_TE_NT 256
#endif
#ifndef COH_TE_MINB_DOUBLE
#define COH_TE_MINB_DOUBLE 4
#endif
#ifndef COH_TE_MINB
#define COH_TE_MINB 5
#endif
constexpr int kNT = COH_TE_NT;  // traces (threads) per block
static_assert(kNT % 128 == 0 && kNT <= 512, "store regions hold 128 threads each");
constexpr uint32_t kStoreBytes = COH_MAX_ARRAYS * kNT * 2u;

// The block's shared memory, one struct so the hot loop can address the table and the
// store with [reg + immediate].  A CTA launched without a cluster is rank 0 of its own
// cluster, so its shared::cta window addresses are plain offsets; the first static
// variable sits after the 1 KB system-reserved area (checked at kernel entry).
struct __align__(16) TraceSmem {
  uint32_t lut[kLutEntries];
  uint16_t store[kStoreBytes / 2];
  unsigned long long cnt[COH_N_COUNTERS];
  uint64_t bytes[COH_MAX_ARRAYS];
};
constexpr uint32_t kSmemBase = 0x400u;
constexpr uint32_t kLutAddr = kSmemBase;
constexpr uint32_t kStoreAddr = kSmemBase + kLutEntries * 4u;
static_assert(kStoreAddr % 16u == 0u, "store alignment");

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

// bnd = 2*bnd + (acc >= 0x2000): with the accumulator clean (steps | transfers << 7 |
// violated << 13), the carry of acc + 0xFFFFE000 is exactly "some array's abstraction is
// violated" (abstraction_correct is false).
__device__ __forceinline__ uint32_t shift_in_violation(uint32_t bnd, uint32_t acc) {
  uint32_t out;
  asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, 0xFFFFE000;\n\taddc.u32 %0, %2, %2;\n\t}"
      : "=r"(out)
      : "r"(acc), "r"(bnd));
  return out;
}

// acc + (e >> 16, signed) on the FMA pipe: hi32(e * 2^16) + acc.
__device__ __forceinline__ uint32_t acc_add(uint32_t acc, uint32_t e) {
  uint32_t out;
  asm("mad.hi.s32 %0, %1, 65536, %2;" : "=r"(out) : "r"(e), "r"(acc));
  return out;
}

// Violation threshold after call c (0..15) of a 16-call flush window: every call adds a
// bias of 1 << 13 (the table's violation delta is stored +1 so no addend is negative),
// so "some array violated" <=> acc >= (c + 2) << 13.  Returned as the u32 addend whose
// carry-out is that test.
__host__ __device__ constexpr uint32_t viol_threshold_addend(int c) { return (uint32_t)(0x100000000ull - ((uint64_t)(c + 2) << 13)); }

// Eight calls (one 128-bit record chunk) in one asm block, so the stop predicate stays
// a predicate: per call one masked OR (slot address), LDS, one masked XOR (table
// address), LDS, a sticky sign test of the entry (slow entries are negative), then the
// predicated accumulate / store / boundary shift.  The run is live at chunk entry (the
// caller branches out after every chunk).  HALF = which half of the 16-call flush
// window the chunk is.  Returns the stop flag.
#define COH_PTX_CALL(W, T)                             \
  "{\n\t"                                              \
  "and.b32 so, " W ", 0x3F00;\n\t"                    \
  "or.b32 so, so, %4;\n\t"                            \
  "ld.shared.u16 sv, [so+%5];\n\t"                    \
  "and.b32 ix, " W ", 0xFC;\n\t"                      \
  "xor.b32 ix, ix, sv;\n\t"                           \
  "ld.shared.u32 ev, [ix+%6];\n\t"                    \
  "setp.lt.or.s32 p, ev, 0, p;\n\t"                   \
  COH_PTX_ACC                                          \
  "st.shared.u16 [so+%5], ev;\n\t"                    \
  "add.cc.u32 cy, %0, " T ";\n\t"                     \
  "addc.u32 %1, %1, %1;\n\t"                          \
  "SKIP:\n\t}\n\t"
#define COH_PTX_PAIR(R, T0, T1)        \
  COH_PTX_CALL(R, T0)                  \
  "mul.hi.u32 th, " R ", 65536;\n\t"  \
  COH_PTX_CALL("th", T1)
#define COH_PTX_CHUNK                                                                       \
  "{\n\t.reg .u32 so, sv, ix, ev, cy, th, an;\n\t.reg .pred p;\n\t"                     \
  "setp.ne.u32 p, 0, 0;\n\t"                                                               \
  COH_PTX_PAIR("%7", "%11", "%12") COH_PTX_PAIR("%8", "%13", "%14")                         \
  COH_PTX_PAIR("%9", "%15", "%16") COH_PTX_PAIR("%10", "%17", "%18")                        \
  "selp.u32 %2, 1, 0, p;\n\t}"
#define COH_PTX_OPERANDS(H)                                                                         \
  : "+r"(acc), "+r"(bnd), "=r"(stop)                                                                \
  : "r"(fuel_left), "r"(toff), "n"(kStoreAddr), "n"(kLutAddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), \
    "n"(viol_threshold_addend(8 * H + 0)), "n"(viol_threshold_addend(8 * H + 1)),                    \
    "n"(viol_threshold_addend(8 * H + 2)), "n"(viol_threshold_addend(8 * H + 3)),                    \
    "n"(viol_threshold_addend(8 * H + 4)), "n"(viol_threshold_addend(8 * H + 5)),                    \
    "n"(viol_threshold_addend(8 * H + 6)), "n"(viol_threshold_addend(8 * H + 7))                     \
  : "memory"

template <bool FUEL, int H>
__device__ __forceinline__ uint32_t run_chunk(const uint4 v, uint32_t toff, uint32_t& acc, uint32_t& bnd,
                                              int fuel_left) {
  uint32_t stop;
  if (FUEL) {  // the call's steps must fit the remaining fuel, else it is the slow call
#define COH_PTX_ACC                                 \
  "mul.hi.s32 cy, ev, 65536;\n\t"                   \
  "add.s32 an, %0, cy;\n\t"                         \
  "and.b32 cy, an, 0x7F;\n\t"                       \
  "setp.gt.or.s32 p, cy, %3, p;\n\t"                \
  "@p bra SKIP;\n\t"                                \
  "mov.u32 %0, an;\n\t"
    asm volatile(COH_PTX_CHUNK COH_PTX_OPERANDS(H));
#undef COH_PTX_ACC
  } else {
#define COH_PTX_ACC "@p bra SKIP;\n\tmul.hi.s32 cy, ev, 65536;\n\tadd.s32 %0, %0, cy;\n\t"
    asm volatile(COH_PTX_CHUNK COH_PTX_OPERANDS(H));
#undef COH_PTX_ACC
  }
  return stop;
}

// 0, computed from x so that the scheduler cannot hoist or sink what depends on it
// (ptxas would otherwise move the ring loads next to their first use).
__device__ __forceinline__ uint32_t pin_zero(uint32_t x) {
  uint32_t z;
  asm volatile("prmt.b32 %0, %1, 0, 0x4444;" : "=r"(z) : "r"(x));
  return z;
}

// FLAGS: kFuel = fuel may run out (fuel < 6 x n_calls), kBytes = non-uniform array
// sizes (per-call byte accumulation), kRing = n_calls % 32 == 0 (the record ring runs on
// into the next trace).
enum : int { kFuel = 1, kBytes = 2, kRing = 4, kDouble = 8 };

template <int FLAGS>
__global__ void __launch_bounds__(kNT, (FLAGS & kDouble) ? COH_TE_MINB_DOUBLE : COH_TE_MINB) k_trace_eval(const KParams p) {
  constexpr bool CHECK_FUEL = FLAGS & kFuel;
  constexpr bool UNIFORM = !(FLAGS & kBytes);
  constexpr bool RING = FLAGS & kRing;
  constexpr bool DOUBLE = FLAGS & kDouble;  // n_calls % 64 == 0: two register rings
  __shared__ TraceSmem sm;
  char* const stb = reinterpret_cast<char*>(sm.store);
  const char* const lutb = reinterpret_cast<const char*>(sm.lut);
  if ((uint32_t)__cvta_generic_to_shared(&sm) != kSmemBase) __trap();  // layout assumption

  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i < (uint32_t)kLutEntries; i += kNT) sm.lut[i] = p.lut[i];
  if (!UNIFORM)
    for (uint32_t i = tid; i < COH_MAX_ARRAYS; i += kNT) sm.bytes[i] = i < p.n_arrays ? p.array_bytes[i] : 0ull;
  constexpr uint32_t kInit = slot_word(COH_STATE_INITIAL);
  // slots are array-major (64 x 256 B per region): u32 word i covers array (i / 64) % 64
  for (uint32_t i = tid; i < kStoreBytes / 4u; i += kNT) {
    const uint32_t w = ((i >> 6) & 63u) < p.n_arrays ? kInit : kPoisonSlot;
    reinterpret_cast<uint32_t*>(sm.store)[i] = w | (w << 16);
  }
  if (tid < COH_N_COUNTERS) sm.cnt[tid] = 0ull;
  __syncthreads();  // the only block barrier: afterwards each thread owns its column

  const uint32_t warp = tid >> 5, lane = tid & 31u;
  // this thread's u16 column: 128 threads share a 16 KB region (64 array rows of 256 B);
  // region r sits at r << 14, so (record & 0x3F00) | toff addresses the slot
  const uint32_t toff = ((warp >> 2) << 14) | ((warp >> 1) & 1u) * 128u + 4u * lane + 2u * (warp & 1u);
  const uint32_t n = p.n_traces;  // < 2^32 (checked by the launcher)
  const uint32_t n_calls = p.n_calls;
  const uint32_t n_chunks = (n_calls + 7u) / 8u;
  const uint32_t n_groups = n_calls / 32u;
  const uint32_t stride = gridDim.x * kNT;
  // chunk c of trace u: 8 calls, one 128-bit streaming load
#define COH_REC(C, U) __ldcs(p.rec + (uint64_t)(C) * n + (U))

  uint4 ring[4];
  uint4 B[4];  // second ring of the DOUBLE variant
  if (DOUBLE)
#pragma unroll
    for (int j = 0; j < 4; ++j) B[j] = make_uint4(0u, 0u, 0u, 0u);
  bool ring_ok = false;  // ring already holds chunks 0..3 of this thread's next trace

  for (uint32_t base = blockIdx.x * kNT; base < n; base += stride) {
    const uint32_t t = base + tid;
    if (t >= n) continue;
    uint32_t acc = 0, steps = 0, xfers = 0, viol_blocks = 0;
    uint64_t tbytes = 0;
    // bnd: shift register of boundary-VIOLATION bits of the current 32-call group,
    // seeded with a sentinel 1: after k calls the sentinel sits at bit k (call 0's bit
    // at k-1); the stored boundary_ok word is its reversed complement.
    uint32_t bnd = 1u, i0 = 0;
    uint32_t status = COH_RUN_DONE, stuck_call = 0, stuck_arr = 0, stuck_eff = 0, stuck_flags = 0;
    uint32_t calls_done = n_calls;
    int fuel_left = p.fuel;
    bool stop = false;
    uint4 stuck_chunk;

    // One call (C++ form: non-uniform byte sizes and the ragged tail).  T = the record in
    // bits 0-15 (bits 16+ may hold the next record), C = its position in the 16-call
    // flush window.  Same semantics as the asm chunk.
#define COH_CALL(T, C)                                                                    \
  {                                                                                       \
    const uint32_t t_ = (T);                                                              \
    const uint32_t so_ = (t_ & 0x3F00u) | toff;                                           \
    const uint32_t s_ = *reinterpret_cast<const uint16_t*>(stb + so_);                    \
    const uint32_t e_ = *reinterpret_cast<const uint32_t*>(lutb + ((t_ & 0xFCu) ^ s_));   \
    const uint32_t an_ = acc + (uint32_t)((int32_t)e_ >> 16);                             \
    stop |= (int32_t)e_ < 0;                                                              \
    if (CHECK_FUEL) stop |= (int)(an_ & kAccSteps) > fuel_left;                           \
    if (!stop) {                                                                          \
      acc = an_;                                                                          \
      *reinterpret_cast<uint16_t*>(stb + so_) = (uint16_t)e_;                             \
      bnd = 2u * bnd + (acc + viol_threshold_addend(C) < acc ? 1u : 0u);                  \
      if (!UNIFORM) tbytes += (uint64_t)((e_ >> 23) & 3u) * sm.bytes[(t_ >> 8) & 63u];     \
    }                                                                                     \
  }
#define COH_PAIR(W, C) \
  COH_CALL(W, C)       \
  COH_CALL(__umulhi((W), 0x10000u), (C) + 1)
#define COH_CHUNK(V, H)                                                                   \
  if (UNIFORM) {                                                                          \
    stop = run_chunk<CHECK_FUEL, H>((V), toff, acc, bnd, fuel_left);                      \
  } else {                                                                                \
    COH_PAIR((V).x, 8 * H) COH_PAIR((V).y, 8 * H + 2) COH_PAIR((V).z, 8 * H + 4)           \
    COH_PAIR((V).w, 8 * H + 6)                                                            \
  }                                                                                       \
  if (__builtin_expect(stop, 0)) {                                                         \
    stuck_chunk = (V); /* the stuck call's chunk, still in registers */                    \
    goto slow_path;                                                                       \
  }
#define COH_FLUSH                                  \
  steps += acc & kAccSteps;                        \
  xfers += (acc >> kAccXferShift) & 0x3Fu;         \
  acc = (acc & kAccKeep) - (16u << kAccViolShift); \
  if (CHECK_FUEL) fuel_left = p.fuel - (int)steps;

    {
      if (!ring_ok) {
#pragma unroll
        for (int j = 0; j < 4; ++j) ring[j] = (uint32_t)j < n_chunks ? COH_REC(j, t) : make_uint4(0u, 0u, 0u, 0u);
      }
      ring_ok = false;
#define COH_GROUP_END(G)                                                          \
  /* 32 calls done: the sentinel was shifted out, call 0's violation bit is 31 */ \
  bnd = ~__brev(bnd);                                                             \
  if (p.bnd) p.bnd[(uint64_t)(G) * n + t] = bnd;                                  \
  viol_blocks += 32u - __popc(bnd);                                               \
  bnd = 1u;
      if (DOUBLE) {
        // Two register rings, A = even groups, B = odd groups.  A group's four loads are
        // issued together right after its predecessor's first chunk, so every first use
        // (which waits for all outstanding loads: they share one scoreboard) has three
        // chunks of lead.  n_groups is even; after the last pair A holds chunks 0..3 of
        // this thread's next trace (RING).
        // Addresses advance by byte increments (one 64-bit add per load, no wide
        // multiply).
        uint4* const A = ring;
        const uint64_t nb = 16ull * n;  // bytes between chunk rows
        const char* gp = reinterpret_cast<const char*>(p.rec + t) + 4u * nb;  // chunk 4(g+1) of trace t
#define COH_LOAD4(R, Q)                                                                 \
  {                                                                                     \
    const char* q_ = (Q);                                                               \
    R[0] = __ldcs(reinterpret_cast<const uint4*>(q_));                                  \
    q_ += nb;                                                                           \
    R[1] = __ldcs(reinterpret_cast<const uint4*>(q_));                                  \
    q_ += nb;                                                                           \
    R[2] = __ldcs(reinterpret_cast<const uint4*>(q_));                                  \
    q_ += nb;                                                                           \
    R[3] = __ldcs(reinterpret_cast<const uint4*>(q_));                                  \
  }
        for (uint32_t g = 0; g < n_groups; g += 2u) {
          i0 = g * 32u;
          COH_CHUNK(A[0], 0)
          COH_LOAD4(B, gp + pin_zero(bnd))  // pin: keeps the loads after chunk 0
          COH_CHUNK(A[1], 1) COH_FLUSH
          COH_CHUNK(A[2], 0)
          COH_CHUNK(A[3], 1) COH_FLUSH
          COH_GROUP_END(g)
          i0 += 32u;
          COH_CHUNK(B[0], 0)
          {
            const bool last = g + 2u >= n_groups;
            const bool nx = RING && last && t + stride < n;
            COH_LOAD4(A, (last ? reinterpret_cast<const char*>(p.rec + (nx ? t + stride : t)) : gp + 4u * nb) +
                             pin_zero(bnd))
            gp += 8u * nb;
          }
          COH_CHUNK(B[1], 1) COH_FLUSH
          COH_CHUNK(B[2], 0)
          COH_CHUNK(B[3], 1) COH_FLUSH
          COH_GROUP_END(g + 1u)
        }
#undef COH_LOAD4
      } else {
        for (uint32_t g = 0; g < n_groups; ++g) {
          i0 = g * 32u;
          // evaluate ring slot J, then refill it with the chunk 4 ahead (in the last
          // group: chunk J of this thread's next trace)
#define COH_STEP(J)                                                                   \
  {                                                                                   \
    COH_CHUNK(ring[J], ((J) & 1))                                                     \
    const uint32_t cn = 4u * (g + 1u) + (uint32_t)(J);                                \
    const bool nx_ = RING && cn >= n_chunks && t + stride < n;                        \
    ring[J] = COH_REC(cn < n_chunks ? cn : (uint32_t)(J), nx_ ? t + stride : t);      \
    if ((J) & 1) { COH_FLUSH }                                                        \
  }
          COH_STEP(0) COH_STEP(1) COH_STEP(2) COH_STEP(3)
#undef COH_STEP
          COH_GROUP_END(g)
        }
      }
#undef COH_GROUP_END
      if (RING) ring_ok = true;
      if (!RING) {
        const uint32_t tail = n_calls - n_groups * 32u;
        if (tail) {
          i0 = n_groups * 32u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t w4[4] = {ring[j].x, ring[j].y, ring[j].z, ring[j].w};
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              if (8u * j + h < tail) COH_CALL(h & 1 ? (w4[h >> 1] >> 16) : w4[h >> 1], 8 * (j & 1) + h)
            }
            if (stop) {
              stuck_chunk = ring[j];
              goto slow_path;
            }
            if (j & 1) { COH_FLUSH }
          }
          const uint32_t word = (~__brev(bnd ^ (1u << tail))) >> (32u - tail);
          viol_blocks += tail - __popc(word);
          if (p.bnd) p.bnd[(uint64_t)n_groups * n + t] = word;
        }
      }
      goto finished;
    }
#undef COH_FLUSH
#undef COH_CHUNK
#undef COH_PAIR
#undef COH_CALL

  slow_path : {
    ring_ok = false;
    uint32_t keep = 0;  // 0; ties the rings to this path (see below)
    if (DOUBLE) {
      // The rings are live on this path too, so the scheduler cannot sink their loads
      // past the slow-path branches (which would leave them no lead before first use).
#pragma unroll
      for (int j = 0; j < 4; ++j) keep ^= ring[j].x ^ B[j].x;  // one word per 128-bit load suffices
      keep = pin_zero(keep);
    }
    // which call: k calls of this 32-group completed (sentinel position)
    const uint32_t k = 31u - __clz(bnd);
    const uint32_t i = i0 + k;
    const uint4 chunk = stuck_chunk;
    const uint32_t q = i & 7u;  // the call within its chunk (selects, no local array)
    const uint32_t wsel = (q & 4u) ? ((q & 2u) ? chunk.w : chunk.z) : ((q & 2u) ? chunk.y : chunk.x);
    const uint32_t r = (wsel >> (16u * (q & 1u))) & 0xFFFFu;
    const uint32_t a = (r >> 8) & 63u, type = (r >> 2) & 63u;
    uint16_t* const sp = reinterpret_cast<uint16_t*>(stb + ((r & 0x3F00u) | toff));
    const uint32_t s = *sp;  // untouched: the store froze before this call
    // the accumulator froze before this call too (its bias does not reach bits 0-12)
    steps += acc & kAccSteps;
    xfers += (acc >> kAccXferShift) & 0x3Fu;
    // exact outcome from the host-compiled slow table (type, state, remaining fuel)
    const int rem_i = p.fuel - (int)steps;
    const uint32_t rem = rem_i <= 0 ? 0u : (rem_i >= 7 ? 7u : (uint32_t)rem_i);
    const bool missing = s == kPoisonSlot;  // array id >= n_arrays
    const uint32_t info = missing ? (uint32_t)COH_RUN_DEFECT : __ldg(p.slow + slow_index(type, slot_state(s), rem));
    const uint32_t so_steps = (info >> 2) & 7u, so_xf = (info >> 5) & 3u;
    if (!missing) *sp = (uint16_t)slot_word((info >> 7) & 15u);
    steps += so_steps;
    xfers += so_xf;
    if (!UNIFORM && !missing) tbytes += (uint64_t)so_xf * sm.bytes[a];
    status = info & 3u;
    stuck_call = i;
    stuck_arr = a;
    stuck_eff = (info >> 11) & 7u;
    stuck_flags = ((info >> 14) & 15u) | keep;
    calls_done = i;
    const uint32_t word = k ? ((~__brev(bnd ^ (1u << k))) >> (32u - k)) : 0u;
    viol_blocks += k - __popc(word);
    if (p.bnd) {
      const uint32_t g = i / 32u;
      p.bnd[(uint64_t)g * n + t] = word;
      for (uint32_t w = g + 1; w < (n_calls + 31u) / 32u; ++w) p.bnd[(uint64_t)w * n + t] = 0u;
    }
  }
  finished : {
    uint32_t sw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int a = 0; a < COH_MAX_ARRAYS; ++a) {
      if (a < (int)p.n_arrays) {
        uint16_t* const wp = reinterpret_cast<uint16_t*>(stb + a * 256 + toff);
        const uint32_t w = *wp;
        *wp = (uint16_t)kInit;  // reset for this thread's next trace
        const int sh = 4 * (a & 7) - 8;  // state nibble at slot bits 8-11
        sw[a >> 3] |= (sh >= 0 ? (w << sh) : (w >> -sh)) & (15u << (4 * (a & 7)));
      }
    }
    const uint64_t tb = UNIFORM ? (uint64_t)xfers * p.bytes_uniform : tbytes;
    uint4* out = reinterpret_cast<uint4*>(p.res + t);
    __stcs(out + 0, make_uint4(sw[0], sw[1], sw[2], sw[3]));
    __stcs(out + 1, make_uint4(sw[4], sw[5], sw[6], sw[7]));
    __stcs(out + 2, make_uint4((uint32_t)tb, (uint32_t)(tb >> 32), steps, xfers));
    __stcs(out + 3, make_uint4(calls_done, viol_blocks, stuck_call,
                               status | (stuck_arr << 8) | (stuck_eff << 16) | (stuck_flags << 24)));
    if (p.counters) {  // fused counter reduction: warp redux, one shared atomic per warp
      const uint32_t m = __activemask();
      const bool leader = (lane == (uint32_t)(__ffs(m) - 1));
      uint32_t v[9] = {status == COH_RUN_STUCK, status == COH_RUN_FUEL_EXHAUSTED, viol_blocks != 0u,
                       status == COH_RUN_DEFECT, steps, xfers, viol_blocks, calls_done, 1u};
      const int slot[9] = {0, 1, 2, 3, 4, 5, 7, 8, 9};
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        v[k] = __reduce_add_sync(m, v[k]);
        if (leader && v[k]) atomicAdd(&sm.cnt[slot[k]], (unsigned long long)v[k]);
      }
      if (UNIFORM) {  // bytes = transfers x size: one multiply by the leader
        if (leader && v[5]) atomicAdd(&sm.cnt[6], (unsigned long long)v[5] * p.bytes_uniform);
      } else if (tb) {  // non-uniform sizes: per-lane shared atomic
        atomicAdd(&sm.cnt[6], (unsigned long long)tb);
      }
    }
  }
  }
#undef COH_REC
  if (p.counters) {
    __syncthreads();
    if (tid < COH_N_COUNTERS && sm.cnt[tid]) atomicAdd(p.counters + tid, sm.cnt[tid]);
  }
}

static bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && *v != '0';
}

template <int F>
static int launch_one(const TraceLaunch& L, const KParams& kp, cudaStream_t s, std::string* err) {
  static int occ = 0;  // resident blocks per SM of this variant
  if (!occ) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trace_eval<F>, kNT, 0);
    if (e != cudaSuccess || occ < 1) {
      *err = std::string("trace_eval occupancy: ") + cudaGetErrorString(e);
      occ = 0;
      return COH_E_CUDA;
    }
  }
  // persistent grid: every block runs the same number of rounds
  const uint64_t need = (L.n_traces + kNT - 1) / kNT;
  const uint64_t cap = (uint64_t)L.sms * (uint64_t)occ;
  const uint64_t rounds = (need + cap - 1) / cap;
  const int grid = (int)((need + rounds - 1) / rounds);
  k_trace_eval<F><<<grid, kNT, 0, s>>>(kp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("trace_eval launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

int trace_eval_occupancy(int* blocks_per_sm, int* threads_per_block, uint32_t n_calls, std::string* err) {
  int b = 0;
  const bool dbl = n_calls % 64u == 0u && n_calls >= 64u && !getenv_flag("COH_TE_SINGLE");
  cudaError_t e = dbl ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_trace_eval<kRing | kDouble>, kNT, 0)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_trace_eval<kRing>, kNT, 0);
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
  if (L.n_traces >= (1ull << 32) - 2u * 148u * kNT * 16u) {
    *err = "trace_eval: n_traces must be < 2^32 per launch";
    return COH_E_ARG;
  }
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
                (L.n_calls % 32u == 0u && L.n_calls >= 32u ? kRing : 0) |
                (L.n_calls % 64u == 0u && L.n_calls >= 64u && !getenv_flag("COH_TE_SINGLE") ? kDouble : 0);
  switch (f) {
#define COH_CASE(F) \
  case F: return launch_one<F>(L, kp, s, err);
    COH_CASE(0) COH_CASE(1) COH_CASE(2) COH_CASE(3) COH_CASE(4) COH_CASE(5) COH_CASE(6) COH_CASE(7)
    COH_CASE(12) COH_CASE(13) COH_CASE(14) COH_CASE(15)
#undef COH_CASE
  }
  return COH_E_ARG;
}

void trace_eval_set_smem_attr() {}

}  // namespace cohb
