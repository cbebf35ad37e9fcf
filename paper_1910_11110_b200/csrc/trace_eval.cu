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
#include <cstring>

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
  uint32_t last;  // this block finished the launch
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
  uint32_t uniform;  // array sizes are all bytes_uniform (else array_bytes)
  uint64_t bytes_uniform;
  const uint64_t* array_bytes;
  const uint32_t* lut;
  const uint32_t* slow;
  coh_trace_result* res;
  uint32_t* bnd;
  unsigned long long* counters;  // optional fused COH_N_COUNTERS reduction (k_trace_eval: written, not added)
  unsigned int* ticket;          // dynamic trace batches handed out after the first round (in *slot)
  LaunchSlot* slot;              // this launch's ticket / counter sums (zero on entry, zeroed again on exit)
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
  COH_PTX_STORE_EARLY                                  \
  "setp.lt.or.s32 p, ev, 0, p;\n\t"                   \
  COH_PTX_ACC                                          \
  COH_PTX_STORE_LATE                                   \
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
    "n"(viol_threshold_addend(8 * H + 6)), "n"(viol_threshold_addend(8 * H + 7))                    \
  : "memory"

template <bool FUEL, int H>
__device__ __forceinline__ uint32_t run_chunk(const uint4 v, uint32_t toff, uint32_t& acc, uint32_t& bnd,
                                              int fuel_left) {
  uint32_t stop;
  if (FUEL) {  // the call's steps must fit the remaining fuel, else it is the slow call
#define COH_PTX_STORE_EARLY ""
#define COH_PTX_STORE_LATE "st.shared.u16 [so+%5], ev;\n\t"
#define COH_PTX_ACC                                 \
  "mul.hi.s32 cy, ev, 65536;\n\t"                   \
  "add.s32 an, %0, cy;\n\t"                         \
  "and.b32 cy, an, 0x7F;\n\t"                       \
  "setp.gt.or.s32 p, cy, %3, p;\n\t"                \
  "@p bra SKIP;\n\t"                                \
  "mov.u32 %0, an;\n\t"
    asm volatile(COH_PTX_CHUNK COH_PTX_OPERANDS(H));
#undef COH_PTX_ACC
#undef COH_PTX_STORE_EARLY
#undef COH_PTX_STORE_LATE
  } else {
#ifdef COH_TE_LATE_STS
#define COH_PTX_STORE_EARLY ""
#define COH_PTX_STORE_LATE "st.shared.u16 [so+%5], ev;\n\t"
#else
    // The store goes out before this call's own stop test, predicated on the stop of the
    // calls before it: a slow entry's low half is the slot word it was read from (the store
    // is unchanged by a stuck call / a missing key), so writing it back is harmless, and the
    // next call's slot load no longer waits for the sign test (one ALU latency less per call
    // on the store -> load chain).  Not with fuel: a call stopped by the fuel has a regular
    // entry.
#define COH_PTX_STORE_EARLY "@!p st.shared.u16 [so+%5], ev;\n\t"
#define COH_PTX_STORE_LATE ""
#endif
#define COH_PTX_ACC "@p bra SKIP;\n\tmul.hi.s32 cy, ev, 65536;\n\tadd.s32 %0, %0, cy;\n\t"
    asm volatile(COH_PTX_CHUNK COH_PTX_OPERANDS(H));
#undef COH_PTX_ACC
#undef COH_PTX_STORE_EARLY
#undef COH_PTX_STORE_LATE
  }
  return stop;
}

// One 128-bit chunk of records.  Read once and never written during the launch: through
// the non-coherent path without allocating in L1 (measured 1.8% faster than ld.global.cs
// on C2, same L1 data-pipe wavefronts).
#ifndef COH_TE_LOAD_HINT
#define COH_TE_LOAD_HINT ""
#endif
__device__ __forceinline__ uint4 rec_load(const uint4* a) {
#ifdef COH_TE_LOAD_CS
  return __ldcs(a);
#else
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate" COH_TE_LOAD_HINT ".v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(a));
  return v;
#endif
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
  constexpr int kRingLen = 4;
  __shared__ TraceSmem sm;
  char* const stb = reinterpret_cast<char*>(sm.store);
  const char* const lutb = reinterpret_cast<const char*>(sm.lut);
  if ((uint32_t)__cvta_generic_to_shared(&sm) != kSmemBase) __trap();  // layout assumption

  const uint32_t tid = threadIdx.x;
  // a COH_BATCH_OVERLAP successor may be scheduled as soon as every block of this launch
  // has started (its blocks then take the SMs this launch's last blocks free)
  asm volatile("griddepcontrol.launch_dependents;" :::);
#ifdef COH_TE_TIMELINE
  unsigned long long tl0, tl1, tl2;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl0));
#endif
  const uint32_t n = p.n_traces;  // < 2^32 (checked by the launcher)
  const uint32_t n_calls = p.n_calls;
  const uint32_t n_chunks = (n_calls + 7u) / 8u;
  // chunk c of trace u: 8 calls, one 128-bit streaming load
#define COH_REC(C, U) rec_load(p.rec + (uint64_t)(C) * n + (U))
  // The first trace's record loads and the table loads go out before the block's set-up,
  // so their latency overlaps it (the launch's fixed cost).
  uint4 ring[kRingLen];
  bool ring_ok = false;  // ring already holds chunks 0..kRingLen-1 of this thread's next trace
  if (blockIdx.x * kNT + tid < n) {
#pragma unroll
    for (int j = 0; j < kRingLen; ++j)
      ring[j] = (uint32_t)j < n_chunks ? COH_REC(j, blockIdx.x * kNT + tid) : make_uint4(0u, 0u, 0u, 0u);
    ring_ok = true;
  }
  {
    constexpr uint32_t kQ = kLutEntries / 4u, kIt = (kQ + kNT - 1) / kNT;
    static_assert(kLutEntries % 4u == 0u, "table in 16-byte pieces");
    uint4 v[kIt];
#pragma unroll
    for (uint32_t j = 0; j < kIt; ++j)
      if (tid + j * kNT < kQ) v[j] = __ldg(reinterpret_cast<const uint4*>(p.lut) + tid + j * kNT);
#pragma unroll
    for (uint32_t j = 0; j < kIt; ++j)
      if (tid + j * kNT < kQ) reinterpret_cast<uint4*>(sm.lut)[tid + j * kNT] = v[j];
  }
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
#ifdef COH_TE_TIMELINE
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl1));
#endif

  const uint32_t warp = tid >> 5, lane = tid & 31u;
  // counters: packed warp sums need n_calls <= 256 (6 steps per call per lane fit 16 bits)
  const bool packed_cnt = n_calls <= 256u;
  uint32_t cnt_acc = 0;  // lane k < 10: warp total of counter k over this warp's traces
  // this thread's u16 column: 128 threads share a 16 KB region (64 array rows of 256 B);
  // region r sits at r << 14, so (record & 0x3F00) | toff addresses the slot
  const uint32_t toff = ((warp >> 2) << 14) | ((warp >> 1) & 1u) * 128u + 4u * lane + 2u * (warp & 1u);
  const uint32_t n_groups = n_calls / 32u;
  const uint32_t stride = gridDim.x * kNT;

  uint4 B[4];  // second ring of the DOUBLE variant
  if (DOUBLE)
#pragma unroll
    for (int j = 0; j < 4; ++j) B[j] = make_uint4(0u, 0u, 0u, 0u);

  // Work distribution: a warp's first two batches of 32 traces are static (the grid
  // covers [0, 2 stride)); later batches come from a global ticket, requested two batches
  // ahead (nobody waits for the atomic), so warps the scheduler favours take more batches
  // and every SM stays busy to the end (static striding left blocks finishing between 118
  // and 176 us of a 182 us launch).  Without a ticket (short launches) striding is static.
  uint32_t req = 0;
  for (uint32_t cur = blockIdx.x * kNT + (tid & ~31u), nxt = cur + stride; cur < n;
       cur = nxt, nxt = p.ticket ? __shfl_sync(0xFFFFFFFFu, req, 0) + 2u * stride : nxt + stride) {
    if (p.ticket && lane == 0) req = atomicAdd(p.ticket, 32u);  // the batch after next
    const uint32_t t = cur + lane;
    const uint32_t tn = nxt + lane;  // this thread's next trace (the ring runs on into it)
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
        for (int j = 0; j < kRingLen; ++j) ring[j] = (uint32_t)j < n_chunks ? COH_REC(j, t) : make_uint4(0u, 0u, 0u, 0u);
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
    R[0] = rec_load(reinterpret_cast<const uint4*>(q_));                                  \
    q_ += nb;                                                                           \
    R[1] = rec_load(reinterpret_cast<const uint4*>(q_));                                  \
    q_ += nb;                                                                           \
    R[2] = rec_load(reinterpret_cast<const uint4*>(q_));                                  \
    q_ += nb;                                                                           \
    R[3] = rec_load(reinterpret_cast<const uint4*>(q_));                                  \
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
            const bool nx = RING && last && tn < n;
            COH_LOAD4(A, (last ? reinterpret_cast<const char*>(p.rec + (nx ? tn : t)) : gp + 4u * nb) +
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
    const bool nx_ = RING && cn >= n_chunks && tn < n;                                \
    ring[J] = COH_REC(cn < n_chunks ? cn : (uint32_t)(J), nx_ ? tn : t);              \
    if ((J) & 1) { COH_FLUSH }                                                        \
  }
          COH_STEP(0) COH_STEP(1) COH_STEP(2) COH_STEP(3)
#undef COH_STEP
          COH_GROUP_END(g)
        }
      }
#undef COH_GROUP_END
      if (RING) ring_ok = true;
      if constexpr (!RING) {
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
    // the final store, nibble-packed, and every slot reset for this thread's next trace
    uint32_t sw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t init;  // kInit in a register (else ptxas rematerialises it before every store)
    asm volatile("mov.u32 %0, %1;" : "=r"(init) : "n"(kInit));
#define COH_SLOT_OUT(A)                                                                \
  {                                                                                    \
    uint16_t* const wp = reinterpret_cast<uint16_t*>(stb + (A) * 256 + toff);          \
    const uint32_t w = *wp;                                                            \
    *wp = (uint16_t)init;                                                              \
    const int sh = 4 * ((A) & 7) - 8; /* state nibble at slot bits 8-11 */             \
    sw[(A) >> 3] |= (sh >= 0 ? (w << sh) : (w >> -sh)) & (15u << (4 * ((A) & 7)));    \
  }
    if (p.n_arrays == COH_MAX_ARRAYS) {  // all 64 arrays (C2): no per-array predicate
#pragma unroll
      for (int a = 0; a < COH_MAX_ARRAYS; ++a) COH_SLOT_OUT(a)
    } else {
#pragma unroll
      for (int a = 0; a < COH_MAX_ARRAYS; ++a)
        if (a < (int)p.n_arrays) COH_SLOT_OUT(a)
    }
#undef COH_SLOT_OUT
    {  // is_unsafe (program.hpp:166-170): a live array whose concrete or abstract pair is (I,I)
      // (bit 0 / bit 2 of ~(nibble | nibble >> 1)); arrays >= n_arrays hold nibble 0
      uint32_t bad = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) bad |= ~(sw[k] | (sw[k] >> 1)) & 0x55555555u;
      if (bad && p.n_arrays < COH_MAX_ARRAYS) {  // (rare) mask the undeclared arrays' empty nibbles
        bad = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // constant word indices: sw stays in registers
          const int live = (int)p.n_arrays - 8 * k;  // arrays of word k that are declared
          const uint32_t m = live >= 8 ? 0x55555555u : live <= 0 ? 0u : 0x55555555u & ((1u << (4 * live)) - 1u);
          bad |= ~(sw[k] | (sw[k] >> 1)) & m;
        }
      }
      if (bad) stuck_flags |= COH_FLAG_UNSAFE;
    }
    const uint64_t tb = UNIFORM ? (uint64_t)xfers * p.bytes_uniform : tbytes;
    uint4* out = reinterpret_cast<uint4*>(p.res + t);
    __stcs(out + 0, make_uint4(sw[0], sw[1], sw[2], sw[3]));
    __stcs(out + 1, make_uint4(sw[4], sw[5], sw[6], sw[7]));
    __stcs(out + 2, make_uint4((uint32_t)tb, (uint32_t)(tb >> 32), steps, xfers));
    __stcs(out + 3, make_uint4(calls_done, viol_blocks, stuck_call,
                               status | (stuck_arr << 8) | (stuck_eff << 16) | (stuck_flags << 24)));
    const uint32_t m = p.counters ? __activemask() : 0u;
    if (packed_cnt && m == 0xFFFFFFFFu) {
      // a full warp: three warp reductions of packed fields (per-warp sums fit their 6 /
      // 16 bits for n_calls <= 256), then lane k keeps counter k's running warp total in
      // a register; the shared atomics happen once per thread, after the last trace
      const uint32_t fl = __reduce_add_sync(
          m, (status == COH_RUN_STUCK) | (uint32_t)(status == COH_RUN_FUEL_EXHAUSTED) << 6 |
                 (uint32_t)(viol_blocks != 0u) << 12 | (uint32_t)(status == COH_RUN_DEFECT) << 18 |
                 (uint32_t)((stuck_flags & COH_FLAG_UNSAFE) != 0u) << 24);
      const uint32_t sx = __reduce_add_sync(m, steps | xfers << 16);
      const uint32_t vc = __reduce_add_sync(m, viol_blocks | calls_done << 16);
      // lanes 0-3 stuck / fuel / violating traces / defect, 4-5 steps / transfers,
      // 6-7 violating blocks / calls done, 8 traces, 9 unsafe
      const uint32_t w = lane < 4u || lane == 9u ? fl : lane < 6u ? sx : vc;
      const uint32_t sh = lane < 4u ? 6u * lane : lane == 9u ? 24u : 16u * (lane & 1u);
      const uint32_t v = lane == 8u ? (uint32_t)__popc(m) : (w >> sh) & (lane < 4u || lane == 9u ? 63u : 0xFFFFu);
      cnt_acc += lane < 10u ? v : 0u;
      if (!UNIFORM && tb) atomicAdd(&sm.cnt[6], (unsigned long long)tb);
    } else if (m) {  // partial warps: per-counter warp reductions, one shared atomic per warp
      const bool leader = (lane == (uint32_t)(__ffs(m) - 1));
      uint32_t v[10] = {status == COH_RUN_STUCK, status == COH_RUN_FUEL_EXHAUSTED, viol_blocks != 0u,
                        status == COH_RUN_DEFECT, steps, xfers, viol_blocks, calls_done, 1u,
                        (stuck_flags & COH_FLAG_UNSAFE) != 0u};
      const int slot[10] = {0, 1, 2, 3, 4, 5, 7, 8, 9, 10};
#pragma unroll
      for (int k = 0; k < 10; ++k) {
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
    if (packed_cnt && lane < 10u && cnt_acc) {
      const int slot = lane < 6u ? (int)lane : (int)lane + 1;  // 6 = bytes, below
      atomicAdd(&sm.cnt[slot], (unsigned long long)cnt_acc);
      if (UNIFORM && lane == 5u) atomicAdd(&sm.cnt[6], (unsigned long long)cnt_acc * p.bytes_uniform);
    }
    __syncthreads();
    if (tid < COH_N_COUNTERS && sm.cnt[tid]) atomicAdd(&p.slot->cnt[tid], sm.cnt[tid]);
  }
  if (p.counters || p.ticket) {  // the last block publishes the sums and zeroes the slot
    __threadfence();
    __syncthreads();
    if (tid == 0) sm.last = atomicAdd(&p.slot->done, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (sm.last) {
      __threadfence();
      if (tid < COH_N_COUNTERS) {
        const unsigned long long v = atomicExch(&p.slot->cnt[tid], 0ull);
        if (p.counters) p.counters[tid] = v;
      }
      if (tid == 0) {
        p.slot->ticket = 0u;
        p.slot->done = 0u;
      }
    }
  }
#ifdef COH_TE_TIMELINE  // per block: entry, after set-up, exit (debug builds only)
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl2));
  if (tid == 0 && p.bnd) {
    unsigned long long* tl = reinterpret_cast<unsigned long long*>(p.bnd) + 3 * blockIdx.x;
    tl[0] = tl0, tl[1] = tl1, tl[2] = tl2;
  }
#endif
}

// ---------------------------------------------------------------------------------
// k_trace_scan — the latency path for few, long single-array traces (BASELINE C1: one
// trace of 1000 calls on one array).  One thread per trace is a chain of n_calls
// dependent table lookups (~50 ns each); here a block evaluates one trace with the calls
// spread over its threads.  Each call is a function on the 16 states of the array, so the
// state entering every call is a prefix composition — an associative scan:
//   1. each thread composes the maps of its kScanCPT consecutive calls (16 start states
//      stepped through the table in parallel; a start state that reaches a slow entry
//      — stuck / malformed / missing key — is flagged);
//   2. a block scan of those maps gives every thread the state entering its first call;
//   3. each thread re-runs its calls from that state (steps, transfers, boundary bits);
//      block scans of the steps find the fuel cut-off, a block min the first slow call
//      (= the stop of run_annotated, modes.hpp:118-121), resolved by the same host-
//      compiled slow table as the per-thread kernel.
// Results are field-for-field those of k_trace_eval (tests run both on the same inputs).
#ifndef COH_SCAN_CPT
#define COH_SCAN_CPT 4
#endif
constexpr int kScanCPT = COH_SCAN_CPT;  // consecutive calls per thread (half or all of a 16-byte chunk)
constexpr int kScanNT = 1024 / kScanCPT;  // threads per trace (1024 calls per pass)
static_assert(kScanCPT == 4 || kScanCPT == 8, "a thread's calls are half or all of one record chunk");
constexpr uint32_t kGroupThreads = 32u / kScanCPT;  // threads per 32-call boundary word
constexpr uint32_t kScanPass = kScanNT * kScanCPT;  // 1024

// A state map: byte s of the four words = the state reached from start state s (bits
// 0-3), bit 4 set when a slow entry was reached on the way.  Composition is four PRMT
// lookups per word (the byte-permute unit indexes 8-byte tables).
struct StateMap {
  uint32_t b[4];
};
__device__ __forceinline__ StateMap identity_map() { return StateMap{{0x03020100u, 0x07060504u, 0x0B0A0908u, 0x0F0E0D0Cu}}; }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// m[i_k] for the four index bytes i_k (0..15) of idx
__device__ __forceinline__ uint32_t lookup4(const StateMap& m, uint32_t idx) {
  const uint32_t pairs = idx | (idx >> 4);                     // bytes 0 and 2: two indices each
  const uint32_t sel = prmt(pairs, 0u, 0x0020u) & 0x7777u;     // four 3-bit byte selectors
  const uint32_t lo = prmt(m.b[0], m.b[1], sel), hi = prmt(m.b[2], m.b[3], sel);
  const uint32_t upper = prmt(idx << 4, 0u, 0xBA98u);          // 0xFF where index bit 3 is set
  return (hi & upper) | (lo & ~upper);
}

__device__ __forceinline__ StateMap compose(const StateMap& a, const StateMap& b) {  // a, then b
  StateMap c;
#pragma unroll
  for (int g = 0; g < 4; ++g) c.b[g] = lookup4(b, a.b[g] & 0x0F0F0F0Fu) | (a.b[g] & 0x10101010u);
  return c;
}

__device__ __forceinline__ uint32_t apply_map(const StateMap& m, uint32_t s) {  // byte s
  const bool up = s & 8u;
  return prmt(up ? m.b[2] : m.b[0], up ? m.b[3] : m.b[1], s & 7u) & 0xFFu;
}

__device__ __forceinline__ StateMap shfl_up_map(const StateMap& m, int o) {
  StateMap r;
#pragma unroll
  for (int g = 0; g < 4; ++g) r.b[g] = __shfl_up_sync(0xFFFFFFFFu, m.b[g], o);
  return r;
}

// bit s: state s violates its abstraction (!leq(abstract, concrete), modes.hpp:71-75)
__host__ __device__ constexpr uint32_t violating_mask() {
  uint32_t m = 0;
  for (uint32_t s = 0; s < 16; ++s) {
    const uint32_t a = s >> 2, c = s & 3u;
    if (!(a == c || (c == 3u && (a == 1u || a == 2u)))) m |= 1u << s;
  }
  return m;
}
constexpr uint32_t kViolMask = violating_mask();

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {  // kScanNT threads; red: kScanNT / 32
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  T t = 0;
#pragma unroll
  for (int w = 0; w < kScanNT / 32; ++w) t += red[w];
  return t;
}

__device__ __forceinline__ uint32_t rec_of(const uint32_t (&w4)[4], uint32_t k) {  // k compile-time after unrolling
  return (w4[k >> 1] >> (16u * (k & 1u))) & 0xFFFFu;
}

#ifdef COH_SCAN_PROFILE
#define COH_TS(K) \
  if (threadIdx.x == 0) ts[K] = clock64();
#else
#define COH_TS(K)
#endif
__global__ void __launch_bounds__(kScanNT) k_trace_scan(const KParams p) {
#ifdef COH_SCAN_PROFILE
  long long ts[8];
  COH_TS(0)
#endif
  __shared__ __align__(16) uint32_t lut[kLutEntries];
  __shared__ StateMap wmap[kScanNT / 32];
  __shared__ uint32_t wred[kScanNT / 32];
  __shared__ unsigned long long wred64[kScanNT / 32];
  __shared__ uint32_t stop_at, s_end, slow_out[5];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t t = blockIdx.x, n = (uint32_t)p.n_traces, nc = p.n_calls;
  const char* const lutb = reinterpret_cast<const char*>(lut);
  // the first pass's records and the table: every load in flight at once
  // this thread's calls: chunk (c0 / 8), all of it (CPT 8) or its half (c0 / 4) & 1 (CPT 4)
  auto load_calls = [&](uint32_t c0) {
    if (c0 >= nc) return make_uint4(0u, 0u, 0u, 0u);
    if (kScanCPT == 8) return __ldg(p.rec + (uint64_t)(c0 / 8u) * n + t);
    const uint2 h = __ldg(reinterpret_cast<const uint2*>(p.rec + (uint64_t)(c0 / 8u) * n + t) + ((c0 >> 2) & 1u));
    return make_uint4(h.x, h.y, 0u, 0u);
  };
  uint4 ch = load_calls(tid * kScanCPT);
  {
    constexpr uint32_t kQ = kLutEntries / 4u, kIt = (kQ + kScanNT - 1) / kScanNT;
    static_assert(kLutEntries % 4u == 0u, "table in 16-byte pieces");
    uint4 v[kIt];
#pragma unroll
    for (uint32_t j = 0; j < kIt; ++j)
      if (tid + j * kScanNT < kQ) v[j] = __ldg(reinterpret_cast<const uint4*>(p.lut) + tid + j * kScanNT);
#pragma unroll
    for (uint32_t j = 0; j < kIt; ++j)
      if (tid + j * kScanNT < kQ) reinterpret_cast<uint4*>(lut)[tid + j * kScanNT] = v[j];
  }
  __syncthreads();
  const uint64_t xbytes = p.uniform ? p.bytes_uniform : p.array_bytes[0];
  uint32_t s_cur = COH_STATE_INITIAL, steps = 0, xfers = 0, viol_blocks = 0, calls_done = nc;
  uint32_t status = COH_RUN_DONE, stuck_call = 0, stuck_arr = 0, stuck_eff = 0, stuck_flags = 0;
  bool stopped = false;
  uint32_t base = 0;
  for (; base < nc && !stopped; base += kScanPass) {
    const uint32_t c0 = base + tid * kScanCPT;
    const uint32_t cnt = c0 < nc ? min((uint32_t)kScanCPT, nc - c0) : 0u;
    if (base) ch = load_calls(c0);
    const uint32_t w4[4] = {ch.x, ch.y, ch.z, ch.w};
    COH_TS(1)
    // 1. this thread's map: the 16 start states stepped through its calls in parallel.
    //    Slot words (internal.hpp) make the table address one XOR, and an entry's low
    //    half is the next slot word; slow entries are negative.
    uint32_t cur[16], sl[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) cur[s] = slot_word((uint32_t)s), sl[s] = 0u;
    uint32_t miss = 0;
#pragma unroll
    for (int k = 0; k < kScanCPT; ++k) {
      if ((uint32_t)k < cnt) {
        const uint32_t r = rec_of(w4, k), tw = r & 0xFCu;
        if (((r >> 8) & 63u) >= p.n_arrays) miss = 0x80000000u;  // missing key
#pragma unroll
        for (int s = 0; s < 16; ++s) {
          const uint32_t e = *reinterpret_cast<const uint32_t*>(lutb + ((cur[s] ^ tw) & 0xFFFFu));
          sl[s] |= e;
          cur[s] = e;
        }
      }
    }
    StateMap m;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      m.b[g] = 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int s = 4 * g + k;
        m.b[g] |= (((cur[s] >> 8) & 15u) | (((sl[s] | miss) >> 31) << 4)) << (8 * k);
      }
    }
    COH_TS(2)
    // 2. inclusive block scan of the maps; exclusive = the map before this thread's calls
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const StateMap y = shfl_up_map(m, o);
      if (lane >= (uint32_t)o) m = compose(y, m);
    }
    if (lane == 31) wmap[warp] = m;
    __syncthreads();
    StateMap pre = identity_map();
    for (uint32_t w = 0; w < warp; ++w) pre = compose(pre, wmap[w]);
    StateMap ex = shfl_up_map(m, 1);
    ex = lane ? compose(pre, ex) : pre;
    const uint32_t v_in = apply_map(ex, s_cur);
    const bool dead = v_in & 0x10u;  // an earlier call of the pass is slow
    COH_TS(3)
    // 3. re-run this thread's calls from the entry state: cumulative steps / transfers
    //    after call k, state before call k, boundary bits
    uint32_t cs[kScanCPT], cx[kScanCPT], sb[kScanCPT];
    uint32_t ok_bits = 0, vbits = 0, first_slow = kScanCPT;
    uint32_t sw = slot_word(v_in & 15u), acc = 0, xacc = 0;
#pragma unroll
    for (int k = 0; k < kScanCPT; ++k) {
      sb[k] = (sw >> 8) & 15u;
      if ((uint32_t)k < cnt && first_slow == kScanCPT && !dead) {
        const uint32_t r = rec_of(w4, k);
        const uint32_t e = *reinterpret_cast<const uint32_t*>(lutb + ((sw ^ (r & 0xFCu)) & 0xFFFFu));
        if ((int32_t)e < 0 || ((r >> 8) & 63u) >= p.n_arrays) {
          first_slow = k;
        } else {
          acc += (e >> 16) & kAccSteps;
          xacc += (e >> (16 + kAccXferShift)) & 0x3Fu;
          sw = e;
          if ((kViolMask >> ((e >> 8) & 15u)) & 1u) vbits |= 1u << k;
          else ok_bits |= 1u << k;
        }
      }
      cs[k] = acc;
      cx[k] = xacc;
    }
    COH_TS(4)
    // fuel: the steps of the pass before this thread's calls (exclusive block scan); a
    // call is the slow one if its steps overrun the fuel left
    uint32_t ps = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, ps, o);
      if (lane >= (uint32_t)o) ps += y;
    }
    if (lane == 31) wred[warp] = ps;
    if (tid == 0) stop_at = 0xFFFFFFFFu;
    __syncthreads();
    uint32_t before = ps - acc;
    for (uint32_t w = 0; w < warp; ++w) before += wred[w];
    const int fuel_left = p.fuel - (int)steps;
    uint32_t stop_k = first_slow;
#pragma unroll
    for (int k = kScanCPT - 1; k >= 0; --k)
      if ((uint32_t)k < first_slow && (int)(before + cs[k]) > fuel_left) stop_k = (uint32_t)k;
    if (stop_k < cnt) atomicMin(&stop_at, c0 + stop_k);
    if (cnt && c0 + cnt == min(nc, base + kScanPass)) s_end = (sw >> 8) & 15u;
    __syncthreads();
    const uint32_t i = stop_at;  // the pass's first slow call, if any
    const uint32_t keep = i == 0xFFFFFFFFu ? cnt : (i <= c0 ? 0u : min(cnt, i - c0));  // completed calls
    const uint32_t km = (1u << keep) - 1u;
    if (p.bnd) {  // boundary words: kGroupThreads threads per 32-call group
      uint32_t word = (ok_bits & km) << (kScanCPT * (tid & (kGroupThreads - 1u)));
#pragma unroll
      for (uint32_t o = 1; o < kGroupThreads; o <<= 1) word |= __shfl_xor_sync(0xFFFFFFFFu, word, o);
      if ((tid & (kGroupThreads - 1u)) == 0u && c0 < nc) p.bnd[(uint64_t)(c0 / 32u) * n + t] = word;
    }
    uint32_t ks = 0, kx = 0, s_slow = 0;  // cs / cx at call keep - 1, state before call keep
#pragma unroll
    for (int k = 0; k < kScanCPT; ++k) {
      if ((uint32_t)k + 1u == keep) ks = cs[k], kx = cx[k];
      if ((uint32_t)k == keep) s_slow = sb[k];
    }
    COH_TS(5)
    const unsigned long long sums = block_sum<unsigned long long>(
        (unsigned long long)ks | ((unsigned long long)kx << 20) | ((unsigned long long)__popc(vbits & km) << 40), wred64);
    steps += (uint32_t)(sums & 0xFFFFFull);
    xfers += (uint32_t)((sums >> 20) & 0xFFFFFull);
    viol_blocks += (uint32_t)(sums >> 40);
    COH_TS(6)
    if (i == 0xFFFFFFFFu) {
      s_cur = s_end;
    } else {  // resolve the slow call from the slow table (as k_trace_eval's slow path)
      stopped = true;
      if (i >= c0 && i < c0 + cnt) {  // keep == i - c0 here
        const uint32_t k = i - c0;
        const uint32_t wk = (k & 4u) ? ((k & 2u) ? w4[3] : w4[2]) : ((k & 2u) ? w4[1] : w4[0]);
        const uint32_t r = (wk >> (16u * (k & 1u))) & 0xFFFFu;
        const uint32_t a = (r >> 8) & 63u, type = (r >> 2) & 63u;
        const int rem_i = p.fuel - (int)steps;
        const uint32_t rem = rem_i <= 0 ? 0u : (rem_i >= 7 ? 7u : (uint32_t)rem_i);
        const bool missing = a >= p.n_arrays;
        const uint32_t info = missing ? (uint32_t)COH_RUN_DEFECT : __ldg(p.slow + slow_index(type, s_slow, rem));
        slow_out[0] = missing ? s_slow : (info >> 7) & 15u;
        slow_out[1] = (info >> 2) & 7u;
        slow_out[2] = (info >> 5) & 3u;
        slow_out[3] = info;
        slow_out[4] = a;
      }
      __syncthreads();
      const uint32_t info = slow_out[3];
      s_cur = slow_out[0];
      steps += slow_out[1];
      xfers += slow_out[2];
      status = info & 3u;
      stuck_call = i;
      stuck_arr = slow_out[4];
      stuck_eff = (info >> 11) & 7u;
      stuck_flags = (info >> 14) & 15u;
      calls_done = i;
    }
    __syncthreads();  // the shared scratch is reused by the next pass
  }
  if (p.bnd)  // groups after the stop's pass: no completed calls
    for (uint32_t g = base / 32u + tid; g < (nc + 31u) / 32u; g += kScanNT) p.bnd[(uint64_t)g * n + t] = 0u;
  if (tid == 0) {
#ifdef COH_SCAN_PROFILE
    COH_TS(7)
    for (int k = 1; k < 8; ++k) reinterpret_cast<long long*>(p.res + t)[k - 1] = ts[k] - ts[k - 1];
    return;
#endif
    const uint64_t tb = (uint64_t)xfers * xbytes;
    if (!(s_cur & 3u) || !(s_cur & 12u)) stuck_flags |= COH_FLAG_UNSAFE;  // is_unsafe
    uint4* out = reinterpret_cast<uint4*>(p.res + t);
    __stcs(out + 0, make_uint4(s_cur, 0u, 0u, 0u));
    __stcs(out + 1, make_uint4(0u, 0u, 0u, 0u));
    __stcs(out + 2, make_uint4((uint32_t)tb, (uint32_t)(tb >> 32), steps, xfers));
    __stcs(out + 3, make_uint4(calls_done, viol_blocks, stuck_call,
                               status | (stuck_arr << 8) | (stuck_eff << 16) | (stuck_flags << 24)));
    if (p.counters) {
      const unsigned long long v[COH_N_COUNTERS] = {
          status == COH_RUN_STUCK, status == COH_RUN_FUEL_EXHAUSTED, viol_blocks != 0u, status == COH_RUN_DEFECT,
          steps, xfers, tb, viol_blocks, calls_done, 1u, (stuck_flags & COH_FLAG_UNSAFE) != 0u};
#pragma unroll
      for (int k = 0; k < COH_N_COUNTERS; ++k)
        if (v[k]) atomicAdd(p.counters + k, v[k]);
    }
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
#ifdef COH_TE_CARVEOUT
    cudaFuncSetAttribute(k_trace_eval<F>, cudaFuncAttributePreferredSharedMemoryCarveout, COH_TE_CARVEOUT);
#endif
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
  if (L.overlap) {  // COH_BATCH_OVERLAP: programmatic dependent of the previous kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kNT);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_trace_eval<F>, kp);
  } else {
    k_trace_eval<F><<<grid, kNT, 0, s>>>(kp);
  }
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
  kp.uniform = L.uniform_bytes ? 1u : 0u;
  kp.bytes_uniform = L.bytes_uniform;
  kp.array_bytes = L.d_array_bytes;
  kp.lut = L.d_lut;
  kp.slow = L.d_slow;
  kp.res = L.results;
  kp.bnd = L.boundary;
  kp.counters = reinterpret_cast<unsigned long long*>(L.counters);
  kp.slot = L.slot;
  kp.ticket = L.dynamic ? &L.slot->ticket : nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Latency path: too few single-array traces to fill the GPU -> a block per trace.
  // COH_TE_PATH=thread|scan forces one path (tests compare both).
  const char* path = std::getenv("COH_TE_PATH");
  bool scan = L.n_arrays == 1u && L.n_calls >= 64u && L.n_traces <= 2ull * (uint64_t)L.sms;
  if (path && std::strcmp(path, "thread") == 0) scan = false;
  if (path && std::strcmp(path, "scan") == 0) scan = L.n_arrays == 1u;
  if (scan) {
    if (L.counters) {  // the scan path adds into the caller's counters
      cudaError_t e = cudaMemsetAsync(L.counters, 0, sizeof(uint64_t) * COH_N_COUNTERS, s);
      if (e != cudaSuccess) {
        *err = std::string("counter memset: ") + cudaGetErrorString(e);
        return COH_E_CUDA;
      }
    }
    k_trace_scan<<<(unsigned)L.n_traces, kScanNT, 0, s>>>(kp);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      *err = std::string("trace_scan launch: ") + cudaGetErrorString(e);
      return COH_E_CUDA;
    }
    return COH_OK;
  }
  const bool ring = L.n_calls % 32u == 0u && L.n_calls >= 32u;
  const int f = (L.check_fuel ? kFuel : 0) | (L.uniform_bytes ? 0 : kBytes) | (ring ? kRing : 0) |
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


}  // namespace cohb
