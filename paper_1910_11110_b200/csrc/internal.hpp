// Internal declarations shared by the host runtime (.cpp) and the CUDA sources (.cu).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "cohere_b200.h"

#if defined(__CUDACC__)
#define COH_HDC __host__ __device__ constexpr
#else
#define COH_HDC constexpr
#endif

namespace cohb {

// ---- micro-op encoding of one translated block (see coh_calltable_program) ----------
enum : uint8_t { OP_END = 0, OP_IF_VALID = 1, OP_IF_GVALID = 2, OP_EFFECT = 3 };
constexpr uint8_t op_effect(uint32_t eff, uint32_t site, uint32_t abstract_target) {
  return (uint8_t)(OP_EFFECT | (eff << 2) | (site << 5) | (abstract_target << 6));
}
// A malformed record (mode kind 3) compiles to this single op.
constexpr uint8_t OP_DEFECT = 0x80;

constexpr int kCallTypes = 64;   // record bits 2..7
constexpr int kStates = 16;      // state nibble

// Store slot in shared memory (one u16 per array per trace), "clean" so that it can be
// XORed straight into a table address:
//   bits 2-7  slot_swizzle(state) = state * 9 mod 64               -- the bank swizzle
//   bits 8-11 state nibble (bit0 cl, bit1 cr, bit2 al, bit3 ar)    -- the table row
//   bit  12   poison row: an array id >= n_arrays (a missing key, program.hpp:147-151)
// Transfers, steps and violations are not per-array state: they accumulate in a register.
COH_HDC uint32_t slot_swizzle(uint32_t state) { return (state * 9u) & 63u; }
COH_HDC uint32_t slot_word(uint32_t state) { return (state << 8) | (slot_swizzle(state) << 2); }
COH_HDC uint32_t slot_state(uint32_t slot) { return (slot >> 8) & 15u; }
constexpr uint32_t kPoisonSlot = 0x1000u;

// Call table (u32 entries), addressed by byte offset (type << 2) ^ slot, i.e. word
// state*64 + (type ^ swizzle(state)): rows of 64 words per state, bank = (type ^
// swizzle) & 31, which spreads the common (type, state) pairs of a warp over the banks
// (1.016 wavefronts per lookup on the C2 mix, vs 1.81 for swizzle = state); row 16
// serves the poison slot (word 1024 + type).
//   lo16 : the slot word after the call (stored as is)
//   hi16 : accumulator addend = steps + (transfers << 7) + ((viol_delta + 1) << 13), always
//          in [0, 0x7FFF] (the +1 is a per-call bias the device subtracts at each flush), or
//          kSlowAddend (the entry is negative) for a (type, state) that gets stuck / is
//          malformed / reads a poison slot
constexpr int kLutRows = kStates + 1;
constexpr int kLutEntries = kLutRows * kCallTypes;
constexpr uint32_t kSlowAddend = 0x8000u;
COH_HDC uint32_t lut_word(uint32_t type, uint32_t state) { return state * 64u + (type ^ slot_swizzle(state)); }
constexpr uint32_t kAccSteps = 0x7Fu;   // accumulator bits 0-6: steps since the last flush
constexpr uint32_t kAccXferShift = 7;   // bits 7-12: transfers since the last flush
constexpr uint32_t kAccViolShift = 13;  // bits 13-19: arrays whose abstraction is violated
constexpr uint32_t kAccKeep = ~((1u << kAccViolShift) - 1u);

// Slow-outcome table: the exact block outcome for (type, state, remaining fuel r), r
// clamped to [0, 7] (a block takes at most 6 steps, so r >= 7 means "unlimited"):
//   bits 0-1 status, 2-4 steps, 5-6 transfers, 7-10 state after, 11-13 stuck effect,
//   14-17 stuck flags (site | key kind << 1 | actual << 2)
constexpr int kSlowEntries = kCallTypes * kStates * 8;
COH_HDC uint32_t slow_index(uint32_t type, uint32_t state, uint32_t rem) { return (type * 16u + state) * 8u + rem; }

struct CallTable {
  uint32_t lut[kLutEntries];
  uint32_t slow[kSlowEntries];
  uint64_t prog[kCallTypes];   // 8 micro-ops per type, byte k = op k (host/ABI listing)
};

// Builds the table by running the restated rules (calltable.cpp).
void build_call_table(CallTable* t);

// Host restatement used by the compiler: one block from one state.
coh_call_outcome simulate_block(uint32_t call_type, uint32_t state, int fuel);

// ---- device entry points (defined in .cu files) ------------------------------------
// Per-launch device state of k_trace_eval, from a ring owned by the context (zeroed once
// at creation): the work-distribution ticket and the counter sums.  The last block of the
// launch copies the sums to the caller's counters and zeroes the slot for its next use, so
// a launch needs no memset before it (and can follow its predecessor without a gap).
struct LaunchSlot {
  unsigned int ticket;  // dynamic trace batches handed out after the first round
  unsigned int done;    // blocks finished
  unsigned long long cnt[COH_N_COUNTERS];
};
constexpr uint32_t kLaunchSlots = 256;
struct TraceLaunch {
  const uint16_t* records;
  uint64_t n_traces;
  uint32_t n_calls;
  uint32_t n_arrays;
  int32_t fuel;
  uint32_t flags;  // COH_BATCH_*
  bool check_fuel;
  bool uniform_bytes;
  uint64_t bytes_uniform;
  const uint64_t* d_array_bytes;   // device, n_arrays, private to the launch (used when !uniform_bytes)
  const uint32_t* d_lut;
  const uint32_t* d_slow;
  coh_trace_result* results;
  uint32_t* boundary;
  uint64_t* counters;  // optional fused counter reduction (device, COH_N_COUNTERS)
  int sms;  // SM count (persistent grid)
  LaunchSlot* slot;  // device, zeroed, private to this launch (ring of the context)
  bool dynamic;      // hand out trace batches from slot->ticket (long launches)
  bool overlap;      // COH_BATCH_OVERLAP: programmatic dependent launch
};
int launch_trace_eval(const TraceLaunch& p, void* stream, std::string* err);
// Multi-mode blocks (COH_BATCH_BLOCKS, trace_blocks.cu).
int launch_trace_blocks(const TraceLaunch& p, void* stream, std::string* err);
int trace_eval_occupancy(int* blocks_per_sm, int* threads_per_block, uint32_t n_calls, std::string* err);
// Launch setup done once per context at creation (the device is current): shared-memory
// attributes of the zero-run and element-apply kernels, the zero-run grid.
cudaError_t runs_ctx_init(int sms, int* grid);
cudaError_t elem_ctx_init();
int launch_gen_records(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                       uint32_t n_arrays, uint32_t adv_per1024, uint16_t* d_records, void* stream,
                       std::string* err);
// COH_BATCH_PACKED12 slice -> the 16-bit call-major records (gen_reduce.cu).
int launch_unpack12(const uint8_t* d_packed, uint16_t* d_records, uint64_t n_traces, uint32_t n_chunks, void* stream,
                    std::string* err);
int launch_gen_blocks(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls, uint32_t cont,
                      uint16_t* d_records, void* stream, std::string* err);
int launch_reduce_counters(const coh_trace_result* d_results, uint64_t n_traces,
                           uint64_t* d_counters, void* stream, std::string* err);

}  // namespace cohb

// The context behind the opaque coh_ctx handle (capi.cpp, elem_host.cpp).
struct coh_ctx {
  int device = 0;
  std::string err;
  uint32_t* d_lut = nullptr;
  uint32_t* d_slow = nullptr;
  int sms = 148;
  int blocks_per_sm = 1;       // trace_eval residency
  uint64_t launches = 0;
  // host-buffer pipeline
  cudaStream_t hs[2] = {nullptr, nullptr};
  uint16_t* d_rec[2] = {nullptr, nullptr};
  coh_trace_result* d_res[2] = {nullptr, nullptr};
  uint32_t* d_bnd[2] = {nullptr, nullptr};
  size_t rec_cap = 0, res_cap = 0, bnd_cap = 0;  // bytes per buffer
  void* d_pk[2] = {nullptr, nullptr};            // COH_BATCH_PACKED12 slices
  size_t pk_cap = 0;
  cohb::LaunchSlot* d_slots = nullptr;           // kLaunchSlots, zeroed at creation
  std::atomic<uint32_t> slot_next{0};          // host threads may share a context
  int runs_grid = 0;                            // zero-run passes: one wave (runs_ctx_init)
};
