// General block programs: bytecode shared by the host compiler (sweep_host.cpp) and the
// device interpreter (sweep.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "cohere_b200.h"

namespace cohb {

// instruction word: bits 0-3 op
//   BC_EFF    bits 4-6 effect, bit 7 site, bits 8-15 key
//   BC_WHOLE  bits 4-6 effect, bit 7 site, bits 8-15 first cell key, bits 16-23 last
//   BC_IF     bits 4-5 cond (0 valid, 1 gvalid, 2 opaque), bits 8-15 key, bits 16-31
//             else target (true -> next instruction)
//   BC_WHILE  as BC_IF, bits 16-31 exit target (the body ends with BC_JMP to the head)
//   BC_JMP    bits 16-31 target (no step)
//   BC_BEND   end of a block: abstraction_correct check (no step)
//   BC_END    program done
enum : uint32_t { BC_EFF = 1, BC_WHOLE = 2, BC_IF = 3, BC_WHILE = 4, BC_JMP = 5, BC_BEND = 6, BC_END = 7 };

// SweepOut packs the completed-block count in 5 bits and boundary_ok in bits 16-23.
constexpr uint32_t kSweepMaxBlocks = 8;

struct SweepProgram {
  std::vector<uint32_t> code;
  std::vector<uint16_t> checks;  // (abstract key | concrete key << 8) pairs for abstraction_correct
  uint32_t n_keys = 0, n_blocks = 0, n_scalars = 0, n_views = 0, buf_len = 0;
};

int sweep_compile(uint64_t seed, const coh_gen_limits& L, SweepProgram* out, std::string* text);

struct SweepMeta {
  uint32_t code_off, n_keys, check_off, n_checks;
};
struct SweepItem {
  uint32_t prog;
  uint32_t bits;   // schedule answers, bit k = k-th (answers 0..31)
  uint32_t len;    // <= 64
  uint32_t pad;    // answers 32..63
};
struct SweepOut {
  uint32_t status_consumed;  // bits 0-1 status, 2-9 consumed, 10 overflowed, 11-15 blocks done,
                             // 16-23 boundary_ok bits, 24-31 stuck key
  uint32_t steps;
  unsigned long long store;  // 2 bits per key (bit0 local, bit1 remote)
  uint32_t stuck;            // effect | site << 3 | key kind (abstract) << 4 | actual << 5
  uint32_t pad;              // 1 when some step left a key (I,I) (is_unsafe, program.hpp:166-172)
};
// One record per reduction step of item 0 (the CLI's --trace): the instruction that fired,
// the rule (0 effect, 1 remote-effect, 2 while-true, 3 while-false, 4 if-true, 5 if-false,
// semantics.hpp:76-79) and the store after the step.
struct SweepTrace {
  uint32_t pc;
  uint32_t rule;
  unsigned long long store;
};
int launch_sweep_run(const uint32_t* code, const SweepMeta* meta, const uint16_t* checks, const SweepItem* items,
                     uint32_t n_items, int32_t fuel, SweepOut* out, void* stream, std::string* err,
                     SweepTrace* trace = nullptr);

}  // namespace cohb
