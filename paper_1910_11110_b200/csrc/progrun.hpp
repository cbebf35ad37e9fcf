// Device interpreter for one general program of any size (the CLI's `run` / `trace`):
// the store is two bit planes over the program's key space (L = local valid, R = remote
// valid, one bit per key), so a whole-view sync is a word-parallel range operation done by
// the whole CTA, and a program's key count is bounded only by device memory.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "cohere_b200.h"

namespace cohb {

// One instruction (16 B).  op: bits 0-3 kind, 4-6 effect, 7 site, 8-9 condition
// (0 valid = local flag, 1 gvalid = remote flag, 2 opaque).
//   PI_EFF    effect on key `a`
//   PI_WHOLE  atomic sync of keys [a, b] (a whole view's cells, ascending)
//   PI_IF     test key `a`; true -> next instruction, false -> `target`
//   PI_WHILE  as PI_IF, false -> `target` (the loop body ends with PI_JMP back here)
//   PI_JMP    -> `target`, no step
//   PI_END    program done
enum : uint32_t { PI_EFF = 1, PI_WHOLE = 2, PI_IF = 3, PI_WHILE = 4, PI_JMP = 5, PI_END = 7 };
struct ProgIns {
  uint32_t op, a, b, target;
};

struct ProgStep {      // one reduction step (trace mode)
  uint32_t pc;         // instruction that fired
  uint32_t rule;       // 0 effect, 1 remote-effect, 2 while-true, 3 while-false, 4 if-true, 5 if-false
  uint32_t delta_end;  // the step's changed keys are deltas[previous delta_end, delta_end)
};
struct ProgDelta {
  uint32_t key, pair;  // pair: bit0 local V, bit1 remote V (after the step)
};

struct ProgRunResult {
  uint32_t status = 0, steps = 0, consumed = 0, overflowed = 0;
  uint32_t stuck_key = 0, stuck_eff = 0, stuck_site = 0, stuck_actual = 0;
  std::vector<uint32_t> L, R;  // final planes (n_keys bits each)
  std::vector<ProgStep> trace;
  std::vector<ProgDelta> deltas;
};

// Runs `code` from initial_store (every key (V,I)) with `fuel` steps and the opaque
// answers `sched` (bit k = k-th answer, `sched_len` <= 64).  Returns COH_OK or COH_E_CUDA.
int prog_run(const std::vector<ProgIns>& code, uint32_t n_keys, int32_t fuel, uint64_t sched, uint32_t sched_len,
             bool trace, ProgRunResult* out, std::string* err);

}  // namespace cohb
