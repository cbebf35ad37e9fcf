// Element-granular path: shared host/device definitions.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "cohere_b200.h"

namespace cohb {

// A stage holds, per buffer, up to kSlots consecutive ops: read-only ops (READ, CHECK)
// followed by at most one writing op (SYNC or WRITE) as the last.  pass1 evaluates every
// read against the stage-start state, decide walks the slots in program order (the first
// stuck op stops the buffer), apply performs the write.
constexpr uint32_t kSlots = 4;

// One device op of one buffer in one stage (16 B).
enum : uint8_t { EOP_NONE = 0, EOP_SYNC = 1, EOP_READ = 2, EOP_WRITE = 3, EOP_CHECK = 4 };
struct ElemOp {
  uint8_t type;
  uint8_t plane;     // SYNC: source plane (0 L, 1 R), the other is set; READ: plane that must be 1;
                     // WRITE: plane set to 1 (the other cleared); CHECK: number of views
  uint16_t call;     // call index
  uint32_t lo, hi;   // absolute cell range, inclusive (CHECK: lo = packed abstract pairs, 2 b/view)
  uint32_t tile0;    // first tile of this op in the stage's tile list
};
static_assert(sizeof(ElemOp) == 16, "ElemOp is 16 bytes");

// One CTA's work item, self-contained so a CTA can start its data loads without a chain
// of dependent descriptor loads: the 2048-word aligned block `tstart` of buffer b, the
// cell range [lo, hi] it applies to (op range, or the view range for CHECK), the op
// type / plane / view / the view's abstract pair, and the stage-local tile index.
struct ElemTile {
  uint32_t b;
  uint32_t tstart;
  uint32_t lo, hi;
  uint8_t type, plane, view, apair;
  uint32_t tloc;     // stage-local index in the pass1 tile list (tcnt / tbase slot)
  uint32_t slot;     // op slot of the buffer in this stage
  uint32_t pad;
};
static_assert(sizeof(ElemTile) == 32, "ElemTile is 32 bytes");

constexpr uint32_t kElemTileWords = 2048;      // 64 Ki cells per plane per CTA
constexpr uint32_t kStageRuns = 256;           // run starts (and ends) a sync tile stages in pass1
constexpr uint32_t kNoCell = 0xFFFFFFFFu;

// Device-side per-buffer state.
struct ElemState {
  uint32_t dead;          // stopped by a device-detected stuck
  uint32_t stuck_op;      // stage * kSlots + slot
  uint32_t stuck_cell;
  uint32_t stuck_pair;    // bit0 L, bit1 R at stuck_cell
  uint32_t calls_done;
  uint32_t violations;
  uint32_t transfers;
  uint32_t pad;
  unsigned long long transfer_cells;
  unsigned long long n_runs;      // run starts emitted (== ends)
};

// Per-stage scratch, per buffer and op slot ([b * kSlots + slot]).
struct ElemScratch {
  uint32_t first_zero;    // atomicMin over the op range (SYNC source / READ plane)
  uint32_t view_flags[COH_MAX_VIEWS];   // CHECK: bit0 some L=0, bit1 some R=0, bit2 some L|R=1
};

// Host plan of a batch.
struct ElemPlan {
  uint32_t n_progs = 0;
  uint32_t max_words = 0;            // words per plane per buffer (multiple of 4)
  uint32_t n_stages = 0;
  std::vector<ElemOp> ops;           // [stage][prog][slot]
  std::vector<ElemTile> tiles;       // all stages concatenated
  std::vector<uint32_t> stage_tile0; // n_stages + 1 offsets into tiles
  std::vector<uint8_t> stage_has_sync;
  std::vector<ElemTile> sync_tiles;        // apply-pass tiles (SYNC and WRITE ops), by stage
  std::vector<uint32_t> stage_sync0;       // n_stages + 1 offsets into sync_tiles
  // host timeline, per program
  struct Timeline {
    std::vector<uint64_t> steps_before;   // per stage (device op) of this program
    std::vector<uint32_t> abs_before;     // abstract pairs (2 b/view) before each device op
    std::vector<uint32_t> op_pos;         // stage * kSlots + slot of each device op
    uint32_t abs_final = 0;
    uint32_t n_ops = 0;
    uint64_t steps_total = 0;             // steps when the host-known sequence ends
    uint8_t term_status = COH_RUN_DONE;   // DONE / STUCK (abstract key) / FUEL_EXHAUSTED
    uint32_t term_call = 0;
    uint8_t term_effect = 0, term_flags = 0;
    uint32_t term_index = 0;
    uint32_t calls_checked = 0;           // CHECK ops emitted
  };
  std::vector<Timeline> tl;
  uint64_t alg_bytes = 0;            // algorithmic bytes of all device ops
};

int elem_compile(const coh_elem_program* progs, uint32_t n, ElemPlan* plan, std::string* err);

// Device view of one stage (elem.cu).
struct ElemDev {
  uint32_t* planes;            // [b][2][W]
  uint32_t W;                  // words per plane (multiple of kElemTileWords)
  const ElemOp* ops;           // this stage, [b][slot]
  const ElemTile* tiles;       // this stage
  const ElemTile* sync_desc;   // this stage: descriptors of the SYNC tiles (apply pass)
  ElemState* st;
  ElemScratch* sc;
  uint32_t* tcnt;              // per tile of this stage: starts, ends, zeros, edge bits
  unsigned long long* tbase;   // per tile: run-start offset, run-end offset
  uint32_t* stage_runs;        // per tile: up to kStageRuns starts, then kStageRuns ends (cells)
  const uint32_t* view_lo;     // [b][16]
  const uint32_t* view_hi;
  uint32_t* boundary;          // [b][bwords]
  uint32_t bwords;
  uint32_t* runs_lo;           // [b][cap]
  uint32_t* runs_hi;
  unsigned long long runs_cap;
  uint32_t n_progs;
  uint32_t stage;
};
int launch_elem_stage(const ElemDev& d, uint32_t n_tiles, uint32_t n_sync_tiles, void* stream, std::string* err);
// pinit: per program {n_cells, frag_log2, frag_seed lo, frag_seed hi} (device)
int launch_elem_init(uint32_t* planes, uint32_t W, const uint32_t* pinit, uint32_t n_progs, void* stream,
                     std::string* err);

}  // namespace cohb
