// The step log of one whole-array trace: run_annotated with TraceMode::Full
// (semantics.hpp:231-235, 279-280), i.e. every reduction step's rule, the statement it
// fired on and the key it changed.  The trace's blocks are lowered, exactly as
// translate_block lays them out (guards in record order, then the bodies), to the program
// interpreter of the CLI (progrun.cu) over 2 keys per array (concrete, abstract), and run
// on the device with step recording.  A debugging view of the same semantics the batched
// kernels evaluate; the tests compare it with the reference's own TraceStep lists.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "internal.hpp"
#include "progrun.hpp"

extern "C" int coh_trace_steps(coh_ctx* ctx, const uint16_t* records, uint32_t n_calls, uint32_t n_arrays,
                               int32_t fuel, uint32_t flags, coh_trace_step* steps, uint32_t cap, uint32_t* n_steps,
                               uint32_t* status) {
  using namespace cohb;
  if (!ctx || (n_calls && !records) || !n_steps || !status || n_arrays < 1 || n_arrays > COH_MAX_ARRAYS ||
      (flags & ~COH_BATCH_BLOCKS) || (cap && !steps))
    return COH_E_ARG;
  if (fuel > (1 << 22)) {
    ctx->err = "coh_trace_steps records at most 4M steps (lower the fuel)";
    return COH_E_ARG;
  }
  struct Origin {
    uint32_t call;
    uint8_t array, head;
  };
  std::vector<ProgIns> code;
  std::vector<Origin> origin;  // per instruction
  auto emit = [&](ProgIns ins, Origin o) {
    code.push_back(ins);
    origin.push_back(o);
  };
  *status = COH_RUN_DONE;
  bool defect = false;
  for (uint32_t b0 = 0; b0 < n_calls && !defect;) {
    uint32_t b1 = b0 + 1;
    if (flags & COH_BATCH_BLOCKS)
      while (b1 < n_calls && (records[b1] & COH_REC_CONT)) ++b1;
    uint64_t seen = 0;
    for (uint32_t i = b0; i < b1; ++i) {  // the DeclBlock constructor's checks
      const uint32_t a = COH_REC_ARRAY(records[i]);
      if (a >= n_arrays || COH_REC_KIND(records[i]) == 3u || ((seen >> a) & 1u)) defect = true;
      seen |= 1ull << a;
    }
    if (defect) break;  // a construction defect: nothing of this block runs
    for (int phase = 0; phase < 2; ++phase)
      for (uint32_t i = b0; i < b1; ++i) {
        const uint16_t r = records[i];
        const uint32_t a = COH_REC_ARRAY(r), kind = COH_REC_KIND(r);
        uint8_t ops[8];
        const int n = coh_calltable_program(COH_REC_TYPE(r), ops);
        const int g = kind == COH_R ? 3 : kind == COH_W ? 1 : 4;
        for (int k = phase ? g : 0; k < (phase ? n : g); ++k) {
          const uint8_t op = ops[k];
          if ((op & 3u) != OP_EFFECT) {  // if (valid(x^)) {} else {sync x; sync x^}
            const uint32_t cond = (op & 3u) == OP_IF_GVALID ? 1u : 0u;
            const size_t at = code.size();
            emit(ProgIns{PI_IF | (cond << 8), 2 * a + 1, 0, (uint32_t)at + 2}, Origin{i, (uint8_t)a, (uint8_t)(0x80u | cond)});
            emit(ProgIns{PI_JMP, 0, 0, (uint32_t)at + 4}, Origin{i, (uint8_t)a, 0});
            continue;
          }
          const uint32_t eff = (op >> 2) & 7u, site = (op >> 5) & 1u, abs = (op >> 6) & 1u;
          emit(ProgIns{PI_EFF | (eff << 4) | (site << 7), 2 * a + abs, 0, 0},
               Origin{i, (uint8_t)a, (uint8_t)(eff | (site << 3) | (abs << 4))});
        }
      }
    b0 = b1;
  }
  code.push_back(ProgIns{PI_END, 0, 0, 0});
  if (cudaSetDevice(ctx->device) != cudaSuccess) {
    ctx->err = "cudaSetDevice failed";
    return COH_E_CUDA;
  }
  ProgRunResult r;
  std::string err;
  const int rc = prog_run(code, 2 * n_arrays, fuel, 0, 0, true, &r, &err);
  if (rc) {
    ctx->err = err;
    return rc;
  }
  ctx->launches++;
  *status = defect && r.status == COH_RUN_DONE ? (uint32_t)COH_RUN_DEFECT : r.status;
  *n_steps = (uint32_t)r.trace.size();
  uint32_t d0 = 0;
  for (size_t s = 0; s < r.trace.size(); ++s) {
    const ProgStep& st = r.trace[s];
    if (s < cap) {
      const Origin& o = origin[st.pc];
      coh_trace_step& out = steps[s];
      out.call = o.call;
      out.rule = (uint8_t)st.rule;
      out.array = o.array;
      out.head = o.head;
      out.delta = 0;
      if (st.delta_end > d0) {  // one key per effect step
        const ProgDelta& d = r.deltas[d0];
        out.delta = (uint8_t)(0x10u | ((d.key & 1u) << 2) | d.pair);
      }
    }
    d0 = st.delta_end;
  }
  return *n_steps > cap ? -(int)*n_steps - 1 : COH_OK;
}
