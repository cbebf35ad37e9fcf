// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// Harness around the UNMODIFIED reference (`cohere`, header-only C++20 under
// /root/reference/proj/include, compiled in place by oracle/Makefile into
// oracle/_ref/libcohere_ref.so).  It turns packed call records into the reference's own
// data model (Declarations with one scalar per array, one DeclBlock per call,
// program.hpp:50-235) and runs the reference evaluator on them:
//
//   mode 0  the run_annotated loop (modes.hpp:105-125) replicated with TraceMode::Full so
//           executed concrete Push/Pull steps (transfers) can be read off the trace heads
//           (legitimate by tests/test_modes.cpp:134-191).
//   mode 1  cohere::run_annotated itself (TraceMode::None): the reference's hot path as
//           shipped; transfers / transfer_bytes are reported as 0.
//
// Output uses the product's result POD (include/cohere_b200.h) so tests compare fields.
#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cohere/cohere.hpp"
#include "cohere_b200.h"

using namespace cohere;

namespace {

const std::vector<std::string>& array_names() {
  static const std::vector<std::string> names = [] {
    std::vector<std::string> v;
    for (int a = 0; a < COH_MAX_ARRAYS; ++a) v.push_back("a" + std::to_string(a));
    return v;
  }();
  return names;
}

// Body variants — the workload definition, not the algorithm.
//   0 canonical: R: r@S  W: w@S  RW: r@S; w@S     1 empty   2 r@O   3 w@O
//   4 r@S   5 w@S; r@O   6 push@S   7 pull@S; w@O
Stmt make_body(const Declarations& d, const std::string& x, uint32_t kind, Site S, uint32_t variant) {
  const Site O = S == Site::Local ? Site::Remote : Site::Local;
  auto e = [&](EffectKind k, Site s) { return Stmt::effect(k, d.scalar_target(x), s); };
  switch (variant) {
    case 0:
      if (kind == 0) return e(EffectKind::Read, S);
      if (kind == 1) return e(EffectKind::Write, S);
      return Stmt::seq(e(EffectKind::Read, S), e(EffectKind::Write, S));
    case 1: return Stmt::noop();
    case 2: return e(EffectKind::Read, O);
    case 3: return e(EffectKind::Write, O);
    case 4: return e(EffectKind::Read, S);
    case 5: return Stmt::seq(e(EffectKind::Write, S), e(EffectKind::Read, O));
    case 6: return e(EffectKind::Push, S);
    case 7: return Stmt::seq(e(EffectKind::Pull, S), e(EffectKind::Write, O));
  }
  return Stmt::noop();
}

DeclBlock make_block(const Declarations& d, uint16_t rec) {
  const std::string& x = array_names()[COH_REC_ARRAY(rec)];
  const uint32_t kind = COH_REC_KIND(rec);
  const Site S = COH_REC_SITE(rec) ? Site::Remote : Site::Local;
  AccessMode m;
  m.kind = static_cast<AccessMode::Kind>(kind);
  m.site = S;
  m.view = x;
  return DeclBlock({m}, make_body(d, x, kind, S, COH_REC_VARIANT(rec)));
}

uint32_t pair_bits(ValidityPair p) {
  return (p.local == Validity::Valid ? 1u : 0u) | (p.remote == Validity::Valid ? 2u : 0u);
}

ValidityPair bits_pair(uint32_t b) {
  return ValidityPair{(b & 1u) ? Validity::Valid : Validity::Invalid,
                      (b & 2u) ? Validity::Valid : Validity::Invalid};
}

bool is_sync(const Stmt& head) {
  if (head.op() != Stmt::Op::Effect) return false;
  const auto& n = head.node();
  return (n.effect == EffectKind::Push || n.effect == EffectKind::Pull) &&
         n.target.kind != Target::Kind::Abstract;
}

void fill_stuck(const std::optional<StuckInfo>& st, coh_trace_result& r) {
  if (!st) return;
  r.stuck_array = (uint8_t)std::stoi(st->key.name.substr(1));
  r.stuck_effect = (uint8_t)st->effect;
  r.stuck_flags = (uint8_t)((st->site == Site::Remote ? 1u : 0u) |
                            (st->key.kind == VarKey::Kind::Abstract ? 2u : 0u) |
                            (pair_bits(st->actual) << 2));
}

// COH_BATCH_BLOCKS: the reference's own multi-mode DeclBlock for records [b0, b1) --
// one AccessMode per record, the body the records' bodies in order (translate_block then
// puts every guard before the body, modes.hpp:53-59).  Returns false when the DeclBlock
// cannot be built (undeclared / malformed / repeated variable: ConstructionError).
bool make_multi_block(const Declarations& d, const uint16_t* recs, uint64_t n_total, uint64_t t, uint32_t b0,
                      uint32_t b1, uint32_t n_arrays, DeclBlock* out, uint32_t* bad_array) {
  std::vector<AccessMode> modes;
  std::vector<Stmt> body;
  uint64_t seen = 0;
  int repeated = -1;  // the first array named twice (reported as the defect's array)
  for (uint32_t i = b0; i < b1; ++i) {
    const uint16_t rec = recs[((uint64_t)(i / 8) * n_total + t) * 8 + i % 8];
    const uint32_t a = COH_REC_ARRAY(rec), kind = COH_REC_KIND(rec);
    if (a >= n_arrays || kind > 2) {
      if (repeated >= 0) break;  // the repeat came first
      *bad_array = a;
      return false;
    }
    if (((seen >> a) & 1u) && repeated < 0) repeated = (int)a;
    seen |= 1ull << a;
    const Site S = COH_REC_SITE(rec) ? Site::Remote : Site::Local;
    AccessMode m;
    m.kind = static_cast<AccessMode::Kind>(kind);
    m.site = S;
    m.view = array_names()[a];
    modes.push_back(m);
    body.push_back(make_body(d, array_names()[a], kind, S, COH_REC_VARIANT(rec)));
  }
  try {
    *out = DeclBlock(std::move(modes), Stmt::seq(body));
  } catch (const ConstructionError&) {  // a variable declared twice in one block (program.hpp:218-225)
    *bad_array = repeated >= 0 ? (uint32_t)repeated : 0u;
    return false;
  }
  if (repeated >= 0) {  // the reference must have refused it
    *bad_array = 0xFFu;
    return false;
  }
  return true;
}

void eval_blocks(const uint16_t* recs, uint64_t n_total, uint64_t t, uint32_t n_calls, uint32_t n_arrays, int32_t fuel,
                 const uint64_t* array_bytes, coh_trace_result& r, std::vector<bool>& bnd) {
  Declarations decls;
  for (uint32_t a = 0; a < n_arrays; ++a) decls.add_scalar({array_names()[a], {}});
  std::memset(&r, 0, sizeof r);
  Store store = initial_store(decls);
  Schedule schedule;
  int steps = 0;
  RunStatus status = RunStatus::Done;
  bnd.clear();
  auto rec_at = [&](uint32_t i) { return recs[((uint64_t)(i / 8) * n_total + t) * 8 + i % 8]; };
  // run_annotated (modes.hpp:105-125) over the blocks, TraceMode::Full for transfers
  for (uint32_t b0 = 0; b0 < n_calls;) {
    uint32_t b1 = b0 + 1;
    while (b1 < n_calls && (rec_at(b1) & COH_REC_CONT)) ++b1;
    DeclBlock block;
    uint32_t bad = 0;
    if (!make_multi_block(decls, recs, n_total, t, b0, b1, n_arrays, &block, &bad)) {
      r.status = COH_RUN_DEFECT;
      r.stuck_call = (uint32_t)bnd.size();
      r.stuck_array = (uint8_t)bad;
      break;
    }
    RunResult rr = run(translate_block(block, decls), std::move(store), fuel - steps, schedule, TraceMode::Full);
    store = std::move(rr.store);
    steps += rr.steps;
    status = rr.status;
    schedule.pos = rr.schedule_consumed;
    for (const auto& ts : rr.trace)
      if (is_sync(ts.head)) {
        r.transfers++;
        const uint32_t a = (uint32_t)std::stoi(ts.head.node().target.name.substr(1));
        r.transfer_bytes += array_bytes ? array_bytes[a] : 1u;
      }
    if (rr.status != RunStatus::Done) {
      r.status = (uint8_t)status;
      r.stuck_call = (uint32_t)bnd.size();
      r.stuck_array = (uint8_t)COH_REC_ARRAY(rec_at(b0));  // fuel exhaustion: the block's first array
      fill_stuck(rr.stuck, r);
      break;
    }
    bnd.push_back(abstraction_correct(store, decls));
    b0 = b1;
  }
  r.steps = (uint32_t)steps;
  r.calls_done = (uint32_t)bnd.size();
  for (bool ok : bnd) r.violations += ok ? 0u : 1u;
  for (uint32_t a = 0; a < n_arrays; ++a) {
    const uint32_t c = pair_bits(store.at(VarKey::scalar(array_names()[a])));
    const uint32_t ab = pair_bits(store.at(VarKey::abstract(array_names()[a])));
    r.state[a / 8] |= (c | (ab << 2)) << (4 * (a % 8));
  }
  if (is_unsafe(store)) r.stuck_flags |= COH_FLAG_UNSAFE;
}

void eval_one(const uint16_t* recs, uint64_t n_total, uint64_t t, uint32_t n_calls,
              uint32_t n_arrays, int32_t fuel, const uint64_t* array_bytes, int mode,
              coh_trace_result& r, std::vector<bool>& bnd) {
  AnnotatedProgram p;
  for (uint32_t a = 0; a < n_arrays; ++a) p.decls.add_scalar({array_names()[a], {}});
  p.blocks.reserve(n_calls);
  for (uint32_t i = 0; i < n_calls; ++i)
    p.blocks.push_back(make_block(p.decls, recs[((uint64_t)(i / 8) * n_total + t) * 8 + i % 8]));

  std::memset(&r, 0, sizeof r);
  RunStatus status;
  Store store;
  std::optional<StuckInfo> stuck;
  if (mode == 1) {
    AnnotatedRun ar = run_annotated(p, fuel, Schedule());
    status = ar.status;
    store = std::move(ar.store);
    stuck = ar.stuck;
    bnd = ar.boundary_ok;
    r.steps = (uint32_t)ar.steps;
  } else {
    // run_annotated (modes.hpp:105-125) with TraceMode::Full for transfer accounting
    Schedule schedule;
    store = initial_store(p.decls);
    int steps = 0;
    status = RunStatus::Done;
    bnd.clear();
    for (const auto& block : p.blocks) {
      RunResult rr = run(translate_block(block, p.decls), std::move(store), fuel - steps,
                         schedule, TraceMode::Full);
      store = std::move(rr.store);
      steps += rr.steps;
      status = rr.status;
      schedule.pos = rr.schedule_consumed;
      for (const auto& ts : rr.trace)
        if (is_sync(ts.head)) {
          r.transfers++;
          const uint32_t a = (uint32_t)std::stoi(ts.head.node().target.name.substr(1));
          r.transfer_bytes += array_bytes ? array_bytes[a] : 1u;
        }
      if (rr.status != RunStatus::Done) {
        stuck = rr.stuck;
        break;
      }
      bnd.push_back(abstraction_correct(store, p.decls));
    }
    r.steps = (uint32_t)steps;
  }
  r.status = (uint8_t)status;
  r.calls_done = (uint32_t)bnd.size();
  for (bool ok : bnd) r.violations += ok ? 0u : 1u;
  if (status != RunStatus::Done) {
    r.stuck_call = r.calls_done;
    const uint64_t i = r.calls_done;
    r.stuck_array = (uint8_t)COH_REC_ARRAY(recs[(i / 8 * n_total + t) * 8 + i % 8]);
    fill_stuck(stuck, r);
  }
  for (uint32_t a = 0; a < n_arrays; ++a) {
    const uint32_t c = pair_bits(store.at(VarKey::scalar(array_names()[a])));
    const uint32_t ab = pair_bits(store.at(VarKey::abstract(array_names()[a])));
    r.state[a / 8] |= (c | (ab << 2)) << (4 * (a % 8));
  }
  if (is_unsafe(store)) r.stuck_flags |= COH_FLAG_UNSAFE;  // program.hpp:166-170
}

}  // namespace

extern "C" {

// Evaluate traces [t_begin, t_end) of a record set laid out for n_total traces.
// out / boundary are indexed relative to t_begin; boundary is word-major
// [(i/32) * (t_end - t_begin) + (t - t_begin)] (may be NULL).  Returns 0 or -1.
// The reference's TraceMode::Full step list for one trace (records in plain call order),
// in coh_trace_step form: run (semantics.hpp:253-287) per block with the trace's shared
// fuel, each TraceStep's rule, head statement and delta (at most one key here).
int ref_trace_steps(const uint16_t* recs, uint32_t n_calls, uint32_t n_arrays, int32_t fuel, uint32_t flags,
                    coh_trace_step* out, uint32_t cap, uint32_t* n_steps, uint32_t* status_out) {
  try {
    Declarations decls;
    for (uint32_t a = 0; a < n_arrays; ++a) decls.add_scalar({array_names()[a], {}});
    Store store = initial_store(decls);
    int steps = 0;
    uint32_t n = 0;
    RunStatus status = RunStatus::Done;
    bool defect = false;
    for (uint32_t b0 = 0; b0 < n_calls;) {
      uint32_t b1 = b0 + 1;
      if (flags & COH_BATCH_BLOCKS)
        while (b1 < n_calls && (recs[b1] & COH_REC_CONT)) ++b1;
      DeclBlock block;
      uint32_t bad = 0;
      if (!make_multi_block(decls, recs, 1, 0, b0, b1, n_arrays, &block, &bad)) {  // one trace, plain order
        defect = true;
        break;
      }
      RunResult rr = run(translate_block(block, decls), std::move(store), fuel - steps, Schedule(), TraceMode::Full);
      store = std::move(rr.store);
      steps += rr.steps;
      status = rr.status;
      for (const auto& ts : rr.trace) {
        coh_trace_step st{};
        const auto& h = ts.head.node();
        std::string name;
        if (ts.head.op() == Stmt::Op::If) {
          name = h.cond.key.name;
          st.head = (uint8_t)(0x80u | (h.cond.kind == Condition::Kind::RemIsValid ? 1u : 0u));
        } else {
          name = h.target.name;
          st.head = (uint8_t)((uint32_t)h.effect | ((h.site == Site::Remote ? 1u : 0u) << 3) |
                              ((h.target.kind == Target::Kind::Abstract ? 1u : 0u) << 4));
        }
        st.array = (uint8_t)std::stoi(name.substr(1));
        for (uint32_t i = b0; i < b1; ++i)  // arrays are distinct within a block
          if (COH_REC_ARRAY(recs[i]) == st.array) st.call = i;
        st.rule = (uint8_t)ts.rule;
        if (!ts.delta.empty())
          st.delta = (uint8_t)(0x10u | ((ts.delta[0].first.kind == VarKey::Kind::Abstract ? 1u : 0u) << 2) |
                               pair_bits(ts.delta[0].second));
        if (n < cap) out[n] = st;
        ++n;
      }
      if (rr.status != RunStatus::Done) break;
      b0 = b1;
    }
    *n_steps = n;
    *status_out = defect && status == RunStatus::Done ? (uint32_t)COH_RUN_DEFECT : (uint32_t)status;
    return 0;
  } catch (...) {
    return -1;
  }
}

// mode 2: COH_BATCH_BLOCKS (records with COH_REC_CONT continue the previous block).
int ref_eval_traces(const uint16_t* records, uint64_t n_total, uint64_t t_begin, uint64_t t_end,
                    uint32_t n_calls, uint32_t n_arrays, int32_t fuel, const uint64_t* array_bytes,
                    coh_trace_result* out, uint32_t* boundary, int n_threads, int mode) {
  if (n_arrays < 1 || n_arrays > COH_MAX_ARRAYS || t_end < t_begin) return -1;
  const uint64_t m = t_end - t_begin;
  const uint32_t n_words = (n_calls + 31) / 32;
  std::atomic<uint64_t> next{0};
  std::atomic<int> failed{0};
  auto worker = [&] {
    std::vector<bool> bnd;
    for (;;) {
      const uint64_t j = next.fetch_add(1);
      if (j >= m) break;
      try {
        if (mode == 2)
          eval_blocks(records, n_total, t_begin + j, n_calls, n_arrays, fuel, array_bytes, out[j], bnd);
        else
          eval_one(records, n_total, t_begin + j, n_calls, n_arrays, fuel, array_bytes, mode, out[j], bnd);
      } catch (...) {
        failed = 1;
        continue;
      }
      if (boundary)
        for (uint32_t w = 0; w < n_words; ++w) {
          uint32_t word = 0;
          for (uint32_t b = 0; b < 32 && w * 32 + b < bnd.size(); ++b)
            if (bnd[w * 32 + b]) word |= 1u << b;
          boundary[(uint64_t)w * m + j] = word;
        }
    }
  };
  n_threads = std::max(1, n_threads);
  std::vector<std::thread> pool;
  for (int k = 1; k < n_threads; ++k) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return failed ? -1 : 0;
}

// One call type (record bits 6..11) from one store state (nibble: cl, cr, al, ar) on a
// single array: translate_block + run(Full) from that store (the SURVEY Appendix A probe).
int ref_call_outcome(uint32_t call_type, uint32_t state, coh_call_outcome* o) {
  if (call_type >= 64 || state >= 16 || !o) return -1;
  std::memset(o, 0, sizeof *o);
  const uint32_t kind = call_type & 3u;
  if (kind > 2) {
    o->status = COH_RUN_DEFECT;
    o->state_after = (uint8_t)state;
    return 0;
  }
  Declarations d;
  d.add_scalar({"a0", {}});
  Store s = initial_store(d);
  s.put(VarKey::scalar("a0"), bits_pair(state & 3u));
  s.put(VarKey::abstract("a0"), bits_pair(state >> 2));
  const uint16_t rec = (uint16_t)(call_type << 2);  // array 0, COH_REC_TYPE = call_type
  DeclBlock b = make_block(d, rec);
  auto viol = [&](const Store& st) { return abstraction_correct(st, d) ? 0 : 1; };
  o->viol_before = (uint8_t)viol(s);
  RunResult r = run(translate_block(b, d), s, 1 << 30, Schedule(), TraceMode::Full);
  o->status = (uint8_t)r.status;
  o->steps = (uint8_t)r.steps;
  for (const auto& ts : r.trace) o->transfers += is_sync(ts.head) ? 1 : 0;
  o->state_after = (uint8_t)(pair_bits(r.store.at(VarKey::scalar("a0"))) |
                             (pair_bits(r.store.at(VarKey::abstract("a0"))) << 2));
  o->viol_after = (uint8_t)viol(r.store);
  if (r.stuck) {
    coh_trace_result tmp;
    std::memset(&tmp, 0, sizeof tmp);
    fill_stuck(r.stuck, tmp);
    o->stuck_effect = tmp.stuck_effect;
    o->stuck_flags = tmp.stuck_flags;
  }
  return 0;
}

// Self-check: mode 0 (replicated loop) and mode 1 (run_annotated) agree on status,
// store planes, steps, calls_done, violations and boundary bits.  Returns mismatches.
int ref_selfcheck(const uint16_t* records, uint64_t n_total, uint32_t n_calls, uint32_t n_arrays,
                  int32_t fuel) {
  int bad = 0;
  std::vector<bool> b0, b1;
  for (uint64_t t = 0; t < n_total; ++t) {
    coh_trace_result r0, r1;
    eval_one(records, n_total, t, n_calls, n_arrays, fuel, nullptr, 0, r0, b0);
    eval_one(records, n_total, t, n_calls, n_arrays, fuel, nullptr, 1, r1, b1);
    r0.transfers = r1.transfers = 0;
    r0.transfer_bytes = r1.transfer_bytes = 0;
    if (std::memcmp(&r0, &r1, sizeof r0) != 0 || b0 != b1) ++bad;
  }
  return bad;
}

// ---------------------------------------------------------------------------------
// Element-granular programs (one buffer "b", views "v0".."vK"): the reference's own
// Declarations / DeclBlock / rewrite_program (overlap closure, overlap.hpp:234-242) /
// translate_block / run(Full) / abstraction_correct, block by block.  Transfer ranges
// are the maximal runs of each whole-view sync step's delta (changed cells, ascending,
// semantics.hpp:125-128, 155-166).  Returns 0, -1 on a construction error, -2 on an
// OverlapInferenceError, -3 when runs_cap is too small.
static int ref_elem_run_impl(const coh_elem_program* P, coh_elem_result* out, uint32_t* plane_l, uint32_t* plane_r,
                             uint8_t* view_abs, uint32_t* boundary, uint32_t* runs, uint64_t runs_cap) {
  try {
    AnnotatedProgram p;
    p.decls.add_buffer({"b", (int)P->n_cells, {}});
    for (uint32_t v = 0; v < P->n_views; ++v)
      p.decls.add_view({"v" + std::to_string(v), "b", (int)P->view_lo[v], (int)P->view_hi[v], {}});
    for (uint32_t c = 0; c < P->n_calls; ++c) {
      const coh_elem_call& call = P->calls[c];
      const std::string x = "v" + std::to_string(call.view);
      AccessMode m;
      m.kind = static_cast<AccessMode::Kind>(call.kind);
      m.site = call.site ? Site::Remote : Site::Local;
      m.view = x;
      std::vector<Stmt> body;
      for (int k = 0; k < call.n_body; ++k) {
        const coh_elem_op& op = call.body[k];
        for (uint32_t i = op.lo; i <= op.hi; ++i)
          body.push_back(Stmt::effect(static_cast<EffectKind>(op.effect), p.decls.element_target(x, (int)i),
                                      op.site ? Site::Remote : Site::Local));
      }
      p.blocks.emplace_back(std::vector<AccessMode>{m}, Stmt::seq(body));
    }
    AnnotatedProgram q = rewrite_program(p, build_registry(p.decls));
    std::memset(out, 0, sizeof *out);
    Store store = initial_store(q.decls);
    for (uint32_t i = 0; i < P->n_cells; ++i)  // pre-fragmented start: these cells coherent
      if ((coh_frag_mask(P->frag_seed, P->frag_log2, i / 32) >> (i % 32)) & 1u)
        store.put(VarKey::element("b", (int)i), ValidityPair{Validity::Valid, Validity::Valid});
    Schedule schedule;
    int64_t steps = 0;
    RunStatus status = RunStatus::Done;
    std::optional<StuckInfo> stuck;
    const uint32_t n_words = (P->n_calls + 31) / 32;
    if (boundary) std::memset(boundary, 0, 4u * n_words);
    uint32_t c = 0;
    for (; c < q.blocks.size(); ++c) {
      RunResult rr = run(translate_block(q.blocks[c], q.decls), std::move(store), (int)(P->fuel - steps),
                         schedule, TraceMode::Full);
      store = std::move(rr.store);
      steps += rr.steps;
      status = rr.status;
      schedule.pos = rr.schedule_consumed;
      for (const auto& ts : rr.trace) {
        if (ts.head.op() != Stmt::Op::Effect) continue;
        const auto& n = ts.head.node();
        if (n.target.kind != Target::Kind::WholeView) continue;
        out->transfers++;
        out->vpu_cells += (uint64_t)(n.target.hi - n.target.lo + 1);
        int64_t run_lo = -2, run_hi = -2;
        auto flush = [&] {
          if (run_lo < 0) return 0;
          if (out->n_runs >= runs_cap) return -3;
          if (runs) {
            runs[2 * out->n_runs] = (uint32_t)run_lo;
            runs[2 * out->n_runs + 1] = (uint32_t)run_hi;
          }
          out->n_runs++;
          out->transfer_cells += (uint64_t)(run_hi - run_lo + 1);
          return 0;
        };
        for (const auto& [key, pair] : ts.delta) {
          (void)pair;
          if (key.index == run_hi + 1) {
            run_hi = key.index;
          } else {
            if (flush()) return -3;
            run_lo = run_hi = key.index;
          }
        }
        if (flush()) return -3;
      }
      if (rr.status != RunStatus::Done) {
        stuck = rr.stuck;
        break;
      }
      const bool ok = abstraction_correct(store, q.decls);
      if (!ok) out->violations++;
      if (ok && boundary) boundary[c / 32] |= 1u << (c % 32);
      out->calls_done++;
    }
    out->status = (uint8_t)status;
    out->steps = (uint64_t)steps;
    if (status != RunStatus::Done) {
      out->stuck_call = c;
      if (stuck) {
        out->stuck_effect = (uint8_t)stuck->effect;
        const bool abs_key = stuck->key.kind == VarKey::Kind::Abstract;
        out->stuck_flags = (uint8_t)((stuck->site == Site::Remote ? 1u : 0u) | (abs_key ? 2u : 0u) |
                                     (pair_bits(stuck->actual) << 2));
        out->stuck_index = abs_key ? (uint32_t)std::stoi(stuck->key.name.substr(1)) : (uint32_t)stuck->key.index;
      }
    }
    const uint32_t n_pw = (P->n_cells + 31) / 32;
    std::memset(plane_l, 0, 4u * n_pw);
    std::memset(plane_r, 0, 4u * n_pw);
    for (uint32_t i = 0; i < P->n_cells; ++i) {
      const uint32_t b = pair_bits(store.at(VarKey::element("b", (int)i)));
      if (b & 1u) plane_l[i / 32] |= 1u << (i % 32);
      if (b & 2u) plane_r[i / 32] |= 1u << (i % 32);
    }
    for (uint32_t v = 0; v < P->n_views; ++v)
      view_abs[v] = (uint8_t)pair_bits(store.at(VarKey::abstract("v" + std::to_string(v))));
    return 0;
  } catch (const OverlapInferenceError&) {
    return -2;
  } catch (const std::exception&) {
    return -1;
  }
}

// The reference builds element bodies as right-nested Stmt chains and normalises /
// destroys them recursively, so large views need a deep stack: run on a pthread with
// a 4 GiB stack (virtual; only touched pages are committed).
struct ElemArgs {
  const coh_elem_program* P;
  coh_elem_result* out;
  uint32_t *plane_l, *plane_r;
  uint8_t* view_abs;
  uint32_t *boundary, *runs;
  uint64_t runs_cap;
  int rc;
};
static void* elem_thread(void* a) {
  ElemArgs* e = static_cast<ElemArgs*>(a);
  e->rc = ref_elem_run_impl(e->P, e->out, e->plane_l, e->plane_r, e->view_abs, e->boundary, e->runs, e->runs_cap);
  return nullptr;
}
int ref_elem_run(const coh_elem_program* P, coh_elem_result* out, uint32_t* plane_l, uint32_t* plane_r,
                 uint8_t* view_abs, uint32_t* boundary, uint32_t* runs, uint64_t runs_cap) {
  ElemArgs a{P, out, plane_l, plane_r, view_abs, boundary, runs, runs_cap, -1};
  pthread_attr_t attr;
  pthread_attr_init(&attr);
  pthread_attr_setstacksize(&attr, (size_t)4 << 30);
  pthread_t th;
  if (pthread_create(&th, &attr, elem_thread, &a) != 0) return -4;
  pthread_join(th, nullptr);
  pthread_attr_destroy(&attr);
  return a.rc;
}

// ---------------------------------------------------------------------------------
// General programs: the reference's own gen_well_declared / run_annotated / sweep.
int ref_gen_program_text(uint64_t seed, char* buf, size_t cap) {
  const std::string t = pretty(gen_well_declared(seed, GenLimits()));
  if (!buf || cap <= t.size()) return -(int)t.size() - 1;
  std::memcpy(buf, t.c_str(), t.size() + 1);
  return 0;
}

static int key_index(const Declarations& d, const VarKey& k) {
  const int S = (int)d.scalars().size(), V = (int)d.views().size();
  auto find = [](const auto& vec, const std::string& n) {
    for (size_t i = 0; i < vec.size(); ++i)
      if (vec[i].name == n) return (int)i;
    return -1;
  };
  switch (k.kind) {
    case VarKey::Kind::Scalar: return find(d.scalars(), k.name);
    case VarKey::Kind::Element: return 2 * S + V + k.index;
    case VarKey::Kind::Abstract: {
      const int s = find(d.scalars(), k.name);
      return s >= 0 ? S + s : 2 * S + find(d.views(), k.name);
    }
  }
  return -1;
}

static uint64_t store_bits(const Store& st, const Declarations& d) {
  uint64_t out = 0;
  for (const auto& [k, pr] : st) out |= (uint64_t)pair_bits(pr) << (2 * key_index(d, k));
  return out;
}

static void sweep_node(const AnnotatedProgram& p, uint64_t seed, std::vector<bool>& prefix, int max_dec, int fuel,
                       std::vector<coh_sweep_leaf>& out) {
  AnnotatedRun r = run_annotated(p, fuel, Schedule(prefix));
  const bool exhausted = r.schedule_consumed >= prefix.size() && r.schedule_overflowed;
  if (exhausted && (int)prefix.size() < max_dec) {
    for (bool bit : {true, false}) {
      prefix.push_back(bit);
      sweep_node(p, seed, prefix, max_dec, fuel, out);
      prefix.pop_back();
    }
    return;
  }
  coh_sweep_leaf lf;
  std::memset(&lf, 0, sizeof lf);
  lf.seed = seed;
  for (size_t i = 0; i < prefix.size(); ++i) lf.schedule |= (prefix[i] ? 1u : 0u) << i;
  lf.sched_len = (uint8_t)prefix.size();
  lf.status = (uint8_t)r.status;
  lf.blocks_done = (uint8_t)r.boundary_ok.size();
  for (size_t b = 0; b < r.boundary_ok.size(); ++b) lf.boundary_ok |= (r.boundary_ok[b] ? 1u : 0u) << b;
  lf.steps = (uint32_t)r.steps;
  lf.consumed = (uint8_t)r.schedule_consumed;
  lf.overflowed = r.schedule_overflowed ? 1 : 0;
  if (r.stuck) {
    lf.stuck_key = (uint8_t)key_index(p.decls, r.stuck->key);
    lf.stuck_info = (uint8_t)((uint32_t)r.stuck->effect | ((r.stuck->site == Site::Remote ? 1u : 0u) << 3) |
                              ((r.stuck->key.kind == VarKey::Kind::Abstract ? 1u : 0u) << 4) |
                              (pair_bits(r.stuck->actual) << 5));
  }
  lf.store = store_bits(r.store, p.decls);
  out.push_back(lf);
}

// Leaves of all_schedules_run over seeds [seed0, seed0+n) (testkit.hpp:465-517 order).
// Returns the number of leaves (may exceed cap) or -1.
int64_t ref_sweep_leaves(uint64_t seed0, uint32_t n, uint32_t max_dec, int32_t fuel, coh_sweep_leaf* leaves,
                         uint64_t cap) {
  std::vector<coh_sweep_leaf> all;
  try {
    for (uint32_t k = 0; k < n; ++k) {
      AnnotatedProgram p = gen_well_declared(seed0 + k, GenLimits());
      std::vector<bool> prefix;
      sweep_node(p, seed0 + k, prefix, (int)max_dec, fuel, all);
    }
  } catch (...) {
    return -1;
  }
  for (uint64_t i = 0; i < all.size() && i < cap; ++i) leaves[i] = all[i];
  return (int64_t)all.size();
}

// The acceptance gate's own aggregate (tests/acceptance.cpp:77-105): runs, outcomes,
// boundary and oracle agreement via all_schedules_run(with_oracle = true).
int ref_sweep_stats(uint64_t seed0, uint32_t n, uint32_t max_dec, int32_t fuel, uint64_t* out6) {
  uint64_t runs = 0, done = 0, stuck = 0, fuelx = 0, bad_bnd = 0, oracle_bad = 0;
  for (uint32_t k = 0; k < n; ++k) {
    AnnotatedProgram p = gen_well_declared(seed0 + k, GenLimits());
    ScheduleSweep sw = all_schedules_run(p, (int)max_dec, fuel, true);
    runs += sw.runs;
    done += sw.outcomes[RunStatus::Done];
    stuck += sw.outcomes[RunStatus::Stuck];
    fuelx += sw.outcomes[RunStatus::FuelExhausted];
    bad_bnd += sw.all_boundaries_ok ? 0 : 1;
    oracle_bad += sw.oracle_agreed ? 0 : 1;
  }
  out6[0] = runs;
  out6[1] = done;
  out6[2] = stuck;
  out6[3] = fuelx;
  out6[4] = bad_bnd;
  out6[5] = oracle_bad;
  return 0;
}

}  // extern "C"
