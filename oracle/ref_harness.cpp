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
}

}  // namespace

extern "C" {

// Evaluate traces [t_begin, t_end) of a record set laid out for n_total traces.
// out / boundary are indexed relative to t_begin; boundary is word-major
// [(i/32) * (t_end - t_begin) + (t - t_begin)] (may be NULL).  Returns 0 or -1.
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
  const uint16_t rec = (uint16_t)(call_type << 6);
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

}  // extern "C"
