// cohere_b200_shim.hpp -- the reference-side binding a maintainer adds next to
// cohere/modes.hpp: whole-array AnnotatedPrograms (program.hpp:237-243) in, AnnotatedRun
// values (modes.hpp:95-103) out, evaluated as one GPU batch through the C ABI
// (include/cohere_b200.h, coh_eval_traces_host).  Header-only; include it after
// "cohere/cohere.hpp" (it uses the reference's own types) and link libcohere_b200.so.
//
//   encode_program   AnnotatedProgram -> call records (COH_REC_CONT between the modes of
//                    one DeclBlock) or a reason it is not expressible as records
//   decode_records   call records -> the AnnotatedProgram they stand for (round trip)
//   run_annotated_batch
//                    many programs, one coh_eval_traces_host call (COH_BATCH_BLOCKS),
//                    results unpacked into AnnotatedRun (status, store, stuck,
//                    boundary_ok, steps) exactly as run_annotated returns them
//
// Expressible programs: declarations are scalars only (at most 64, the whole arrays); every
// block body is, mode by mode in declaration order, one of the record body variants on
// that mode's own scalar (canonical `r`/`w`/`r; w` at the mode's site, empty,
// `r`@other site, `w`@other, `r`@site, `w; r`@other, `push`@site, `pull; w`@other).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "cohere_b200.h"

namespace cohere::b200 {

namespace detail {
// Body variant v of a mode (kind k, site s) as (effect, site) pairs; the same table the
// device compiles (calltable.cpp body_ops).
inline std::vector<std::pair<EffectKind, Site>> variant_body(uint32_t kind, Site s, uint32_t v) {
  const Site o = s == Site::Local ? Site::Remote : Site::Local;
  using E = EffectKind;
  switch (v) {
    case 0:
      if (kind == 0) return {{E::Read, s}};
      if (kind == 1) return {{E::Write, s}};
      return {{E::Read, s}, {E::Write, s}};
    case 1: return {};
    case 2: return {{E::Read, o}};
    case 3: return {{E::Write, o}};
    case 4: return {{E::Read, s}};
    case 5: return {{E::Write, s}, {E::Read, o}};
    case 6: return {{E::Push, s}};
    default: return {{E::Pull, s}, {E::Write, o}};
  }
}

// The effects of a normalized straight-line body; false if it branches or loops.
inline bool flatten(const Stmt& s, std::vector<const Stmt::Node*>& out) {
  switch (s.op()) {
    case Stmt::Op::Noop: return true;
    case Stmt::Op::Effect: out.push_back(&s.node()); return true;
    case Stmt::Op::Seq: return flatten(s.seq_a(), out) && flatten(s.seq_b(), out);
    default: return false;
  }
}
}  // namespace detail

// Records of one program (one trace); n_arrays = its scalar count.  Returns "" or why the
// program cannot be expressed as records.
inline std::string encode_program(const AnnotatedProgram& p, std::vector<uint16_t>* recs, uint32_t* n_arrays) {
  const auto& sc = p.decls.scalars();
  if (sc.empty() || sc.size() > COH_MAX_ARRAYS) return "needs 1..64 scalar declarations";
  if (!p.decls.buffers().empty() || !p.decls.views().empty()) return "buffers / views are the element path";
  auto index_of = [&](const std::string& n) -> int {
    for (size_t i = 0; i < sc.size(); ++i)
      if (sc[i].name == n) return (int)i;
    return -1;
  };
  recs->clear();
  for (const DeclBlock& b : p.blocks) {
    if (b.modes.empty()) return "a block without modes has no record";
    std::vector<const Stmt::Node*> fx;
    if (!detail::flatten(normalize(b.body), fx)) return "a body with if / while";
    size_t at = 0;
    for (size_t m = 0; m < b.modes.size(); ++m) {
      const AccessMode& md = b.modes[m];
      const int a = index_of(md.view);
      if (a < 0) return "mode on an undeclared scalar '" + md.view + "'";
      // this mode's segment: the effects on its own scalar, then the first matching variant
      size_t end = at;
      while (end < fx.size() && fx[end]->target.kind == Target::Kind::Scalar && fx[end]->target.name == md.view) ++end;
      const uint32_t kind = (uint32_t)md.kind;
      int variant = -1;
      for (uint32_t v = 0; v < COH_N_VARIANTS && variant < 0; ++v) {
        const auto want = detail::variant_body(kind, md.site, v);
        bool same = want.size() == end - at;
        for (size_t k = 0; same && k < want.size(); ++k)
          same = fx[at + k]->effect == want[k].first && fx[at + k]->site == want[k].second;
        if (same) variant = (int)v;
      }
      if (variant < 0) return "the body of '" + md.view + "' is not a record variant";
      uint16_t r = COH_MAKE_REC((uint32_t)a, kind, md.site == Site::Remote ? 1u : 0u, (uint32_t)variant);
      if (m) r |= COH_REC_CONT;
      recs->push_back(r);
      at = end;
    }
    if (at != fx.size()) return "body effects outside the block's modes' segments";
  }
  *n_arrays = (uint32_t)sc.size();
  return "";
}

// The program a record sequence stands for (scalars a0..a{n-1}).
inline AnnotatedProgram decode_records(const std::vector<uint16_t>& recs, uint32_t n_arrays,
                                       const std::vector<std::string>& names) {
  AnnotatedProgram p;
  for (uint32_t a = 0; a < n_arrays; ++a) p.decls.add_scalar({names[a], {}});
  for (size_t i = 0; i < recs.size();) {
    std::vector<AccessMode> modes;
    std::vector<Stmt> body;
    do {
      const uint16_t r = recs[i];
      AccessMode m;
      m.kind = static_cast<AccessMode::Kind>(COH_REC_KIND(r));
      m.site = COH_REC_SITE(r) ? Site::Remote : Site::Local;
      m.view = names[COH_REC_ARRAY(r)];
      for (const auto& [e, s] : detail::variant_body(COH_REC_KIND(r), m.site, COH_REC_VARIANT(r)))
        body.push_back(Stmt::effect(e, p.decls.scalar_target(m.view), s));
      modes.push_back(m);
      ++i;
    } while (i < recs.size() && (recs[i] & COH_REC_CONT));
    p.blocks.emplace_back(std::move(modes), normalize(Stmt::seq(body)));
  }
  return p;
}

// run_annotated (modes.hpp:105) for many whole-array programs: one device batch per
// distinct record count (a batch's traces share their length); fuel is shared across each
// program's blocks as in the reference.
inline std::vector<AnnotatedRun> run_annotated_batch(coh_ctx* ctx, const std::vector<AnnotatedProgram>& progs,
                                                     int fuel);

namespace detail {
inline void run_same_length(coh_ctx* ctx, const std::vector<AnnotatedProgram>& all, const std::vector<size_t>& idx,
                            const std::vector<std::vector<uint16_t>>& enc, uint32_t arrays, int fuel,
                            std::vector<AnnotatedRun>& result);
}  // namespace detail

inline std::vector<AnnotatedRun> run_annotated_batch(coh_ctx* ctx, const std::vector<AnnotatedProgram>& progs,
                                                     int fuel) {
  std::vector<std::vector<uint16_t>> enc(progs.size());
  std::vector<std::pair<size_t, std::vector<size_t>>> groups;  // record count -> programs
  uint32_t arrays = 1;
  for (size_t t = 0; t < progs.size(); ++t) {
    uint32_t na = 0;
    const std::string why = encode_program(progs[t], &enc[t], &na);
    if (!why.empty()) throw std::invalid_argument("program " + std::to_string(t) + ": " + why);
    arrays = na > arrays ? na : arrays;
    size_t g = 0;
    while (g < groups.size() && groups[g].first != enc[t].size()) ++g;
    if (g == groups.size()) groups.push_back({enc[t].size(), {}});
    groups[g].second.push_back(t);
  }
  std::vector<AnnotatedRun> out(progs.size());
  for (const auto& grp : groups) detail::run_same_length(ctx, progs, grp.second, enc, arrays, fuel, out);
  return out;
}

inline void detail::run_same_length(coh_ctx* ctx, const std::vector<AnnotatedProgram>& all,
                                    const std::vector<size_t>& idx, const std::vector<std::vector<uint16_t>>& enc,
                                    uint32_t arrays, int fuel, std::vector<AnnotatedRun>& result) {
  const uint64_t n = idx.size();
  const uint32_t calls = n ? (uint32_t)enc[idx[0]].size() : 0u;
  std::vector<AnnotatedProgram> progs;
  std::vector<std::vector<uint16_t>> tr;
  for (size_t k : idx) {
    progs.push_back(all[k]);
    tr.push_back(enc[k]);
  }
  std::vector<uint16_t> rec(coh_records_elems(n, calls));
  for (uint64_t t = 0; t < n; ++t)
    for (uint32_t i = 0; i < calls; ++i) rec[((uint64_t)(i / 8) * n + t) * 8 + i % 8] = tr[t][i];
  coh_trace_batch b{rec.data(), n, calls, arrays, fuel, COH_BATCH_BLOCKS, nullptr};
  std::vector<coh_trace_result> res(n);
  std::vector<uint32_t> bnd((size_t)coh_boundary_words(calls) * n);
  if (n && coh_eval_traces_host(ctx, &b, res.data(), bnd.data()) != COH_OK)
    throw std::runtime_error(coh_last_error(ctx));
  for (uint64_t t = 0; t < n; ++t) {
    const coh_trace_result& r = res[t];
    AnnotatedRun& ar = result[idx[t]];
    if (r.status == COH_RUN_DEFECT) throw std::logic_error("program " + std::to_string(t) + ": defect");
    ar.status = static_cast<RunStatus>(r.status);
    ar.steps = (int)r.steps;
    for (uint32_t i = 0; i < r.calls_done; ++i) ar.boundary_ok.push_back((bnd[(size_t)(i / 32) * n + t] >> (i % 32)) & 1u);
    const auto& sc = progs[t].decls.scalars();
    auto pair = [](uint32_t b2) {
      return ValidityPair{(b2 & 1u) ? Validity::Valid : Validity::Invalid, (b2 & 2u) ? Validity::Valid : Validity::Invalid};
    };
    for (size_t a = 0; a < sc.size(); ++a) {
      const uint32_t nib = coh_result_nibble(&r, (uint32_t)a);
      ar.store.put(VarKey::scalar(sc[a].name), pair(nib & 3u));
      ar.store.put(VarKey::abstract(sc[a].name), pair(nib >> 2));
    }
    if (r.status == COH_RUN_STUCK) {
      StuckInfo s;
      const std::string& x = sc[r.stuck_array].name;
      s.key = (r.stuck_flags & 2u) ? VarKey::abstract(x) : VarKey::scalar(x);
      s.effect = static_cast<EffectKind>(r.stuck_effect);
      s.site = (r.stuck_flags & 1u) ? Site::Remote : Site::Local;
      s.actual = pair((r.stuck_flags >> 2) & 3u);
      ar.stuck = s;
    }
  }
}

}  // namespace cohere::b200
