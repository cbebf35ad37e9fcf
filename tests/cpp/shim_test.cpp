// TEST INFRASTRUCTURE: the INTEGRATION.md shim (include/cohere_b200_shim.hpp) compiled
// against the unmodified reference headers.  Random whole-array AnnotatedPrograms (1..64
// scalars, multi-mode blocks, record-variant bodies) built with the reference's own
// types:
//   shim_test encode   encode_program -> decode_records gives back an equal program
//   shim_test run      run_annotated_batch on the GPU == cohere::run_annotated, field by field
// Built by oracle/Makefile into oracle/_ref/shim_test (only where /root/reference exists).
#include <cstdio>
#include <cstring>
#include <random>

#include "cohere/cohere.hpp"
#include "cohere_b200_shim.hpp"

using namespace cohere;

static AnnotatedProgram random_program(uint64_t seed, uint32_t n_blocks) {
  std::mt19937_64 rng(seed);
  const uint32_t S = 1 + (uint32_t)(rng() % 64);
  AnnotatedProgram p;
  for (uint32_t a = 0; a < S; ++a) p.decls.add_scalar({"s" + std::to_string(a), {}});
  for (uint32_t b = 0; b < n_blocks; ++b) {
    const uint32_t k = 1 + (uint32_t)(rng() % std::min<uint32_t>(3, S));
    std::vector<AccessMode> modes;
    std::vector<Stmt> body;
    std::vector<uint32_t> used;
    while (modes.size() < k) {
      const uint32_t a = (uint32_t)(rng() % S);
      bool dup = false;
      for (uint32_t u : used) dup |= u == a;
      if (dup) continue;
      used.push_back(a);
      AccessMode m;
      m.kind = static_cast<AccessMode::Kind>(rng() % 3);
      m.site = (rng() & 1) ? Site::Remote : Site::Local;
      m.view = "s" + std::to_string(a);
      const uint32_t v = (rng() % 8 < 6) ? 0u : (uint32_t)(rng() % 8);
      for (const auto& [e, s] : b200::detail::variant_body((uint32_t)m.kind, m.site, v))
        body.push_back(Stmt::effect(e, p.decls.scalar_target(m.view), s));
      modes.push_back(m);
    }
    p.blocks.emplace_back(std::move(modes), normalize(Stmt::seq(body)));
  }
  return p;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "encode";
  const uint32_t n = 600;
  std::vector<AnnotatedProgram> progs;
  for (uint32_t i = 0; i < n; ++i) progs.push_back(random_program(1000 + i, 40));
  int bad = 0;
  if (mode == "encode") {
    for (uint32_t i = 0; i < n; ++i) {
      std::vector<uint16_t> recs;
      uint32_t na = 0;
      const std::string why = b200::encode_program(progs[i], &recs, &na);
      std::vector<std::string> names;
      for (const auto& s : progs[i].decls.scalars()) names.push_back(s.name);
      if (!why.empty() || !(b200::decode_records(recs, na, names) == progs[i])) ++bad;
    }
    std::printf("encode: %u programs, %d mismatches\n", n, bad);
    return bad ? 1 : 0;
  }
  coh_ctx* ctx = nullptr;
  if (coh_ctx_create(0, &ctx) != COH_OK) {
    std::printf("no CUDA device\n");
    return 2;
  }
  for (int fuel : {10000, 90}) {
    const std::vector<AnnotatedRun> got = b200::run_annotated_batch(ctx, progs, fuel);
    for (uint32_t i = 0; i < n; ++i) {
      const AnnotatedRun want = run_annotated(progs[i], fuel, Schedule());
      const AnnotatedRun& g = got[i];
      bool same = g.status == want.status && g.steps == want.steps && g.boundary_ok == want.boundary_ok &&
                  g.store == want.store && g.stuck.has_value() == want.stuck.has_value();
      if (same && want.stuck)
        same = g.stuck->key == want.stuck->key && g.stuck->effect == want.stuck->effect &&
               g.stuck->site == want.stuck->site && g.stuck->actual == want.stuck->actual;
      if (!same && bad++ < 5) std::printf("mismatch: program %u fuel %d\n", i, fuel);
    }
  }
  coh_ctx_destroy(ctx);
  std::printf("run: %u programs x 2 fuels, %d mismatches\n", n, bad);
  return bad ? 1 : 0;
}
