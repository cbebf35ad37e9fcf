// General block programs: opaque if/while with schedules, several
// modes per block, scalars + one buffer with overlapping views, element bodies.  Host side:
//   * a restatement of the test kit's program generator gen_well_declared
//     (testkit.hpp:291-447: std::mt19937_64 seeded seed*0x9E3779B97F4A7C15+1, modulo
//     draws, the same draw order) so the acceptance corpus can be generated natively;
//   * the block-level overlap closure infer_overlap_closure (overlap.hpp:182-230);
//   * translate_block (modes.hpp:31-59) into a compact bytecode for the device
//     interpreter (sweep.cu);
//   * a renderer in the reference's canonical `pretty` form (pretty.hpp:41-148), used by
//     the tests to pin the generator against the reference text, program by program.
#include <algorithm>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"
#include "sweep.hpp"

namespace cohb {
namespace {

// ---- a small statement tree (normalised: a block is a list of primitive statements) ----
struct GTarget {
  uint8_t kind = 0;  // 0 scalar, 1 abstract, 2 element, 3 whole view
  uint8_t var = 0;   // scalar index, or view index (abstract of a view: var = view, is_view)
  bool is_view = false;
  uint32_t offset = 0;  // element: view-relative index
};
struct GCond {
  uint8_t kind = 2;  // 0 valid, 1 gvalid, 2 opaque
  GTarget key;       // scalar (concrete) or abstract key
};
struct GStmt {
  uint8_t kind = 0;  // 0 effect, 1 if, 2 while
  uint8_t eff = 0, site = 0;
  GTarget t;
  GCond c;
  std::vector<GStmt> a, b;  // then / body, else
};
using GList = std::vector<GStmt>;

struct GMode {
  uint8_t kind, site;
  bool is_view;
  uint8_t var;
  bool shadow;
};
struct GBlock {
  std::vector<GMode> modes;
  GList body;
};
struct GProgram {
  uint32_t n_scalars = 0;
  bool has_buffer = false;
  uint32_t buf_len = 0;
  std::vector<uint32_t> vlo, vhi;
  std::vector<GBlock> blocks;
};

struct Rng {
  std::mt19937_64 eng;
  explicit Rng(uint64_t seed) : eng(seed) {}
  uint32_t pick(uint32_t n) { return n ? (uint32_t)(eng() % n) : 0; }
  bool percent(uint32_t p) { return pick(100) < p; }
};

struct GVar {
  bool is_view;
  uint8_t var;
  uint32_t length;
  uint8_t kind, site;
};

void append(GList& out, GList&& x) {
  for (auto& s : x) out.push_back(std::move(s));
}

// gen_extra (testkit.hpp:309-360); returns a normalised list
GList gen_extra(Rng& rng, const std::vector<GVar>& vars, int depth, int& opaque_budget, int& loops_left) {
  auto effect = [&]() -> GList {
    if (vars.empty()) return {};
    const GVar& v = vars[rng.pick((uint32_t)vars.size())];
    const bool can_read = v.kind != COH_W, can_write = v.kind != COH_R;
    const bool write = can_write && (!can_read || rng.percent(40));
    GStmt s;
    s.kind = 0;
    s.eff = write ? COH_WRITE : COH_READ;
    s.site = v.site;
    if (v.is_view) {
      s.t.kind = 2;
      s.t.is_view = true;
      s.t.var = v.var;
      s.t.offset = rng.pick(v.length);
    } else {
      s.t.kind = 0;
      s.t.var = v.var;
    }
    return {s};
  };
  auto condition = [&]() -> GCond {
    GCond c;
    if (opaque_budget > 0 && rng.percent(60)) {
      --opaque_budget;
      c.kind = 2;
      return c;
    }
    if (!vars.empty()) {
      const GVar& v = vars[rng.pick((uint32_t)vars.size())];
      c.key.is_view = v.is_view;
      c.key.var = v.var;
      c.key.kind = v.is_view ? 1 : 0;  // abstract(view) or scalar (concrete)
      c.kind = rng.percent(50) ? 0 : 1;
      return c;
    }
    if (opaque_budget > 0) {
      --opaque_budget;
      c.kind = 2;
      return c;
    }
    c.kind = 0;  // unreachable with non-empty vars (testkit.hpp:338)
    return c;
  };
  const uint32_t roll = rng.pick(10);
  if (depth > 0 && roll < 2) {
    GList then_s = gen_extra(rng, vars, depth - 1, opaque_budget, loops_left);
    GList else_s;
    if (rng.percent(60)) else_s = gen_extra(rng, vars, depth - 1, opaque_budget, loops_left);
    GStmt s;
    s.kind = 1;
    s.c = condition();
    s.a = std::move(then_s);
    s.b = std::move(else_s);
    return {s};
  }
  if (depth > 0 && roll < 4 && loops_left > 0 && opaque_budget > 0) {
    --loops_left;
    --opaque_budget;
    GStmt s;
    s.kind = 2;
    s.c.kind = 2;
    s.a = gen_extra(rng, vars, depth - 1, opaque_budget, loops_left);
    return {s};
  }
  if (roll < 8) return effect();
  GList a = effect();
  GList b = effect();
  append(a, std::move(b));
  return a;
}

// infer_overlap_closure for one block (overlap.hpp:182-230): W/RW on a view x make every
// overlapping y (name-sorted query) need RW at x's site (W skips y with a same-site W);
// an existing R is upgraded in place, others appended as shadows in declaration order.
bool close_block(const GProgram& p, std::vector<GMode>& modes) {
  auto overl = [&](uint32_t x, uint32_t y) { return x != y && p.vlo[x] <= p.vhi[y] && p.vlo[y] <= p.vhi[x]; };
  std::map<std::string, uint8_t> needed;  // view name -> site (map: name order)
  const std::vector<GMode> declared = modes;
  for (const auto& m : declared) {
    if (m.kind == COH_R || m.shadow || !m.is_view) continue;
    for (uint32_t y = 0; y < p.vlo.size(); ++y) {
      if (!overl(m.var, y)) continue;
      if (m.kind == COH_W) {
        bool same = false;
        for (const auto& o : declared)
          if (o.is_view && o.var == y && o.kind == COH_W && o.site == m.site) same = true;
        if (same) continue;
      }
      const std::string name = "v" + std::to_string(y);
      auto it = needed.find(name);
      if (it == needed.end()) needed.emplace(name, m.site);
      else if (it->second != m.site) return false;  // OverlapInferenceError
    }
  }
  std::vector<std::pair<uint32_t, uint8_t>> shadows;
  for (const auto& [name, site] : needed) {
    const uint32_t y = (uint32_t)std::stoul(name.substr(1));
    GMode* existing = nullptr;
    for (auto& m : modes)
      if (m.is_view && m.var == y) existing = &m;
    if (existing) {
      if (existing->site != site) return false;
      if (existing->kind == COH_R) existing->kind = COH_RW;
    } else {
      shadows.emplace_back(y, site);
    }
  }
  for (uint32_t v = 0; v < p.vlo.size(); ++v)
    for (const auto& [y, site] : shadows)
      if (y == v) modes.push_back(GMode{COH_RW, site, true, (uint8_t)y, true});
  return true;
}

// gen_well_declared (testkit.hpp:364-447) with the default GenLimits (:279-287)
GProgram generate(uint64_t seed, const coh_gen_limits& L, bool* ok) {
  Rng rng(seed * 0x9E3779B97F4A7C15ull + 1);
  GProgram p;
  p.n_scalars = 1 + rng.pick(L.max_vars);
  if (L.allow_arrays) {
    const uint32_t len = 2 + rng.pick(L.max_buffer_len - 1);
    p.has_buffer = true;
    p.buf_len = len;
    const uint32_t n_views = 1 + rng.pick(L.max_vars);
    for (uint32_t i = 0; i < n_views; ++i) {
      uint32_t lo, hi;
      if (L.allow_overlaps) {
        lo = rng.pick(len);
        hi = lo + rng.pick(len - lo);
      } else {
        const uint32_t used = p.vlo.empty() ? 0 : p.vhi.back() + 1;
        if (used >= len) break;
        lo = used;
        hi = lo + rng.pick(len - lo);
      }
      p.vlo.push_back(lo);
      p.vhi.push_back(hi);
    }
  }
  const uint32_t n_blocks = 1 + rng.pick(L.max_blocks);
  int opaque_budget = 3;
  for (uint32_t bi = 0; bi < n_blocks; ++bi) {
    const uint8_t buffer_site = rng.percent(50) ? COH_LOCAL : COH_REMOTE;
    std::vector<GVar> chosen;
    std::vector<GMode> modes;
    for (uint32_t s = 0; s < p.n_scalars; ++s) {
      if (!rng.percent(60)) continue;
      GVar v{false, (uint8_t)s, 1, 0, 0};
      v.site = rng.percent(50) ? COH_LOCAL : COH_REMOTE;
      v.kind = (uint8_t)rng.pick(3);
      chosen.push_back(v);
      modes.push_back(GMode{v.kind, v.site, false, v.var, false});
    }
    for (uint32_t vi = 0; vi < p.vlo.size(); ++vi) {
      if (!rng.percent(55)) continue;
      GVar v{true, (uint8_t)vi, p.vhi[vi] - p.vlo[vi] + 1, 0, buffer_site};
      v.kind = (uint8_t)rng.pick(3);
      chosen.push_back(v);
      modes.push_back(GMode{v.kind, v.site, true, v.var, false});
    }
    GList body;
    for (const auto& v : chosen) {
      if (v.kind != COH_W) continue;
      if (v.is_view) {
        for (uint32_t i = 0; i < v.length; ++i) {
          GStmt s;
          s.eff = COH_WRITE;
          s.site = v.site;
          s.t.kind = 2;
          s.t.is_view = true;
          s.t.var = v.var;
          s.t.offset = i;
          body.push_back(s);
        }
      } else {
        GStmt s;
        s.eff = COH_WRITE;
        s.site = v.site;
        s.t.kind = 0;
        s.t.var = v.var;
        body.push_back(s);
      }
    }
    int loops_left = (int)L.max_loop_unroll;
    const uint32_t n_extras = rng.pick(4);
    for (uint32_t i = 0; i < n_extras && !chosen.empty(); ++i)
      append(body, gen_extra(rng, chosen, (int)L.max_body_depth, opaque_budget, loops_left));
    p.blocks.push_back(GBlock{modes, std::move(body)});
  }
  *ok = true;
  if (!p.vlo.empty())
    for (auto& b : p.blocks)
      if (!close_block(p, b.modes)) *ok = false;
  return p;
}

// ---- rendering in the reference's pretty() form ---------------------------------------
std::string name_of(const GTarget& t, bool abstract_key) {
  const std::string base = t.is_view ? "v" + std::to_string(t.var) : "s" + std::to_string(t.var);
  return abstract_key ? base + "^" : base;
}

std::string target_str(const GTarget& t) {
  switch (t.kind) {
    case 0: return "s" + std::to_string(t.var);
    case 1: return name_of(t, true);
    case 2: return "v" + std::to_string(t.var) + "[" + std::to_string(t.offset) + "]";
    default: return "v" + std::to_string(t.var);
  }
}

const char* eff_word(uint32_t e) {
  static const char* n[] = {"push", "pull", "r", "w", "noop"};
  return n[e];
}

void render(const GList& l, int indent, std::string& out) {
  const std::string pad(2 * (size_t)indent, ' ');
  for (const auto& s : l) {
    if (s.kind == 0) {
      out += pad + (s.site ? "g" : "") + eff_word(s.eff) + " " + target_str(s.t) + ";\n";
      continue;
    }
    std::string cond;
    if (s.c.kind == 2) cond = "opaque";
    else cond = std::string(s.c.kind == 0 ? "valid(" : "gvalid(") + (s.c.key.kind == 1 ? name_of(s.c.key, true) : name_of(s.c.key, false)) + ")";
    out += pad + (s.kind == 1 ? "if (" : "while (") + cond + ") {\n";
    render(s.a, indent + 1, out);
    if (s.kind == 1 && !s.b.empty()) {
      out += pad + "} else {\n";
      render(s.b, indent + 1, out);
    }
    out += pad + "}\n";
  }
}

std::string pretty(const GProgram& p) {
  std::string out;
  for (uint32_t s = 0; s < p.n_scalars; ++s) out += "scalar s" + std::to_string(s) + "\n";
  if (p.has_buffer) out += "buffer b0[" + std::to_string(p.buf_len) + "]\n";
  for (uint32_t v = 0; v < p.vlo.size(); ++v)
    out += "view v" + std::to_string(v) + " = b0[" + std::to_string(p.vlo[v]) + ":" + std::to_string(p.vhi[v]) + "]\n";
  for (const auto& b : p.blocks) {
    if (!out.empty()) out += "\n";
    std::string header;
    for (const auto& m : b.modes) {
      if (!header.empty()) header += ", ";
      header += std::string(m.site ? "G" : "") + (m.kind == COH_R ? "R" : m.kind == COH_W ? "W" : "RW") + "(" +
                (m.is_view ? "v" : "s") + std::to_string(m.var) + ")";
      if (m.shadow) header += " /*shadow*/";
    }
    out += header + (header.empty() ? "{\n" : " {\n");
    render(b.body, 1, out);
    out += "}\n";
  }
  return out;
}

// ---- bytecode -----------------------------------------------------------------------
// keys: s_i concrete = i, s_i^ = S + i, v_j^ = 2S + j, b0[c] = 2S + V + c
struct Emitter {
  const GProgram& p;
  std::vector<uint32_t> code;
  uint32_t S, V;
  explicit Emitter(const GProgram& q) : p(q), S(q.n_scalars), V((uint32_t)q.vlo.size()) {}
  uint32_t key(const GTarget& t) const {
    switch (t.kind) {
      case 0: return t.var;
      case 1: return t.is_view ? 2 * S + t.var : S + t.var;
      default: return 2 * S + V + p.vlo[t.var] + t.offset;  // element
    }
  }
  void eff(uint32_t e, uint32_t site, uint32_t k) { code.push_back(BC_EFF | (e << 4) | (site << 7) | (k << 8)); }
  void list(const GList& l) {
    for (const auto& s : l) {
      if (s.kind == 0) {
        eff(s.eff, s.site, key(s.t));
        continue;
      }
      const uint32_t ck = s.c.kind == 2 ? 0 : key(s.c.key);
      const uint32_t head = (uint32_t)code.size();
      code.push_back((s.kind == 1 ? BC_IF : BC_WHILE) | ((uint32_t)s.c.kind << 4) | (ck << 8));
      list(s.a);
      if (s.kind == 1) {
        if (!s.b.empty()) {
          const uint32_t j = (uint32_t)code.size();
          code.push_back(BC_JMP);
          code[head] |= (uint32_t)code.size() << 16;  // else target
          list(s.b);
          code[j] |= (uint32_t)code.size() << 16;
        } else {
          code[head] |= (uint32_t)code.size() << 16;
        }
      } else {
        code.push_back(BC_JMP | (head << 16));
        code[head] |= (uint32_t)code.size() << 16;  // exit target
      }
    }
  }
  // translate_mode (modes.hpp:31-50)
  void mode(const GMode& m) {
    const uint32_t sync = m.site ? COH_PUSH : COH_PULL;
    const uint32_t abs_key = m.is_view ? 2 * S + m.var : S + m.var;
    if (m.kind == COH_R || m.kind == COH_RW) {
      const uint32_t head = (uint32_t)code.size();
      code.push_back(BC_IF | ((uint32_t)(m.site ? 1 : 0) << 4) | (abs_key << 8));
      const uint32_t j = (uint32_t)code.size();
      code.push_back(BC_JMP);  // then-branch empty: skip the sync pair
      code[head] |= (uint32_t)code.size() << 16;
      if (m.is_view) {
        const uint32_t lo = 2 * S + V + p.vlo[m.var], hi = 2 * S + V + p.vhi[m.var];
        code.push_back(BC_WHOLE | (sync << 4) | (0u << 7) | (lo << 8) | (hi << 16));
      } else {
        eff(sync, COH_LOCAL, m.var);
      }
      eff(sync, COH_LOCAL, abs_key);
      code[j] |= (uint32_t)code.size() << 16;
    }
    if (m.kind == COH_W || m.kind == COH_RW) eff(COH_WRITE, m.site, abs_key);
  }
};

}  // namespace

int sweep_compile(uint64_t seed, const coh_gen_limits& L, SweepProgram* out, std::string* text) {
  bool ok = true;
  GProgram p = generate(seed, L, &ok);
  if (text) *text = pretty(p);
  if (!ok) return COH_E_OVERLAP_CONFLICT;
  Emitter e(p);
  for (const auto& b : p.blocks) {
    for (const auto& m : b.modes) e.mode(m);
    e.list(b.body);
    e.code.push_back(BC_BEND);
  }
  e.code.push_back(BC_END);
  out->code = std::move(e.code);
  out->n_keys = 2 * e.S + e.V + (p.has_buffer ? p.buf_len : 0);
  out->n_blocks = (uint32_t)p.blocks.size();
  out->checks.clear();
  for (uint32_t s = 0; s < e.S; ++s) out->checks.push_back((uint16_t)((e.S + s) | (s << 8)));
  for (uint32_t v = 0; v < e.V; ++v)
    for (uint32_t c = p.vlo[v]; c <= p.vhi[v]; ++c)
      out->checks.push_back((uint16_t)((2 * e.S + v) | ((2 * e.S + e.V + c) << 8)));
  out->n_scalars = e.S;
  out->n_views = e.V;
  out->buf_len = p.has_buffer ? p.buf_len : 0;
  return COH_OK;
}

}  // namespace cohb

extern "C" int coh_gen_program_text(uint64_t seed, const coh_gen_limits* limits, char* buf, size_t cap) {
  coh_gen_limits L = limits ? *limits : coh_gen_limits{3, 2, 3, 6, 2, 1, 1, 0};
  std::string text;
  cohb::SweepProgram sp;
  const int rc = cohb::sweep_compile(seed, L, &sp, &text);
  if (!buf || cap <= text.size()) return -(int)text.size() - 1;
  std::memcpy(buf, text.c_str(), text.size() + 1);
  return rc;
}

// ---- the schedule sweep (all_schedules_run / sweep_explore, testkit.hpp:465-517) -------
namespace {
struct DevMem {
  void* p = nullptr;
  ~DevMem() { cudaFree(p); }
};
}  // namespace

extern "C" int coh_sweep(coh_ctx* ctx, uint64_t seed0, uint32_t n_seeds, const coh_gen_limits* limits,
                         uint32_t max_decisions, int32_t fuel, coh_sweep_leaf* leaves, uint64_t leaves_cap,
                         coh_sweep_stats* stats) {
  using namespace cohb;
  if (!ctx || max_decisions > 24) return COH_E_ARG;
  const coh_gen_limits L = limits ? *limits : coh_gen_limits{3, 2, 3, 6, 2, 1, 1, 0};
  if (L.max_blocks > kSweepMaxBlocks) {  // SweepOut carries 5 block bits and 8 boundary bits
    ctx->err = "coh_sweep: max_blocks must be <= " + std::to_string(kSweepMaxBlocks);
    return COH_E_ARG;
  }
  coh_sweep_stats st{};
  std::vector<uint32_t> code;
  std::vector<uint16_t> checks;
  std::vector<SweepMeta> meta;
  std::vector<uint64_t> seeds;
  std::vector<uint32_t> nS, nV;
  // program generation + bytecode compile on all host threads (seed slices), then
  // concatenated in seed order
  const uint32_t n_th = std::max(1u, std::min<uint32_t>(std::thread::hardware_concurrency(), (n_seeds + 255) / 256));
  std::vector<std::vector<SweepProgram>> part(n_th);
  std::vector<std::vector<uint64_t>> part_seed(n_th);
  std::vector<uint64_t> part_conflicts(n_th, 0);
  std::vector<int> part_err(n_th, 0);
  {
    std::vector<std::thread> pool;
    for (uint32_t th = 0; th < n_th; ++th)
      pool.emplace_back([&, th] {
        const uint32_t k0 = (uint32_t)((uint64_t)n_seeds * th / n_th), k1 = (uint32_t)((uint64_t)n_seeds * (th + 1) / n_th);
        for (uint32_t k = k0; k < k1; ++k) {
          SweepProgram sp;
          if (sweep_compile(seed0 + k, L, &sp, nullptr) != COH_OK) {
            part_conflicts[th]++;  // OverlapInferenceError: the reference generator would throw
            continue;
          }
          if (sp.n_keys > 32 || sp.code.size() > 65535) {
            part_err[th] = (int)(k - k0) + 1;
            return;
          }
          part[th].push_back(std::move(sp));
          part_seed[th].push_back(seed0 + k);
        }
      });
    for (auto& t : pool) t.join();
  }
  for (uint32_t th = 0; th < n_th; ++th) {
    if (part_err[th]) {
      ctx->err = "a generated program exceeds the 32-key / 64K-instruction interpreter";
      return COH_E_CONSTRUCTION;
    }
    st.conflicts += part_conflicts[th];
    for (size_t j = 0; j < part[th].size(); ++j) {
      const SweepProgram& sp = part[th][j];
      meta.push_back(SweepMeta{(uint32_t)code.size(), sp.n_keys, (uint32_t)checks.size(), (uint32_t)sp.checks.size()});
      code.insert(code.end(), sp.code.begin(), sp.code.end());
      checks.insert(checks.end(), sp.checks.begin(), sp.checks.end());
      seeds.push_back(part_seed[th][j]);
      nS.push_back(sp.n_scalars);
      nV.push_back(sp.n_views);
    }
  }
  st.programs = meta.size();
  DevMem d_code, d_meta, d_checks, d_items, d_out;
#define COH_S(x)                                                  \
  do {                                                            \
    cudaError_t e_ = (x);                                         \
    if (e_ != cudaSuccess) {                                      \
      ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_); \
      return COH_E_CUDA;                                          \
    }                                                             \
  } while (0)
  if (!ctx->hs[0]) COH_S(cudaStreamCreateWithFlags(&ctx->hs[0], cudaStreamNonBlocking));
  cudaStream_t s = ctx->hs[0];
  COH_S(cudaMalloc(&d_code.p, std::max<size_t>(code.size() * 4, 16)));
  COH_S(cudaMalloc(&d_meta.p, std::max<size_t>(meta.size() * sizeof(SweepMeta), 16)));
  COH_S(cudaMalloc(&d_checks.p, std::max<size_t>(checks.size() * 2, 16)));
  if (!code.empty()) COH_S(cudaMemcpyAsync(d_code.p, code.data(), code.size() * 4, cudaMemcpyHostToDevice, s));
  if (!meta.empty()) COH_S(cudaMemcpyAsync(d_meta.p, meta.data(), meta.size() * sizeof(SweepMeta), cudaMemcpyHostToDevice, s));
  if (!checks.empty()) COH_S(cudaMemcpyAsync(d_checks.p, checks.data(), checks.size() * 2, cudaMemcpyHostToDevice, s));
  std::vector<SweepItem> frontier(meta.size());
  for (uint32_t p = 0; p < meta.size(); ++p) frontier[p] = SweepItem{p, 0, 0, 0};
  size_t cap = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float total_ms = 0.f;
  uint64_t n_leaves = 0;
  std::vector<SweepOut> out;
  for (uint32_t level = 0; !frontier.empty(); ++level) {
    const size_t n = frontier.size();
    if (n > cap) {
      cudaFree(d_items.p);
      cudaFree(d_out.p);
      d_items.p = d_out.p = nullptr;
      cap = n * 2;
      COH_S(cudaMalloc(&d_items.p, cap * sizeof(SweepItem)));
      COH_S(cudaMalloc(&d_out.p, cap * sizeof(SweepOut)));
    }
    COH_S(cudaMemcpyAsync(d_items.p, frontier.data(), n * sizeof(SweepItem), cudaMemcpyHostToDevice, s));
    std::string err;
    COH_S(cudaEventRecord(e0, s));
    int rc = launch_sweep_run(static_cast<uint32_t*>(d_code.p), static_cast<SweepMeta*>(d_meta.p),
                              static_cast<uint16_t*>(d_checks.p), static_cast<SweepItem*>(d_items.p), (uint32_t)n,
                              fuel, static_cast<SweepOut*>(d_out.p), s, &err);
    if (rc) {
      ctx->err = err;
      return rc;
    }
    COH_S(cudaEventRecord(e1, s));
    out.resize(n);
    COH_S(cudaMemcpyAsync(out.data(), d_out.p, n * sizeof(SweepOut), cudaMemcpyDeviceToHost, s));
    COH_S(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    total_ms += ms;
    st.launches++;
    ctx->launches++;
    std::vector<SweepItem> next;
    for (size_t k = 0; k < n; ++k) {
      const SweepItem& it = frontier[k];
      const SweepOut& o = out[k];
      st.nodes++;
      const uint32_t consumed = (o.status_consumed >> 2) & 0xFFu, overflowed = (o.status_consumed >> 10) & 1u;
      // sweep_explore: a run that consumed its whole prefix and wanted more branches
      if (consumed >= it.len && overflowed && it.len < max_decisions) {
        next.push_back(SweepItem{it.prog, it.bits | (1u << it.len), it.len + 1, 0});  // answer 1 first
        next.push_back(SweepItem{it.prog, it.bits, it.len + 1, 0});
        continue;
      }
      const uint32_t status = o.status_consumed & 3u;
      st.runs++;
      if (status == COH_RUN_DONE) st.done++;
      else if (status == COH_RUN_STUCK) st.stuck++;
      else st.fuel_exhausted++;
      const uint32_t blocks = (o.status_consumed >> 11) & 31u, bnd = (o.status_consumed >> 16) & 0xFFu;
      if (bnd != (blocks >= 8 ? 0xFFu : ((1u << blocks) - 1u))) st.runs_with_violation++;
      if (leaves && n_leaves < leaves_cap) {
        coh_sweep_leaf& lf = leaves[n_leaves];
        lf.seed = seeds[it.prog];
        lf.schedule = it.bits;
        lf.sched_len = (uint8_t)it.len;
        lf.status = (uint8_t)status;
        lf.blocks_done = (uint8_t)blocks;
        lf.boundary_ok = (uint8_t)bnd;
        lf.steps = o.steps;
        lf.consumed = (uint8_t)consumed;
        lf.overflowed = (uint8_t)overflowed;
        lf.stuck_key = status == COH_RUN_STUCK ? (uint8_t)(o.status_consumed >> 24) : 0;
        const uint32_t S = nS[it.prog], V = nV[it.prog];
        const bool abs_key = lf.stuck_key >= S && lf.stuck_key < 2 * S + V;
        lf.stuck_info = status == COH_RUN_STUCK ? (uint8_t)(o.stuck | (abs_key ? 16u : 0u)) : 0;
        lf.store = o.store;
      }
      n_leaves++;
    }
    frontier.swap(next);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  st.device_ms = total_ms;
  if (stats) *stats = st;
  return COH_OK;
#undef COH_S
}

// ---- acceptance criterion 1 (tests/acceptance.cpp:107-138) ---------------------------
// enumerate_raw_programs (testkit.hpp:241-268): every straight-line program of length
// <= max_len over the ten effect forms (push, pull, r, w, noop x local, remote) on one
// scalar, run from initial_store on the GPU block interpreter; counts of outcomes and of
// programs that ever reach an unsafe (I,I) key.
extern "C" int coh_enum_straight_line(coh_ctx* ctx, uint32_t max_len, int32_t fuel, coh_enum_stats* stats,
                                      uint8_t* statuses, uint64_t statuses_cap) {
  using namespace cohb;
  if (!ctx || !stats || max_len > 8) return COH_E_ARG;
  std::vector<uint32_t> code;
  std::vector<SweepMeta> meta;
  std::vector<uint32_t> prog;  // current program: form indices
  // breadth-first by length, forms in the reference's order (kind-major, then site)
  std::vector<std::vector<uint32_t>> frontier = {{}};
  auto emit = [&](const std::vector<uint32_t>& p) {
    meta.push_back(SweepMeta{(uint32_t)code.size(), 2u, 0u, 0u});  // keys: x = 0, x^ = 1
    for (uint32_t f : p) code.push_back(BC_EFF | ((f / 2) << 4) | ((f % 2) << 7) | (0u << 8));
    code.push_back(BC_END);
  };
  emit({});
  for (uint32_t len = 1; len <= max_len; ++len) {
    std::vector<std::vector<uint32_t>> next;
    for (const auto& pre : frontier)
      for (uint32_t f = 0; f < 10; ++f) {
        std::vector<uint32_t> p = pre;
        p.push_back(f);
        emit(p);
        next.push_back(std::move(p));
      }
    frontier.swap(next);
  }
  const uint32_t n = (uint32_t)meta.size();
  std::vector<SweepItem> items(n);
  for (uint32_t i = 0; i < n; ++i) items[i] = SweepItem{i, 0, 0, 0};
  DevMem d_code, d_meta, d_checks, d_items, d_out;
  cudaStream_t s = nullptr;
#define COH_S(x)                                                  \
  do {                                                            \
    cudaError_t e_ = (x);                                         \
    if (e_ != cudaSuccess) {                                      \
      ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_); \
      return COH_E_CUDA;                                          \
    }                                                             \
  } while (0)
  COH_S(cudaMalloc(&d_code.p, code.size() * 4));
  COH_S(cudaMalloc(&d_meta.p, meta.size() * sizeof(SweepMeta)));
  COH_S(cudaMalloc(&d_checks.p, 16));
  COH_S(cudaMalloc(&d_items.p, items.size() * sizeof(SweepItem)));
  COH_S(cudaMalloc(&d_out.p, items.size() * sizeof(SweepOut)));
  COH_S(cudaMemcpy(d_code.p, code.data(), code.size() * 4, cudaMemcpyHostToDevice));
  COH_S(cudaMemcpy(d_meta.p, meta.data(), meta.size() * sizeof(SweepMeta), cudaMemcpyHostToDevice));
  COH_S(cudaMemcpy(d_items.p, items.data(), items.size() * sizeof(SweepItem), cudaMemcpyHostToDevice));
  std::string err;
  int rc = launch_sweep_run(static_cast<uint32_t*>(d_code.p), static_cast<SweepMeta*>(d_meta.p),
                            static_cast<uint16_t*>(d_checks.p), static_cast<SweepItem*>(d_items.p), n, fuel,
                            static_cast<SweepOut*>(d_out.p), s, &err);
  if (rc) {
    ctx->err = err;
    return rc;
  }
  std::vector<SweepOut> out(n);
  COH_S(cudaMemcpy(out.data(), d_out.p, n * sizeof(SweepOut), cudaMemcpyDeviceToHost));
#undef COH_S
  ctx->launches++;
  coh_enum_stats st{};
  st.programs = n;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t status = out[i].status_consumed & 3u;
    if (status == COH_RUN_DONE) st.done++;
    else if (status == COH_RUN_STUCK) st.stuck++;
    else st.fuel_exhausted++;
    st.unsafe += out[i].pad ? 1 : 0;
    st.steps += out[i].steps;
    if (statuses && i < statuses_cap) statuses[i] = (uint8_t)status;
  }
  *stats = st;
  return COH_OK;
}
