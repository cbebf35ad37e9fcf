// Element-granular path, host side: program generator, overlap closure, and the compiler
// that turns each program into a per-buffer list of device ops plus a host-known step
// timeline.  Everything that depends only on abstract keys runs here (the abstract pairs
// of views evolve independently of concrete cells, which can only stop a run by getting
// stuck); every concrete cell operation runs on the device.
//
//   overlap closure   infer_overlap_closure, overlap.hpp:182-230 (+ overlaps :17-20)
//   translation       translate_mode / translate_block, modes.hpp:31-59
//   stepping / fuel   run, semantics.hpp:253-287 (Done before fuel; If = one step;
//                     an element range op = one step per cell)
//   abstract effects  effect_signature / apply_signature, validity.hpp:79-120 (swap rule
//                     semantics.hpp:109-130)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "elem.hpp"
#include "gen_common.h"
#include "internal.hpp"

namespace cohb {
namespace {

int apply_pair(uint32_t eff, uint32_t site, uint32_t p) {
  uint32_t q = site ? (((p & 1u) << 1) | (p >> 1)) : p;
  int r;
  switch (eff) {
    case COH_PUSH: r = (q & 1u) ? 3 : -1; break;
    case COH_PULL: r = (q & 2u) ? 3 : -1; break;
    case COH_READ: r = (q & 1u) ? (int)q : -1; break;
    case COH_WRITE: r = 1; break;
    default: r = (int)q; break;
  }
  if (r < 0) return -1;
  return site ? (int)((((uint32_t)r & 1u) << 1) | ((uint32_t)r >> 1)) : r;
}

bool overlaps(const coh_elem_program& P, uint32_t x, uint32_t y) {
  return x != y && P.view_lo[x] <= P.view_hi[y] && P.view_lo[y] <= P.view_hi[x];
}

struct Mode {
  uint32_t view, kind, site;
};

// infer_overlap_closure for a block with one declared mode: W/RW on x adds RW@site on
// every overlapping view, appended in view-declaration order (overlap.hpp:212-228); an R
// infers nothing.  (With a single declared mode no cross-site conflict can arise.)
std::vector<Mode> closure(const coh_elem_program& P, const coh_elem_call& c) {
  std::vector<Mode> m{{c.view, c.kind, c.site}};
  if (c.kind == COH_R) return m;
  for (uint32_t y = 0; y < P.n_views; ++y)
    if (overlaps(P, c.view, y)) m.push_back({y, (uint32_t)COH_RW, c.site});
  return m;
}

}  // namespace

int elem_compile(const coh_elem_program* progs, uint32_t n, ElemPlan* plan, std::string* err) {
  plan->n_progs = n;
  plan->tl.assign(n, {});
  uint32_t max_cells = 1;
  std::vector<std::vector<ElemOp>> per(n);
  uint64_t alg = 0;
  for (uint32_t b = 0; b < n; ++b) {
    const coh_elem_program& P = progs[b];
    if (P.n_cells == 0 || P.n_views > COH_MAX_VIEWS) {
      *err = "element program " + std::to_string(b) + ": n_cells must be >= 1 and n_views <= 16";
      return COH_E_CONSTRUCTION;
    }
    if (P.frag_log2 > 32) {  // coh_frag_mask: rho = 2^-frag_log2 down to 2^-32
      *err = "element program " + std::to_string(b) + ": frag_log2 must be <= 32";
      return COH_E_CONSTRUCTION;
    }
    if (P.n_calls > COH_ELEM_MAX_CALLS) {  // ElemOp::call and the stuck call index are 16-bit
      *err = "element program " + std::to_string(b) + ": more than " + std::to_string(COH_ELEM_MAX_CALLS) + " calls";
      return COH_E_CONSTRUCTION;
    }
    for (uint32_t v = 0; v < P.n_views; ++v)
      if (P.view_lo[v] > P.view_hi[v] || P.view_hi[v] >= P.n_cells) {
        *err = "view v" + std::to_string(v) + " range does not fit its buffer";  // program.hpp:65-68
        return COH_E_CONSTRUCTION;
      }
    max_cells = std::max(max_cells, P.n_cells);
    ElemPlan::Timeline& T = plan->tl[b];
    std::vector<ElemOp>& ops = per[b];
    uint32_t abs[COH_MAX_VIEWS];
    for (uint32_t v = 0; v < P.n_views; ++v) abs[v] = 1;  // initial_store: (V,I)
    uint64_t steps = 0;
    const uint64_t fuel = P.fuel < 0 ? 0 : (uint64_t)P.fuel;
    bool stop = false;
    auto fuel_out = [&](uint32_t c) {
      if (steps < fuel) return false;
      T.term_status = COH_RUN_FUEL_EXHAUSTED;
      T.term_call = c;
      stop = true;
      return true;
    };
    auto emit = [&](uint8_t type, uint8_t plane, uint32_t c, uint32_t lo, uint32_t hi) {
      ops.push_back(ElemOp{type, plane, (uint16_t)c, lo, hi, 0});
      T.steps_before.push_back(steps);
      uint32_t packed = 0;
      for (uint32_t v = 0; v < P.n_views; ++v) packed |= abs[v] << (2 * v);
      T.abs_before.push_back(packed);
    };
    for (uint32_t c = 0; c < P.n_calls && !stop; ++c) {
      const coh_elem_call& call = P.calls[c];
      if (call.view >= P.n_views || call.kind > COH_RW || call.n_body > 2) {
        *err = "call " + std::to_string(c) + " of program " + std::to_string(b) + " is malformed";
        return COH_E_CONSTRUCTION;
      }
      for (const Mode& m : closure(P, call)) {
        const uint32_t v = m.view, lo = P.view_lo[v], hi = P.view_hi[v];
        if (m.kind == COH_R || m.kind == COH_RW) {
          if (fuel_out(c)) break;
          steps++;  // if (valid(v^)) / if (gvalid(v^))
          const bool valid = m.site ? (abs[v] >> 1) & 1u : abs[v] & 1u;
          if (!valid) {
            // concrete whole-view sync, Local site (ast.hpp:144): pull needs R, sets L;
            // push needs L, sets R
            const uint32_t sync = m.site ? COH_PUSH : COH_PULL;
            if (fuel_out(c)) break;
            emit(EOP_SYNC, sync == COH_PULL ? 1 : 0, c, lo, hi);
            const uint64_t mcells = (uint64_t)(hi - lo + 1);
            alg += 3 * ((mcells + 7) / 8);  // read src + read dst + write dst (+ 8 B per run at run time)
            steps++;
            if (fuel_out(c)) break;
            const int after = apply_pair(sync, COH_LOCAL, abs[v]);
            if (after < 0) {
              T.term_status = COH_RUN_STUCK;
              T.term_call = c;
              T.term_effect = (uint8_t)sync;
              T.term_flags = (uint8_t)(0u | (1u << 1) | (abs[v] << 2));
              T.term_index = v;
              stop = true;
              break;
            }
            abs[v] = (uint32_t)after;
            steps++;
          }
        }
        if (m.kind == COH_W || m.kind == COH_RW) {
          if (fuel_out(c)) break;
          abs[v] = (uint32_t)apply_pair(COH_WRITE, m.site, abs[v]);  // w v^ never fails
          steps++;
        }
      }
      if (stop) break;
      for (uint32_t k = 0; k < call.n_body && !stop; ++k) {
        const coh_elem_op& op = call.body[k];
        const uint32_t vlo = P.view_lo[call.view], len = P.view_hi[call.view] - vlo + 1;
        if (op.lo > op.hi || op.hi >= len || (op.effect != COH_READ && op.effect != COH_WRITE)) {
          *err = "body op of call " + std::to_string(c) + " is malformed";
          return COH_E_CONSTRUCTION;
        }
        uint64_t m = (uint64_t)(op.hi - op.lo + 1);
        if (fuel_out(c)) break;
        const uint64_t avail = fuel - steps;
        const bool trunc = avail < m;
        if (trunc) m = avail;
        const uint32_t lo = vlo + op.lo, hi = lo + (uint32_t)m - 1;
        // the plane a read needs / a write sets: local site -> L, remote -> R
        emit(op.effect == COH_READ ? EOP_READ : EOP_WRITE, op.site ? 1 : 0, c, lo, hi);
        alg += (op.effect == COH_READ ? 1 : 2) * ((m + 7) / 8);
        steps += m;
        if (trunc) {
          T.term_status = COH_RUN_FUEL_EXHAUSTED;
          T.term_call = c;
          stop = true;
        }
      }
      if (stop) break;
      // abstraction_correct after the completed block: pack every view's abstract pair
      uint32_t packed = 0;
      for (uint32_t v = 0; v < P.n_views; ++v) {
        packed |= abs[v] << (2 * v);
        const uint64_t mv = (uint64_t)(P.view_hi[v] - P.view_lo[v] + 1);
        alg += ((abs[v] == 1u || abs[v] == 2u) ? 1 : 2) * ((mv + 7) / 8);
      }
      emit(EOP_CHECK, (uint8_t)P.n_views, c, packed, 0);
      T.calls_checked++;
    }
    T.n_ops = (uint32_t)ops.size();
    T.steps_total = steps;
    T.abs_final = 0;
    for (uint32_t v = 0; v < P.n_views; ++v) T.abs_final |= abs[v] << (2 * v);
  }
  // stages: per buffer, runs of read-only ops closed by at most one writing op
  std::vector<std::vector<std::vector<ElemOp>>> st_ops(n);  // [b][stage] -> ops in order
  for (uint32_t b = 0; b < n; ++b) {
    std::vector<ElemOp> cur;
    plan->tl[b].op_pos.clear();
    for (const ElemOp& op : per[b]) {
      const bool writes = op.type == EOP_SYNC || op.type == EOP_WRITE;
      cur.push_back(op);
      plan->tl[b].op_pos.push_back((uint32_t)st_ops[b].size() * kSlots + (uint32_t)cur.size() - 1);
      if (writes || cur.size() == kSlots) {
        st_ops[b].push_back(cur);
        cur.clear();
      }
    }
    if (!cur.empty()) st_ops[b].push_back(cur);
  }
  uint32_t n_stages = 0;
  for (auto& v : st_ops) n_stages = std::max(n_stages, (uint32_t)v.size());
  plan->n_stages = n_stages;
  plan->max_words = ((max_cells + 31) / 32 + 3) & ~3u;
  plan->ops.assign((size_t)n_stages * n * kSlots, ElemOp{EOP_NONE, 0, 0, 0, 0, 0});
  plan->tiles.clear();
  plan->stage_tile0.assign(n_stages + 1, 0);
  plan->stage_has_sync.assign(n_stages, 0);
  plan->sync_tiles.clear();
  plan->stage_sync0.assign(n_stages + 1, 0);
  for (uint32_t s = 0; s < n_stages; ++s) {
    plan->stage_tile0[s] = (uint32_t)plan->tiles.size();
    plan->stage_sync0[s] = (uint32_t)plan->sync_tiles.size();
    for (uint32_t b = 0; b < n; ++b) {
      if (s >= st_ops[b].size()) continue;
      for (uint32_t slot = 0; slot < st_ops[b][s].size(); ++slot) {
        ElemOp op = st_ops[b][s][slot];
        op.tile0 = (uint32_t)plan->tiles.size() - plan->stage_tile0[s];  // stage-local (pass1 list)
        auto make_tiles = [&](uint32_t lo, uint32_t hi, uint32_t view, uint32_t apair, std::vector<ElemTile>& dst,
                              bool pass1) {
          const uint32_t w_lo = lo / 32, w_hi = hi / 32;
          for (uint32_t t0 = (w_lo / kElemTileWords) * kElemTileWords; t0 <= w_hi; t0 += kElemTileWords) {
            ElemTile t{};
            t.b = b;
            t.tstart = t0;
            t.lo = lo;
            t.hi = hi;
            t.type = op.type;
            t.plane = op.plane;
            t.view = (uint8_t)view;
            t.apair = (uint8_t)apair;
            t.tloc = pass1 ? (uint32_t)plan->tiles.size() - plan->stage_tile0[s] : 0u;
            t.slot = slot;
            dst.push_back(t);
          }
        };
        if (op.type == EOP_CHECK) {
          for (uint32_t v = 0; v < progs[b].n_views; ++v)
            make_tiles(progs[b].view_lo[v], progs[b].view_hi[v], v, (op.lo >> (2 * v)) & 3u, plan->tiles, true);
        } else if (op.type == EOP_WRITE) {
          make_tiles(op.lo, op.hi, 0, 0, plan->sync_tiles, false);  // apply pass only
        } else {
          const size_t first = plan->tiles.size();
          make_tiles(op.lo, op.hi, 0, 0, plan->tiles, true);
          if (op.type == EOP_SYNC) {
            plan->stage_has_sync[s] = 1;
            for (size_t k = first; k < plan->tiles.size(); ++k) plan->sync_tiles.push_back(plan->tiles[k]);
          }
        }
        plan->ops[((size_t)s * n + b) * kSlots + slot] = op;
      }
    }
  }
  plan->stage_tile0[n_stages] = (uint32_t)plan->tiles.size();
  plan->stage_sync0[n_stages] = (uint32_t)plan->sync_tiles.size();
  // initial_store writes both planes of every cell (L = 1, R = 0)
  for (uint32_t b = 0; b < n; ++b) alg += 2 * (((uint64_t)progs[b].n_cells + 7) / 8);
  plan->alg_bytes = alg;
  return COH_OK;
}

}  // namespace cohb

// ---- generator ------------------------------------------------------------------------
// Views follow the acceptance pattern lo ~ U[0,n), hi = lo + U[0, n-lo)
// (tests/acceptance.cpp:235-236).  Calls: view ~ U[0,V), kind ~ U{R,W,RW}, site ~ U{L,R};
// adversarial with probability adv_per1024/1024, else the canonical body:
//   R: r x[0..len-1]@S   W: w x[0..len-1]@S   RW: r x[0..len-1]@S; w x[a..b]@S
// adversarial variants: 1 empty, 2 r x[a..b]@O, 3 w x[a..b]@S (partial write),
//   4 w x[a..b]@O, 5 r x[0..len-1]@S; w x[a..b]@O
extern "C" int coh_elem_gen(uint64_t seed, uint64_t prog_id, uint32_t n_cells, uint32_t n_views,
                            uint32_t n_calls, uint32_t adv_per1024, uint32_t* view_lo, uint32_t* view_hi,
                            coh_elem_call* calls) {
  if (n_cells == 0 || n_views == 0 || n_views > COH_MAX_VIEWS) return COH_E_ARG;
  uint64_t k = 0;
  auto h = [&]() { return coh_splitmix64(seed ^ (prog_id << 24) ^ (k++)); };
  for (uint32_t v = 0; v < n_views; ++v) {
    const uint32_t lo = (uint32_t)(h() % n_cells);
    view_lo[v] = lo;
    view_hi[v] = lo + (uint32_t)(h() % (uint64_t)(n_cells - lo));
  }
  for (uint32_t c = 0; c < n_calls; ++c) {
    const uint64_t x = h();
    coh_elem_call& cl = calls[c];
    std::memset(&cl, 0, sizeof cl);
    cl.view = (uint32_t)(x % n_views);
    cl.kind = (uint8_t)((x >> 8) % 3);
    cl.site = (uint8_t)((x >> 10) & 1);
    const bool adv = ((x >> 16) & 1023u) < adv_per1024;
    const uint32_t variant = adv ? 1u + (uint32_t)((x >> 26) % 5) : 0u;
    const uint32_t len = view_hi[cl.view] - view_lo[cl.view] + 1;
    const uint32_t a = (uint32_t)(h() % len);
    const uint32_t b = a + (uint32_t)(h() % (uint64_t)(len - a));
    const uint8_t S = cl.site, O = (uint8_t)(cl.site ^ 1);
    auto op = [&](uint8_t eff, uint8_t site, uint32_t lo, uint32_t hi) {
      coh_elem_op& o = cl.body[cl.n_body++];
      o.effect = eff;
      o.site = site;
      o.lo = lo;
      o.hi = hi;
    };
    switch (variant) {
      case 0:
        if (cl.kind == COH_R) op(COH_READ, S, 0, len - 1);
        else if (cl.kind == COH_W) op(COH_WRITE, S, 0, len - 1);
        else { op(COH_READ, S, 0, len - 1); op(COH_WRITE, S, a, b); }
        break;
      case 1: break;
      case 2: op(COH_READ, O, a, b); break;
      case 3: op(COH_WRITE, S, a, b); break;
      case 4: op(COH_WRITE, O, a, b); break;
      default: op(COH_READ, S, 0, len - 1); op(COH_WRITE, O, a, b); break;
    }
  }
  return COH_OK;
}

// ---- C ABI: compile, execute stage by stage, finalise ----------------------------------
namespace {

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
  template <typename T>
  T* as() { return static_cast<T*>(p); }
};

}  // namespace

#define COH_E(x)                                            \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) {                                \
      *err = std::string(#x) + ": " + cudaGetErrorString(e_); \
      return COH_E_CUDA;                                    \
    }                                                       \
  } while (0)

namespace {
using namespace cohb;

// One group of programs (buffers) with its own plan, device state and stage chain.  The
// buffers of different groups are independent, so their stage chains run concurrently on
// separate streams (branches of one CUDA graph): one chain's per-stage launch, dependency
// and drain latency is filled by the other's streaming.
struct ElemGroup {
  const coh_elem_program* progs = nullptr;
  uint32_t n = 0, b0 = 0;  // programs [b0, b0 + n) of the batch
  ElemPlan plan;
  uint32_t W = 0, bwords = 1;
  uint64_t runs_cap = 0, launches = 0;
  DevBuf planes, ops, tiles, stiles, st, sc, tcnt, tbase, stage_buf, vlo, vhi, ncell, bnd, rlo, rhi;

  int compile(std::string* err) {
    int rc = elem_compile(progs, n, &plan, err);
    if (rc) return rc;
    W = ((plan.max_words + kElemTileWords - 1) / kElemTileWords) * kElemTileWords;
    for (uint32_t b = 0; b < n; ++b) bwords = std::max(bwords, (progs[b].n_calls + 31) / 32);
    return COH_OK;
  }

  int prepare(cudaStream_t s, std::string* err) {  // allocations and uploads (outside the graph)
    uint32_t max_tiles = 1;
    for (uint32_t g = 0; g < plan.n_stages; ++g)
      max_tiles = std::max(max_tiles, plan.stage_tile0[g + 1] - plan.stage_tile0[g]);
    auto alloc = [&](DevBuf& d, size_t bytes) { return cudaMalloc(&d.p, std::max<size_t>(bytes, 16)); };
    COH_E(alloc(planes, (size_t)n * 2 * W * 4));
    COH_E(alloc(ops, plan.ops.size() * sizeof(ElemOp)));
    COH_E(alloc(tiles, plan.tiles.size() * sizeof(ElemTile)));
    COH_E(alloc(stiles, plan.sync_tiles.size() * sizeof(ElemTile)));
    COH_E(alloc(st, (size_t)n * sizeof(ElemState)));
    COH_E(alloc(sc, (size_t)n * kSlots * sizeof(ElemScratch)));
    COH_E(alloc(tcnt, (size_t)max_tiles * 4 * 4));
    COH_E(alloc(tbase, (size_t)max_tiles * 2 * 8));
    if (runs_cap) COH_E(alloc(stage_buf, (size_t)max_tiles * 2 * kStageRuns * 4));
    COH_E(alloc(vlo, (size_t)n * COH_MAX_VIEWS * 4));
    COH_E(alloc(vhi, (size_t)n * COH_MAX_VIEWS * 4));
    COH_E(alloc(ncell, (size_t)n * 16));
    COH_E(alloc(bnd, (size_t)n * bwords * 4));
    if (runs_cap) {
      COH_E(alloc(rlo, (size_t)n * runs_cap * 4));
      COH_E(alloc(rhi, (size_t)n * runs_cap * 4));
    }
    std::vector<uint32_t> h_vlo((size_t)n * COH_MAX_VIEWS, 0), h_vhi((size_t)n * COH_MAX_VIEWS, 0), h_nc(4 * (size_t)n);
    for (uint32_t b = 0; b < n; ++b) {
      h_nc[4 * b] = progs[b].n_cells;
      h_nc[4 * b + 1] = progs[b].frag_log2;
      h_nc[4 * b + 2] = (uint32_t)progs[b].frag_seed;
      h_nc[4 * b + 3] = (uint32_t)(progs[b].frag_seed >> 32);
      for (uint32_t v = 0; v < progs[b].n_views; ++v) {
        h_vlo[(size_t)b * COH_MAX_VIEWS + v] = progs[b].view_lo[v];
        h_vhi[(size_t)b * COH_MAX_VIEWS + v] = progs[b].view_hi[v];
      }
    }
    std::vector<ElemScratch> h_sc((size_t)n * kSlots);
    for (auto& x : h_sc) {
      x.first_zero = kNoCell;
      for (auto& f : x.view_flags) f = 0;
    }
    COH_E(cudaMemcpyAsync(ops.p, plan.ops.data(), plan.ops.size() * sizeof(ElemOp), cudaMemcpyHostToDevice, s));
    if (!plan.tiles.empty())
      COH_E(cudaMemcpyAsync(tiles.p, plan.tiles.data(), plan.tiles.size() * sizeof(ElemTile), cudaMemcpyHostToDevice,
                            s));
    if (!plan.sync_tiles.empty())
      COH_E(cudaMemcpyAsync(stiles.p, plan.sync_tiles.data(), plan.sync_tiles.size() * sizeof(ElemTile),
                            cudaMemcpyHostToDevice, s));
    COH_E(cudaMemcpyAsync(vlo.p, h_vlo.data(), h_vlo.size() * 4, cudaMemcpyHostToDevice, s));
    COH_E(cudaMemcpyAsync(vhi.p, h_vhi.data(), h_vhi.size() * 4, cudaMemcpyHostToDevice, s));
    COH_E(cudaMemcpyAsync(ncell.p, h_nc.data(), h_nc.size() * 4, cudaMemcpyHostToDevice, s));
    COH_E(cudaMemcpyAsync(sc.p, h_sc.data(), h_sc.size() * sizeof(ElemScratch), cudaMemcpyHostToDevice, s));
    COH_E(cudaMemsetAsync(st.p, 0, (size_t)n * sizeof(ElemState), s));
    COH_E(cudaMemsetAsync(bnd.p, 0, (size_t)n * bwords * 4, s));
    return cudaStreamSynchronize(s) == cudaSuccess ? COH_OK : COH_E_CUDA;  // host vectors die here
  }

  int enqueue(cudaStream_t s, std::string* err) {  // init + every stage (captured into the graph)
    launches = 1;
    int r = launch_elem_init(planes.as<uint32_t>(), W, ncell.as<uint32_t>(), n, s, err);
    for (uint32_t stg = 0; stg < plan.n_stages && r == COH_OK; ++stg) {
      ElemDev d;
      d.planes = planes.as<uint32_t>();
      d.W = W;
      d.ops = ops.as<ElemOp>() + (size_t)stg * n * kSlots;
      d.tiles = tiles.as<ElemTile>() + plan.stage_tile0[stg];
      d.sync_desc = stiles.as<ElemTile>() + plan.stage_sync0[stg];
      d.st = st.as<ElemState>();
      d.sc = sc.as<ElemScratch>();
      d.tcnt = tcnt.as<uint32_t>();
      d.tbase = tbase.as<unsigned long long>();
      d.stage_runs = stage_buf.as<uint32_t>();
      d.view_lo = vlo.as<uint32_t>();
      d.view_hi = vhi.as<uint32_t>();
      d.boundary = bnd.as<uint32_t>();
      d.bwords = bwords;
      d.runs_lo = rlo.as<uint32_t>();
      d.runs_hi = rhi.as<uint32_t>();
      d.runs_cap = runs_cap;
      d.n_progs = n;
      d.stage = stg;
      const uint32_t nt = plan.stage_tile0[stg + 1] - plan.stage_tile0[stg];
      const uint32_t ns = plan.stage_sync0[stg + 1] - plan.stage_sync0[stg];
      r = launch_elem_stage(d, nt, ns, s, err);
      launches += (nt ? 2 : 0) + (ns ? 1 : 0);
    }
    return r;
  }
};

}  // namespace

static int elem_eval_impl(coh_ctx* ctx, const coh_elem_program* progs, uint32_t n, coh_elem_result* results,
                          uint32_t* planes_out, uint32_t plane_words, uint8_t* view_abs_out, uint32_t* boundary_out,
                          uint32_t boundary_words, uint32_t* runs_out, uint64_t runs_cap, coh_elem_stats* stats,
                          std::string* err) {
  std::string& err_s = *err;
  // concurrent stage chains (one per group of >= 32 buffers, up to kChains)
  constexpr uint32_t kChains = 6;
  const char* gv = std::getenv("COH_ELEM_CHAINS");
  const uint32_t gmax = gv ? std::max(1, std::min((int)kChains, std::atoi(gv))) : kChains;
  const uint32_t G = std::max(1u, std::min(gmax, n / 32u));
  std::vector<ElemGroup> grp(G);
  for (uint32_t g = 0; g < G; ++g) {
    grp[g].b0 = (uint32_t)((uint64_t)n * g / G);
    grp[g].n = (uint32_t)((uint64_t)n * (g + 1) / G) - grp[g].b0;
    grp[g].progs = progs + grp[g].b0;
    grp[g].runs_cap = runs_cap;
    int rc = grp[g].compile(err);
    if (rc) {
      ctx->err = err_s;
      return rc;
    }
  }
  if (planes_out) {  // plane_words must hold every program's cells
    uint32_t need = 0;
    for (uint32_t b = 0; b < n; ++b) need = std::max(need, (progs[b].n_cells + 31) / 32);
    if (plane_words < need) {
      ctx->err = "plane_words too small";
      return COH_E_ARG;
    }
  }
  uint32_t bwords = 1;
  for (auto& g : grp) bwords = std::max(bwords, g.bwords);
  if (boundary_out && boundary_words < bwords) {
    ctx->err = "boundary_words too small";
    return COH_E_ARG;
  }
  if (!ctx->hs[0] && cudaStreamCreateWithFlags(&ctx->hs[0], cudaStreamNonBlocking) != cudaSuccess) {
    ctx->err = "stream create";
    return COH_E_CUDA;
  }
  struct Streams {  // the chains' extra streams (branches of the captured graph)
    cudaStream_t s[kChains] = {};
    ~Streams() {
      for (uint32_t k = 1; k < kChains; ++k)
        if (s[k]) cudaStreamDestroy(s[k]);
    }
  } st_;
  st_.s[0] = ctx->hs[0];
  for (uint32_t k = 1; k < G; ++k) COH_E(cudaStreamCreateWithFlags(&st_.s[k], cudaStreamNonBlocking));
  cudaStream_t* strm = st_.s;
  cudaStream_t s = strm[0];
  for (auto& g : grp) {
    const int rc = g.prepare(s, err);
    if (rc) {
      ctx->err = err_s.empty() ? std::string("element upload failed") : err_s;
      return rc;
    }
  }
  cudaEvent_t e0, e1, fork, join[kChains];
  COH_E(cudaEventCreate(&e0));
  COH_E(cudaEventCreate(&e1));
  COH_E(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  for (uint32_t k = 0; k < kChains; ++k) COH_E(cudaEventCreateWithFlags(&join[k], cudaEventDisableTiming));
  // The stage sequences are static once compiled: capture them into one CUDA graph (the
  // groups g > 0 fork onto their own streams and join back) so launch gaps disappear.
  auto enqueue_all = [&]() -> int {
    COH_E(cudaEventRecord(fork, s));
    for (uint32_t g = 1; g < G; ++g) COH_E(cudaStreamWaitEvent(strm[g], fork, 0));
    for (uint32_t g = 0; g < G; ++g) {
      const int r = grp[g].enqueue(strm[g], err);
      if (r) return r;
    }
    for (uint32_t g = 1; g < G; ++g) {
      COH_E(cudaEventRecord(join[g], strm[g]));
      COH_E(cudaStreamWaitEvent(s, join[g], 0));
    }
    return COH_OK;
  };
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int rc = COH_OK;
  bool graphed = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (graphed) {
    rc = enqueue_all();
    graphed = cudaStreamEndCapture(s, &graph) == cudaSuccess && rc == COH_OK &&
              cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    cudaGetLastError();
  }
  COH_E(cudaEventRecord(e0, s));
  if (graphed) {
    COH_E(cudaGraphLaunch(exec, s));
  } else {
    rc = enqueue_all();  // capture unavailable: plain stream launches
  }
  COH_E(cudaEventRecord(e1, s));
  if (rc) {
    ctx->err = err_s;
    cudaDeviceSynchronize();
    return rc;
  }
  // downloads, per group
  std::vector<std::vector<ElemState>> h_st(G);
  std::vector<std::vector<uint32_t>> h_bnd(G), h_rlo(G), h_rhi(G);
  for (uint32_t gi = 0; gi < G; ++gi) {
    ElemGroup& g = grp[gi];
    h_st[gi].resize(g.n);
    COH_E(cudaMemcpyAsync(h_st[gi].data(), g.st.p, (size_t)g.n * sizeof(ElemState), cudaMemcpyDeviceToHost, s));
    if (boundary_out) {
      h_bnd[gi].resize((size_t)g.n * g.bwords);
      COH_E(cudaMemcpyAsync(h_bnd[gi].data(), g.bnd.p, h_bnd[gi].size() * 4, cudaMemcpyDeviceToHost, s));
    }
    if (planes_out)
      COH_E(cudaMemcpy2DAsync(planes_out + (size_t)g.b0 * 2 * plane_words, (size_t)plane_words * 4, g.planes.p,
                              (size_t)g.W * 4, (size_t)std::min(plane_words, g.W) * 4, (size_t)2 * g.n,
                              cudaMemcpyDeviceToHost, s));
    if (runs_out && runs_cap) {
      h_rlo[gi].resize((size_t)g.n * runs_cap);
      h_rhi[gi].resize((size_t)g.n * runs_cap);
      COH_E(cudaMemcpyAsync(h_rlo[gi].data(), g.rlo.p, h_rlo[gi].size() * 4, cudaMemcpyDeviceToHost, s));
      COH_E(cudaMemcpyAsync(h_rhi[gi].data(), g.rhi.p, h_rhi[gi].size() * 4, cudaMemcpyDeviceToHost, s));
    }
  }
  COH_E(cudaStreamSynchronize(s));
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(fork);
  for (uint32_t k = 0; k < kChains; ++k) cudaEventDestroy(join[k]);
  uint64_t launches = 0, alg = 0, n_tiles = 0;
  uint32_t stages = 0;
  for (uint32_t gi = 0; gi < G; ++gi) {
    ElemGroup& g = grp[gi];
    launches += g.launches;
    alg += g.plan.alg_bytes;
    n_tiles += g.plan.tiles.size();
    stages = std::max(stages, g.plan.n_stages);
    const uint32_t n_g = g.n;
    for (uint32_t bl = 0; bl < n_g; ++bl) {
      const uint32_t b = g.b0 + bl;  // batch index
      const ElemPlan::Timeline& T = g.plan.tl[bl];
      const ElemState& S = h_st[gi][bl];
      coh_elem_result& r = results[b];
      std::memset(&r, 0, sizeof r);
      r.calls_done = S.calls_done;
      r.violations = S.violations;
      r.transfers = S.transfers;
      r.transfer_cells = S.transfer_cells;
      r.n_runs = S.n_runs;
      alg += 8 * std::min<uint64_t>(S.n_runs, runs_cap);  // ranges actually written (8 B each)
      uint32_t abs_final = T.abs_final;
      uint32_t executed_ops = T.n_ops;
      if (S.dead) {
        const uint32_t stage = S.stuck_op / kSlots, slot = S.stuck_op % kSlots;
        const ElemOp& op = g.plan.ops[((size_t)stage * n_g + bl) * kSlots + slot];
        uint32_t k = 0;
        while (k < T.op_pos.size() && T.op_pos[k] != S.stuck_op) ++k;
        executed_ops = k;
        r.status = COH_RUN_STUCK;
        r.stuck_call = op.call;
        r.stuck_index = S.stuck_cell;
        const uint32_t site = op.type == EOP_READ ? op.plane : 0u;
        r.stuck_effect = (uint8_t)(op.type == EOP_READ ? COH_READ : (op.plane ? COH_PULL : COH_PUSH));
        r.stuck_flags = (uint8_t)(site | (S.stuck_pair << 2));
        r.steps = T.steps_before[k] + (op.type == EOP_READ ? (uint64_t)(S.stuck_cell - op.lo) : 0u);
        abs_final = T.abs_before[k];
      } else {
        r.status = T.term_status;
        r.steps = T.steps_total;
        if (T.term_status != COH_RUN_DONE) {
          r.stuck_call = T.term_call;
          r.stuck_effect = T.term_effect;
          r.stuck_flags = T.term_flags;
          r.stuck_index = T.term_index;
        }
      }
      // VectorPU-faithful transfer size: the whole view range of every executed sync
      for (uint32_t k = 0; k < executed_ops; ++k) {
        const uint32_t pos = T.op_pos[k];
        const ElemOp& op = g.plan.ops[((size_t)(pos / kSlots) * n_g + bl) * kSlots + pos % kSlots];
        if (op.type == EOP_SYNC) r.vpu_cells += (uint64_t)(op.hi - op.lo + 1);
      }
      if (view_abs_out)
        for (uint32_t v = 0; v < COH_MAX_VIEWS; ++v)
          view_abs_out[(size_t)b * COH_MAX_VIEWS + v] =
              v < progs[b].n_views ? (uint8_t)((abs_final >> (2 * v)) & 3u) : 0;
      if (boundary_out)
        for (uint32_t w = 0; w < boundary_words; ++w)
          boundary_out[(size_t)b * boundary_words + w] = w < g.bwords ? h_bnd[gi][(size_t)bl * g.bwords + w] : 0u;
      if (runs_out && runs_cap) {
        const uint64_t m = std::min<uint64_t>(S.n_runs, runs_cap);
        for (uint64_t k = 0; k < m; ++k) {
          runs_out[((size_t)b * runs_cap + k) * 2] = h_rlo[gi][(size_t)bl * runs_cap + k];
          runs_out[((size_t)b * runs_cap + k) * 2 + 1] = h_rhi[gi][(size_t)bl * runs_cap + k];
        }
      }
    }
  }
  ctx->launches += launches;
  if (stats) {
    stats->device_ms = ms;
    stats->alg_bytes = alg;
    stats->launches = launches;
    stats->tiles = n_tiles;
    stats->stages = stages;
    stats->pad = 0;
  }
  return COH_OK;
}
#undef COH_E

extern "C" int coh_elem_eval(coh_ctx* ctx, const coh_elem_program* progs, uint32_t n,
                             coh_elem_result* results, uint32_t* planes_out, uint32_t plane_words,
                             uint8_t* view_abs_out, uint32_t* boundary_out, uint32_t boundary_words,
                             uint32_t* runs_out, uint64_t runs_cap, coh_elem_stats* stats) {
  if (!ctx) return COH_E_ARG;
  if (n && (!progs || !results)) {
    ctx->err = "progs/results is NULL";
    return COH_E_ARG;
  }
  if (n == 0) return COH_OK;
  std::string err;
  const int rc = elem_eval_impl(ctx, progs, n, results, planes_out, plane_words, view_abs_out, boundary_out,
                                boundary_words, runs_out, runs_cap, stats, &err);
  if (rc && !err.empty()) ctx->err = err;
  return rc;
}
