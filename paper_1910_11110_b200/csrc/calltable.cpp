// Host call-table compiler: restates the reference's per-cell rules and the Fig. 3
// translation for one whole-array call, and tabulates every (call type, start state)
// outcome so the device evaluates a call with one table lookup.
//
//   per-cell rules   validity.hpp:73-120 (signature table + unification),
//                    semantics.hpp:109-130 (remote = swap, apply, swap)
//   translation      modes.hpp:31-59 (R x -> if valid(x^) {} else {pull x; pull x^};
//                    GR x -> if gvalid(x^) {} else {push x; push x^}; the syncs are
//                    Local-site, ast.hpp:144 default; W/GW -> w x^ at the mode site;
//                    RW = guard then w x^; guards then the body)
//   stepping         semantics.hpp:253-287 (Done before fuel, Stuck takes no step)
//   boundary check   modes.hpp:71-90 (leq / abstraction_correct)
#include <cstring>

#include "internal.hpp"

namespace cohb {
namespace {

// pair: bit0 local Valid, bit1 remote Valid
inline uint32_t swap_pair(uint32_t p) { return ((p & 1u) << 1) | ((p >> 1) & 1u); }

// effect_signature / apply_signature, local form (validity.hpp:79-120).
// Returns 0..3 or -1 for NoUnify.
int apply_local(uint32_t eff, uint32_t p) {
  switch (eff) {
    case COH_PUSH: return (p & 1u) ? 3 : -1;   // (V,X) -> (V,V)
    case COH_PULL: return (p & 2u) ? 3 : -1;   // (X,V) -> (V,V)
    case COH_READ: return (p & 1u) ? (int)p : -1;  // (V,X) -> (V,X)
    case COH_WRITE: return 1;                  // (X,Y) -> (V,I)
    case COH_NOOP: return (int)p;
  }
  return -1;
}

// apply_effect_at (semantics.hpp:109-130): remote effects unify against the swapped
// pair and store the swapped postcondition.
int apply_cell(uint32_t eff, uint32_t site, uint32_t p) {
  if (site == COH_LOCAL) return apply_local(eff, p);
  int r = apply_local(eff, swap_pair(p));
  return r < 0 ? -1 : (int)swap_pair((uint32_t)r);
}

// leq (modes.hpp:71-75): equal, or concrete (V,V) under a one-sided abstract flag.
bool leq(uint32_t abs_pair, uint32_t conc) {
  if (abs_pair == conc) return true;
  return conc == 3u && (abs_pair == 1u || abs_pair == 2u);
}
bool violating(uint32_t state) { return !leq(state >> 2, state & 3u); }

// Body variants.  S = the mode's site, O = the opposite site.
//   0 canonical well-declared body: R: r@S   W: w@S   RW: r@S; w@S
//   1 empty   2 r@O   3 w@O   4 r@S   5 w@S; r@O   6 push@S   7 pull@S; w@O
int body_ops(uint32_t kind, uint32_t site, uint32_t variant, uint8_t* out) {
  const uint32_t S = site, O = site ^ 1u;
  int n = 0;
  auto eff = [&](uint32_t e, uint32_t s) { out[n++] = op_effect(e, s, 0); };
  switch (variant) {
    case 0:
      if (kind == COH_R) eff(COH_READ, S);
      else if (kind == COH_W) eff(COH_WRITE, S);
      else { eff(COH_READ, S); eff(COH_WRITE, S); }
      break;
    case 1: break;
    case 2: eff(COH_READ, O); break;
    case 3: eff(COH_WRITE, O); break;
    case 4: eff(COH_READ, S); break;
    case 5: eff(COH_WRITE, S); eff(COH_READ, O); break;
    case 6: eff(COH_PUSH, S); break;
    case 7: eff(COH_PULL, S); eff(COH_WRITE, O); break;
  }
  return n;
}

// translate_mode + translate_block (modes.hpp:31-59) for one mode on one array.
int block_ops(uint32_t call_type, uint8_t ops[8]) {
  std::memset(ops, 0, 8);
  const uint32_t kind = call_type & 3u, site = (call_type >> 2) & 1u, variant = (call_type >> 3) & 7u;
  if (kind > COH_RW) {
    ops[0] = OP_DEFECT;
    return 1;
  }
  int n = 0;
  const uint32_t sync = site == COH_REMOTE ? COH_PUSH : COH_PULL;
  if (kind == COH_R || kind == COH_RW) {
    ops[n++] = site == COH_REMOTE ? OP_IF_GVALID : OP_IF_VALID;
    ops[n++] = op_effect(sync, COH_LOCAL, 0);  // push/pull x (concrete)
    ops[n++] = op_effect(sync, COH_LOCAL, 1);  // push/pull x^
  }
  if (kind == COH_W || kind == COH_RW) ops[n++] = op_effect(COH_WRITE, site, 1);  // w x^ @site
  n += body_ops(kind, site, variant, ops + n);
  return n;
}

}  // namespace

coh_call_outcome simulate_block(uint32_t call_type, uint32_t state, int fuel) {
  coh_call_outcome o;
  std::memset(&o, 0, sizeof o);
  uint8_t ops[8];
  const int n = block_ops(call_type, ops);
  o.viol_before = violating(state);
  uint32_t s = state & 15u;
  int k = 0;
  o.status = COH_RUN_DONE;
  while (true) {
    if (k >= n) break;                  // program is Noop: Done (checked before fuel)
    const uint8_t op = ops[k];
    if (op == OP_DEFECT) {              // malformed record: a construction defect
      o.status = COH_RUN_DEFECT;
      break;
    }
    if ((int)o.steps >= fuel) {         // semantics.hpp:262-265
      o.status = COH_RUN_FUEL_EXHAUSTED;
      break;
    }
    const uint32_t kindop = op & 3u;
    if (kindop == OP_IF_VALID || kindop == OP_IF_GVALID) {
      // eval_condition (semantics.hpp:43-54) on x^: valid -> empty then-branch;
      // else the two sync statements follow.
      const bool taken = kindop == OP_IF_VALID ? ((s >> 2) & 1u) : ((s >> 3) & 1u);
      o.steps++;
      k += taken ? 3 : 1;
      continue;
    }
    const uint32_t eff = (op >> 2) & 7u, site = (op >> 5) & 1u, abs_t = (op >> 6) & 1u;
    const uint32_t shift = abs_t ? 2u : 0u;
    const uint32_t before = (s >> shift) & 3u;
    const int after = apply_cell(eff, site, before);
    if (after < 0) {                    // Stuck: no step consumed, store untouched
      o.status = COH_RUN_STUCK;
      o.stuck_effect = (uint8_t)eff;
      o.stuck_flags = (uint8_t)(site | (abs_t << 1) | (before << 2));
      break;
    }
    s = (s & ~(3u << shift)) | ((uint32_t)after << shift);
    o.steps++;
    if (!abs_t && (eff == COH_PUSH || eff == COH_PULL)) o.transfers++;
    k++;
  }
  o.state_after = (uint8_t)s;
  o.viol_after = violating(s);
  return o;
}

void build_call_table(CallTable* t) {
  for (uint32_t type = 0; type < (uint32_t)kCallTypes; ++type) {
    uint8_t ops[8];
    block_ops(type, ops);
    uint64_t prog = 0;
    for (int k = 0; k < 8; ++k) prog |= (uint64_t)ops[k] << (8 * k);
    t->prog[type] = prog;
    t->lut[kStates * 64u + type] = kPoisonSlot | (kSlowAddend << 16);  // poison row
    for (uint32_t s = 0; s < (uint32_t)kStates; ++s) {
      const coh_call_outcome o = simulate_block(type, s, 1 << 30);
      uint32_t lo, hi;
      if (o.status != COH_RUN_DONE) {
        lo = slot_word(s);
        hi = kSlowAddend;
      } else {
        lo = slot_word(o.state_after);
        hi = ((uint32_t)o.steps + ((uint32_t)o.transfers << kAccXferShift) +
              (uint32_t)(((int)o.viol_after - (int)o.viol_before + 1) * (1 << kAccViolShift))) & 0xFFFFu;
      }
      t->lut[lut_word(type, s)] = lo | (hi << 16);
      for (uint32_t rem = 0; rem < 8; ++rem) {
        const coh_call_outcome q = simulate_block(type, s, rem == 7 ? (1 << 30) : (int)rem);
        t->slow[slow_index(type, s, rem)] =
            (uint32_t)q.status | ((uint32_t)q.steps << 2) | ((uint32_t)q.transfers << 5) |
            ((uint32_t)q.state_after << 7) | ((uint32_t)q.stuck_effect << 11) | ((uint32_t)q.stuck_flags << 14);
      }
    }
  }
}

}  // namespace cohb

extern "C" int coh_calltable_describe(uint32_t call_type, uint32_t state, coh_call_outcome* out) {
  if (call_type >= (uint32_t)cohb::kCallTypes || state >= 16u || !out) return COH_E_ARG;
  *out = cohb::simulate_block(call_type, state, 1 << 30);
  return COH_OK;
}

extern "C" int coh_calltable_program(uint32_t call_type, uint8_t ops[8]) {
  if (call_type >= (uint32_t)cohb::kCallTypes || !ops) return -COH_E_ARG;
  return cohb::block_ops(call_type, ops);
}
