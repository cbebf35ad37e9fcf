/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.  The product path
 * (paper_1910_11110_b200/) never links or calls it.
 *
 * Plain-C restatement of the reference evaluator (/root/reference/proj/include/cohere)
 * for the whole-array trace path, written statement by statement from the reference:
 *
 *   orc_apply_cell      validity.hpp:73-120 (signature table, unification) and the
 *                       swap rule of apply_effect_at, semantics.hpp:109-130
 *   orc_leq             modes.hpp:71-75
 *   translate_call      translate_mode / translate_block, modes.hpp:31-59 (guards use
 *                       Local-site syncs, ast.hpp:144 Stmt::effect default)
 *   run_block           run, semantics.hpp:253-287 (Done before fuel, Stuck takes no
 *                       step, If = one step, eval_condition semantics.hpp:43-54)
 *   orc_eval_traces     run_annotated, modes.hpp:105-125 + abstraction_correct
 *                       modes.hpp:79-90 (full O(arrays) scan after every block)
 *
 * Pinned against the reference: tests/golden/ fixtures were produced by oracle/_ref (the
 * reference compiled from its own headers) by tests/golden/make_golden.py, and
 * tests/test_oracle.py checks this file against every one of them.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "cohere_b200.h"

/* pair bits: bit0 local Valid, bit1 remote Valid.  Returns -1 on NoUnify. */
int orc_apply_cell(int eff, int site, int pair) {
  int p = pair;
  if (site == COH_REMOTE) p = ((p & 1) << 1) | ((p >> 1) & 1); /* swapped(before) */
  int r;
  switch (eff) {
    case COH_PUSH: r = (p & 1) ? 3 : -1; break;  /* push : (V,X) -> (V,V) */
    case COH_PULL: r = (p & 2) ? 3 : -1; break;  /* pull : (X,V) -> (V,V) */
    case COH_READ: r = (p & 1) ? p : -1; break;  /* r    : (V,X) -> (V,X) */
    case COH_WRITE: r = 1; break;                /* w    : (X,Y) -> (V,I) */
    case COH_NOOP: r = p; break;                 /* noop : (X,Y) -> (X,Y) */
    default: return -1;
  }
  if (r < 0) return -1;
  if (site == COH_REMOTE) r = ((r & 1) << 1) | ((r >> 1) & 1); /* swapped(post) */
  return r;
}

/* leq(abstract, concrete), modes.hpp:71-75 */
int orc_leq(int abs_pair, int conc) {
  if (abs_pair == conc) return 1;
  return conc == 3 && (abs_pair == 1 || abs_pair == 2);
}

/* statement of a translated block: kind 0 = effect, 1 = if (valid(x^)) {} else {next 2},
 * 2 = if (gvalid(x^)) {} else {next 2} */
typedef struct {
  int kind, eff, site, abstract_target;
} orc_stmt;

static int push_eff(orc_stmt* s, int n, int eff, int site, int abs_t) {
  s[n].kind = 0;
  s[n].eff = eff;
  s[n].site = site;
  s[n].abstract_target = abs_t;
  return n + 1;
}

/* Fig. 3 translation of one mode on one array + the body variant. */
static int translate_call(uint16_t rec, orc_stmt* s) {
  const int kind = (int)COH_REC_KIND(rec), site = (int)COH_REC_SITE(rec);
  const int var = (int)COH_REC_VARIANT(rec), S = site, O = site ^ 1;
  const int sync = site == COH_REMOTE ? COH_PUSH : COH_PULL;
  int n = 0;
  if (kind == 3) return -1;
  if (kind == COH_R || kind == COH_RW) { /* ensure_valid, modes.hpp:36-41 */
    s[n].kind = site == COH_REMOTE ? 2 : 1;
    n++;
    n = push_eff(s, n, sync, COH_LOCAL, 0);
    n = push_eff(s, n, sync, COH_LOCAL, 1);
  }
  if (kind == COH_W || kind == COH_RW) n = push_eff(s, n, COH_WRITE, site, 1); /* mark_written */
  switch (var) {
    case 0:
      if (kind == COH_R) n = push_eff(s, n, COH_READ, S, 0);
      else if (kind == COH_W) n = push_eff(s, n, COH_WRITE, S, 0);
      else { n = push_eff(s, n, COH_READ, S, 0); n = push_eff(s, n, COH_WRITE, S, 0); }
      break;
    case 1: break;
    case 2: n = push_eff(s, n, COH_READ, O, 0); break;
    case 3: n = push_eff(s, n, COH_WRITE, O, 0); break;
    case 4: n = push_eff(s, n, COH_READ, S, 0); break;
    case 5: n = push_eff(s, n, COH_WRITE, S, 0); n = push_eff(s, n, COH_READ, O, 0); break;
    case 6: n = push_eff(s, n, COH_PUSH, S, 0); break;
    case 7: n = push_eff(s, n, COH_PULL, S, 0); n = push_eff(s, n, COH_WRITE, O, 0); break;
  }
  return n;
}

typedef struct {
  int status, steps, transfers, stuck_eff, stuck_flags;
} orc_block_out;

/* run() over one translated block on one array's (concrete, abstract) pairs. */
static void run_block(const orc_stmt* s, int n, int* conc, int* abst, int fuel, orc_block_out* o) {
  int k = 0;
  memset(o, 0, sizeof *o);
  if (n < 0) { o->status = COH_RUN_DEFECT; return; }
  for (;;) {
    if (k >= n) { o->status = COH_RUN_DONE; return; }
    if (o->steps >= fuel) { o->status = COH_RUN_FUEL_EXHAUSTED; return; }
    if (s[k].kind != 0) {
      const int flag = s[k].kind == 1 ? (*abst & 1) : ((*abst >> 1) & 1);
      o->steps++;
      k += flag ? 3 : 1;
      continue;
    }
    int* cell = s[k].abstract_target ? abst : conc;
    const int after = orc_apply_cell(s[k].eff, s[k].site, *cell);
    if (after < 0) {
      o->status = COH_RUN_STUCK;
      o->stuck_eff = s[k].eff;
      o->stuck_flags = s[k].site | (s[k].abstract_target << 1) | (*cell << 2);
      return;
    }
    *cell = after;
    o->steps++;
    if (!s[k].abstract_target && (s[k].eff == COH_PUSH || s[k].eff == COH_PULL)) o->transfers++;
    k++;
  }
}

/* One block from a state nibble (cl, cr, al, ar): the call-table KAT. */
int orc_call_outcome(uint32_t call_type, uint32_t state, coh_call_outcome* out) {
  orc_stmt s[8];
  const int n = translate_call((uint16_t)(call_type << 2), s); /* COH_REC_TYPE */
  int conc = (int)(state & 3u), abst = (int)(state >> 2);
  orc_block_out o;
  memset(out, 0, sizeof *out);
  out->viol_before = !orc_leq(abst, conc);
  run_block(s, n, &conc, &abst, 1 << 30, &o);
  out->status = (uint8_t)o.status;
  out->steps = (uint8_t)o.steps;
  out->transfers = (uint8_t)o.transfers;
  out->state_after = (uint8_t)(conc | (abst << 2));
  out->viol_after = !orc_leq(abst, conc);
  out->stuck_effect = (uint8_t)o.stuck_eff;
  out->stuck_flags = (uint8_t)o.stuck_flags;
  return 0;
}

/* One record's statements split as translate_block interleaves them for a multi-mode
 * block: the mode's guard (ensure_valid + mark_written, modes.hpp:36-48) and its body. */
static int split_call(uint16_t rec, orc_stmt* guard, int* n_guard, orc_stmt* body) {
  orc_stmt s[8];
  const int n = translate_call(rec, s);
  if (n < 0) return -1;
  const int kind = (int)COH_REC_KIND(rec);
  const int g = kind == COH_R ? 3 : kind == COH_W ? 1 : 4;
  memcpy(guard, s, sizeof(orc_stmt) * (size_t)g);
  memcpy(body, s + g, sizeof(orc_stmt) * (size_t)(n - g));
  *n_guard = g;
  return n - g;
}

/* run() over a block's statement list, each statement on its own array (the if-guards
 * skip the two syncs that follow them when the flag is valid). */
typedef struct {
  orc_stmt s;
  int a;
} orc_astmt;

static void run_multi(const orc_astmt* s, int n, int* conc, int* abst, int fuel, orc_block_out* o, int* stuck_a,
                      const uint64_t* array_bytes, uint64_t* tbytes) {
  int k = 0;
  memset(o, 0, sizeof *o);
  for (;;) {
    if (k >= n) { o->status = COH_RUN_DONE; return; }
    if (o->steps >= fuel) { o->status = COH_RUN_FUEL_EXHAUSTED; return; }
    const int a = s[k].a;
    if (s[k].s.kind != 0) {
      const int flag = s[k].s.kind == 1 ? (abst[a] & 1) : ((abst[a] >> 1) & 1);
      o->steps++;
      k += flag ? 3 : 1;
      continue;
    }
    int* cell = s[k].s.abstract_target ? &abst[a] : &conc[a];
    const int after = orc_apply_cell(s[k].s.eff, s[k].s.site, *cell);
    if (after < 0) {
      o->status = COH_RUN_STUCK;
      o->stuck_eff = s[k].s.eff;
      o->stuck_flags = s[k].s.site | (s[k].s.abstract_target << 1) | (*cell << 2);
      *stuck_a = a;
      return;
    }
    *cell = after;
    o->steps++;
    if (!s[k].s.abstract_target && (s[k].s.eff == COH_PUSH || s[k].s.eff == COH_PULL)) {
      o->transfers++;
      *tbytes += array_bytes ? array_bytes[a] : 1u;
    }
    k++;
  }
}

/* flags & COH_BATCH_BLOCKS: a record with COH_REC_CONT continues the previous record's
 * block (a DeclBlock with several modes, program.hpp:212-235): its arrays must be
 * distinct and declared (else a construction defect at that block), and it runs as
 * translate_block lays it out (modes.hpp:53-59): all guards in record order, then all
 * bodies in record order.  Without the flag every record is its own block. */
int orc_eval_traces_ex(const uint16_t* records, uint64_t n_total, uint64_t t_begin, uint64_t t_end,
                       uint32_t n_calls, uint32_t n_arrays, int32_t fuel, const uint64_t* array_bytes,
                       uint32_t flags, coh_trace_result* out, uint32_t* boundary) {
  if (n_arrays < 1 || n_arrays > COH_MAX_ARRAYS || t_end < t_begin) return -1;
  const uint64_t m = t_end - t_begin;
  const uint32_t n_words = (n_calls + 31) / 32;
  orc_astmt* prog = (orc_astmt*)malloc(sizeof(orc_astmt) * 8u * (n_calls ? n_calls : 1u));
  if (!prog) return -1;
  for (uint64_t j = 0; j < m; ++j) {
    const uint64_t t = t_begin + j;
    int conc[COH_MAX_ARRAYS], abst[COH_MAX_ARRAYS];
    coh_trace_result* r = &out[j];
    memset(r, 0, sizeof *r);
    for (uint32_t a = 0; a < n_arrays; ++a) conc[a] = abst[a] = 1; /* initial_store: (V,I) */
    if (boundary)
      for (uint32_t w = 0; w < n_words; ++w) boundary[(uint64_t)w * m + j] = 0;
    int steps = 0, status = COH_RUN_DONE;
    uint32_t blk = 0;
#define ORC_REC(i) records[((uint64_t)((i) / 8) * n_total + t) * 8 + (i) % 8]
    for (uint32_t b0 = 0; b0 < n_calls; ++blk) {
      uint32_t b1 = b0 + 1;
      if (flags & COH_BATCH_BLOCKS)
        while (b1 < n_calls && (ORC_REC(b1) & COH_REC_CONT)) ++b1;
      /* DeclBlock construction: every mode declared, well formed, on a distinct array */
      uint64_t seen = 0;
      int defect = -1;
      for (uint32_t i = b0; i < b1 && defect < 0; ++i) {
        const uint16_t rec = ORC_REC(i);
        const uint32_t a = COH_REC_ARRAY(rec);
        if (a >= n_arrays || COH_REC_KIND(rec) == 3 || ((seen >> a) & 1u)) defect = (int)a;
        seen |= 1ull << a;
      }
      if (defect >= 0) {
        status = COH_RUN_DEFECT;
        r->stuck_call = blk;
        r->stuck_array = (uint8_t)defect;
        break;
      }
      int n = 0;
      orc_stmt g[8], bd[8];
      for (uint32_t i = b0; i < b1; ++i) { /* guards */
        int ng = 0;
        split_call(ORC_REC(i), g, &ng, bd);
        for (int k = 0; k < ng; ++k) prog[n].s = g[k], prog[n++].a = (int)COH_REC_ARRAY(ORC_REC(i));
      }
      for (uint32_t i = b0; i < b1; ++i) { /* bodies */
        int ng = 0;
        const int nb = split_call(ORC_REC(i), g, &ng, bd);
        for (int k = 0; k < nb; ++k) prog[n].s = bd[k], prog[n++].a = (int)COH_REC_ARRAY(ORC_REC(i));
      }
      orc_block_out o;
      int stuck_a = (int)COH_REC_ARRAY(ORC_REC(b0)); /* fuel exhaustion: the block's first array */
      run_multi(prog, n, conc, abst, fuel - steps, &o, &stuck_a, array_bytes, &r->transfer_bytes);
      r->transfers += (uint32_t)o.transfers;
      steps += o.steps;
      if (o.status != COH_RUN_DONE) {
        status = o.status;
        r->stuck_call = blk;
        r->stuck_array = (uint8_t)stuck_a;
        r->stuck_effect = (uint8_t)o.stuck_eff;
        r->stuck_flags = (uint8_t)o.stuck_flags;
        break;
      }
      int ok = 1;
      for (uint32_t b = 0; b < n_arrays; ++b)
        if (!orc_leq(abst[b], conc[b])) { ok = 0; break; }
      r->calls_done++;
      if (!ok) r->violations++;
      if (ok && boundary) boundary[(uint64_t)(blk / 32) * m + j] |= 1u << (blk % 32);
      b0 = b1;
    }
#undef ORC_REC
    r->status = (uint8_t)status;
    r->steps = (uint32_t)steps;
    for (uint32_t a = 0; a < n_arrays; ++a) {
      r->state[a / 8] |= (uint32_t)(conc[a] | (abst[a] << 2)) << (4 * (a % 8));
      if (conc[a] == 0 || abst[a] == 0) r->stuck_flags |= COH_FLAG_UNSAFE; /* is_unsafe, program.hpp:166-170 */
    }
  }
  free(prog);
  return 0;
}

int orc_eval_traces(const uint16_t* records, uint64_t n_total, uint64_t t_begin, uint64_t t_end,
                    uint32_t n_calls, uint32_t n_arrays, int32_t fuel, const uint64_t* array_bytes,
                    coh_trace_result* out, uint32_t* boundary) {
  return orc_eval_traces_ex(records, n_total, t_begin, t_end, n_calls, n_arrays, fuel, array_bytes, 0, out,
                            boundary);
}

/* Generator restatement (include/cohere_b200.h) for record-checksum parity. */
static uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

int orc_gen_records(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                    uint32_t n_arrays, uint32_t adv_per1024, uint16_t* recs) {
  const uint32_t n_chunks = (n_calls + 7) / 8;
  for (uint32_t c = 0; c < n_chunks; ++c)
    for (uint64_t t = 0; t < n_traces; ++t)
      for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t i = c * 8 + k;
        uint16_t v = 0;
        if (i < n_calls) {
          const uint64_t h = orc_splitmix64(seed ^ ((trace0 + t) << 20) ^ (uint64_t)i);
          const uint32_t arr = (uint32_t)(((h & 0xFFFFFFFFull) * n_arrays) >> 32);
          const uint32_t kind = (uint32_t)((((h >> 32) & 0xFFFFull) * 3ull) >> 16);
          const uint32_t site = (uint32_t)((h >> 48) & 1ull);
          const uint32_t adv = (uint32_t)((h >> 49) & 0x3FFull) < adv_per1024;
          const uint32_t var = adv ? 1u + (uint32_t)((((h >> 59) & 0x1Full) * 7ull) >> 5) : 0u;
          v = COH_MAKE_REC(arr, kind, site, var);
        }
        recs[((uint64_t)c * n_traces + t) * 8 + k] = v;
      }
  return 0;
}

/* ===================================================================================
 * Element-granular programs (restatement, bit planes):
 *   overlap closure     infer_overlap_closure, overlap.hpp:182-230 (one declared mode
 *                       per call: W/RW on x appends RW@site on every overlapping view in
 *                       declaration order; overlaps() overlap.hpp:17-20)
 *   translation         translate_mode/translate_block, modes.hpp:31-59 (whole-view sync
 *                       of the concrete range, then the abstract key)
 *   whole-view sync     semantics.hpp:155-166: atomic over [lo,hi] ascending, first
 *                       failing cell is the stuck key, delta = changed cells
 *   element effects     program.hpp:94-101 + apply_effect_at, one step per cell
 *   boundary check      abstraction_correct, modes.hpp:79-90 (every view, every cell)
 */
#include <stdlib.h>

static int bit_get(const uint8_t* p, uint32_t i) { return p[i]; }

typedef struct {
  uint8_t* L;
  uint8_t* R;
  uint8_t abs[COH_MAX_VIEWS];
  int64_t steps;
  int64_t fuel;
  coh_elem_result* out;
  uint32_t* runs;
  uint64_t runs_cap;
  int overflow;
} orc_elem_state;

/* one step budget check: 1 = ok to step, 0 = fuel exhausted */
static int fuel_ok(orc_elem_state* st) { return st->steps < st->fuel; }

static void set_stuck(orc_elem_state* st, int eff, int site, int abs_key, uint32_t index, int actual) {
  st->out->status = COH_RUN_STUCK;
  st->out->stuck_effect = (uint8_t)eff;
  st->out->stuck_flags = (uint8_t)(site | (abs_key << 1) | (actual << 2));
  st->out->stuck_index = index;
}

/* returns 0 to continue, 1 when the run stops (stuck / fuel) */
static int abstract_effect(orc_elem_state* st, uint32_t v, int eff, int site) {
  if (!fuel_ok(st)) { st->out->status = COH_RUN_FUEL_EXHAUSTED; return 1; }
  const int after = orc_apply_cell(eff, site, st->abs[v]);
  if (after < 0) { set_stuck(st, eff, site, 1, v, st->abs[v]); return 1; }
  st->abs[v] = (uint8_t)after;
  st->steps++;
  return 0;
}

static int whole_view_sync(orc_elem_state* st, uint32_t lo, uint32_t hi, int eff, int site) {
  if (!fuel_ok(st)) { st->out->status = COH_RUN_FUEL_EXHAUSTED; return 1; }
  /* unify every cell first (atomic: a failure leaves the store untouched) */
  for (uint32_t i = lo; i <= hi; ++i) {
    const int pair = bit_get(st->L, i) | (bit_get(st->R, i) << 1);
    if (orc_apply_cell(eff, site, pair) < 0) { set_stuck(st, eff, site, 0, i, pair); return 1; }
  }
  int64_t run_lo = -1;
  for (uint32_t i = lo; i <= hi + 1; ++i) {
    int changed = 0;
    if (i <= hi) {
      const int pair = bit_get(st->L, i) | (bit_get(st->R, i) << 1);
      const int after = orc_apply_cell(eff, site, pair);
      changed = after != pair;
      st->L[i] = (uint8_t)(after & 1);
      st->R[i] = (uint8_t)((after >> 1) & 1);
    }
    if (changed && run_lo < 0) run_lo = i;
    if (!changed && run_lo >= 0) {
      if (st->out->n_runs < st->runs_cap) {
        if (st->runs) {
          st->runs[2 * st->out->n_runs] = (uint32_t)run_lo;
          st->runs[2 * st->out->n_runs + 1] = i - 1;
        }
      } else {
        st->overflow = 1;
      }
      st->out->n_runs++;
      st->out->transfer_cells += (uint64_t)(i - run_lo);
      run_lo = -1;
    }
  }
  st->out->transfers++;
  st->out->vpu_cells += (uint64_t)(hi - lo + 1);
  st->steps++;
  return 0;
}

static int element_range(orc_elem_state* st, uint32_t lo, uint32_t hi, int eff, int site) {
  for (uint32_t i = lo; i <= hi; ++i) {
    if (!fuel_ok(st)) { st->out->status = COH_RUN_FUEL_EXHAUSTED; return 1; }
    const int pair = bit_get(st->L, i) | (bit_get(st->R, i) << 1);
    const int after = orc_apply_cell(eff, site, pair);
    if (after < 0) { set_stuck(st, eff, site, 0, i, pair); return 1; }
    st->L[i] = (uint8_t)(after & 1);
    st->R[i] = (uint8_t)((after >> 1) & 1);
    st->steps++;
  }
  return 0;
}

/* translate_mode (modes.hpp:31-50) executed directly */
static int run_mode(orc_elem_state* st, const coh_elem_program* P, uint32_t v, int kind, int site) {
  const int sync = site == COH_REMOTE ? COH_PUSH : COH_PULL;
  if (kind == COH_R || kind == COH_RW) {
    if (!fuel_ok(st)) { st->out->status = COH_RUN_FUEL_EXHAUSTED; return 1; }
    const int flag = site == COH_REMOTE ? (st->abs[v] >> 1) & 1 : st->abs[v] & 1;
    st->steps++; /* the if step */
    if (!flag) {
      if (whole_view_sync(st, P->view_lo[v], P->view_hi[v], sync, COH_LOCAL)) return 1;
      if (abstract_effect(st, v, sync, COH_LOCAL)) return 1;
    }
  }
  if (kind == COH_W || kind == COH_RW)
    if (abstract_effect(st, v, COH_WRITE, site)) return 1;
  return 0;
}

int orc_elem_run(const coh_elem_program* P, coh_elem_result* out, uint32_t* plane_l, uint32_t* plane_r,
                 uint8_t* view_abs, uint32_t* boundary, uint32_t* runs, uint64_t runs_cap) {
  if (P->n_views > COH_MAX_VIEWS) return -1;
  for (uint32_t v = 0; v < P->n_views; ++v)
    if (P->view_lo[v] > P->view_hi[v] || P->view_hi[v] >= P->n_cells) return -1;
  orc_elem_state st;
  memset(&st, 0, sizeof st);
  memset(out, 0, sizeof *out);
  st.L = (uint8_t*)malloc(P->n_cells);
  st.R = (uint8_t*)malloc(P->n_cells);
  memset(st.L, 1, P->n_cells); /* initial_store: (V,I) */
  memset(st.R, 0, P->n_cells);
  if (P->frag_log2 > 32) return -1;
  for (uint32_t i = 0; i < P->n_cells; ++i) /* pre-fragmented cells start coherent, (V,V) */
    if ((coh_frag_mask(P->frag_seed, P->frag_log2, i / 32) >> (i % 32)) & 1u) st.R[i] = 1;
  for (uint32_t v = 0; v < P->n_views; ++v) st.abs[v] = 1;
  st.fuel = P->fuel;
  st.out = out;
  st.runs = runs;
  st.runs_cap = runs_cap;
  const uint32_t n_words = (P->n_calls + 31) / 32;
  if (boundary) memset(boundary, 0, 4u * n_words);
  int rc = 0;
  uint32_t c;
  for (c = 0; c < P->n_calls; ++c) {
    const coh_elem_call* call = &P->calls[c];
    const uint32_t x = call->view;
    if (x >= P->n_views) { rc = -1; break; }
    /* closure: declared mode, then shadow RW on overlapping views (declaration order) */
    if (run_mode(&st, P, x, call->kind, call->site)) break;
    int stopped = 0;
    if (call->kind != COH_R)
      for (uint32_t y = 0; y < P->n_views && !stopped; ++y)
        if (y != x && P->view_lo[x] <= P->view_hi[y] && P->view_lo[y] <= P->view_hi[x])
          stopped = run_mode(&st, P, y, COH_RW, call->site);
    if (stopped) break;
    for (int k = 0; k < call->n_body && !stopped; ++k) {
      const coh_elem_op* op = &call->body[k];
      stopped = element_range(&st, P->view_lo[x] + op->lo, P->view_lo[x] + op->hi, op->effect, op->site);
    }
    if (stopped) break;
    int ok = 1;
    for (uint32_t v = 0; v < P->n_views && ok; ++v)
      for (uint32_t i = P->view_lo[v]; i <= P->view_hi[v]; ++i) {
        const int pair = st.L[i] | (st.R[i] << 1);
        if (!orc_leq(st.abs[v], pair)) { ok = 0; break; }
      }
    out->calls_done++;
    if (!ok) out->violations++;
    if (ok && boundary) boundary[c / 32] |= 1u << (c % 32);
  }
  if (out->status != COH_RUN_DONE) out->stuck_call = c;
  out->steps = (uint64_t)st.steps;
  const uint32_t n_pw = (P->n_cells + 31) / 32;
  memset(plane_l, 0, 4u * n_pw);
  memset(plane_r, 0, 4u * n_pw);
  for (uint32_t i = 0; i < P->n_cells; ++i) {
    if (st.L[i]) plane_l[i / 32] |= 1u << (i % 32);
    if (st.R[i]) plane_r[i / 32] |= 1u << (i % 32);
  }
  for (uint32_t v = 0; v < P->n_views; ++v) view_abs[v] = st.abs[v];
  free(st.L);
  free(st.R);
  if (rc) return rc;
  return st.overflow ? -3 : 0;
}
