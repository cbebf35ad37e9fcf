// Device interpreter for one general program of any size (the CLI's `run` / `trace`),
// following run (semantics.hpp:253-287: Done checked before fuel, Stuck takes no step,
// opaque conditions read the schedule and answer false once it is exhausted) over
// step_inplace (semantics.hpp:138-191: effects through the local / swapped-remote rules,
// whole-view syncs atomic over their cells, If/While one step each).
//
// The CTA runs the instruction stream in lockstep: every thread decodes the same
// instruction and evaluates the same (uniform) condition or effect outcome; thread 0
// commits single-key effects, and a whole-view sync is a range operation on the bit planes
// shared by all threads (first failing cell by a shared atomicMin, then a word-parallel
// set of the destination plane).
#include <cuda_runtime.h>

#include <algorithm>

#include "progrun.hpp"

namespace cohb {
namespace {

constexpr uint32_t kThreads = 256;
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct ProgOut {
  uint32_t status, steps, consumed, overflowed;
  uint32_t stuck_key, stuck_eff, stuck_site, stuck_actual;
  uint32_t n_deltas, pad;
};

// validity.hpp:73-120 on one pair (bit0 local, bit1 remote); a remote effect applies to
// the swapped pair and swaps the result back (semantics.hpp:109-130).  -1 = no unifier.
__device__ __forceinline__ int effect_on(uint32_t eff, uint32_t site, uint32_t p) {
  const uint32_t q = site ? ((p >> 1) | ((p & 1u) << 1)) : p;
  uint32_t r;
  if (eff == COH_PUSH) {
    if (!(q & 1u)) return -1;
    r = 3u;
  } else if (eff == COH_PULL) {
    if (!(q & 2u)) return -1;
    r = 3u;
  } else if (eff == COH_READ) {
    if (!(q & 1u)) return -1;
    r = q;
  } else if (eff == COH_WRITE) {
    r = 1u;
  } else {
    r = q;
  }
  return (int)(site ? ((r >> 1) | ((r & 1u) << 1)) : r);
}

__device__ __forceinline__ uint32_t pair_of(const uint32_t* L, const uint32_t* R, uint32_t k) {
  return ((L[k >> 5] >> (k & 31u)) & 1u) | (((R[k >> 5] >> (k & 31u)) & 1u) << 1);
}

// cells of word w inside [lo, hi]
__device__ __forceinline__ uint32_t range_mask(uint32_t w, uint32_t lo, uint32_t hi) {
  uint32_t m = 0xFFFFFFFFu;
  if (w == (lo >> 5)) m &= 0xFFFFFFFFu << (lo & 31u);
  if (w == (hi >> 5)) m &= 0xFFFFFFFFu >> (31u - (hi & 31u));
  return m;
}

__global__ void __launch_bounds__(kThreads) k_prog_run(const ProgIns* __restrict__ code, uint32_t* L, uint32_t* R,
                                                       int32_t fuel, unsigned long long sched, uint32_t sched_len,
                                                       ProgStep* trace, ProgDelta* deltas, uint32_t delta_cap,
                                                       ProgOut* out) {
  __shared__ uint32_t s_fail;
  const uint32_t tid = threadIdx.x;
  uint32_t pc = 0, steps = 0, cursor = 0, overflow = 0, status = COH_RUN_DONE, nd = 0;
  uint32_t sk = 0, se = 0, ss = 0, sa = 0;
  for (;;) {
    const ProgIns ins = code[pc];
    const uint32_t kind = ins.op & 15u;
    if (kind == PI_END) break;
    if (kind == PI_JMP) {
      pc = ins.target;
      continue;
    }
    if ((int32_t)steps >= fuel) {
      status = COH_RUN_FUEL_EXHAUSTED;
      break;
    }
    if (kind == PI_IF || kind == PI_WHILE) {
      const uint32_t cond = (ins.op >> 8) & 3u;
      uint32_t bit;
      if (cond == 2u) {
        if (cursor < sched_len) {
          bit = (uint32_t)(sched >> cursor) & 1u;
          ++cursor;
        } else {
          overflow = 1u;
          bit = 0u;
        }
      } else {
        bit = (pair_of(L, R, ins.a) >> cond) & 1u;
      }
      if (trace && tid == 0) trace[steps] = ProgStep{pc, (kind == PI_WHILE ? 2u : 4u) + (bit ? 0u : 1u), nd};
      ++steps;
      pc = bit ? pc + 1 : ins.target;
      continue;
    }
    const uint32_t eff = (ins.op >> 4) & 7u, site = (ins.op >> 7) & 1u;
    if (kind == PI_EFF) {
      const uint32_t before = pair_of(L, R, ins.a);
      const int after = effect_on(eff, site, before);
      if (after < 0) {
        status = COH_RUN_STUCK;
        sk = ins.a, se = eff, ss = site, sa = before;
        break;
      }
      __syncthreads();  // every thread has read the key
      if (tid == 0 && (uint32_t)after != before) {
        const uint32_t w = ins.a >> 5, b = 1u << (ins.a & 31u);
        L[w] = (after & 1) ? (L[w] | b) : (L[w] & ~b);
        R[w] = (after & 2) ? (R[w] | b) : (R[w] & ~b);
        if (deltas) {
          if (nd < delta_cap) deltas[nd] = ProgDelta{ins.a, (uint32_t)after};
          ++nd;
        }
      }
      __syncthreads();  // the new pair is visible to the CTA
    } else {            // PI_WHOLE: push/pull over the view's cells [a, b]
      const uint32_t lo = ins.a, hi = ins.b;
      // local push / remote pull need L and set R; local pull / remote push need R and set L
      const bool need_local = (eff == COH_PUSH) == (site == 0u);
      const uint32_t* need = need_local ? L : R;
      uint32_t* dst = need_local ? R : L;
      if (tid == 0) s_fail = kNone;
      __syncthreads();
      for (uint32_t w = (lo >> 5) + tid; w <= (hi >> 5); w += kThreads) {
        const uint32_t miss = ~need[w] & range_mask(w, lo, hi);
        if (miss) atomicMin(&s_fail, (w << 5) + (uint32_t)(__ffs(miss) - 1));
      }
      __syncthreads();
      const uint32_t fail = s_fail;
      if (fail != kNone) {  // the first failing cell, ascending; the store is untouched
        status = COH_RUN_STUCK;
        sk = fail, se = eff, ss = site, sa = pair_of(L, R, fail);
        break;
      }
      if (deltas && tid == 0) {  // changed cells (destination bit was 0), ascending, now (V,V)
        for (uint32_t w = lo >> 5; w <= (hi >> 5); ++w) {
          uint32_t ch = ~dst[w] & range_mask(w, lo, hi);
          while (ch) {
            const uint32_t b = (uint32_t)(__ffs(ch) - 1);
            ch &= ch - 1u;
            if (nd < delta_cap) deltas[nd] = ProgDelta{(w << 5) + b, 3u};
            ++nd;
          }
        }
      }
      __syncthreads();
      for (uint32_t w = (lo >> 5) + tid; w <= (hi >> 5); w += kThreads) dst[w] |= range_mask(w, lo, hi);
      __syncthreads();
    }
    if (trace && tid == 0) trace[steps] = ProgStep{pc, site, nd};
    ++steps;
    ++pc;
  }
  if (tid == 0) *out = ProgOut{status, steps, cursor, overflow, sk, se, ss, sa, nd, 0u};
}

struct DevMem {
  void* p = nullptr;
  ~DevMem() { cudaFree(p); }
};

}  // namespace

int prog_run(const std::vector<ProgIns>& code, uint32_t n_keys, int32_t fuel, uint64_t sched, uint32_t sched_len,
             bool trace, ProgRunResult* r, std::string* err) {
  const size_t words = std::max<size_t>(1, ((size_t)n_keys + 31) / 32);
  uint32_t cap = trace ? (1u << 20) : 0u;
  for (;;) {
    DevMem d_code, d_L, d_R, d_trace, d_delta, d_out;
    cudaError_t e;
#define COH_PR(x)                                          \
  if ((e = (x)) != cudaSuccess) {                          \
    *err = std::string(#x ": ") + cudaGetErrorString(e);   \
    return COH_E_CUDA;                                     \
  }
    COH_PR(cudaMalloc(&d_code.p, code.size() * sizeof(ProgIns)));
    COH_PR(cudaMalloc(&d_L.p, words * 4));
    COH_PR(cudaMalloc(&d_R.p, words * 4));
    COH_PR(cudaMalloc(&d_out.p, sizeof(ProgOut)));
    if (trace) {
      COH_PR(cudaMalloc(&d_trace.p, std::max<size_t>(1, (size_t)fuel) * sizeof(ProgStep)));
      COH_PR(cudaMalloc(&d_delta.p, (size_t)cap * sizeof(ProgDelta)));
    }
    COH_PR(cudaMemcpy(d_code.p, code.data(), code.size() * sizeof(ProgIns), cudaMemcpyHostToDevice));
    COH_PR(cudaMemset(d_L.p, 0xFF, words * 4));  // initial_store (program.hpp:174-184): every key (V,I)
    COH_PR(cudaMemset(d_R.p, 0x00, words * 4));
    k_prog_run<<<1, kThreads>>>(static_cast<const ProgIns*>(d_code.p), static_cast<uint32_t*>(d_L.p),
                                static_cast<uint32_t*>(d_R.p), fuel, sched, sched_len,
                                static_cast<ProgStep*>(d_trace.p), static_cast<ProgDelta*>(d_delta.p), cap,
                                static_cast<ProgOut*>(d_out.p));
    COH_PR(cudaGetLastError());
    ProgOut o;
    COH_PR(cudaMemcpy(&o, d_out.p, sizeof o, cudaMemcpyDeviceToHost));
    if (trace && o.n_deltas > cap) {  // the changed-key log did not fit: once more with room for all
      cap = o.n_deltas;
      continue;
    }
    r->status = o.status;
    r->steps = o.steps;
    r->consumed = o.consumed;
    r->overflowed = o.overflowed;
    r->stuck_key = o.stuck_key;
    r->stuck_eff = o.stuck_eff;
    r->stuck_site = o.stuck_site;
    r->stuck_actual = o.stuck_actual;
    r->L.resize(words);
    r->R.resize(words);
    COH_PR(cudaMemcpy(r->L.data(), d_L.p, words * 4, cudaMemcpyDeviceToHost));
    COH_PR(cudaMemcpy(r->R.data(), d_R.p, words * 4, cudaMemcpyDeviceToHost));
    if (trace) {
      r->trace.resize(o.steps);
      r->deltas.resize(o.n_deltas);
      if (o.steps) COH_PR(cudaMemcpy(r->trace.data(), d_trace.p, o.steps * sizeof(ProgStep), cudaMemcpyDeviceToHost));
      if (o.n_deltas)
        COH_PR(cudaMemcpy(r->deltas.data(), d_delta.p, o.n_deltas * sizeof(ProgDelta), cudaMemcpyDeviceToHost));
    }
#undef COH_PR
    return COH_OK;
  }
}

}  // namespace cohb
