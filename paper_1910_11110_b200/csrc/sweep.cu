// Device interpreter of general block programs: one thread runs one (program, schedule
// prefix) through run_annotated semantics (modes.hpp:105-125 over run, semantics.hpp:
// 253-287): effects and whole-view syncs (atomic, semantics.hpp:155-166) on a 2-bit-per-
// key store held in one 64-bit register, If/While one step each, opaque conditions read
// the schedule (exhausted -> false + overflow, semantics.hpp:39-43), fuel shared across
// blocks with Done checked before fuel, abstraction_correct after every block.
#include <cuda_runtime.h>

#include "internal.hpp"
#include "sweep.hpp"

namespace cohb {
namespace {

__device__ __forceinline__ int apply_pair_d(uint32_t eff, uint32_t site, uint32_t p) {
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

__device__ __forceinline__ bool leq_d(uint32_t a, uint32_t c) {
  return a == c || (c == 3u && (a == 1u || a == 2u));
}

__global__ void k_sweep_run(const uint32_t* __restrict__ code, const SweepMeta* __restrict__ meta,
                            const uint16_t* __restrict__ checks, const SweepItem* __restrict__ items,
                            uint32_t n_items, int32_t fuel, SweepOut* __restrict__ out,
                            SweepTrace* __restrict__ trace) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const SweepItem it = items[i];
  if (i != 0) trace = nullptr;
  const unsigned long long sbits = (unsigned long long)it.bits | ((unsigned long long)it.pad << 32);
  const SweepMeta m = meta[it.prog];
  const uint32_t* prog = code + m.code_off;
  unsigned long long store = 0x5555555555555555ull;  // initial_store: every key (V,I)
  if (m.n_keys < 32) store &= (1ull << (2 * m.n_keys)) - 1ull;
  uint32_t pc = 0, steps = 0, cursor = 0, overflow = 0, bnd = 0, blocks = 0, status = COH_RUN_DONE;
  uint32_t stuck_key = 0, stuck = 0, unsafe = 0;  // unsafe: some step left a key (I,I) (is_unsafe)
  for (;;) {
    const uint32_t ins = prog[pc];
    const uint32_t op = ins & 15u;
    if (op == BC_END) break;
    if (op == BC_JMP) {
      pc = ins >> 16;
      continue;
    }
    if (op == BC_BEND) {  // abstraction_correct (modes.hpp:79-90)
      bool ok = true;
      for (uint32_t k = 0; k < m.n_checks; ++k) {
        const uint32_t c = checks[m.check_off + k];
        const uint32_t a = (uint32_t)(store >> (2 * (c & 0xFFu))) & 3u, v = (uint32_t)(store >> (2 * (c >> 8))) & 3u;
        ok = ok && leq_d(a, v);
      }
      bnd |= (ok ? 1u : 0u) << blocks;
      ++blocks;
      ++pc;
      continue;
    }
    if ((int)steps >= fuel) {  // Done (BC_END) is checked first; every other op is a step
      status = COH_RUN_FUEL_EXHAUSTED;
      break;
    }
    if (op == BC_IF || op == BC_WHILE) {
      const uint32_t ck = (ins >> 4) & 3u, key = (ins >> 8) & 0xFFu;
      uint32_t bit;
      if (ck == 2u) {
        if (cursor < it.len) bit = (uint32_t)(sbits >> cursor++) & 1u;
        else { overflow = 1; bit = 0; }
      } else {
        bit = (uint32_t)(store >> (2 * key + ck)) & 1u;  // valid: local flag, gvalid: remote
      }
      if (trace) trace[steps] = SweepTrace{pc, (op == BC_WHILE ? 2u : 4u) + (bit ? 0u : 1u), store};
      ++steps;
      pc = bit ? pc + 1 : (ins >> 16);
      continue;
    }
    const uint32_t eff = (ins >> 4) & 7u, site = (ins >> 7) & 1u;
    if (op == BC_EFF) {
      const uint32_t key = (ins >> 8) & 0xFFu;
      const uint32_t before = (uint32_t)(store >> (2 * key)) & 3u;
      const int after = apply_pair_d(eff, site, before);
      if (after < 0) {
        status = COH_RUN_STUCK;
        stuck_key = key;
        stuck = eff | (site << 3) | (before << 5);
        break;
      }
      store = (store & ~(3ull << (2 * key))) | ((unsigned long long)after << (2 * key));
      unsafe |= after == 0;
    } else {  // BC_WHOLE: atomic over the cells, ascending
      const uint32_t lo = (ins >> 8) & 0xFFu, hi = (ins >> 16) & 0xFFu;
      bool fail = false;
      for (uint32_t k = lo; k <= hi; ++k) {
        const uint32_t before = (uint32_t)(store >> (2 * k)) & 3u;
        if (apply_pair_d(eff, site, before) < 0) {
          status = COH_RUN_STUCK;
          stuck_key = k;
          stuck = eff | (site << 3) | (before << 5);
          fail = true;
          break;
        }
      }
      if (fail) break;
      for (uint32_t k = lo; k <= hi; ++k) {
        const uint32_t before = (uint32_t)(store >> (2 * k)) & 3u;
        const uint32_t after = (uint32_t)apply_pair_d(eff, site, before);
        store = (store & ~(3ull << (2 * k))) | ((unsigned long long)after << (2 * k));
        unsafe |= after == 0;
      }
    }
    if (trace) trace[steps] = SweepTrace{pc, site, store};
    ++steps;
    ++pc;
  }
  SweepOut o;
  o.status_consumed = status | (cursor << 2) | (overflow << 10) | (blocks << 11) | (bnd << 16) | (stuck_key << 24);
  o.steps = steps;
  o.store = store;
  o.stuck = stuck;
  o.pad = unsafe;
  out[i] = o;
}

}  // namespace

int launch_sweep_run(const uint32_t* code, const SweepMeta* meta, const uint16_t* checks, const SweepItem* items,
                     uint32_t n_items, int32_t fuel, SweepOut* out, void* stream, std::string* err,
                     SweepTrace* trace) {
  if (!n_items) return COH_OK;
  k_sweep_run<<<(n_items + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(code, meta, checks, items,
                                                                                   n_items, fuel, out, trace);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("sweep launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

}  // namespace cohb
