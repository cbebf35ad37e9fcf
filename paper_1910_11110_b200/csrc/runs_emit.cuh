// Cooperative emission of run starts / ends for a warp step (shared by the zero-run
// primitive, bitmap.cu, and the element path's sync apply, elem.cu).
#pragma once

#include <cstdint>

namespace cohb {

#ifndef COH_DENSE_STEP
#define COH_DENSE_STEP 64
#endif
constexpr uint32_t kDenseStep = COH_DENSE_STEP;  // runs per warp step above which the warp stages them

// Dense warp steps, staged: a step (32 lanes x 4 words = 4096 cells) has at most 2048
// run starts (or ends).  Every lane writes its own set bits' cells, in ascending order,
// into the warp's shared-memory buffer at S_lane + rank (independent per lane: no
// shuffles on the critical path), then the warp copies the step's T cells to out[base ..)
// with coalesced 128-byte stores.  A buffer of B entries takes the step in passes of B
// positions.  Buffer index o is stored at o ^ ((o >> 5) & 31): lanes whose offsets are
// ~32 apart (the dense case) then hit different banks.
constexpr uint32_t kStageBuf = 2048;  // u32 entries per warp per pass (default)
__device__ __forceinline__ uint32_t stage_swz(uint32_t o) { return o ^ ((o >> 5) & 31u); }

template <uint32_t B = kStageBuf>
__device__ __forceinline__ void emit_staged(const uint32_t* m, uint32_t S, uint32_t T, uint32_t cb, uint64_t base,
                                            uint32_t* out, uint64_t cap, uint32_t* buf) {
  if (base >= cap) return;  // warp-uniform: nothing of this step fits (e.g. a full staging chunk)
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t lim = T < cap - base ? T : cap - base;
  const uint32_t mine = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
  for (uint32_t p0 = 0; p0 < lim; p0 += B) {  // warp-uniform passes of B positions
    uint32_t o = S;
    if (S < p0 + B && S + mine > p0) {  // this lane has positions in the pass
#pragma unroll
      for (int k = 0; k < 4; ++k)
        for (uint32_t x = m[k]; x; x &= x - 1, ++o)
          if (o - p0 < B) buf[stage_swz(o - p0)] = cb + 32u * k + (uint32_t)(__ffs(x) - 1);
    }
    __syncwarp();
    const uint32_t n = lim - p0 < B ? (uint32_t)(lim - p0) : B;
    for (uint32_t p = lane; p < n; p += 32) out[base + p0 + p] = buf[stage_swz(p)];
    __syncwarp();  // the buffer is free again
  }
}

// The same for one warp step whose lanes cover consecutive 128-cell spans (lane L's first
// cell = lane 0's + 128 L): entries are u16 offsets from lane 0's first cell, so a whole
// step (at most 2048 starts or ends) fits one pass of a ~4 KB buffer -- no lane re-walks
// its bits for a second pass.  Each lane fills its slots [S, S + n) from the top, highest
// bit first (one FLO per bit, no lowest-bit isolation).  Entry o is stored at o + (o >> 5)
// (one pad slot per 32): lanes whose slots are ~32 apart (the dense case) land in
// different banks, and the copy-out reads 32 consecutive slots per warp load.
constexpr uint32_t kStageBuf16 = 2048 + 64;  // u16 slots per warp
__device__ __forceinline__ uint32_t stage_skew(uint32_t o) { return o + (o >> 5); }

__device__ __forceinline__ void emit_dense16(const uint32_t* m, uint32_t S, uint32_t T, uint32_t cb, uint64_t base,
                                             uint32_t* out, uint64_t cap, uint16_t* buf) {
  if (base >= cap) return;  // warp-uniform: nothing of this step fits
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cell0 = __shfl_sync(0xFFFFFFFFu, cb, 0);
  const uint32_t rel = cb - cell0;
  uint32_t o = S + __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
#pragma unroll
  for (int k = 3; k >= 0; --k) {
    const uint32_t rk = rel + 32u * k;
    for (uint32_t x = m[k]; x;) {
      const uint32_t pos = 31u - __clz(x);
      buf[stage_skew(--o)] = (uint16_t)(rk + pos);
      x ^= 1u << pos;
    }
  }
  __syncwarp();
  const uint32_t n = (uint64_t)T < cap - base ? T : (uint32_t)(cap - base);
  uint32_t* const ob = out + base;
  uint32_t p = lane;
  for (; p + 96u < n; p += 128u) {  // four coalesced stores per lane per round
    const uint32_t v0 = buf[stage_skew(p)], v1 = buf[stage_skew(p + 32u)], v2 = buf[stage_skew(p + 64u)],
                   v3 = buf[stage_skew(p + 96u)];
    ob[p] = cell0 + v0;
    ob[p + 32u] = cell0 + v1;
    ob[p + 64u] = cell0 + v2;
    ob[p + 96u] = cell0 + v3;
  }
  for (; p < n; p += 32u) ob[p] = cell0 + buf[stage_skew(p)];
  __syncwarp();  // the buffer is free again
}

// Sparse emission of one lane's starts (or ends) m[0..3] at out[pos ..) (pos = the lane's
// first position): the lowest set bit of every word goes out without a loop (its position
// is known from the popcounts of the words before it), the rare further bits of a word in
// a warp-uniform second round.  (The zero-run walker's form: a loop per bit, below, costs
// it 17 us at rho 2^-16 -- its register allocation shifts.)
__device__ __forceinline__ void emit_sparse(const uint32_t* m, uint64_t pos, uint32_t cb, uint32_t* out, uint64_t cap) {
  uint32_t rest = 0;
  uint64_t p = pos;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (m[k] && p < cap) out[p] = cb + 32u * k + (uint32_t)(__ffs(m[k]) - 1);
    rest |= m[k] & (m[k] - 1u);
    p += (uint32_t)__popc(m[k]);
  }
  if (!__any_sync(0xFFFFFFFFu, rest != 0u)) return;
  p = pos;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t x = m[k] & (m[k] - 1u);
    uint64_t q = p + 1u;
    for (; x; x &= x - 1u, ++q)
      if (q < cap) out[q] = cb + 32u * k + (uint32_t)(__ffs(x) - 1);
    p += (uint32_t)__popc(m[k]);
  }
}

// The same for the element path's apply (2% faster there at rho 2^-8 and 1/2): the lane's
// n bits, one loop trip per bit, lowest first, over its 128 cells as two 64-bit words (the
// warp runs max-n trips, 1-3 on a sparse step; the positions need no per-store test).
__device__ __forceinline__ void emit_sparse_bits(const uint32_t* m, uint32_t n, uint64_t pos, uint32_t cb,
                                                 uint32_t* out, uint64_t cap) {
  const uint32_t nn = pos >= cap ? 0u : (cap - pos < n ? (uint32_t)(cap - pos) : n);
  uint64_t lo = (uint64_t)m[1] << 32 | m[0], hi = (uint64_t)m[3] << 32 | m[2];
  uint32_t* const o = out + pos;
  for (uint32_t j = 0; j < nn; ++j) {
    const bool in_lo = lo != 0ull;
    const uint64_t x = in_lo ? lo : hi;
    o[j] = cb + (in_lo ? 0u : 64u) + (uint32_t)(__ffsll((long long)x) - 1);
    if (in_lo) lo &= lo - 1ull;
    else hi &= hi - 1ull;
  }
}

// Positions of one warp step's starts / ends (st / en: the lane's four words, ns / ne their
// popcounts): the lane's exclusive offsets xs / xe and the step totals Ts / Te.  Ballots
// when every lane holds at most one of each (sparse planes), else a warp scan of both
// counts packed in one word (a step has at most 2048 of each).
__device__ __forceinline__ void step_positions(uint32_t ns, uint32_t ne, uint32_t& xs, uint32_t& xe, uint32_t& Ts,
                                               uint32_t& Te) {
  const uint32_t lane = threadIdx.x & 31;
  if (__all_sync(0xFFFFFFFFu, (ns | ne) <= 1u)) {
    const uint32_t bs = __ballot_sync(0xFFFFFFFFu, ns != 0u), be = __ballot_sync(0xFFFFFFFFu, ne != 0u);
    const uint32_t lt = (1u << lane) - 1u;
    xs = __popc(bs & lt), xe = __popc(be & lt), Ts = __popc(bs), Te = __popc(be);
    return;
  }
  const uint32_t nse = ns | (ne << 16);
  uint32_t pse = nse;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(0xFFFFFFFFu, pse, o);
    if (lane >= (uint32_t)o) pse += a;
  }
  xs = (pse - nse) & 0xFFFFu, xe = (pse - nse) >> 16;
  const uint32_t T = __shfl_sync(0xFFFFFFFFu, pse, 31);
  Ts = T & 0xFFFFu, Te = T >> 16;
}

}  // namespace cohb
