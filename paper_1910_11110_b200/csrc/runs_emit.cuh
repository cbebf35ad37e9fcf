// Cooperative emission of run starts / ends for a warp step (shared by the zero-run
// primitive, bitmap.cu, and the element path's sync apply, elem.cu).
#pragma once

#include <cstdint>

namespace cohb {

#ifndef COH_DENSE_STEP
#define COH_DENSE_STEP 64
#endif
constexpr uint32_t kDenseStep = COH_DENSE_STEP;  // runs per warp step above which the warp writes cooperatively

// Dense steps: the warp writes the step's T positions [base, base + T) together, 32
// consecutive positions per store.  Position p belongs to the lane L with S_L <= p <
// S_L + n_L (S = the exclusive scan of the lanes' counts; found by a binary search over
// shuffled S) and is the (p - S_L)-th set bit of L's four mask words, at cell cb_L + 32 k
// + bit.  Positions at or past `cap` are neither computed nor written.
__device__ __forceinline__ void emit_dense(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3, uint32_t S, uint32_t T,
                                           uint64_t cb, uint64_t base, uint32_t* out, uint64_t cap) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t lim = base >= cap ? 0 : (T < cap - base ? T : cap - base);  // warp-uniform
  for (uint32_t k = 0; k * 32 < lim; ++k) {
    const uint32_t p = k * 32 + lane;
    uint32_t L = 0;
#pragma unroll
    for (uint32_t b = 16; b; b >>= 1)
      if (__shfl_sync(0xFFFFFFFFu, S, L + b) <= p) L += b;
    uint32_t rr = p - __shfl_sync(0xFFFFFFFFu, S, L);
    const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, m0, L), w1 = __shfl_sync(0xFFFFFFFFu, m1, L);
    const uint32_t w2 = __shfl_sync(0xFFFFFFFFu, m2, L), w3 = __shfl_sync(0xFFFFFFFFu, m3, L);
    const uint64_t c = __shfl_sync(0xFFFFFFFFu, cb, L);
    // the word holding the rr-th set bit, then the bit (binary search by popcount)
    uint32_t w = w0, wi = 0, cnt = __popc(w0);
    if (rr >= cnt) { rr -= cnt; w = w1; wi = 1; cnt = __popc(w1); }
    if (wi == 1 && rr >= cnt) { rr -= cnt; w = w2; wi = 2; cnt = __popc(w2); }
    if (wi == 2 && rr >= cnt) { rr -= cnt; w = w3; wi = 3; }
    uint32_t pos = 0;
#pragma unroll
    for (uint32_t sh = 16; sh; sh >>= 1) {
      const uint32_t low = __popc(w & ((1u << sh) - 1u));
      if (rr >= low) {
        rr -= low;
        w >>= sh;
        pos += sh;
      }
    }
    if (p < lim) out[base + p] = (uint32_t)(c + 32u * wi + pos);
  }
}


}  // namespace cohb

namespace cohb {

// Dense warp steps, staged: a step (32 lanes x 4 words = 4096 cells) has at most 2048
// run starts (or ends).  Every lane writes its own set bits' cells, in ascending order,
// into the warp's shared-memory buffer at S_lane + rank (independent per lane: no
// shuffles on the critical path), then the warp copies the step's T cells to out[base ..)
// with coalesced 128-byte stores.  A buffer of B entries takes the step in passes of B
// positions.  Buffer index o is stored at o ^ ((o >> 5) & 31): lanes whose offsets are
// ~32 apart (the dense case) then hit different banks.
constexpr uint32_t kStageBuf = 2048;  // u32 entries per warp (the element apply)
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

}  // namespace cohb
