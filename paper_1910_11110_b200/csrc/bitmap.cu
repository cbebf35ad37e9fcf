// Bit-plane primitives (coh_bitmap_{range_set, range_clear,
// first_zero, extract_zero_runs, view_check}), batched over ranges, stream-ordered.
//
// Semantics (from validity.hpp:79-120 / semantics.hpp:155-166 /
// modes.hpp:79-90): a plane is a run of 32-bit words, cell i = bit i%32 of word i/32.
//   range_set / range_clear   w x[i] on a range: the plane's bits [lo, hi] := 1 / 0
//   first_zero                the stuck cell of a whole-view sync: the first cell of
//                             [lo, hi] whose bit is 0 (the reference checks ascending)
//   extract_zero_runs         the transfer ranges of a whole-view sync: maximal runs of
//                             0 bits of the destination plane in [lo, hi], ascending
//   view_check                abstraction_correct for one view: (V,I) <=> L == 1 on the
//                             range, (I,V) <=> R == 1, (V,V) <=> both, (I,I) <=> L == R == 0
//
// Streaming decomposition: the aligned 16-byte quads covering all ranges form one flat
// index space (a single-block scan gives each range's first flat quad).  Every warp owns a
// contiguous chunk of it and walks it 32 quads per step, lane i on quad i (a coalesced
// 512-byte access), four steps in flight; a lane finds its range once by binary search and
// then only advances.  Per-range results (first zero, view flags) accumulate in registers
// and are flushed with one atomic when the range changes (warp-reduced when the whole warp
// agrees), so the loop has no barriers and stays HBM-bound.  Zero runs: a collect pass over
// warp chunks (counts + staged runs), a scan of the chunk counts, and a place pass putting
// each start / end at its global ascending position (the k-th start and the k-th end are
// the same run: runs never cross ranges).
#include <cuda_runtime.h>

#include <string>

#include "internal.hpp"
#include "runs_emit.cuh"

namespace cohb {
namespace {

constexpr uint32_t kBT = 256;   // threads per block
constexpr int kU = 4;           // warp steps in flight
#ifndef COH_RUNS_RU
#define COH_RUNS_RU 4
#endif
#ifndef COH_RUNS_MINB
#define COH_RUNS_MINB 3
#endif
constexpr int kRU = COH_RUNS_RU;  // warp steps in flight in the zero-run walker (chunk_runs)
#ifndef COH_RUNS_PF
#define COH_RUNS_PF 1
#endif
constexpr int kRunsPf = COH_RUNS_PF;  // walker iterations between an L2 prefetch and its loads
constexpr uint32_t kRunsBuf = kStageBuf16 / 2;  // dense-step staging per warp, u32 words (kStageBuf16 u16 slots)
constexpr size_t kRunsSmem = (size_t)(kBT / 32) * kRunsBuf * 4u;  // both zero-run passes: dense staging
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct Flat {
  const coh_bitmap_range* r;
  const uint64_t* qp;  // n + 1: first flat quad of each range (qp[n] = total)
  uint32_t n;
};

__device__ __forceinline__ uint64_t qa_first(const coh_bitmap_range& R) { return (R.word_off + (R.lo >> 5)) >> 2; }
__device__ __forceinline__ uint64_t qa_last(const coh_bitmap_range& R) { return (R.word_off + (R.hi >> 5)) >> 2; }
// The flat space gives every range whole 128-byte lines (8 quads): a warp step of 32 quads
// then writes / reads exactly four full lines, so no L2 sector is ever half-written by two
// different steps (which costs a DRAM read-fill).  The padding quads are never touched.
__device__ __forceinline__ uint64_t qa_base(const coh_bitmap_range& R) { return qa_first(R) & ~7ull; }
__device__ __forceinline__ uint64_t qa_end(const coh_bitmap_range& R) { return qa_last(R) | 7ull; }

// Mask of the cells of plane-relative word w inside [lo, hi].
__device__ __forceinline__ uint32_t cell_mask(uint64_t w, uint32_t lo, uint32_t hi) {
  const uint64_t wl = lo >> 5, wh = hi >> 5;
  if (w < wl || w > wh) return 0u;
  uint32_t m = 0xFFFFFFFFu;
  if (w == wl) m &= 0xFFFFFFFFu << (lo & 31u);
  if (w == wh) m &= 0xFFFFFFFFu >> (31u - (hi & 31u));
  return m;
}

__device__ __forceinline__ uint32_t find_range(const Flat& F, uint64_t f) {  // last r with qp[r] <= f
  uint32_t a = 0, b = F.n;
  while (b - a > 1) {
    const uint32_t m = (a + b) >> 1;
    if (F.qp[m] <= f) a = m;
    else b = m;
  }
  return a;
}

// The warp's chunk of the flat quad space: [f0, f1), f0 a multiple of 32.
__device__ __forceinline__ void warp_chunk(uint64_t Q, uint64_t& f0, uint64_t& f1, uint64_t& wid) {
  const uint64_t warps = (uint64_t)gridDim.x * (kBT / 32);
  wid = ((uint64_t)blockIdx.x * kBT + threadIdx.x) >> 5;
  const uint64_t per = (((Q + warps - 1) / warps) + 31) & ~31ull;
  f0 = wid * per;
  f1 = f0 + per < Q ? f0 + per : Q;
}

// True (warp-uniform) when the iteration's 32 x kU quads [base, base + 32 kU) are all
// interior quads of the lanes' current range: then every lane is in that one range (a
// lane's range only advances, and the iteration lies inside it), and the walkers skip
// per-quad range tracking (its 64-bit compares dominate the instruction count).
template <int U = kU>
__device__ __forceinline__ bool interior_iteration(uint64_t base, uint64_t f1, uint64_t qend, uint64_t qa0,
                                                   uint64_t qtf, uint64_t qtl) {
  const uint64_t e = base + 32ull * U;
  return __all_sync(0xFFFFFFFFu, e <= f1 && e <= qend && qa0 + base > qtf && qa0 + e - 1 < qtl);
}

// Walks this lane's quads of the warp chunk (lane + 32 j), kU steps per iteration so the
// loads of several steps are in flight.  body(r, R, qa, interior) for each valid quad;
// interior = neither the first nor the last quad of its range, i.e. all four words lie
// wholly inside [lo, hi] (the fast path: no masks).
template <class Body>
__device__ __forceinline__ void walk(const Flat& F, uint64_t f0, uint64_t f1, Body&& body) {
  const uint32_t lane = threadIdx.x & 31;
  if (f0 >= f1) return;
  uint32_t r = find_range(F, f0 + lane < f1 ? f0 + lane : f1 - 1);
  uint64_t qbeg = F.qp[r], qend = F.qp[r + 1];
  coh_bitmap_range R = F.r[r];
  uint64_t qa0 = qa_base(R) - qbeg, qtf = qa_first(R), qtl = qa_last(R);
  for (uint64_t base = f0; base < f1; base += 32ull * kU) {
    if (interior_iteration(base, f1, qend, qa0, qtf, qtl)) {
#pragma unroll
      for (int u = 0; u < kU; ++u) body(r, R, qa0 + base + 32ull * u + lane, true);
      continue;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t f = base + 32ull * u + lane;
      if (f >= f1) break;
      if (f >= qend) {  // monotone advance (empty ranges skipped)
        do {
          ++r;
          qbeg = qend;
          qend = F.qp[r + 1];
        } while (f >= qend);
        R = F.r[r];
        qa0 = qa_base(R) - qbeg, qtf = qa_first(R), qtl = qa_last(R);
      }
      const uint64_t qa = qa0 + f;
      if (qa >= qtf && qa <= qtl) body(r, R, qa, qa != qtf && qa != qtl);
    }
  }
}

// walk() for reading kernels: the kU quads of an iteration are located and their 16-byte
// words (from NP planes) loaded first, then processed, so all kU x NP loads are in flight
// together.  body(r, qa, interior, v[NP]); edge quads re-read their range record (L1 hit).
template <int NP, class Body>
__device__ __forceinline__ void walk_pf(const Flat& F, uint64_t f0, uint64_t f1, const uint32_t* const (&planes)[NP],
                                        Body&& body) {
  const uint32_t lane = threadIdx.x & 31;
  if (f0 >= f1) return;
  uint32_t r = find_range(F, f0 + lane < f1 ? f0 + lane : f1 - 1);
  uint64_t qbeg = F.qp[r], qend = F.qp[r + 1];
  coh_bitmap_range R0 = F.r[r];
  uint64_t qa0 = qa_base(R0) - qbeg, qtf = qa_first(R0), qtl = qa_last(R0);
  for (uint64_t base = f0; base < f1; base += 32ull * kU) {
    uint4 v[kU][NP];
    if (interior_iteration(base, f1, qend, qa0, qtf, qtl)) {
      const uint64_t qb = qa0 + base + lane;
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int p = 0; p < NP; ++p) v[u][p] = __ldcs(reinterpret_cast<const uint4*>(planes[p]) + qb + 32ull * u);
#pragma unroll
      for (int u = 0; u < kU; ++u) body(r, qb + 32ull * u, true, v[u]);
      continue;
    }
    uint32_t rr[kU];
    uint64_t qa[kU];
    bool in[kU], ok[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t f = base + 32ull * u + lane;
      bool live = f < f1;
      if (live && f >= qend) {
        do {
          ++r;
          qbeg = qend;
          qend = F.qp[r + 1];
        } while (f >= qend);
        const coh_bitmap_range R = F.r[r];
        qa0 = qa_base(R) - qbeg, qtf = qa_first(R), qtl = qa_last(R);
      }
      rr[u] = r;
      qa[u] = qa0 + f;
      ok[u] = live && qa[u] >= qtf && qa[u] <= qtl;
      in[u] = qa[u] != qtf && qa[u] != qtl;
#pragma unroll
      for (int p = 0; p < NP; ++p)
        v[u][p] = ok[u] ? __ldcs(reinterpret_cast<const uint4*>(planes[p]) + qa[u]) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (ok[u]) body(rr[u], qa[u], in[u], v[u]);
  }
}

__global__ void __launch_bounds__(1024) k_quad_prefix(const coh_bitmap_range* r, uint32_t n, uint64_t* prefix) {
  __shared__ uint64_t warp_sum[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t base = 0; base <= n; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    uint64_t v = 0;
    if (i < n && r[i].lo <= r[i].hi) v = qa_end(r[i]) - qa_base(r[i]) + 1;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) warp_sum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = warp_sum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= (uint32_t)o) w += y;
      }
      warp_sum[lane] = w;
    }
    __syncthreads();
    if (i <= n) prefix[i] = carry + (warp ? warp_sum[warp - 1] : 0) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sum[31];
    __syncthreads();
  }
}

// Up to kFusedRanges ranges, every block scans the range list itself into shared memory
// (F.qp == nullptr on entry) instead of a separate single-block prefix launch.
constexpr uint32_t kFusedRanges = 1023;
__device__ __forceinline__ void shared_prefix(Flat& F, uint64_t* s_qp) {
  if (F.qp) return;
  __shared__ uint64_t wsum[kBT / 32];
  constexpr uint32_t kPer = (kFusedRanges + 1) / kBT;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t v[kPer], sum = 0;
#pragma unroll
  for (uint32_t j = 0; j < kPer; ++j) {
    const uint32_t i = tid * kPer + j;
    v[j] = 0;
    if (i < F.n) {
      const coh_bitmap_range R = F.r[i];
      if (R.lo <= R.hi) v[j] = qa_end(R) - qa_base(R) + 1;
    }
    sum += v[j];
  }
  uint64_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  uint64_t e = x - sum;
  for (uint32_t w = 0; w < warp; ++w) e += wsum[w];
#pragma unroll
  for (uint32_t j = 0; j < kPer; ++j) {
    const uint32_t i = tid * kPer + j;
    if (i <= F.n) s_qp[i] = e;
    e += v[j];
  }
  __syncthreads();
  F.qp = s_qp;
}
#define COH_BM_PROLOGUE               \
  __shared__ uint64_t s_qp_[kFusedRanges + 1]; \
  Flat F = Fg;                        \
  shared_prefix(F, s_qp_);

template <bool SET>
__global__ void __launch_bounds__(kBT) k_range_set(uint32_t* words, Flat Fg) {
  COH_BM_PROLOGUE
  uint64_t f0, f1, wid;
  warp_chunk(F.qp[F.n], f0, f1, wid);
  walk(F, f0, f1, [&](uint32_t, const coh_bitmap_range& R, uint64_t qa, bool interior) {
    if (interior) {
      const uint32_t v = SET ? 0xFFFFFFFFu : 0u;
      reinterpret_cast<uint4*>(words)[qa] = make_uint4(v, v, v, v);
      return;
    }
    uint32_t m[4];
    bool full = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      m[k] = cell_mask(qa * 4 + k - R.word_off, R.lo, R.hi);
      full &= m[k] == 0xFFFFFFFFu;
    }
    if (full) {
      const uint32_t v = SET ? 0xFFFFFFFFu : 0u;
      reinterpret_cast<uint4*>(words)[qa] = make_uint4(v, v, v, v);
      return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // range edges: another range may share the word
      if (!m[k]) continue;
      if (SET) atomicOr(words + qa * 4 + k, m[k]);
      else atomicAnd(words + qa * 4 + k, ~m[k]);
    }
  });
}

// Per-range accumulation with flushes on range change; OP: 0 = min (first zero), 1 = or.
template <int OP>
struct Acc {
  uint32_t r = kNone, v = OP == 0 ? kNone : 0u;
  uint32_t* out;
  __device__ __forceinline__ void add(uint32_t rr, uint32_t x) {
    if (rr != r) {
      flush_lane();
      r = rr;
    }
    v = OP == 0 ? min(v, x) : (v | x);
  }
  __device__ __forceinline__ void flush_lane() {
    if (r == kNone) return;
    if (OP == 0 && v != kNone) atomicMin(out + r, v);
    if (OP == 1 && v) atomicOr(out + r, v);
    v = OP == 0 ? kNone : 0u;
  }
  __device__ __forceinline__ void finish() {  // warp-reduced when every lane holds the same range
    const uint32_t r0 = __shfl_sync(0xFFFFFFFFu, r, 0);
    if (__all_sync(0xFFFFFFFFu, r == r0)) {
      if (r0 == kNone) return;
      const uint32_t w = OP == 0 ? __reduce_min_sync(0xFFFFFFFFu, v) : __reduce_or_sync(0xFFFFFFFFu, v);
      if ((threadIdx.x & 31) == 0) {
        if (OP == 0 && w != kNone) atomicMin(out + r0, w);
        if (OP == 1 && w) atomicOr(out + r0, w);
      }
    } else {
      flush_lane();
    }
  }
};

__global__ void __launch_bounds__(kBT) k_first_zero(const uint32_t* words, Flat Fg, uint32_t* first) {
  COH_BM_PROLOGUE
  uint64_t f0, f1, wid;
  warp_chunk(F.qp[F.n], f0, f1, wid);
  Acc<0> acc;
  acc.out = first;
  const uint32_t* const planes[1] = {words};
  walk_pf<1>(F, f0, f1, planes, [&](uint32_t r, uint64_t qa, bool interior, const uint4 (&vv)[1]) {
    const uint4 v = vv[0];
    if (interior && (v.x & v.y & v.z & v.w) == 0xFFFFFFFFu) return;  // no zero: nothing to record
    const coh_bitmap_range R = F.r[r];
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
    uint32_t best = kNone;
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      const uint64_t wr = qa * 4 + k - R.word_off;
      const uint32_t z = ~w4[k] & cell_mask(wr, R.lo, R.hi);
      if (z) best = (uint32_t)(wr * 32 + (__ffs(z) - 1));
    }
    acc.add(r, best);
  });
  acc.finish();
}

__global__ void __launch_bounds__(kBT) k_view_flags(const uint32_t* L, const uint32_t* Rp, Flat Fg, uint32_t* flags) {
  COH_BM_PROLOGUE
  uint64_t f0, f1, wid;
  warp_chunk(F.qp[F.n], f0, f1, wid);
  Acc<1> acc;
  acc.out = flags;
  const uint32_t* const planes[2] = {L, Rp};
  walk_pf<2>(F, f0, f1, planes, [&](uint32_t r, uint64_t qa, bool interior, const uint4 (&v)[2]) {
    const uint4 a = v[0], b = v[1];
    if (interior) {  // whole words: AND / OR folds
      const uint32_t land = a.x & a.y & a.z & a.w, rand_ = b.x & b.y & b.z & b.w;
      const uint32_t lor = a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w;
      acc.add(r, (~land ? 1u : 0u) | (~rand_ ? 2u : 0u) | (lor ? 4u : 0u));
      return;
    }
    const coh_bitmap_range R = F.r[r];
    const uint32_t la[4] = {a.x, a.y, a.z, a.w}, ra[4] = {b.x, b.y, b.z, b.w};
    uint32_t f = 0;  // bit0 some L == 0, bit1 some R == 0, bit2 some L | R == 1
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t m = cell_mask(qa * 4 + k - R.word_off, R.lo, R.hi);
      f |= ((~la[k] & m) ? 1u : 0u) | ((~ra[k] & m) ? 2u : 0u) | (((la[k] | ra[k]) & m) ? 4u : 0u);
    }
    acc.add(r, f);
  });
  acc.finish();
}

__global__ void k_view_finish(const uint32_t* flags, const uint8_t* abs_pair, uint32_t n, uint8_t* ok) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t f = flags[i], a = abs_pair[i] & 3u;  // bit0 local V, bit1 remote V
  const bool L1 = !(f & 1u), R1 = !(f & 2u), none = !(f & 4u);
  ok[i] = a == 1u ? L1 : a == 2u ? R1 : a == 3u ? (L1 && R1) : none;
}

// Run starts / ends of one quad, given the plane words just before and after it: a start
// is a 0 cell whose predecessor (in the range) is not 0, an end a 0 cell whose successor is
// not 0.  Interior quads (neither first nor last of their range) need no masks.
__device__ __forceinline__ void runs_of(const coh_bitmap_range* Rp, uint64_t qa, bool interior, const uint4 v,
                                        uint32_t pw, uint32_t nw, uint32_t st[4], uint32_t en[4]) {
  uint32_t z[4], zp, zn;
  if (interior) {
    if ((v.x | v.y | v.z | v.w) == 0u) {  // all 0: a start iff the cell before is set, an end iff the one after
      st[0] = pw >> 31;
      en[3] = (nw & 1u) << 31;
      st[1] = st[2] = st[3] = en[0] = en[1] = en[2] = 0u;
      return;
    }
    z[0] = ~v.x, z[1] = ~v.y, z[2] = ~v.z, z[3] = ~v.w;
    zp = ~pw, zn = ~nw;
  } else {
    const coh_bitmap_range R = *Rp;
    const uint64_t wr0 = qa * 4 - R.word_off;  // plane-relative word of v.x (may wrap: masks are 0)
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) z[k] = ~w4[k] & cell_mask(wr0 + k, R.lo, R.hi);
    zp = ~pw & cell_mask(wr0 - 1, R.lo, R.hi);
    zn = ~nw & cell_mask(wr0 + 4, R.lo, R.hi);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t prev = k ? z[k - 1] : zp, next = k < 3 ? z[k + 1] : zn;
    st[k] = z[k] & ~((z[k] << 1) | (prev >> 31));
    en[k] = z[k] & ~((z[k] >> 1) | (next << 31));
  }
}

// Walks the warp chunk [f0, f1) in steps of 32 quads (kU steps' loads in flight) and calls
// visit(u, ok, f, r, qa, qbeg, st, en) warp-synchronously for every step (all lanes, ok =
// the lane has a quad).  Neighbour words come from the adjacent lanes by shuffle; only the
// chunk / iteration edges load them.
template <class Visit>
__device__ __forceinline__ void chunk_runs(const uint32_t* words, const Flat& F, uint64_t f0, uint64_t f1,
                                           Visit&& visit) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t r = find_range(F, f0 + lane < f1 ? f0 + lane : f1 - 1);
  uint64_t qbeg = F.qp[r], qend = F.qp[r + 1];
  coh_bitmap_range R0 = F.r[r];
  uint64_t qa0 = qa_base(R0) - qbeg, qtf = qa_first(R0), qtl = qa_last(R0);
  uint32_t carry = 0;
  bool carry_ok = false;
  for (uint64_t base = f0; base < f1; base += 32ull * kRU) {
    // Fast iteration (warp-uniform): all 32 x kRU quads are interior quads of one range
    // (then every lane is in the same range, see the monotone advance below), so no
    // per-quad range tracking, masks or edge loads.
    if (interior_iteration<kRU>(base, f1, qend, qa0, qtf, qtl)) {
      const uint64_t qb = qa0 + base + lane;
#ifndef COH_RUNS_NO_PF
      {  // L2 prefetch of the iteration kRunsPf ahead (16 lanes x one 128-byte line), when it
         // still lies in this chunk and range: the loads then wait on L2, not HBM.  (Loading
         // the next iteration into a second register ring instead was measured no faster.)
        const uint64_t b2 = base + 32ull * kRU * kRunsPf;
        if (lane < 4u * kRU && b2 + 32ull * kRU <= f1 && b2 + 32ull * kRU <= qend)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(words) + qa0 + b2 + 8u * lane));
      }
#endif
      uint4 v[kRU];
#pragma unroll
      for (int u = 0; u < kRU; ++u) v[u] = __ldcg(reinterpret_cast<const uint4*>(words) + qb + 32ull * u);
      // the word after the iteration (inside the range: the iteration's quads are interior),
      // loaded with the others so that no step waits on it
      const uint32_t nw_it = __ldg(words + (qa0 + base + 32ull * kRU) * 4);
      const uint32_t pw_it = carry_ok ? carry : __ldg(words + (qa0 + base) * 4 - 1);
      {  // whole-iteration fast exits (one vote pair for kRU steps): no zero cell at all, or
         // all zero cells with set cells on neither side (one run continues through)
        uint32_t o = 0u, a = 0xFFFFFFFFu;
#pragma unroll
        for (int u = 0; u < kRU; ++u) {
          o |= v[u].x | v[u].y | v[u].z | v[u].w;
          a &= v[u].x & v[u].y & v[u].z & v[u].w;
        }
        if (__all_sync(0xFFFFFFFFu, a == 0xFFFFFFFFu) ||
            (__all_sync(0xFFFFFFFFu, o == 0u) && !((pw_it >> 31) | (nw_it & 1u)))) {
          carry = __shfl_sync(0xFFFFFFFFu, v[kRU - 1].w, 31);
          carry_ok = true;
          continue;
        }
      }

#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        const uint32_t a4 = v[u].x & v[u].y & v[u].z & v[u].w;
        if (__all_sync(0xFFFFFFFFu, a4 == 0xFFFFFFFFu)) continue;
        // the words just before and after the step (warp-uniform; the iteration lies
        // inside the range, so both exist)
        const uint32_t pw0 = u ? __shfl_sync(0xFFFFFFFFu, v[u ? u - 1 : 0].w, 31) : pw_it;
        const uint32_t nw31 = u < kRU - 1 ? __shfl_sync(0xFFFFFFFFu, v[u < kRU - 1 ? u + 1 : 0].x, 0) : nw_it;
        if (__all_sync(0xFFFFFFFFu, (v[u].x | v[u].y | v[u].z | v[u].w) == 0u) && !((pw0 >> 31) | (nw31 & 1u)))
          continue;  // one zero run continues through the step
        uint32_t pw = __shfl_up_sync(0xFFFFFFFFu, v[u].w, 1);
        uint32_t nw = __shfl_down_sync(0xFFFFFFFFu, v[u].x, 1);
        const uint64_t qa = qb + 32ull * u;
        if (lane == 0) pw = pw0;
        if (lane == 31) nw = nw31;
        uint32_t st[4] = {0, 0, 0, 0}, en[4] = {0, 0, 0, 0};
        if (a4 != 0xFFFFFFFFu) runs_of(F.r + r, qa, true, v[u], pw, nw, st, en);
        visit(true, base + 32ull * u + lane, r, qa, false, st, en);
      }
      carry = __shfl_sync(0xFFFFFFFFu, v[kRU - 1].w, 31);
      carry_ok = true;
      continue;
    }
    // General iteration (range edges, chunk ends): one quad per lane at a time, with
    // per-lane range tracking and masks; edge neighbours are loaded, not shuffled.
#pragma unroll 1
    for (int u = 0; u < kRU; ++u) {
      const uint64_t f = base + 32ull * u + lane;
      const bool live = f < f1;
      if (live && f >= qend) {
        do {
          ++r;
          qbeg = qend;
          qend = F.qp[r + 1];
        } while (f >= qend);
        const coh_bitmap_range R = F.r[r];
        qa0 = qa_base(R) - qbeg, qtf = qa_first(R), qtl = qa_last(R);
      }
      const uint64_t qa = qa0 + f;
      const bool ok = live && qa >= qtf && qa <= qtl;
      const bool first = qa == qtf, last = qa == qtl, in = ok && !first && !last;
      const uint4 v = ok ? __ldcg(reinterpret_cast<const uint4*>(words) + qa) : make_uint4(~0u, ~0u, ~0u, ~0u);
      uint32_t pw = __shfl_up_sync(0xFFFFFFFFu, v.w, 1);
      uint32_t nw = __shfl_down_sync(0xFFFFFFFFu, v.x, 1);
      if (lane == 0) pw = carry;
      if (ok) {  // neighbours the shuffles could not supply (inside the range only; else masked)
        if (lane == 0 && !carry_ok && !first) pw = __ldg(words + qa * 4 - 1);
        if ((lane == 31 || f + 1 >= f1) && !last) nw = __ldg(words + qa * 4 + 4);
      }
      uint32_t st[4] = {0, 0, 0, 0}, en[4] = {0, 0, 0, 0};
      if (ok && !(in && (v.x & v.y & v.z & v.w) == 0xFFFFFFFFu)) runs_of(F.r + r, qa, in, v, pw, nw, st, en);
      visit(ok, f, r, qa, live && f == qbeg, st, en);
      carry = __shfl_sync(0xFFFFFFFFu, v.w, 31);
      carry_ok = true;
    }
  }
}

// Run extraction.  Collect: each warp walks its chunk once, counting run starts and ends
// (separately: a run may start in one chunk and end in a later one) and staging the first
// kRunCap of each, chunk-local and ascending, in scratch, plus the chunk-local start count
// at the first quad of every range that begins in the chunk.  An exclusive scan of the
// chunk counts gives every chunk its global offsets.  Place: each warp copies its staged
// runs to their global positions; only a chunk with more than kRunCap runs walks its
// quads again.  Sparse planes (the usual sync destination) are therefore read once.
// (Measured alternatives on B200: a single-pass decoupled look-back over ticketed chunks
// -- the first wave's look-backs walk back over thousands of aggregates; a count-only
// first pass with a step bitmap and a place pass visiting the marked steps -- the place
// pass then waits on a dependent chain of loads per marked step, 54 us at rho = 2^-16
// against 16 us for copying staged runs; one cooperative kernel with a grid barrier
// between the passes -- no faster than the two launches.)
constexpr uint32_t kRunCap = 4096;
// Places the starts / ends of one warp step at chunk-relative (STAGE) or global positions
// s.., e.. (warp-synchronous; s and e advance by the warp's totals).  STAGE also records,
// at the first flat quad of a range (at_start), the chunk-local start count before it.
template <bool STAGE>
__device__ __forceinline__ void place_step(const Flat& F, uint64_t f, uint32_t r, uint64_t qa, bool at_start,
                                           const uint32_t* st, const uint32_t* en, uint64_t& gs, uint64_t& ge,
                                           uint32_t* out_s, uint32_t* out_e, uint64_t cap, uint32_t* off_local,
                                           uint32_t* wbuf) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t ns = __popc(st[0]) + __popc(st[1]) + __popc(st[2]) + __popc(st[3]);
  const uint32_t ne = __popc(en[0]) + __popc(en[1]) + __popc(en[2]) + __popc(en[3]);
  if (!__any_sync(0xFFFFFFFFu, ns || ne || (STAGE && at_start))) return;  // nothing to place in this step
  uint32_t xs, xe, Ts, Te;  // exclusive positions of the lane's first start / end, step totals
  step_positions(ns, ne, xs, xe, Ts, Te);
  if (STAGE && at_start)  // the first flat quad of range r (and of the empty ranges just before it)
    for (int64_t q = r; q >= 0 && F.qp[q] == f; --q) off_local[q] = (uint32_t)(gs + xs);
  const uint32_t cb = (uint32_t)((qa * 4 - F.r[r].word_off) * 32);  // the lane's first cell
  if (Ts + Te > kDenseStep) {  // staged in shared memory, written with coalesced stores
    if (__all_sync(0xFFFFFFFFu, cb - __shfl_sync(0xFFFFFFFFu, cb, 0) < 4096u)) {  // lanes on consecutive quads
      emit_dense16(st, xs, Ts, cb, gs, out_s, cap, reinterpret_cast<uint16_t*>(wbuf));
      emit_dense16(en, xe, Te, cb, ge, out_e, cap, reinterpret_cast<uint16_t*>(wbuf));
    } else {  // lanes in different ranges (edge steps): u32 entries, in passes
      emit_staged<kRunsBuf>(st, xs, Ts, cb, gs, out_s, cap, wbuf);
      emit_staged<kRunsBuf>(en, xe, Te, cb, ge, out_e, cap, wbuf);
    }
  } else {  // sparse step: each lane writes its few runs
    if (__any_sync(0xFFFFFFFFu, ns != 0u)) emit_sparse(st, gs + xs, cb, out_s, cap);
    if (__any_sync(0xFFFFFFFFu, ne != 0u)) emit_sparse(en, ge + xe, cb, out_e, cap);
  }
  gs += Ts;
  ge += Te;
}

// Collect pass.  Per warp chunk: start / end counts (chunk_s, chunk_e) and staged runs;
// per block: its totals (block_s, block_e).  Every place block scans the block totals
// itself (a few hundred entries), so neither a ticket nor a zeroing memset is needed.  The
// place pass is launched as its programmatic dependent: it may start (and scan the range
// list) while the last collect blocks finish.
struct RunCounts {
  uint64_t *chunk_s, *chunk_e, *block_s, *block_e;
  uint64_t *chunk_xs, *chunk_xe;  // exclusive prefix of the chunk counts inside their block
};

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__global__ void __launch_bounds__(kBT, COH_RUNS_MINB) k_runs_collect(const uint32_t* words, Flat Fg, RunCounts C,
                                                                     uint32_t* stage, uint32_t* off_local) {
  griddep_launch();
  COH_BM_PROLOGUE
  extern __shared__ uint32_t runs_smem[];  // kBT / 32 warps x kRunsBuf: dense run staging
  uint32_t* const wbuf = runs_smem + (threadIdx.x >> 5) * kRunsBuf;
  __shared__ uint64_t ws[2][kBT / 32];
  uint64_t f0, f1, wid;
  warp_chunk(F.qp[F.n], f0, f1, wid);
  uint64_t ls = 0, le = 0;
  if (f0 < f1) {
    uint32_t* const ss = stage + wid * (2 * kRunCap);
    chunk_runs(words, F, f0, f1,
               [&](bool, uint64_t f, uint32_t r, uint64_t qa, bool at_start, const uint32_t* st, const uint32_t* en) {
                 place_step<true>(F, f, r, qa, at_start, st, en, ls, le, ss, ss + kRunCap, kRunCap, off_local, wbuf);
               });
  }
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    C.chunk_s[wid] = ls;
    C.chunk_e[wid] = le;
    ws[0][warp] = ls;
    ws[1][warp] = le;
  }
  __syncthreads();
  if (lane == 0) {  // the chunk's offsets inside the block (the place pass then loads one word)
    uint64_t xs = 0, xe = 0;
    for (uint32_t w = 0; w < warp; ++w) {
      xs += ws[0][w];
      xe += ws[1][w];
    }
    C.chunk_xs[wid] = xs;
    C.chunk_xe[wid] = xe;
    if (warp == kBT / 32 - 1) {
      C.block_s[blockIdx.x] = xs + ls;
      C.block_e[blockIdx.x] = xe + le;
    }
  }
}

// Exclusive scans of a[0..n) and b[0..n) into sa / sb (n + 1 entries, the last = totals),
// one block of kBT threads, n <= kBT * kPer.
constexpr uint32_t kMaxCollectBlocks = 2048;  // count-pass blocks (one wave)
__device__ void block_scan2(const uint64_t* a, const uint64_t* b, uint32_t n, uint64_t* sa, uint64_t* sb) {
  constexpr uint32_t kPer = kMaxCollectBlocks / kBT;
  __shared__ uint64_t wsum[2][kBT / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t va[kPer], vb[kPer], xa = 0, xb = 0;
#pragma unroll
  for (uint32_t j = 0; j < kPer; ++j) {
    const uint32_t i = tid * kPer + j;
    va[j] = i < n ? a[i] : 0;
    vb[j] = i < n ? b[i] : 0;
    xa += va[j];
    xb += vb[j];
  }
  const uint64_t ta = xa, tb = xb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t ya = __shfl_up_sync(0xFFFFFFFFu, xa, o), yb = __shfl_up_sync(0xFFFFFFFFu, xb, o);
    if (lane >= (uint32_t)o) {
      xa += ya;
      xb += yb;
    }
  }
  if (lane == 31) {
    wsum[0][warp] = xa;
    wsum[1][warp] = xb;
  }
  __syncthreads();
  uint64_t ea = xa - ta, eb = xb - tb;
  for (uint32_t w = 0; w < warp; ++w) {
    ea += wsum[0][w];
    eb += wsum[1][w];
  }
#pragma unroll
  for (uint32_t j = 0; j < kPer; ++j) {
    const uint32_t i = tid * kPer + j;
    if (i <= n) {
      sa[i] = ea;
      sb[i] = eb;
    }
    ea += va[j];
    eb += vb[j];
  }
  __syncthreads();
}

// global start / end offsets of warp chunk wid (bs / be: exclusive scans of the block totals)
__device__ __forceinline__ void chunk_offsets(const RunCounts& C, const uint64_t* bs, const uint64_t* be, uint64_t wid,
                                              uint64_t& gs, uint64_t& ge) {
  const uint64_t blk = wid / (kBT / 32);
  gs = bs[blk] + __ldcg(C.chunk_xs + wid);
  ge = be[blk] + __ldcg(C.chunk_xe + wid);
}

// One warp copies n staged entries to out[at ..) (clipped at cap): eight independent L2
// loads in flight per lane, coalesced stores (a chunk stages up to kRunCap entries; one
// load at a time left the copy latency-bound at 1.8 TB/s).
__device__ __forceinline__ void copy_staged(const uint32_t* src, uint32_t n, uint32_t* out, uint64_t at, uint64_t cap) {
  if (at >= cap) return;
  const uint32_t m = (uint64_t)n < cap - at ? n : (uint32_t)(cap - at);
  uint32_t* const dst = out + at;
  uint32_t i = threadIdx.x & 31;
  for (; i + 224u < m; i += 256u) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(src + i + 32u * k);
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[i + 32u * k] = v[k];
  }
  for (; i < m; i += 32u) dst[i] = __ldcg(src + i);
}

// Place pass, plus run_off[i] = global index of range i's first run: its chunk's offset +
// the chunk-local count staged by the collect pass; ranges starting at the end get the
// total.  Dynamic shared memory: kBT / 32 warps x kRunsBuf (dense run staging), then the
// exclusive scans of the collect blocks' totals (gridDim.x + 1 each).
__global__ void __launch_bounds__(kBT, COH_RUNS_MINB) k_runs_place(const uint32_t* words, Flat Fg, RunCounts C,
                                                                   const uint32_t* stage, const uint32_t* off_local,
                                                                   uint32_t* run_start, uint32_t* run_end, uint64_t cap,
                                                                   uint64_t* run_off) {
  COH_BM_PROLOGUE  // the range list is an input of both passes: scanned before the wait
  griddep_wait();  // the collect pass is complete and its writes are visible
  extern __shared__ __align__(16) uint32_t runs_smem[];
  uint32_t* const wbuf = runs_smem + (threadIdx.x >> 5) * kRunsBuf;
  uint64_t* const bs = reinterpret_cast<uint64_t*>(runs_smem + (kBT / 32) * kRunsBuf);
  uint64_t* const be = bs + gridDim.x + 1;
  const uint64_t Q = F.qp[F.n], n_chunks = (uint64_t)gridDim.x * (kBT / 32);
  uint64_t f0, f1, wid;
  warp_chunk(Q, f0, f1, wid);
  // this warp's chunk words, loaded ahead of the block scan (independent of it)
  const uint64_t cs = __ldcg(C.chunk_s + wid), ce = __ldcg(C.chunk_e + wid);
  const uint64_t xs = __ldcg(C.chunk_xs + wid), xe = __ldcg(C.chunk_xe + wid);
  block_scan2(C.block_s, C.block_e, gridDim.x, bs, be);
  const uint64_t cper = (((Q + n_chunks - 1) / n_chunks) + 31) & ~31ull;  // as warp_chunk
  for (uint64_t i = (uint64_t)blockIdx.x * kBT + threadIdx.x; i <= F.n; i += (uint64_t)gridDim.x * kBT) {
    const uint64_t f = F.qp[i];
    uint64_t gs = bs[gridDim.x], ge;
    if (f < Q) {
      chunk_offsets(C, bs, be, f / cper, gs, ge);
      gs += off_local[i];
    }
    run_off[i] = gs;
  }
  if (f0 >= f1) return;
  const uint64_t blk = wid / (kBT / 32);
  uint64_t gs = bs[blk] + xs, ge = be[blk] + xe;
  if (cs <= kRunCap && ce <= kRunCap) {  // staged by the collect pass: copy
    const uint32_t* const ss = stage + wid * (2 * kRunCap);
    copy_staged(ss, (uint32_t)cs, run_start, gs, cap);
    copy_staged(ss + kRunCap, (uint32_t)ce, run_end, ge, cap);
    return;
  }
  chunk_runs(words, F, f0, f1,
             [&](bool, uint64_t f, uint32_t r, uint64_t qa, bool at_start, const uint32_t* st, const uint32_t* en) {
               place_step<false>(F, f, r, qa, at_start, st, en, gs, ge, run_start, run_end, cap, nullptr, wbuf);
             });
}

struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

int grid_for(coh_ctx* ctx) { return ctx->sms * 8; }

int fail(coh_ctx* ctx, const char* what, cudaError_t e) {
  ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
  return COH_E_CUDA;
}

int check(coh_ctx* ctx, const char* what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? COH_OK : fail(ctx, what, e);
}

}  // namespace

cudaError_t runs_ctx_init(int sms, int* grid) {
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_runs_collect, kBT, kRunsSmem);
  if (e != cudaSuccess) return e;
  const int g = sms * (occ > 0 ? occ : 1);
  if (g > (int)kMaxCollectBlocks) return cudaErrorInvalidConfiguration;
  if ((e = cudaFuncSetAttribute(k_runs_collect, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRunsSmem)) !=
      cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_runs_place, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kRunsSmem + sizeof(uint64_t) * 2 * ((size_t)g + 1)))) != cudaSuccess)
    return e;
  *grid = g;
  return cudaSuccess;
}

}  // namespace cohb

using namespace cohb;

// flat quad prefix of the ranges, in stream-ordered scratch
#define COH_BM_FLAT(ctx, d_r, n, s)                                                             \
  Scratch pre_;                                                                               \
  pre_.s = s;                                                                                 \
  if (n > kFusedRanges) { /* else each block scans the ranges itself (shared_prefix) */        \
    const cudaError_t e_ = cudaMallocAsync(&pre_.p, sizeof(uint64_t) * ((size_t)n + 1), s);   \
    if (e_ != cudaSuccess) return fail(ctx, "bitmap scratch", e_);                           \
    k_quad_prefix<<<1, 1024, 0, s>>>(d_r, n, static_cast<uint64_t*>(pre_.p));                 \
    ctx->launches++;                                                                          \
  }                                                                                           \
  const Flat F{d_r, static_cast<uint64_t*>(pre_.p), n};

static int range_fill(coh_ctx* ctx, uint32_t* d_words, const coh_bitmap_range* d_r, uint32_t n, bool set, void* stream) {
  if (!ctx || (n && (!d_words || !d_r))) return COH_E_ARG;
  if (!n) return COH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  COH_BM_FLAT(ctx, d_r, n, s)
  if (set) k_range_set<true><<<grid_for(ctx), kBT, 0, s>>>(d_words, F);
  else k_range_set<false><<<grid_for(ctx), kBT, 0, s>>>(d_words, F);
  ctx->launches++;
  return check(ctx, "range set/clear");
}

extern "C" int coh_bitmap_range_set(coh_ctx* ctx, uint32_t* d_words, const coh_bitmap_range* d_ranges, uint32_t n,
                                    void* stream) {
  return range_fill(ctx, d_words, d_ranges, n, true, stream);
}

extern "C" int coh_bitmap_range_clear(coh_ctx* ctx, uint32_t* d_words, const coh_bitmap_range* d_ranges, uint32_t n,
                                      void* stream) {
  return range_fill(ctx, d_words, d_ranges, n, false, stream);
}

extern "C" int coh_bitmap_first_zero(coh_ctx* ctx, const uint32_t* d_words, const coh_bitmap_range* d_ranges, uint32_t n,
                                     uint32_t* d_first, void* stream) {
  if (!ctx || (n && (!d_words || !d_ranges || !d_first))) return COH_E_ARG;
  if (!n) return COH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_first, 0xFF, sizeof(uint32_t) * n, s);
  if (e != cudaSuccess) return fail(ctx, "first_zero init", e);
  COH_BM_FLAT(ctx, d_ranges, n, s)
  k_first_zero<<<grid_for(ctx), kBT, 0, s>>>(d_words, F, d_first);
  ctx->launches++;
  return check(ctx, "first_zero");
}

extern "C" int coh_bitmap_view_check(coh_ctx* ctx, const uint32_t* d_L, const uint32_t* d_R,
                                     const coh_bitmap_range* d_ranges, const uint8_t* d_abs_pair, uint32_t n,
                                     uint8_t* d_ok, void* stream) {
  if (!ctx || (n && (!d_L || !d_R || !d_ranges || !d_abs_pair || !d_ok))) return COH_E_ARG;
  if (!n) return COH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch fl;
  fl.s = s;
  cudaError_t e = cudaMallocAsync(&fl.p, sizeof(uint32_t) * n, s);
  if (e != cudaSuccess) return fail(ctx, "view_check scratch", e);
  if ((e = cudaMemsetAsync(fl.p, 0, sizeof(uint32_t) * n, s)) != cudaSuccess) return fail(ctx, "view_check init", e);
  COH_BM_FLAT(ctx, d_ranges, n, s)
  k_view_flags<<<grid_for(ctx), kBT, 0, s>>>(d_L, d_R, F, static_cast<uint32_t*>(fl.p));
  k_view_finish<<<(n + 255) / 256, 256, 0, s>>>(static_cast<uint32_t*>(fl.p), d_abs_pair, n, d_ok);
  ctx->launches += 2;
  return check(ctx, "view_check");
}

extern "C" int coh_bitmap_extract_zero_runs(coh_ctx* ctx, const uint32_t* d_words, const coh_bitmap_range* d_ranges,
                                            uint32_t n, uint32_t* d_run_start, uint32_t* d_run_end, uint64_t cap,
                                            uint64_t* d_run_off, void* stream) {
  if (!ctx || (n && (!d_words || !d_ranges || !d_run_off || (cap && (!d_run_start || !d_run_end))))) return COH_E_ARG;
  if (!n) return COH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  COH_BM_FLAT(ctx, d_ranges, n, s)
  // one wave of the collect pass (the place pass reuses its warp -> chunk mapping); grid and
  // shared-memory attributes are set up once per context (runs_ctx_init)
  const int grid = ctx->runs_grid;
  if (grid <= 0 || grid > (int)kMaxCollectBlocks) return fail(ctx, "zero_runs grid", cudaErrorInvalidConfiguration);
  const uint64_t n_chunks = (uint64_t)grid * (kBT / 32);
  // scratch: run counts (see RunCounts, all written by the collect pass), staged runs,
  // chunk-local range offsets
  const size_t counts_b = (sizeof(uint64_t) * (4 * n_chunks + 2 * (size_t)grid) + 255u) & ~(size_t)255u;  // stage: whole lines
  const size_t stage_b = sizeof(uint32_t) * 2 * kRunCap * n_chunks;
  Scratch co;
  co.s = s;
  cudaError_t e = cudaMallocAsync(&co.p, counts_b + stage_b + sizeof(uint32_t) * ((size_t)n + 1), s);
  if (e != cudaSuccess) return fail(ctx, "zero_runs scratch", e);
  RunCounts C;
  C.chunk_s = static_cast<uint64_t*>(co.p);
  C.chunk_e = C.chunk_s + n_chunks;
  C.block_s = C.chunk_e + n_chunks;
  C.block_e = C.block_s + grid;
  C.chunk_xs = C.block_e + grid;
  C.chunk_xe = C.chunk_xs + n_chunks;
  uint32_t* stage = reinterpret_cast<uint32_t*>(static_cast<char*>(co.p) + counts_b);
  uint32_t* off_local = stage + 2 * kRunCap * n_chunks;
  const size_t place_smem = kRunsSmem + sizeof(uint64_t) * 2 * ((size_t)grid + 1);
  k_runs_collect<<<grid, kBT, kRunsSmem, s>>>(d_words, F, C, stage, off_local);
  {  // the place pass as the collect pass's programmatic dependent
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBT);
    cfg.dynamicSmemBytes = place_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const Flat Fc = F;
    const uint32_t* stage_c = stage;
    const uint32_t* off_c = off_local;
    e = cudaLaunchKernelEx(&cfg, k_runs_place, d_words, Fc, C, stage_c, off_c, d_run_start, d_run_end, cap, d_run_off);
    if (e != cudaSuccess) return fail(ctx, "zero_runs place launch", e);
  }
  ctx->launches += 2;
  return check(ctx, "zero_runs");
}
