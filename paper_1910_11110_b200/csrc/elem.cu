// Element-granular path, device side: validity bit planes (L = local valid, R = remote
// valid; bit i of word i/32) for many buffers, executed stage by stage (op k of every
// buffer in stage k).  Per stage:
//   pass1  one CTA per 64 Ki-cell tile: SYNC -> first zero of the source plane
//          (stuck cell) + zero-run starts/ends/zeros of the destination; READ -> first
//          zero; WRITE -> applied directly (cannot fail); CHECK -> per-view
//          all-ones / all-zero flags (abstraction_correct, modes.hpp:79-90)
//   decide one thread per buffer: stuck (whole-view sync is atomic, semantics.hpp:
//          155-166: nothing is written when any cell fails), run offsets (exclusive
//          scan over the op's tiles), boundary bit
//   apply  SYNC tiles that passed: write the transfer ranges (maximal runs of cells the
//          sync changes, ascending) and set the destination plane
// Words move as 128-bit loads (8 consecutive words per thread), warp/block reductions
// via shuffles; every kernel is HBM-streaming.
#include <cuda_runtime.h>

#include <string>

#include "elem.hpp"
#include "gen_common.h"
#include "internal.hpp"
#include "runs_emit.cuh"

namespace cohb {

constexpr int kET = 256;                   // threads per tile CTA
constexpr int kWPT = kElemTileWords / kET; // 8 words per thread
static_assert(kWPT == 8, "8 words per thread");


// Programmatic dependent launch: a stage kernel may be scheduled while its predecessor
// drains; it reads only host-built descriptors before waiting for the predecessor's
// results (griddepcontrol.wait = cudaGridDependencySynchronize) and lets its own successor
// launch early.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ uint32_t word_mask(uint32_t w, uint32_t lo, uint32_t hi) {
  const uint32_t wl = lo >> 5, wh = hi >> 5;
  if (w < wl || w > wh) return 0u;
  uint32_t m = 0xFFFFFFFFu;
  if (w == wl) m &= 0xFFFFFFFFu << (lo & 31u);
  if (w == wh) m &= 0xFFFFFFFFu >> (31u - (hi & 31u));
  return m;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = 0;
#pragma unroll
  for (int k = 0; k < kET / 32; ++k) s += red[k];
  return s;
}

__device__ __forceinline__ uint32_t block_or(uint32_t v, uint32_t* red) {
  v = __reduce_or_sync(0xffffffffu, v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kET / 32; ++k) s |= red[k];
  return s;
}

__device__ __forceinline__ uint32_t block_min(uint32_t v, uint32_t* red) {
  v = __reduce_min_sync(0xffffffffu, v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  uint32_t s = 0xFFFFFFFFu;
#pragma unroll
  for (int k = 0; k < kET / 32; ++k) s = min(s, red[k]);
  return s;
}

// Exclusive block scan of per-thread counts; returns this thread's prefix.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = x;
  __syncthreads();
  uint32_t base = 0;
  for (int k = 0; k < warp; ++k) base += red[k];
  return base + x - v;
}

__device__ __forceinline__ void load8(const uint32_t* p, uint32_t (&w)[kWPT]) {
  const uint4 a = __ldcg(reinterpret_cast<const uint4*>(p));
  const uint4 b = __ldcg(reinterpret_cast<const uint4*>(p) + 1);
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
  w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}
__device__ __forceinline__ void store8(uint32_t* p, const uint32_t (&w)[kWPT]) {
  reinterpret_cast<uint4*>(p)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  reinterpret_cast<uint4*>(p)[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// Zero-run starts / ends of z (zeros of the destination inside the range) for this
// thread's 8 words, given the neighbouring bits.
__device__ __forceinline__ void run_edges(const uint32_t (&z)[kWPT], uint32_t prev_top, uint32_t next_bot,
                                          uint32_t (&st)[kWPT], uint32_t (&en)[kWPT]) {
#pragma unroll
  for (int k = 0; k < kWPT; ++k) {
    const uint32_t pt = k ? (z[k - 1] >> 31) : prev_top;
    const uint32_t nb = k < kWPT - 1 ? (z[k + 1] & 1u) : next_bot;
    st[k] = z[k] & ~((z[k] << 1) | pt);
    en[k] = z[k] & ~((z[k] >> 1) | (nb << 31));
  }
}

// A tile is "full" when every word of its aligned 2048-word block lies strictly inside
// the op range: then every mask is all-ones and the per-word mask work disappears
// (uniform per CTA, so no divergence).
__device__ __forceinline__ bool tile_full(uint32_t tstart, uint32_t lo, uint32_t hi) {
  return tstart * 32u >= lo && (tstart + kElemTileWords) * 32u - 1u <= hi;
}

__device__ __forceinline__ void masks8(uint32_t base, uint32_t lo, uint32_t hi, bool full, uint32_t (&m)[kWPT]) {
#pragma unroll
  for (int k = 0; k < kWPT; ++k) m[k] = full ? 0xFFFFFFFFu : word_mask(base + k, lo, hi);
}

__device__ __forceinline__ void store8_const(uint32_t* p, uint32_t v) {
  const uint4 q = make_uint4(v, v, v, v);
  __stcg(reinterpret_cast<uint4*>(p), q);
  __stcg(reinterpret_cast<uint4*>(p) + 1, q);
}

__global__ void __launch_bounds__(kET, 8) k_elem_pass1(const ElemDev d) {
  __shared__ uint32_t red[kET / 32];
  __shared__ uint32_t s_first[kET], s_last[kET];
  __shared__ uint32_t s_next;
  const ElemTile tile = d.tiles[blockIdx.x];
  griddep_wait();
  griddep_launch();
  const uint32_t b = tile.b;
  uint32_t* Lp = d.planes + (size_t)b * 2u * d.W;
  uint32_t* Rp = Lp + d.W;
  const uint32_t tstart = tile.tstart;
  const uint32_t base = tstart + threadIdx.x * kWPT;
  const int tloc = (int)(blockIdx.x);  // index of this tile within the stage
  const uint32_t lane = threadIdx.x & 31;
  struct {
    uint8_t type, plane;
  } op{tile.type, tile.plane};
  if (op.type == EOP_CHECK) {
    // abstraction_correct for one view over this tile: which of "some L=0", "some R=0",
    // "some L|R=1" occur.  Violations are rare: warp OR, atomic only when non-zero.
    // (Loads are issued before the dead-flag check: reads are harmless.)
    const uint32_t lo = tile.lo, hi = tile.hi, a = tile.apair;
    uint32_t l[kWPT], r[kWPT], m[kWPT];
    if (a != 2u) load8(Lp + base, l);   // (I,V) needs only R
    if (a != 1u) load8(Rp + base, r);   // (V,I) needs only L
    masks8(base, lo, hi, tile_full(tstart, lo, hi), m);
    uint32_t f = 0;
    if (tile_full(tstart, lo, hi)) {  // interior tile: AND / OR reductions, no per-word masks
      uint32_t al = 0xFFFFFFFFu, ar = 0xFFFFFFFFu, o = 0u;
#pragma unroll
      for (int k = 0; k < kWPT; ++k) {
        if (a != 2u) al &= l[k];
        if (a != 1u) ar &= r[k];
        if (a == 0u) o |= l[k] | r[k];
      }
      f = (a != 2u && al != 0xFFFFFFFFu ? 1u : 0u) | (a != 1u && ar != 0xFFFFFFFFu ? 2u : 0u) | (o ? 4u : 0u);
    } else {
#pragma unroll
      for (int k = 0; k < kWPT; ++k) {
        if (a != 2u && (~l[k] & m[k])) f |= 1u;
        if (a != 1u && (~r[k] & m[k])) f |= 2u;
        if (a == 0u && ((l[k] | r[k]) & m[k])) f |= 4u;
      }
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0 && f && !d.st[b].dead) atomicOr(&d.sc[b * kSlots + tile.slot].view_flags[tile.view], f);
    return;
  }
  const uint32_t lo = tile.lo, hi = tile.hi;
  const bool full = tile_full(tstart, lo, hi);
  uint32_t m[kWPT];
  masks8(base, lo, hi, full, m);
  // SYNC / READ: first zero of the required (source) plane; rare -> warp min + atomic
  const uint32_t* src = op.plane ? Rp : Lp;
  uint32_t v[kWPT];
  load8(src + base, v);
  uint32_t fz = kNoCell;
  uint32_t all = 0xFFFFFFFFu;
#pragma unroll
  for (int k = 0; k < kWPT; ++k) all &= v[k] | ~m[k];
  if (all != 0xFFFFFFFFu) {  // some required bit is 0 here: locate the first one
#pragma unroll
    for (int k = kWPT - 1; k >= 0; --k) {
      const uint32_t z = ~v[k] & m[k];
      if (z) fz = (base + k) * 32u + (__ffs(z) - 1);
    }
  }
  fz = __reduce_min_sync(0xffffffffu, fz);
  if (lane == 0 && fz != kNoCell) atomicMin(&d.sc[b * kSlots + tile.slot].first_zero, fz);  // ignored if dead
  if (op.type != EOP_SYNC) return;
  // destination zero runs: counts for the offsets, and the tile's edge bits
  const uint32_t* dst = op.plane ? Lp : Rp;
  uint32_t z[kWPT], sts[kWPT], ens[kWPT];
  load8(dst + base, v);
#pragma unroll
  for (int k = 0; k < kWPT; ++k) z[k] = ~v[k] & m[k];
  s_first[threadIdx.x] = z[0];
  s_last[threadIdx.x] = z[kWPT - 1];
  uint32_t edge_prev = 0;
  if (threadIdx.x == 0 && tstart > 0) {
    const uint32_t w = tstart - 1;
    edge_prev = (~dst[w] & word_mask(w, lo, hi)) >> 31;
  }
  if (threadIdx.x == kET - 1) {
    uint32_t edge_next = 0;
    if (tstart + kElemTileWords < d.W) {
      const uint32_t w = tstart + kElemTileWords;
      edge_next = ~dst[w] & word_mask(w, lo, hi) & 1u;
    }
    s_next = edge_next;
  }
  __syncthreads();
  const uint32_t pt = threadIdx.x ? (s_last[threadIdx.x - 1] >> 31) : edge_prev;
  const uint32_t nb = threadIdx.x < kET - 1 ? (s_first[threadIdx.x + 1] & 1u) : s_next;
  uint32_t ns = 0, ne = 0, nz = 0;
  uint32_t zor = 0u, zand = 0xFFFFFFFFu;
#pragma unroll
  for (int k = 0; k < kWPT; ++k) {
    zor |= z[k];
    zand &= z[k];
  }
  if (zor == 0u) {
    // destination already valid on these 8 words: no changed cells, no run edges
  } else if (zand == 0xFFFFFFFFu) {
    // all 256 cells change: a run can only start at the first bit / end at the last
    nz = 32u * kWPT;
    ns = pt ? 0u : 1u;
    ne = nb ? 0u : 1u;
  } else {
    run_edges(z, pt, nb, sts, ens);
#pragma unroll
    for (int k = 0; k < kWPT; ++k) {
      ns += __popc(sts[k]);
      ne += __popc(ens[k]);
      nz += __popc(z[k]);
    }
  }
  const uint32_t my_s = ns, my_e = ne;
  ns = block_sum(ns, red);
  ne = block_sum(ne, red);
  nz = block_sum(nz, red);
  if (threadIdx.x == 0)
    *reinterpret_cast<uint4*>(d.tcnt + 4 * tloc) = make_uint4(ns, ne, nz, edge_prev | (s_next << 1));
  // Sparse tiles stage their run cells (tile-local order = ascending) so that apply can
  // write the destination without reading it again (block-uniform condition).
  if (d.stage_runs && (ns | ne) && ns <= kStageRuns && ne <= kStageRuns) {
    uint32_t os = block_excl_scan(my_s, red);
    uint32_t oe = block_excl_scan(my_e, red);
    uint32_t* const stg = d.stage_runs + (size_t)tloc * 2u * kStageRuns;
    if (zand == 0xFFFFFFFFu) {  // all 256 cells change: only the first / last cell can be edges
      if (my_s) stg[os] = base * 32u;
      if (my_e) stg[kStageRuns + oe] = (base + kWPT) * 32u - 1u;
    } else if (zor != 0u) {
      run_edges(z, pt, nb, sts, ens);  // recomputed: keeps them dead across the block sums
#pragma unroll
      for (int k = 0; k < kWPT; ++k) {
        for (uint32_t x = sts[k]; x; x &= x - 1) stg[os++] = (base + k) * 32u + (__ffs(x) - 1);
        for (uint32_t x = ens[k]; x; x &= x - 1) stg[kStageRuns + oe++] = (base + k) * 32u + (__ffs(x) - 1);
      }
    }
  }
}

// One warp per buffer: walks the buffer's ops of this stage in program order — stuck
// detection (the first stuck op stops the buffer; a whole-view sync is atomic), run-offset
// scan over a SYNC's tiles (shuffle scan, loads issued in batches), boundary bits — and
// resets the scratch.
constexpr int kDecideWarps = 4;
__global__ void __launch_bounds__(32 * kDecideWarps) k_elem_decide(const ElemDev d) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t b = blockIdx.x * kDecideWarps + (threadIdx.x >> 5);
  griddep_wait();
  griddep_launch();
  if (b >= d.n_progs) return;
  ElemState* __restrict__ st = d.st + b;
  uint32_t dead = st->dead;
  for (uint32_t slot = 0; slot < kSlots; ++slot) {
    const ElemOp op = d.ops[b * kSlots + slot];
    if (op.type == EOP_NONE) break;
    ElemScratch* __restrict__ sc = d.sc + b * kSlots + slot;
    const uint32_t fz0 = sc->first_zero;
    const uint32_t vf = lane < COH_MAX_VIEWS ? sc->view_flags[lane] : 0u;
    __syncwarp();
    if (lane == 0) sc->first_zero = kNoCell;
    if (lane < COH_MAX_VIEWS) sc->view_flags[lane] = 0;
    if (dead) continue;  // keep resetting the scratch of the remaining slots
    if (op.type == EOP_SYNC || op.type == EOP_READ) {
      if (fz0 != kNoCell) {
        if (lane == 0) {
          const uint32_t* Lp = d.planes + (size_t)b * 2u * d.W;
          const uint32_t* Rp = Lp + d.W;
          st->dead = 1;
          st->stuck_op = d.stage * kSlots + slot;
          st->stuck_cell = fz0;
          st->stuck_pair = ((Lp[fz0 >> 5] >> (fz0 & 31u)) & 1u) | (((Rp[fz0 >> 5] >> (fz0 & 31u)) & 1u) << 1);
        }
        dead = 1;
      } else if (op.type == EOP_SYNC) {
        const uint32_t t0 = op.tile0;  // stage-local tile index
        const uint32_t n_t = ((op.hi >> 5) / kElemTileWords) - ((op.lo >> 5) / kElemTileWords) + 1;
        const unsigned long long run0 = st->n_runs;
        unsigned long long cs = 0, ce = 0, zeros = 0;
        for (uint32_t k0 = 0; k0 < n_t; k0 += 32 * 8) {
          uint4 c[8];  // issue every load of the batch before the dependent scan
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t k = k0 + 32u * j + lane;
            c[j] = k < n_t ? __ldg(reinterpret_cast<const uint4*>(d.tcnt) + (t0 + k)) : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t k = k0 + 32u * j + lane;
            const uint32_t ns = c[j].x, ne = c[j].y;
            uint32_t xs = ns, xe = ne;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t ys = __shfl_up_sync(0xffffffffu, xs, o), ye = __shfl_up_sync(0xffffffffu, xe, o);
              if (lane >= (uint32_t)o) {
                xs += ys;
                xe += ye;
              }
            }
            if (k < n_t) {
              d.tbase[2 * (t0 + k)] = run0 + cs + xs - ns;
              d.tbase[2 * (t0 + k) + 1] = run0 + ce + xe - ne;
            }
            cs += __shfl_sync(0xffffffffu, xs, 31);
            ce += __shfl_sync(0xffffffffu, xe, 31);
            zeros += __reduce_add_sync(0xffffffffu, c[j].z);
          }
        }
        if (lane == 0) {
          st->n_runs = run0 + cs;
          st->transfers += 1;
          st->transfer_cells += zeros;
        }
      }
    } else if (op.type == EOP_CHECK) {
      bool okv = true;
      if (lane < op.plane) {
        const uint32_t a = (op.lo >> (2 * lane)) & 3u, f = vf;
        // leq(a, cell) for every cell of the view:
        // (V,I): L all 1; (I,V): R all 1; (V,V): both; (I,I): L|R all 0
        okv = a == 1u ? !(f & 1u) : a == 2u ? !(f & 2u) : a == 3u ? !(f & 3u) : !(f & 4u);
      }
      const bool ok = __all_sync(0xffffffffu, okv);
      if (lane == 0) {
        st->calls_done += 1;
        if (!ok) st->violations += 1;
        else if (d.boundary) d.boundary[(size_t)b * d.bwords + op.call / 32] |= 1u << (op.call % 32);
      }
    }
    __syncwarp();
  }
}

// Warp-per-tile over this stage's SYNC tiles (self-contained descriptors): each warp loads
// its descriptor, then the two device-side inputs together (stuck flag, run counts).
// Tiles without run edges (almost all) are a coalesced read-modify-write or, when the
// tile lies inside the range, a pure store of ones; edge tiles emit their transfer runs
// with a warp scan (lane l owns words [64 l, 64 l + 63] of the tile).
constexpr int kApplyWarps = 8;
constexpr int kApplyU = 4;  // warp steps of an edge tile loaded together
constexpr int kWPL = kElemTileWords / 32;  // 64 words per lane
__global__ void __launch_bounds__(32 * kApplyWarps, 3) k_elem_apply(const ElemDev d, uint32_t n_sync_tiles) {
  extern __shared__ uint16_t apply_smem[];  // kApplyWarps x kStageBuf16: dense run staging
  const uint32_t lane = threadIdx.x & 31;
  uint16_t* const wbuf = apply_smem + (threadIdx.x >> 5) * kStageBuf16;
  const uint32_t gw = blockIdx.x * kApplyWarps + (threadIdx.x >> 5), nw = gridDim.x * kApplyWarps;
  // descriptors are host-built: the first one loads while the predecessor drains
  ElemTile next = gw < n_sync_tiles ? d.sync_desc[gw] : ElemTile{};
  griddep_wait();
  griddep_launch();
  for (uint32_t it = gw; it < n_sync_tiles; it += nw) {
    const ElemTile tile = next;
    if (it + nw < n_sync_tiles) next = d.sync_desc[it + nw];
    const uint32_t b = tile.b, tloc = tile.tloc;
    const uint32_t dead = d.st[b].dead;
    const uint4 cnt = tile.type == EOP_SYNC ? *reinterpret_cast<const uint4*>(d.tcnt + 4 * tloc) : make_uint4(0u, 0u, 0u, 0u);
    if (dead) continue;  // warp-uniform (also set by an earlier op of this stage)
    uint32_t* Lp = d.planes + (size_t)b * 2u * d.W;
    if (tile.type == EOP_WRITE) {  // w x[i] @site over the range: set one plane, clear the other
      uint4* sp4 = reinterpret_cast<uint4*>((tile.plane ? Lp + d.W : Lp) + tile.tstart);
      uint4* cp4 = reinterpret_cast<uint4*>((tile.plane ? Lp : Lp + d.W) + tile.tstart);
      if (tile_full(tile.tstart, tile.lo, tile.hi)) {
#pragma unroll
        for (int j = 0; j < kElemTileWords / 128; ++j) {
          __stcg(sp4 + lane + 32 * j, make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu));
          __stcg(cp4 + lane + 32 * j, make_uint4(0u, 0u, 0u, 0u));
        }
      } else {
        for (int j = 0; j < kElemTileWords / 128; ++j) {
          const uint32_t w = tile.tstart + 4u * (lane + 32u * j);
          const uint32_t m0 = word_mask(w, tile.lo, tile.hi), m1 = word_mask(w + 1, tile.lo, tile.hi),
                         m2 = word_mask(w + 2, tile.lo, tile.hi), m3 = word_mask(w + 3, tile.lo, tile.hi);
          if ((m0 | m1 | m2 | m3) == 0u) continue;
          uint4 a = __ldcg(sp4 + lane + 32 * j), c = __ldcg(cp4 + lane + 32 * j);
          a.x |= m0; a.y |= m1; a.z |= m2; a.w |= m3;
          c.x &= ~m0; c.y &= ~m1; c.z &= ~m2; c.w &= ~m3;
          __stcg(sp4 + lane + 32 * j, a);
          __stcg(cp4 + lane + 32 * j, c);
        }
      }
      continue;
    }
    uint32_t* dst = tile.plane ? Lp : Lp + d.W;
    const uint32_t tstart = tile.tstart;
    const bool full = tile_full(tstart, tile.lo, tile.hi);
    uint4* dst4 = reinterpret_cast<uint4*>(dst + tstart);
    if (!(d.runs_cap && (cnt.x | cnt.y))) {
      // no runs to emit: dst |= mask over the tile, 512 contiguous bytes per instruction
      if (full) {
#pragma unroll
        for (int j = 0; j < kElemTileWords / 128; ++j)
          __stcg(dst4 + lane + 32 * j, make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu));
      } else {
        for (int j = 0; j < kElemTileWords / 128; ++j) {
          const uint32_t w = tstart + 4u * (lane + 32u * j);
          uint4 q = __ldcg(dst4 + lane + 32 * j);
          q.x |= word_mask(w, tile.lo, tile.hi);
          q.y |= word_mask(w + 1, tile.lo, tile.hi);
          q.z |= word_mask(w + 2, tile.lo, tile.hi);
          q.w |= word_mask(w + 3, tile.lo, tile.hi);
          __stcg(dst4 + lane + 32 * j, q);
        }
      }
      continue;
    }
    if (full && cnt.x <= kStageRuns && cnt.y <= kStageRuns) {
      // sparse interior tile: pass1 staged its runs; the destination becomes all ones
      // without being read again
#pragma unroll
      for (int j = 0; j < kElemTileWords / 128; ++j)
        __stcg(dst4 + lane + 32 * j, make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu));
      const uint32_t* stg = d.stage_runs + (size_t)tloc * 2u * kStageRuns;
      const uint64_t gs = d.tbase[2 * tloc], ge = d.tbase[2 * tloc + 1];
      const size_t arena = (size_t)b * d.runs_cap;
      for (uint32_t k = lane; k < cnt.x; k += 32)
        if (gs + k < d.runs_cap) d.runs_lo[arena + gs + k] = __ldcg(stg + k);
      for (uint32_t k = lane; k < cnt.y; k += 32)
        if (ge + k < d.runs_cap) d.runs_hi[arena + ge + k] = __ldcg(stg + kStageRuns + k);
      continue;
    }
    // edge tile: 16 warp steps of 32 quads (lane l on quad l: 512 contiguous bytes), kApplyU
    // steps loaded together.  Run starts / ends come from each quad and its neighbour words
    // (adjacent lanes by shuffle; across steps the carried last word; outside the tile the
    // edge bits pass1 read before anything was written), are placed by a warp scan
    // (sparse: each lane writes its few; dense: coalesced cooperative stores), and the
    // destination quad is written back with the range bits set.
    uint64_t gs = d.tbase[2 * tloc], ge = d.tbase[2 * tloc + 1];
    uint32_t* const out_s = d.runs_lo + (size_t)b * d.runs_cap;
    uint32_t* const out_e = d.runs_hi + (size_t)b * d.runs_cap;
    uint32_t carry = (cnt.w & 1u) << 31;  // z of the cell before the tile, as a word's top bit
    for (uint32_t s0 = 0; s0 < kElemTileWords / 128; s0 += kApplyU) {
      uint4 v[kApplyU];
#pragma unroll
      for (int u = 0; u < kApplyU; ++u) v[u] = __ldcg(dst4 + 32 * (s0 + u) + lane);
      // lane 31's successor word for the batch's last step: the next batch's first word, or
      // the cell after the tile (pass1's edge bit)
      const uint32_t wn = tstart + 128u * (s0 + kApplyU);
      const uint32_t z_after = s0 + kApplyU < kElemTileWords / 128
                                   ? ~__ldcg(dst + wn) & (full ? 0xFFFFFFFFu : word_mask(wn, tile.lo, tile.hi))
                                   : (cnt.w >> 1) & 1u;
#pragma unroll
      for (int u = 0; u < kApplyU; ++u) {
        const uint32_t w0 = tstart + 4u * (32u * (s0 + u) + lane);
        uint32_t m[4], z[4];
        const uint32_t vv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          m[k] = full ? 0xFFFFFFFFu : word_mask(w0 + k, tile.lo, tile.hi);
          z[k] = ~vv[k] & m[k];
        }
        uint32_t zp = __shfl_up_sync(0xffffffffu, z[3], 1);
        uint32_t zn = __shfl_down_sync(0xffffffffu, z[0], 1);
        // lane 0's first word of the next step (all lanes shuffle; lane 31 uses it)
        const uint32_t nx = __shfl_sync(0xffffffffu, v[u + 1 < kApplyU ? u + 1 : u].x, 0);
        if (lane == 0) zp = carry;
        if (lane == 31)
          zn = u + 1 < kApplyU ? ~nx & (full ? 0xFFFFFFFFu : word_mask(w0 + 4u, tile.lo, tile.hi)) : z_after;
        uint32_t st[4], en[4], ns = 0, ne = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t prev = k ? z[k - 1] : zp, next = k < 3 ? z[k + 1] : zn;
          st[k] = z[k] & ~((z[k] << 1) | (prev >> 31));
          en[k] = z[k] & ~((z[k] >> 1) | (next << 31));
          ns += __popc(st[k]);
          ne += __popc(en[k]);
        }
        if (__any_sync(0xffffffffu, ns | ne)) {
          uint32_t xs, xe, Ts, Te;
          step_positions(ns, ne, xs, xe, Ts, Te);
          if (Ts + Te > kDenseStep) {  // lanes on consecutive quads: u16 staging, one pass
            emit_dense16(st, xs, Ts, w0 * 32u, gs, out_s, d.runs_cap, wbuf);
            emit_dense16(en, xe, Te, w0 * 32u, ge, out_e, d.runs_cap, wbuf);
          } else {
            if (__any_sync(0xffffffffu, ns != 0u)) emit_sparse_bits(st, ns, gs + xs, w0 * 32u, out_s, d.runs_cap);
            if (__any_sync(0xffffffffu, ne != 0u)) emit_sparse_bits(en, ne, ge + xe, w0 * 32u, out_e, d.runs_cap);
          }
          gs += Ts;
          ge += Te;
        }
        carry = __shfl_sync(0xffffffffu, z[3], 31);
        __stcg(dst4 + 32 * (s0 + u) + lane, make_uint4(vv[0] | m[0], vv[1] | m[1], vv[2] | m[2], vv[3] | m[3]));
      }
    }
  }
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), uint32_t grid, uint32_t block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

cudaError_t elem_ctx_init() {  // at context creation: the apply kernel's dynamic shared memory
  return cudaFuncSetAttribute(k_elem_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)((size_t)kApplyWarps * kStageBuf16 * 2u));
}

int launch_elem_stage(const ElemDev& d, uint32_t n_tiles, uint32_t n_sync_tiles, void* stream, std::string* err) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  constexpr size_t kApplySmem = (size_t)kApplyWarps * kStageBuf16 * 2u;
  if (n_tiles && e == cudaSuccess) e = launch_pdl(k_elem_pass1, n_tiles, kET, 0, s, d);
  if (n_tiles && e == cudaSuccess)  // a stage with only WRITE ops has nothing to decide (writes cannot get stuck)
    e = launch_pdl(k_elem_decide, (d.n_progs + kDecideWarps - 1) / kDecideWarps, 32 * kDecideWarps, 0, s, d);
  if (n_sync_tiles && e == cudaSuccess) {
    const uint32_t blocks = (n_sync_tiles + kApplyWarps - 1) / kApplyWarps;
    e = launch_pdl(k_elem_apply, blocks < 148u * 16u ? blocks : 148u * 16u, 32 * kApplyWarps, kApplySmem, s, d,
                   n_sync_tiles);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("element stage launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

// Initial store: every cell (V,I) -> L = 1 on [0, n_cells), R = 0 (program.hpp:174-184),
// except the pre-fragmented cells (coh_frag_mask), which start coherent: (V,V), R = 1.  pinit[b] =
// {n_cells, frag_log2, frag_seed lo, frag_seed hi}.  128-bit stores, one 4-word group
// per thread iteration.
__global__ void __launch_bounds__(256) k_elem_init(uint32_t* planes, uint32_t W, const uint4* __restrict__ pinit) {
  const uint32_t b = blockIdx.y;  // one buffer per grid row: no index division
  const uint4 pi = pinit[b];
  const uint32_t n = pi.x;
  const uint64_t seed = (uint64_t)pi.z | ((uint64_t)pi.w << 32);
  uint4* const L4 = reinterpret_cast<uint4*>(planes + (size_t)b * 2u * W);
  uint4* const R4 = L4 + W / 4u;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < W / 4u; q += gridDim.x * blockDim.x) {
    uint32_t l[4], r[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t w = 4u * q + k;
      l[k] = (w + 1) * 32u <= n ? 0xFFFFFFFFu : (w * 32u < n ? (0xFFFFFFFFu >> (32u - (n - w * 32u))) : 0u);
    }
    if (pi.y) {  // coh_frag_mask of the four words (one draw each when rho <= 2^-6)
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = l[k] ? coh_frag_word(seed, pi.y, 4u * q + k) & l[k] : 0u;
    }
    __stcg(L4 + q, make_uint4(l[0], l[1], l[2], l[3]));
    __stcg(R4 + q, make_uint4(r[0], r[1], r[2], r[3]));
  }
}

int launch_elem_init(uint32_t* planes, uint32_t W, const uint32_t* pinit, uint32_t n_progs, void* stream,
                     std::string* err) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // ~8 quads per thread: enough blocks to fill the GPU for any buffer count
  const uint32_t per_row = (W / 4u + 256u * 8u - 1u) / (256u * 8u);
  k_elem_init<<<dim3(per_row, n_progs), 256, 0, s>>>(planes, W, reinterpret_cast<const uint4*>(pinit));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("element init launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

}  // namespace cohb
