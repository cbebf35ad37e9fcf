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
// Work decomposition: every range is cut into tiles of 2048 words (64 Ki cells); a
// persistent grid (a multiple of the SM count) strides over the global tile list and
// finds a tile's range by binary search over the per-range tile prefix.  A thread owns
// two aligned 16-byte quads of a tile; interior quads move as 128-bit loads / stores,
// partial words at range edges use atomics (two ranges may share an edge word).  Run
// extraction is count -> CUB scan over tiles -> write, so runs land ascending with no
// sort.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <string>

#include "internal.hpp"

namespace cohb {
namespace {

constexpr uint32_t kBT = 256;               // threads per tile
constexpr uint32_t kTileWords = 2048;       // 8 words per thread = 2 quads
constexpr uint32_t kTileQuads = kTileWords / 4;

struct Tiles {
  const coh_bitmap_range* r;
  const uint64_t* prefix;  // n + 1 entries: tile index of each range's first tile
  uint32_t n;
};

__device__ __forceinline__ uint32_t range_of_tile(const Tiles& T, uint64_t tile) {
  uint32_t a = 0, b = T.n;  // last r with prefix[r] <= tile
  while (b - a > 1) {
    const uint32_t m = (a + b) >> 1;
    if (T.prefix[m] <= tile) a = m;
    else b = m;
  }
  return a;
}

// Mask of the cells of absolute word w (plane-relative) inside [lo, hi].
__device__ __forceinline__ uint32_t cell_mask(uint64_t w, uint32_t lo, uint32_t hi) {
  const uint64_t wl = lo >> 5, wh = hi >> 5;
  if (w < wl || w > wh) return 0u;
  uint32_t m = 0xFFFFFFFFu;
  if (w == wl) m &= 0xFFFFFFFFu << (lo & 31u);
  if (w == wh) m &= 0xFFFFFFFFu >> (31u - (hi & 31u));
  return m;
}

// The tile's quads: quad q of a range = absolute (device) quad index qa0 + q, where qa0 is
// the aligned quad holding the range's first word.  Returns false past the range.
struct TileGeom {
  uint32_t r;
  uint64_t qa_first, qa_last;  // absolute quad indices (d_words as uint4*) covering the range
  uint64_t tile_in_range;
};
__device__ __forceinline__ TileGeom geom(const Tiles& T, uint64_t tile) {
  TileGeom g;
  g.r = range_of_tile(T, tile);
  const coh_bitmap_range R = T.r[g.r];
  g.qa_first = (R.word_off + (R.lo >> 5)) >> 2;
  g.qa_last = (R.word_off + (R.hi >> 5)) >> 2;
  g.tile_in_range = tile - T.prefix[g.r];
  return g;
}

template <bool SET>
__global__ void __launch_bounds__(kBT) k_range_set(uint32_t* words, Tiles T) {
  const uint64_t n_tiles = T.prefix[T.n];
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const TileGeom g = geom(T, tile);
    const coh_bitmap_range R = T.r[g.r];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t qa = g.qa_first + g.tile_in_range * kTileQuads + h * kBT + threadIdx.x;
      if (qa > g.qa_last) continue;
      uint32_t m[4];
      bool full = true;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        m[k] = cell_mask(qa * 4 + k - R.word_off, R.lo, R.hi);
        full &= m[k] == 0xFFFFFFFFu;
      }
      uint4* p = reinterpret_cast<uint4*>(words) + qa;
      if (full) {
        const uint32_t v = SET ? 0xFFFFFFFFu : 0u;
        __stcg(p, make_uint4(v, v, v, v));
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!m[k]) continue;
          uint32_t* w = words + qa * 4 + k;
          if (m[k] == 0xFFFFFFFFu) *w = SET ? 0xFFFFFFFFu : 0u;
          else if (SET) atomicOr(w, m[k]);
          else atomicAnd(w, ~m[k]);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kBT) k_first_zero(const uint32_t* words, Tiles T, uint32_t* first) {
  __shared__ uint32_t red[kBT / 32];
  const uint64_t n_tiles = T.prefix[T.n];
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const TileGeom g = geom(T, tile);
    const coh_bitmap_range R = T.r[g.r];
    uint32_t best = 0xFFFFFFFFu;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t qa = g.qa_first + g.tile_in_range * kTileQuads + h * kBT + threadIdx.x;
      if (qa > g.qa_last) continue;
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(words) + qa);
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 3; k >= 0; --k) {  // keep the lowest
        const uint64_t wr = qa * 4 + k - R.word_off;
        const uint32_t z = ~w4[k] & cell_mask(wr, R.lo, R.hi);
        if (z) best = (uint32_t)(wr * 32 + (__ffs(z) - 1));
      }
      if (best != 0xFFFFFFFFu) break;  // quad h = 0 is below quad h = 1
    }
    best = __reduce_min_sync(0xFFFFFFFFu, best);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t b = red[0];
      for (uint32_t k = 1; k < kBT / 32; ++k) b = min(b, red[k]);
      if (b != 0xFFFFFFFFu) atomicMin(first + g.r, b);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBT) k_view_flags(const uint32_t* L, const uint32_t* Rp, Tiles T, uint32_t* flags) {
  const uint64_t n_tiles = T.prefix[T.n];
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const TileGeom g = geom(T, tile);
    const coh_bitmap_range R = T.r[g.r];
    uint32_t f = 0;  // bit0 some L == 0, bit1 some R == 0, bit2 some L | R == 1
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t qa = g.qa_first + g.tile_in_range * kTileQuads + h * kBT + threadIdx.x;
      if (qa > g.qa_last) continue;
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(L) + qa), b = __ldcs(reinterpret_cast<const uint4*>(Rp) + qa);
      const uint32_t la[4] = {a.x, a.y, a.z, a.w}, ra[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t m = cell_mask(qa * 4 + k - R.word_off, R.lo, R.hi);
        f |= ((~la[k] & m) ? 1u : 0u) | ((~ra[k] & m) ? 2u : 0u) | (((la[k] | ra[k]) & m) ? 4u : 0u);
      }
    }
    f = __reduce_or_sync(0xFFFFFFFFu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags + g.r, f);
  }
}

__global__ void k_view_finish(const uint32_t* flags, const uint8_t* abs_pair, uint32_t n, uint8_t* ok) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t f = flags[i], a = abs_pair[i] & 3u;  // bit0 local V, bit1 remote V
  const bool L1 = !(f & 1u), R1 = !(f & 2u), none = !(f & 4u);
  ok[i] = a == 1u ? L1 : a == 2u ? R1 : a == 3u ? (L1 && R1) : none;
}

// Zero runs.  Per thread: its 8 words (2 quads) and the cells just outside them.
struct RunBits {
  uint32_t starts[8], ends[8];
  uint32_t n_starts[2], n_ends[2];  // per quad (the quads of a thread are 256 quads apart)
};
__device__ __forceinline__ void run_bits(const uint32_t* words, const coh_bitmap_range& R, uint64_t qa_first,
                                         uint64_t qa_last, uint64_t qa0, RunBits& b) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    b.n_starts[h] = b.n_ends[h] = 0;
    const uint64_t qa = qa0 + h * kBT;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      b.starts[h * 4 + k] = b.ends[h * 4 + k] = 0;
    }
    if (qa > qa_last) continue;
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(words) + qa);
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
    // neighbours: the word before this quad and the word after it (plane-relative)
    const uint64_t wr0 = qa * 4 - R.word_off;
    const uint32_t prev = (qa * 4 > R.word_off && wr0 >= 1) ? words[qa * 4 - 1] : 0xFFFFFFFFu;
    const uint32_t next = words[qa * 4 + 4 - ((qa * 4 + 4) > (R.word_off + (R.hi >> 5)) ? 1 : 0)];
    uint32_t zp = ~prev & cell_mask(wr0 - 1, R.lo, R.hi);  // zeros of the previous word (in range)
    if (wr0 == 0) zp = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t wr = wr0 + k;
      const uint32_t z = ~w4[k] & cell_mask(wr, R.lo, R.hi);
      const uint32_t zn = k < 3 ? (~w4[k + 1] & cell_mask(wr + 1, R.lo, R.hi))
                                : (~next & cell_mask(wr + 1, R.lo, R.hi));
      const uint32_t before = (z << 1) | (zp >> 31);   // zero at cell - 1
      const uint32_t after = (z >> 1) | (zn << 31);    // zero at cell + 1
      b.starts[h * 4 + k] = z & ~before;
      b.ends[h * 4 + k] = z & ~after;
      b.n_starts[h] += __popc(b.starts[h * 4 + k]);
      b.n_ends[h] += __popc(b.ends[h * 4 + k]);
      zp = z;
    }
  }
}

__device__ __forceinline__ uint32_t block_excl(uint32_t v, uint32_t* red, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) red[warp] = x;
  __syncthreads();
  uint32_t base = 0, tot = 0;
  for (uint32_t k = 0; k < kBT / 32; ++k) {
    if (k < warp) base += red[k];
    tot += red[k];
  }
  __syncthreads();
  *total = tot;
  return base + x - v;
}

__global__ void __launch_bounds__(kBT) k_runs_count(const uint32_t* words, Tiles T, uint64_t* tile_runs) {
  __shared__ uint32_t red[kBT / 32];
  const uint64_t n_tiles = T.prefix[T.n];
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const TileGeom g = geom(T, tile);
    const coh_bitmap_range R = T.r[g.r];
    RunBits b;
    run_bits(words, R, g.qa_first, g.qa_last, g.qa_first + g.tile_in_range * kTileQuads + threadIdx.x, b);
    uint32_t total;
    block_excl(b.n_starts[0] + b.n_starts[1], red, &total);
    if (threadIdx.x == 0) tile_runs[tile] = total;
  }
}

__global__ void __launch_bounds__(kBT) k_runs_write(const uint32_t* words, Tiles T, const uint64_t* tile_off,
                                                    uint32_t* run_start, uint32_t* run_end, uint64_t cap) {
  __shared__ uint32_t red[kBT / 32];
  const uint64_t n_tiles = T.prefix[T.n];
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const TileGeom g = geom(T, tile);
    const coh_bitmap_range R = T.r[g.r];
    const uint64_t qa0 = g.qa_first + g.tile_in_range * kTileQuads + threadIdx.x;
    RunBits b;
    run_bits(words, R, g.qa_first, g.qa_last, qa0, b);
    // cell order inside a tile: all first quads (threads 0..255), then all second quads
    uint32_t ts0, te0, ts1, te1;
    const uint32_t ps0 = block_excl(b.n_starts[0], red, &ts0);
    const uint32_t pe0 = block_excl(b.n_ends[0], red, &te0);
    const uint32_t ps1 = block_excl(b.n_starts[1], red, &ts1);
    const uint32_t pe1 = block_excl(b.n_ends[1], red, &te1);
    // runs of this range started before this tile, and one still open across its start
    const uint64_t range_base = tile_off[T.prefix[g.r]];
    const uint64_t starts_before = tile_off[tile] - range_base;
    uint64_t open = 0;
    if (g.tile_in_range > 0) {  // the tile's first cell and the cell before it both zero
      const uint64_t w = (g.qa_first + g.tile_in_range * kTileQuads) * 4;  // absolute first word of the tile
      const uint64_t wr = w - R.word_off;
      const uint32_t z0 = ~words[w] & cell_mask(wr, R.lo, R.hi), zm = ~words[w - 1] & cell_mask(wr - 1, R.lo, R.hi);
      open = ((z0 & 1u) && (zm >> 31)) ? 1 : 0;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint64_t gs = tile_off[tile] + (h ? ts0 + ps1 : ps0);
      uint64_t ge = range_base + starts_before - open + (h ? te0 + pe1 : pe0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t wr = (qa0 + h * kBT) * 4 + k - R.word_off;
        uint32_t s = b.starts[h * 4 + k], e = b.ends[h * 4 + k];
        while (s) {
          const uint32_t bit = __ffs(s) - 1;
          if (gs < cap) run_start[gs] = (uint32_t)(wr * 32 + bit);
          ++gs;
          s &= s - 1;
        }
        while (e) {
          const uint32_t bit = __ffs(e) - 1;
          if (ge < cap) run_end[ge] = (uint32_t)(wr * 32 + bit);
          ++ge;
          e &= e - 1;
        }
      }
    }
  }
}

__global__ void k_range_run_off(const uint64_t* prefix, const uint64_t* tile_off, uint32_t n, uint64_t* run_off) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) run_off[i] = tile_off[prefix[i]];
}

struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

int grid_for(coh_ctx* ctx) { return ctx->sms * 8; }

// Tile prefix for the ranges: prefix[n + 1] (exclusive scan of per-range tile counts), one
// single-block launch (a running carry over chunks of 1024 ranges).
__global__ void __launch_bounds__(1024) k_tile_prefix(const coh_bitmap_range* r, uint32_t n, uint64_t* prefix) {
  __shared__ uint64_t warp_sum[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t base = 0; base <= n; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    uint64_t v = 0;
    if (i < n) {
      const uint64_t q0 = (r[i].word_off + (r[i].lo >> 5)) >> 2, q1 = (r[i].word_off + (r[i].hi >> 5)) >> 2;
      v = r[i].lo <= r[i].hi ? (q1 - q0 + kTileQuads) / kTileQuads : 0;
    }
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
      warp_sum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const uint64_t excl = carry + (warp ? warp_sum[warp - 1] : 0) + x - v;
    if (i <= n) prefix[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sum[31];
    __syncthreads();
  }
}

int tile_prefix(coh_ctx* ctx, const coh_bitmap_range* d_r, uint32_t n, uint64_t* d_prefix, cudaStream_t s) {
  k_tile_prefix<<<1, 1024, 0, s>>>(d_r, n, d_prefix);
  ctx->launches += 1;
  return cudaGetLastError() == cudaSuccess ? COH_OK : COH_E_CUDA;
}

int check(coh_ctx* ctx, const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return COH_OK;
  ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
  return COH_E_CUDA;
}

}  // namespace
}  // namespace cohb

using namespace cohb;

#define COH_BM_PREFIX(ctx, d_r, n, s, T)                                                   \
  Scratch pre_;                                                                          \
  pre_.s = s;                                                                            \
  if (cudaMallocAsync(&pre_.p, sizeof(uint64_t) * ((size_t)n + 1), s) != cudaSuccess)    \
    return check(ctx, "bitmap scratch"), COH_E_CUDA;                                     \
  if (tile_prefix(ctx, d_r, n, static_cast<uint64_t*>(pre_.p), s)) return check(ctx, "bitmap prefix"), COH_E_CUDA; \
  const Tiles T{d_r, static_cast<uint64_t*>(pre_.p), n};

static int range_fill(coh_ctx* ctx, uint32_t* d_words, const coh_bitmap_range* d_r, uint32_t n, bool set, void* stream) {
  if (!ctx || (n && (!d_words || !d_r))) return COH_E_ARG;
  if (!n) return COH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  COH_BM_PREFIX(ctx, d_r, n, s, T)
  if (set) k_range_set<true><<<grid_for(ctx), kBT, 0, s>>>(d_words, T);
  else k_range_set<false><<<grid_for(ctx), kBT, 0, s>>>(d_words, T);
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
  if (cudaMemsetAsync(d_first, 0xFF, sizeof(uint32_t) * n, s) != cudaSuccess) return check(ctx, "first_zero init");
  COH_BM_PREFIX(ctx, d_ranges, n, s, T)
  k_first_zero<<<grid_for(ctx), kBT, 0, s>>>(d_words, T, d_first);
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
  if (cudaMallocAsync(&fl.p, sizeof(uint32_t) * n, s) != cudaSuccess) return check(ctx, "view_check scratch");
  if (cudaMemsetAsync(fl.p, 0, sizeof(uint32_t) * n, s) != cudaSuccess) return check(ctx, "view_check init");
  COH_BM_PREFIX(ctx, d_ranges, n, s, T)
  k_view_flags<<<grid_for(ctx), kBT, 0, s>>>(d_L, d_R, T, static_cast<uint32_t*>(fl.p));
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
  COH_BM_PREFIX(ctx, d_ranges, n, s, T)
  // tiles in total: read back once (sizes the per-tile count array)
  uint64_t n_tiles = 0;
  if (cudaMemcpyAsync(&n_tiles, T.prefix + n, sizeof n_tiles, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return check(ctx, "zero_runs tiles");
  Scratch tr;
  tr.s = s;
  if (cudaMallocAsync(&tr.p, sizeof(uint64_t) * (n_tiles + 1), s) != cudaSuccess) return check(ctx, "zero_runs scratch");
  uint64_t* tile_off = static_cast<uint64_t*>(tr.p);
  if (cudaMemsetAsync(tile_off + n_tiles, 0, sizeof(uint64_t), s) != cudaSuccess) return check(ctx, "zero_runs init");
  k_runs_count<<<grid_for(ctx), kBT, 0, s>>>(d_words, T, tile_off);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, tile_off, tile_off, (int)(n_tiles + 1), s);
  Scratch sc;
  sc.s = s;
  if (cudaMallocAsync(&sc.p, tmp, s) != cudaSuccess) return check(ctx, "zero_runs scan scratch");
  cub::DeviceScan::ExclusiveSum(sc.p, tmp, tile_off, tile_off, (int)(n_tiles + 1), s);
  k_range_run_off<<<(n + 1 + 255) / 256, 256, 0, s>>>(T.prefix, tile_off, n, d_run_off);
  k_runs_write<<<grid_for(ctx), kBT, 0, s>>>(d_words, T, tile_off, d_run_start, d_run_end, cap);
  ctx->launches += 4;
  return check(ctx, "zero_runs");
}
