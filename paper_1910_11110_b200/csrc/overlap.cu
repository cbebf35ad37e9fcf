// Batched overlap registry and mode closure.
//
// Replaces, for many views and many blocks at once:
//   OverlapRegistry::insert / query (overlap.hpp:33-175): views of a buffer whose
//     inclusive ranges intersect the probe's, the probe excluded, name-sorted;
//   infer_overlap_closure (overlap.hpp:177-230): per block, W x adds same-site RW on every
//     overlapping y without a same-site W, RW x on every overlapping y; a declared R is
//     upgraded in place, others appended as shadows in view declaration order; a view
//     needed at both sites (or against its declared site) is an OverlapInferenceError.
//
// Device layout (coh_registry): the views sorted by (buffer, lo) — CUB radix sort of a
// 64-bit key — as struct-of-arrays lo / hi / view id, plus an implicit max-hi segment
// tree over that order.  A query is two binary searches (the buffer's range, then the last
// view starting at or before the probe's hi) and an output-sensitive descent of the tree
// that skips every subtree whose largest hi ends before the probe's lo: O((k + 1) log n)
// for k hits, the stabbing-plus-start-index bound of the reference's segment-tree backend.
//
// Closure: one thread per block (blocks carry a handful of modes); hits of each declared
// W/RW view are ordered by name rank, folded into a small `needed` table in the reference's
// iteration order (so the same OverlapInferenceError view is reported), then upgrades and
// shadows are emitted.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <string>

#include "internal.hpp"

namespace cohb {
namespace {

constexpr uint32_t kMaxNeeded = 64;   // per-block `needed` table (status -2 beyond)
constexpr uint32_t kMaxModes = 64;    // declared modes per block
constexpr int kStack = 64;            // tree descent stack (depth <= 2 * log2 n)

struct RegDev {
  uint32_t n, P;               // views, leaves (power of two >= n)
  const uint64_t* key;         // sorted (buffer << 32 | lo)
  const int32_t* lo;           // sorted order
  const int32_t* hi;
  const uint32_t* view;        // sorted position -> view index
  const int32_t* tree;         // 2P nodes, node 1 = root, max hi (INT_MIN for padding)
  const coh_view* views;       // by view index
  const uint64_t* hoff;        // optional CSR of every view's hits (n + 1 offsets) ...
  const uint32_t* hits;        // ... name-rank ordered, probe excluded (nullptr: use the tree)
};

__device__ __forceinline__ uint32_t lower_bound_key(const uint64_t* key, uint32_t n, uint64_t k) {
  uint32_t a = 0, b = n;
  while (a < b) {
    const uint32_t m = (a + b) >> 1;
    if (key[m] < k) a = m + 1;
    else b = m;
  }
  return a;
}

// Visits, in sorted order, every position i in [lo_i, hi_i) with hi[i] >= qlo.
template <class F>
__device__ void enumerate(const RegDev& r, uint32_t lo_i, uint32_t hi_i, int32_t qlo, F&& f) {
  if (lo_i >= hi_i) return;
  uint32_t stack[kStack];
  int sp = 0;
  // node, node range [nl, nr) packed: push root
  uint32_t node = 1, nl = 0, nr = r.P;
  for (;;) {
    bool descend = false;
    if (nr > lo_i && nl < hi_i && r.tree[node] >= qlo) {
      if (nr - nl == 1) {
        f(nl);
      } else {
        descend = true;
      }
    }
    if (descend) {
      const uint32_t mid = (nl + nr) >> 1;
      // push right child, continue with left (keeps ascending order)
      stack[sp++] = (2 * node + 1);
      stack[sp++] = mid;
      node = 2 * node;
      nr = mid;
      continue;
    }
    if (sp == 0) break;
    nl = stack[--sp];
    node = stack[--sp];
    // right child range: [nl, nl + size) with size from the node's level
    const uint32_t level = 31u - __clz(node);
    nr = nl + (r.P >> level);
  }
}

__global__ void k_build_tree_leaves(uint32_t n, uint32_t P, const int32_t* hi, int32_t* tree) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) tree[P + i] = i < n ? hi[i] : INT32_MIN;
}
__global__ void k_build_tree_level(uint32_t first, uint32_t count, int32_t* tree) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) {
    const uint32_t node = first + i;
    tree[node] = max(tree[2 * node], tree[2 * node + 1]);
  }
}
// The top levels (nodes < first) in one block: level by level with block barriers.
__global__ void __launch_bounds__(1024) k_build_tree_top(uint32_t first, int32_t* tree) {
  for (uint32_t f = first; f >= 1; f >>= 1) {
    for (uint32_t i = threadIdx.x; i < f; i += blockDim.x) tree[f + i] = max(tree[2 * (f + i)], tree[2 * (f + i) + 1]);
    __syncthreads();
  }
}
__global__ void k_make_keys(const coh_view* views, uint32_t n, uint64_t* key, uint32_t* idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    key[i] = ((uint64_t)views[i].buffer << 32) | (uint32_t)views[i].lo;
    idx[i] = i;
  }
}
__global__ void k_gather(const coh_view* views, const uint32_t* order, uint32_t n, int32_t* lo, int32_t* hi) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const coh_view v = views[order[i]];
    lo[i] = v.lo;
    hi[i] = v.hi;
  }
}

// Hits of view p, in sorted (buffer, lo) order, probe excluded.
template <class F>
__device__ void query_view(const RegDev& r, uint32_t p, F&& f) {
  const coh_view v = r.views[p];
  const uint32_t bs = lower_bound_key(r.key, r.n, (uint64_t)v.buffer << 32);
  // last view of this buffer starting at or before v.hi
  const uint32_t be = lower_bound_key(r.key, r.n, ((uint64_t)v.buffer << 32) | ((uint64_t)(uint32_t)v.hi + 1ull));
  enumerate(r, bs, be, v.lo, [&](uint32_t i) {
    const uint32_t y = r.view[i];
    if (y != p) f(y);
  });
}

// Registry build, second half: every view's hits once, as a CSR in name-rank order, so a
// closure reads a short contiguous list instead of descending the tree per mode.
__global__ void k_count_hits(RegDev r, uint64_t* cnt) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= r.n) return;
  uint32_t c = 0;
  query_view(r, v, [&](uint32_t) { ++c; });
  cnt[v] = c;
}

__global__ void k_fill_hits(RegDev r, const uint64_t* off, uint32_t* hits) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= r.n) return;
  uint32_t* h = hits + off[v];
  uint32_t k = 0;
  query_view(r, v, [&](uint32_t y) {  // insertion by name rank (std::set<std::string> order)
    const uint32_t ry = r.views[y].name_rank;
    uint32_t j = k++;
    while (j > 0 && r.views[h[j - 1]].name_rank > ry) {
      h[j] = h[j - 1];
      --j;
    }
    h[j] = y;
  });
}

__global__ void k_query(RegDev r, const uint32_t* probes, uint32_t n_probes, uint32_t* hits, uint32_t stride,
                        uint32_t* count) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_probes) return;
  uint32_t c = 0;
  uint32_t* out = hits + (uint64_t)q * stride;
  if (r.hits) {  // the precomputed list, already name-ordered
    const uint64_t a = r.hoff[probes[q]], e = r.hoff[probes[q] + 1];
    for (uint64_t i = a; i < e; ++i, ++c)
      if (c < stride) out[c] = r.hits[i];
    count[q] = c;
    return;
  }
  query_view(r, probes[q], [&](uint32_t y) {
    // insertion by name rank (the reference returns std::set<std::string> order)
    if (c < stride) {
      const uint32_t ry = r.views[y].name_rank;
      uint32_t k = c;
      while (k > 0 && r.views[out[k - 1]].name_rank > ry) {
        out[k] = out[k - 1];
        --k;
      }
      out[k] = y;
    }
    ++c;
  });
  count[q] = c;
}

__global__ void k_closure(RegDev r, const coh_mode* modes, const uint32_t* off, uint32_t n_blocks, coh_mode* out,
                          uint32_t stride, uint32_t* out_count, int32_t* status) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  const uint32_t m0 = off[b], m1 = off[b + 1];
  const uint32_t nm = m1 - m0;
  coh_mode* o = out + (uint64_t)b * stride;
  if (nm > kMaxModes || nm > stride) {
    status[b] = -2;
    out_count[b] = 0;
    return;
  }
  // needed: (view, site) in name-rank order of first insertion handled via rank sort
  uint32_t nv[kMaxNeeded];
  uint8_t ns[kMaxNeeded];
  uint32_t nn = 0;
  int32_t st = -1;
  for (uint32_t k = m0; k < m1 && st == -1; ++k) {
    const coh_mode m = modes[k];
    if (m.kind == COH_R || (m.flags & 2u) || !(m.flags & 1u)) continue;  // R, shadow, scalar
    // this mode's hits, name-ordered: collect then insertion-sort by rank
    uint32_t hv[kMaxNeeded];
    uint32_t nh = 0;
    bool over = false;
    auto skip = [&](uint32_t y) {  // a W skips y with a same-site W (the declared set)
      if (m.kind != COH_W) return false;
      for (uint32_t q = m0; q < m1; ++q) {
        const coh_mode o2 = modes[q];
        if ((o2.flags & 1u) && o2.var == y && o2.kind == COH_W && o2.site == m.site) return true;
      }
      return false;
    };
    if (r.hits) {  // the precomputed, already name-ordered list
      for (uint64_t i = r.hoff[m.var], e = r.hoff[m.var + 1]; i < e && !over; ++i) {
        const uint32_t y = r.hits[i];
        if (skip(y)) continue;
        if (nh == kMaxNeeded) over = true;
        else hv[nh++] = y;
      }
    } else {
      query_view(r, m.var, [&](uint32_t y) {
        if (skip(y)) return;
        if (nh == kMaxNeeded) {
          over = true;
          return;
        }
        const uint32_t ry = r.views[y].name_rank;
        uint32_t j = nh++;
        while (j > 0 && r.views[hv[j - 1]].name_rank > ry) {
          hv[j] = hv[j - 1];
          --j;
        }
        hv[j] = y;
      });
    }
    if (over) {
      st = -2;
      break;
    }
    for (uint32_t h = 0; h < nh && st == -1; ++h) {  // needed.emplace(y, site), first conflict throws
      uint32_t j = 0;
      while (j < nn && nv[j] != hv[h]) ++j;
      if (j < nn) {
        if (ns[j] != m.site) st = (int32_t)hv[h];
      } else if (nn == kMaxNeeded) {
        st = -2;
      } else {
        nv[nn] = hv[h];
        ns[nn] = m.site;
        ++nn;
      }
    }
  }
  if (st != -1) {
    status[b] = st;
    out_count[b] = 0;
    return;
  }
  // needed in name order (std::map): upgrade / conflict against the declared entries
  for (uint32_t i = 1; i < nn; ++i)
    for (uint32_t j = i; j > 0 && r.views[nv[j - 1]].name_rank > r.views[nv[j]].name_rank; --j) {
      const uint32_t tv = nv[j];
      nv[j] = nv[j - 1];
      nv[j - 1] = tv;
      const uint8_t ts = ns[j];
      ns[j] = ns[j - 1];
      ns[j - 1] = ts;
    }
  for (uint32_t k = 0; k < nm; ++k) o[k] = modes[m0 + k];
  uint32_t cnt = nm;
  uint32_t sh_v[kMaxNeeded];
  uint8_t sh_s[kMaxNeeded];
  uint32_t nsh = 0;
  for (uint32_t i = 0; i < nn && st == -1; ++i) {
    int32_t ex = -1;  // the last declared entry naming this view
    for (uint32_t k = 0; k < nm; ++k)
      if ((o[k].flags & 1u) && o[k].var == nv[i]) ex = (int32_t)k;
    if (ex >= 0) {
      if (o[ex].site != ns[i]) st = (int32_t)nv[i];
      else if (o[ex].kind == COH_R) o[ex].kind = COH_RW;
    } else {
      sh_v[nsh] = nv[i];
      sh_s[nsh] = ns[i];
      ++nsh;
    }
  }
  if (st != -1) {
    status[b] = st;
    out_count[b] = 0;
    return;
  }
  // shadows in view declaration order (= view index)
  for (uint32_t i = 1; i < nsh; ++i)
    for (uint32_t j = i; j > 0 && sh_v[j - 1] > sh_v[j]; --j) {
      const uint32_t tv = sh_v[j];
      sh_v[j] = sh_v[j - 1];
      sh_v[j - 1] = tv;
      const uint8_t ts = sh_s[j];
      sh_s[j] = sh_s[j - 1];
      sh_s[j - 1] = ts;
    }
  if (cnt + nsh > stride) {
    status[b] = -2;
    out_count[b] = 0;
    return;
  }
  for (uint32_t i = 0; i < nsh; ++i) {
    coh_mode s;
    s.var = sh_v[i];
    s.kind = COH_RW;
    s.site = sh_s[i];
    s.flags = 3u;  // view | shadow
    s.pad = 0;
    o[cnt++] = s;
  }
  out_count[b] = cnt;
  status[b] = -1;
}

}  // namespace
}  // namespace cohb

struct coh_registry {
  int device = 0;
  cudaStream_t stream = nullptr;  // the build stream; the memory is stream-ordered
  uint32_t n = 0, P = 1;
  void* mem = nullptr;  // one allocation: keys, lo, hi, view, tree, views copy
  void* csr = nullptr;  // the hits CSR (offsets, then hits), when it fits kMaxCsrHits
  cohb::RegDev dev{};
  std::string err;
};

namespace {
int fail(coh_ctx* ctx, const char* what, cudaError_t e) {
  if (ctx) ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
  return COH_E_CUDA;
}
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
}  // namespace

extern "C" int coh_registry_build(coh_ctx* ctx, const coh_view* d_views, uint32_t n_views, coh_registry** out,
                                  void* stream) {
  using namespace cohb;
  if (!ctx || !out || (n_views && !d_views) || n_views > (1u << 30)) return COH_E_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  coh_registry* r = new coh_registry();
  r->device = ctx->device;
  r->n = n_views;
  while (r->P < n_views) r->P <<= 1;
  const uint32_t n = n_views ? n_views : 1, P = r->P;
  // layout
  size_t o_key = 0, o_key2 = align256(o_key + 8ull * n), o_idx = align256(o_key2 + 8ull * n),
         o_view = align256(o_idx + 4ull * n), o_lo = align256(o_view + 4ull * n), o_hi = align256(o_lo + 4ull * n),
         o_tree = align256(o_hi + 4ull * n), o_views = align256(o_tree + 8ull * P), o_tmp = align256(o_views + sizeof(coh_view) * n);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n, 0, 64, s);
  const size_t total = o_tmp + tmp_bytes;
  r->stream = s;
  cudaError_t e = cudaMallocAsync(&r->mem, total, s);
  if (e != cudaSuccess) {
    delete r;
    return fail(ctx, "registry alloc", e);
  }
  char* base = static_cast<char*>(r->mem);
  uint64_t* key_in = reinterpret_cast<uint64_t*>(base + o_key);
  uint64_t* key = reinterpret_cast<uint64_t*>(base + o_key2);
  uint32_t* idx = reinterpret_cast<uint32_t*>(base + o_idx);
  uint32_t* view = reinterpret_cast<uint32_t*>(base + o_view);
  int32_t* lo = reinterpret_cast<int32_t*>(base + o_lo);
  int32_t* hi = reinterpret_cast<int32_t*>(base + o_hi);
  int32_t* tree = reinterpret_cast<int32_t*>(base + o_tree);
  coh_view* views = reinterpret_cast<coh_view*>(base + o_views);
  if (n_views) {
    if ((e = cudaMemcpyAsync(views, d_views, sizeof(coh_view) * n_views, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return fail(ctx, "registry copy", e);
    k_make_keys<<<(n_views + 255) / 256, 256, 0, s>>>(views, n_views, key_in, idx);
    cub::DeviceRadixSort::SortPairs(base + o_tmp, tmp_bytes, key_in, key, idx, view, (int)n_views, 0, 64, s);
    k_gather<<<(n_views + 255) / 256, 256, 0, s>>>(views, view, n_views, lo, hi);
  }
  k_build_tree_leaves<<<(P + 255) / 256, 256, 0, s>>>(n_views, P, hi, tree);
  uint32_t first = P >> 1;
  for (; first > 1024; first >>= 1) k_build_tree_level<<<(first + 255) / 256, 256, 0, s>>>(first, first, tree);
  if (first >= 1) k_build_tree_top<<<1, 1024, 0, s>>>(first, tree);
  if ((e = cudaGetLastError()) != cudaSuccess) {
    cudaFreeAsync(r->mem, s);
    delete r;
    return fail(ctx, "registry build", e);
  }
  ctx->launches += (n_views ? 4 : 2) + (uint64_t)(P > 2048 ? 31 - __builtin_clz(P / 2048) : 0);  // + the CUB sort
  r->dev = RegDev{n_views, P, key, lo, hi, view, tree, views, nullptr, nullptr};
  if (n_views) {  // every view's hits, once (closures then read contiguous lists); on any
                  // failure the registry simply keeps answering from the tree
    constexpr uint64_t kMaxCsrHits = 1ull << 26;
    const size_t o_tmp2 = align256(8ull * (n_views + 1));
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)n_views + 1, s);
    void* cmem = nullptr;
    uint64_t total = ~0ull;
    if (cudaMallocAsync(&cmem, o_tmp2 + scan_bytes, s) == cudaSuccess) {
      uint64_t* off = static_cast<uint64_t*>(cmem);
      cudaMemsetAsync(off + n_views, 0, 8, s);
      k_count_hits<<<(n_views + 255) / 256, 256, 0, s>>>(r->dev, off);
      cub::DeviceScan::ExclusiveSum(static_cast<char*>(cmem) + o_tmp2, scan_bytes, off, off, (int)n_views + 1, s);
      if (cudaMemcpyAsync(&total, off + n_views, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        total = ~0ull;
      void* csr = nullptr;
      const size_t o_hits = align256(8ull * (n_views + 1));
      if (total <= kMaxCsrHits && cudaMallocAsync(&csr, o_hits + 4 * std::max<uint64_t>(total, 1), s) == cudaSuccess) {
        uint64_t* hoff = static_cast<uint64_t*>(csr);
        uint32_t* hits = reinterpret_cast<uint32_t*>(static_cast<char*>(csr) + o_hits);
        cudaMemcpyAsync(hoff, off, 8ull * (n_views + 1), cudaMemcpyDeviceToDevice, s);
        k_fill_hits<<<(n_views + 255) / 256, 256, 0, s>>>(r->dev, hoff, hits);
        r->csr = csr;
        r->dev.hoff = hoff;
        r->dev.hits = hits;
        ctx->launches += 1;
      }
      cudaFreeAsync(cmem, s);
      ctx->launches += 2;
    }
    if (cudaGetLastError() != cudaSuccess && r->csr) {  // fall back to the tree
      cudaFreeAsync(r->csr, s);
      r->csr = nullptr;
      r->dev.hoff = nullptr;
      r->dev.hits = nullptr;
    }
  }
  *out = r;
  return COH_OK;
}

extern "C" void coh_registry_destroy(coh_registry* r) {
  if (!r) return;
  if (r->csr) cudaFreeAsync(r->csr, r->stream);
  cudaFreeAsync(r->mem, r->stream);
  delete r;
}

extern "C" int coh_registry_query(coh_ctx* ctx, const coh_registry* r, const uint32_t* d_probes, uint32_t n_probes,
                                  uint32_t* d_hits, uint32_t hits_stride, uint32_t* d_hit_count, void* stream) {
  if (!ctx || !r || (n_probes && (!d_probes || !d_hits || !d_hit_count))) return COH_E_ARG;
  if (!n_probes) return COH_OK;
  cohb::k_query<<<(n_probes + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(r->dev, d_probes, n_probes,
                                                                                        d_hits, hits_stride, d_hit_count);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, "registry query", e);
  ctx->launches++;
  return COH_OK;
}

extern "C" int coh_overlap_closure(coh_ctx* ctx, const coh_registry* r, const coh_mode* d_modes,
                                   const uint32_t* d_block_off, uint32_t n_blocks, coh_mode* d_out, uint32_t out_stride,
                                   uint32_t* d_out_count, int32_t* d_status, void* stream) {
  if (!ctx || !r || (n_blocks && (!d_modes || !d_block_off || !d_out || !d_out_count || !d_status))) return COH_E_ARG;
  if (!n_blocks) return COH_OK;
  cohb::k_closure<<<(n_blocks + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      r->dev, d_modes, d_block_off, n_blocks, d_out, out_stride, d_out_count, d_status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, "overlap closure", e);
  ctx->launches++;
  return COH_OK;
}
