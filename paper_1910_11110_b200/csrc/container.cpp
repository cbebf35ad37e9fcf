// Coherent-container runtime (config C5): VectorPU's coherence control
// (coherent_on_{cpu,gpu}_{r,w,rw}, download/upload) rebuilt on the
// calculus.  Each vector keeps the calculus state of its whole-array variable — concrete
// pair (which copies really hold the data) and abstract pair (the flags VectorPU keeps,
// PAPER.md:1211) — and a component call executes exactly the translated block
// (modes.hpp:31-59): for every argument in order, the guard on the abstract flag decides
// whether to copy (`pull x` = cudaMemcpyAsync D2H for a CPU component, `push x` = H2D for
// a GPU component), then `w x^` for W/RW; then the component runs (CPU: on the calling
// thread once its own arguments' copies have landed; GPU: launched on the component
// stream); then its body effects (R: `r x`, W: `w x`, RW: both, at the component's site).
// Uploads and downloads run on two side streams; per vector, events on its last device-
// and host-copy operations order each copy and component after exactly the work on the
// same vector, so copies of independent vectors overlap each other and the components.  A step that cannot
// unify (data valid nowhere the component needs it) is the calculus' Stuck and comes back
// as COH_E_DEFECT with the StuckInfo text in coh_last_error; nothing is copied for it.
//
// Unlike VectorPU, whose flags start (true, true), vectors start at
// the calculus' initial store (V,I)/(V,I) (program.hpp:174-184) so the copies issued are
// exactly the ones the evaluator predicts for the same call sequence.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace {

int apply_pair(uint32_t eff, uint32_t site, uint32_t p) {
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

const char* eff_name(uint32_t e) {
  static const char* n[] = {"push", "pull", "r", "w", "noop"};
  return e < 5 ? n[e] : "?";
}

std::string pair_str(uint32_t p) {
  return std::string("(") + ((p & 1u) ? "V" : "I") + "," + ((p & 2u) ? "V" : "I") + ")";
}

}  // namespace

struct RtVector {
  size_t bytes = 0;
  void* host = nullptr;
  void* dev = nullptr;
  uint32_t conc = 1, abst = 1;  // pairs: bit0 local (CPU) valid, bit1 remote (GPU) valid
  // Stream-ordering state (side streams): the last enqueued operation touching each copy.
  cudaEvent_t dev_last = nullptr;   // a GPU component, an upload (writes) or a download (reads)
  cudaEvent_t host_last = nullptr;  // an upload (reads the host copy) or a download (writes it)
  bool dev_pending = false, host_pending = false, host_written = false;
};

// A mother vector with element-granular validity (views, pvector<T>): planes L, R in one
// device allocation (words [0, W) and [W, 2W), W a multiple of 4 for the 16-byte quads of
// the bit-plane primitives), views with their abstract pairs, and the small device /
// pinned scratch the per-call primitives use.
struct RtBuffer {
  uint32_t n_cells = 0, elem_bytes = 0, W = 0;
  void* host = nullptr;
  void* dev = nullptr;
  uint32_t* planes = nullptr;
  std::vector<uint32_t> lo, hi, abst;  // views, declaration order
  coh_bitmap_range* d_rng = nullptr;   // [2]
  uint32_t* d_first = nullptr;         // [1]
  uint64_t* d_off = nullptr;           // [2]
  uint32_t* d_runs = nullptr;          // [2][cap]
  uint64_t cap = 0;
  uint32_t* h_io = nullptr;            // pinned readback: first zero [0], run offsets [2..5], runs [8..]
};

struct coh_rt {
  coh_ctx* ctx = nullptr;
  std::vector<RtVector> vec;
  std::vector<RtBuffer> buf;
  std::vector<coh_rt_copy> log;
  cudaStream_t stream = nullptr;              // GPU components (and the view path)
  cudaStream_t up = nullptr, down = nullptr;  // side streams: uploads (H2D), downloads (D2H)
  cudaStream_t host = nullptr;                // async mode: CPU components as host functions
  bool async_host = false;
  coh_rt_stats stats{};
  std::vector<cudaEvent_t> ev_free;                           // event pool
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_open;  // copies not yet harvested
};

namespace {
cudaEvent_t take_event(coh_rt* rt) {
  if (!rt->ev_free.empty()) {
    cudaEvent_t e = rt->ev_free.back();
    rt->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// After a stream synchronisation every recorded copy has completed: add their durations.
void harvest(coh_rt* rt) {
  for (auto& pr : rt->ev_open) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) rt->stats.copy_ms += ms;
    rt->ev_free.push_back(pr.first);
    rt->ev_free.push_back(pr.second);
  }
  rt->ev_open.clear();
}
}  // namespace

extern "C" {

int coh_rt_create(coh_ctx* ctx, coh_rt** out) {
  if (!ctx || !out) return COH_E_ARG;
  coh_rt* rt = new coh_rt();
  rt->ctx = ctx;
  if (cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&rt->up, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&rt->down, cudaStreamNonBlocking) != cudaSuccess) {
    if (rt->stream) cudaStreamDestroy(rt->stream);
    if (rt->up) cudaStreamDestroy(rt->up);
    delete rt;
    ctx->err = "coh_rt_create: stream";
    return COH_E_CUDA;
  }
  *out = rt;
  return COH_OK;
}

void coh_rt_destroy(coh_rt* rt) {
  if (!rt) return;
  cudaStreamSynchronize(rt->stream);
  cudaStreamSynchronize(rt->up);
  cudaStreamSynchronize(rt->down);
  if (rt->host) cudaStreamSynchronize(rt->host);
  harvest(rt);
  for (cudaEvent_t e : rt->ev_free) cudaEventDestroy(e);
  for (auto& v : rt->vec) {
    cudaFreeHost(v.host);
    cudaFree(v.dev);
    cudaEventDestroy(v.dev_last);
    cudaEventDestroy(v.host_last);
  }
  for (auto& b : rt->buf) {
    cudaFreeHost(b.host);
    cudaFreeHost(b.h_io);
    cudaFree(b.dev);
    cudaFree(b.planes);
    cudaFree(b.d_rng);
    cudaFree(b.d_first);
    cudaFree(b.d_off);
    cudaFree(b.d_runs);
  }
  cudaStreamDestroy(rt->stream);
  cudaStreamDestroy(rt->up);
  cudaStreamDestroy(rt->down);
  if (rt->host) cudaStreamDestroy(rt->host);
  delete rt;
}

int coh_rt_vector(coh_rt* rt, size_t bytes, uint32_t* id) {
  if (!rt || !id || bytes == 0) return COH_E_ARG;
  RtVector v;
  v.bytes = bytes;
  if (cudaHostAlloc(&v.host, bytes, cudaHostAllocDefault) != cudaSuccess) {
    rt->ctx->err = "coh_rt_vector: pinned host allocation of " + std::to_string(bytes) + " bytes";
    return COH_E_CUDA;
  }
  if (cudaMalloc(&v.dev, bytes) != cudaSuccess) {
    cudaFreeHost(v.host);
    rt->ctx->err = "coh_rt_vector: device allocation of " + std::to_string(bytes) + " bytes";
    return COH_E_CUDA;
  }
  cudaEventCreateWithFlags(&v.dev_last, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&v.host_last, cudaEventDisableTiming);
  *id = (uint32_t)rt->vec.size();
  rt->vec.push_back(v);
  return COH_OK;
}

void* coh_rt_host_ptr(coh_rt* rt, uint32_t id) { return rt && id < rt->vec.size() ? rt->vec[id].host : nullptr; }
void* coh_rt_device_ptr(coh_rt* rt, uint32_t id) { return rt && id < rt->vec.size() ? rt->vec[id].dev : nullptr; }
void* coh_rt_stream(coh_rt* rt) { return rt ? rt->stream : nullptr; }

int coh_rt_state(coh_rt* rt, uint32_t id, uint8_t* nibble) {
  if (!rt || id >= rt->vec.size() || !nibble) return COH_E_ARG;
  *nibble = (uint8_t)(rt->vec[id].conc | (rt->vec[id].abst << 2));
  return COH_OK;
}

int coh_rt_call(coh_rt* rt, uint32_t site, const coh_rt_arg* args, uint32_t n_args, coh_rt_fn fn, void* user) {
  if (!rt || (n_args && !args) || site > COH_REMOTE) return COH_E_ARG;
  // DeclBlock: a variable appears at most once per block (program.hpp:218-225)
  for (uint32_t i = 0; i < n_args; ++i) {
    if (args[i].vec >= rt->vec.size() || args[i].kind > COH_RW) {
      rt->ctx->err = "coh_rt_call: bad argument " + std::to_string(i);
      return COH_E_CONSTRUCTION;
    }
    for (uint32_t j = i + 1; j < n_args; ++j)
      if (args[i].vec == args[j].vec) {
        rt->ctx->err = "variable 'x" + std::to_string(args[i].vec) + "' declared twice in one block";
        return COH_E_CONSTRUCTION;
      }
  }
  auto stuck = [&](uint32_t eff, uint32_t s, uint32_t vec, bool abstract, uint32_t actual) {
    rt->ctx->err = std::string("stuck: ") + (s ? "g" : "") + eff_name(eff) + " x" + std::to_string(vec) +
                   (abstract ? "^" : "") + ": have " + pair_str(actual);
    rt->stats.stuck_calls++;
    return COH_E_DEFECT;
  };
  // guards (translate_mode, modes.hpp:31-50): syncs are Local-site effects
  const uint32_t sync = site == COH_REMOTE ? COH_PUSH : COH_PULL;
  for (uint32_t i = 0; i < n_args; ++i) {
    RtVector& v = rt->vec[args[i].vec];
    const uint32_t kind = args[i].kind;
    if (kind == COH_R || kind == COH_RW) {
      const bool valid = site == COH_REMOTE ? (v.abst >> 1) & 1u : v.abst & 1u;
      if (!valid) {
        const int c = apply_pair(sync, COH_LOCAL, v.conc);
        if (c < 0) return stuck(sync, COH_LOCAL, args[i].vec, false, v.conc);
        const int a = apply_pair(sync, COH_LOCAL, v.abst);
        if (a < 0) return stuck(sync, COH_LOCAL, args[i].vec, true, v.abst);
        // the transfer: upload for a GPU component (push), download for a CPU one (pull),
        // each on its side stream, ordered only after the operations that last touched
        // this vector's two copies (other vectors' copies and components overlap it)
        cudaStream_t cs = sync == COH_PUSH ? rt->up : rt->down;
        if (v.dev_pending) cudaStreamWaitEvent(cs, v.dev_last, 0);
        if (v.host_pending) cudaStreamWaitEvent(cs, v.host_last, 0);
        const cudaEvent_t e0 = take_event(rt), e1 = take_event(rt);
        cudaEventRecord(e0, cs);
        cudaError_t e = sync == COH_PUSH ? cudaMemcpyAsync(v.dev, v.host, v.bytes, cudaMemcpyHostToDevice, cs)
                                         : cudaMemcpyAsync(v.host, v.dev, v.bytes, cudaMemcpyDeviceToHost, cs);
        cudaEventRecord(e1, cs);
        rt->ev_open.emplace_back(e0, e1);
        cudaEventRecord(v.dev_last, cs);
        cudaEventRecord(v.host_last, cs);
        v.dev_pending = v.host_pending = true;
        v.host_written = sync == COH_PULL;
        if (e != cudaSuccess) {
          rt->ctx->err = std::string("coh_rt_call copy: ") + cudaGetErrorString(e);
          return COH_E_CUDA;
        }
        if (sync == COH_PUSH) {
          rt->stats.h2d_bytes += v.bytes;
          rt->stats.h2d_copies++;
        } else {
          rt->stats.d2h_bytes += v.bytes;
          rt->stats.d2h_copies++;
        }
        v.conc = (uint32_t)c;
        v.abst = (uint32_t)a;
      } else {
        rt->stats.syncs_elided++;
      }
    }
    if (kind == COH_W || kind == COH_RW) v.abst = (uint32_t)apply_pair(COH_WRITE, site, v.abst);
  }
  // body: the component reads (R/RW) and writes (W/RW) every cell at its site
  for (uint32_t i = 0; i < n_args; ++i) {
    RtVector& v = rt->vec[args[i].vec];
    if (args[i].kind != COH_W && apply_pair(COH_READ, site, v.conc) < 0)
      return stuck(COH_READ, site, args[i].vec, false, v.conc);
  }
  if (site == COH_REMOTE) {
    // the component stream waits for the last operation on each argument's device copy
    // (its upload, an earlier component, or a download still reading it)
    for (uint32_t i = 0; i < n_args; ++i) {
      RtVector& v = rt->vec[args[i].vec];
      if (v.dev_pending) cudaStreamWaitEvent(rt->stream, v.dev_last, 0);
    }
    if (fn) fn(user, rt->stream);
    for (uint32_t i = 0; i < n_args; ++i) {
      RtVector& v = rt->vec[args[i].vec];
      cudaEventRecord(v.dev_last, rt->stream);
      v.dev_pending = true;
    }
  } else if (fn && rt->async_host) {
    // stream-ordered CPU component: the host stream waits for the last operation on each
    // argument's host copy (its download, an upload still reading it, an earlier CPU
    // component), then runs the component on the driver's host-function thread
    for (uint32_t i = 0; i < n_args; ++i) {
      RtVector& v = rt->vec[args[i].vec];
      if (v.host_pending) cudaStreamWaitEvent(rt->host, v.host_last, 0);
    }
    struct Pack {
      coh_rt_fn fn;
      void* user;
    };
    Pack* pk = new Pack{fn, user};
    const cudaError_t e = cudaLaunchHostFunc(
        rt->host,
        [](void* p) {
          Pack* q = static_cast<Pack*>(p);
          q->fn(q->user, nullptr);
          delete q;
        },
        pk);
    if (e != cudaSuccess) {
      delete pk;
      rt->ctx->err = std::string("coh_rt_call host function: ") + cudaGetErrorString(e);
      return COH_E_CUDA;
    }
    for (uint32_t i = 0; i < n_args; ++i) {
      RtVector& v = rt->vec[args[i].vec];
      cudaEventRecord(v.host_last, rt->host);
      v.host_pending = true;
      v.host_written = true;
    }
  } else if (fn) {
    // the host thread waits only for its arguments: their downloads (read after write),
    // and for an argument it writes, an upload still reading the host copy
    for (uint32_t i = 0; i < n_args; ++i) {
      RtVector& v = rt->vec[args[i].vec];
      if (v.host_pending && (v.host_written || args[i].kind != COH_R)) {
        const cudaError_t e = cudaEventSynchronize(v.host_last);
        if (e != cudaSuccess) {
          rt->ctx->err = std::string("coh_rt_call sync: ") + cudaGetErrorString(e);
          return COH_E_CUDA;
        }
        v.host_pending = false;
      }
    }
    fn(user, nullptr);
  }
  for (uint32_t i = 0; i < n_args; ++i) {
    RtVector& v = rt->vec[args[i].vec];
    if (args[i].kind != COH_R) v.conc = (uint32_t)apply_pair(COH_WRITE, site, v.conc);
  }
  rt->stats.calls++;
  return COH_OK;
}

int coh_rt_sync(coh_rt* rt) {
  if (!rt) return COH_E_ARG;
  cudaError_t e = cudaStreamSynchronize(rt->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(rt->up);
  if (e == cudaSuccess) e = cudaStreamSynchronize(rt->down);
  if (e == cudaSuccess && rt->host) e = cudaStreamSynchronize(rt->host);
  for (auto& v : rt->vec) v.dev_pending = v.host_pending = false;
  if (e != cudaSuccess) {
    rt->ctx->err = std::string("coh_rt_sync: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  harvest(rt);
  return COH_OK;
}

int coh_rt_set_async(coh_rt* rt, int on) {
  if (!rt) return COH_E_ARG;
  if (on && !rt->host && cudaStreamCreateWithFlags(&rt->host, cudaStreamNonBlocking) != cudaSuccess) {
    rt->ctx->err = "coh_rt_set_async: stream";
    return COH_E_CUDA;
  }
  rt->async_host = on != 0;
  return COH_OK;
}

int coh_rt_get_stats(const coh_rt* rt, coh_rt_stats* out) {
  if (!rt || !out) return COH_E_ARG;
  *out = rt->stats;
  return COH_OK;
}

// ---- views: element-granular validity (pvector<T>) -----------------

int coh_rt_buffer(coh_rt* rt, uint32_t n_cells, uint32_t elem_bytes, uint32_t* id) {
  if (!rt || !id || n_cells == 0 || elem_bytes == 0) return COH_E_ARG;
  RtBuffer b;
  b.n_cells = n_cells;
  b.elem_bytes = elem_bytes;
  b.W = ((n_cells + 31u) / 32u + 3u) & ~3u;
  b.cap = (uint64_t)n_cells / 2u + 2u;  // at most one run per two cells
  const size_t bytes = (size_t)n_cells * elem_bytes;
  bool ok = cudaHostAlloc(&b.host, bytes, cudaHostAllocDefault) == cudaSuccess &&
            cudaMalloc(&b.dev, bytes) == cudaSuccess &&
            cudaMalloc(reinterpret_cast<void**>(&b.planes), (size_t)2 * b.W * 4) == cudaSuccess &&
            cudaMalloc(reinterpret_cast<void**>(&b.d_rng), 2 * sizeof(coh_bitmap_range)) == cudaSuccess &&
            cudaMalloc(reinterpret_cast<void**>(&b.d_first), 16) == cudaSuccess &&
            cudaMalloc(reinterpret_cast<void**>(&b.d_off), 16) == cudaSuccess &&
            cudaMalloc(reinterpret_cast<void**>(&b.d_runs), (size_t)2 * b.cap * 4) == cudaSuccess &&
            cudaHostAlloc(reinterpret_cast<void**>(&b.h_io), (size_t)(8 + 2 * b.cap) * 4, cudaHostAllocDefault) ==
                cudaSuccess;
  // initial_store (program.hpp:174-184): every cell (V,I) -> L = 1, R = 0 (bits past
  // n_cells stay 0)
  ok = ok && cudaMemsetAsync(b.planes, 0, (size_t)2 * b.W * 4, rt->stream) == cudaSuccess;
  if (ok) {
    const coh_bitmap_range all{0, 0, n_cells - 1};
    ok = cudaMemcpyAsync(b.d_rng, &all, sizeof all, cudaMemcpyHostToDevice, rt->stream) == cudaSuccess &&
         coh_bitmap_range_set(rt->ctx, b.planes, b.d_rng, 1, rt->stream) == COH_OK;
  }
  if (!ok) {
    cudaFreeHost(b.host);
    cudaFreeHost(b.h_io);
    cudaFree(b.dev);
    cudaFree(b.planes);
    cudaFree(b.d_rng);
    cudaFree(b.d_first);
    cudaFree(b.d_off);
    cudaFree(b.d_runs);
    rt->ctx->err = "coh_rt_buffer: allocation of " + std::to_string(bytes) + " bytes";
    return COH_E_CUDA;
  }
  *id = (uint32_t)rt->buf.size();
  rt->buf.push_back(b);
  return COH_OK;
}

int coh_rt_view(coh_rt* rt, uint32_t buffer, uint32_t lo, uint32_t hi, uint32_t* view_index) {
  if (!rt || !view_index || buffer >= rt->buf.size()) return COH_E_ARG;
  RtBuffer& b = rt->buf[buffer];
  if (lo > hi || hi >= b.n_cells) {  // program.hpp:65-68
    rt->ctx->err = "view range does not fit its buffer";
    return COH_E_CONSTRUCTION;
  }
  if (b.lo.size() >= COH_MAX_VIEWS) {
    rt->ctx->err = "too many views on one buffer";
    return COH_E_CONSTRUCTION;
  }
  *view_index = (uint32_t)b.lo.size();
  b.lo.push_back(lo);
  b.hi.push_back(hi);
  b.abst.push_back(1u);  // v^ starts (V,I)
  return COH_OK;
}

int coh_rt_view_state(coh_rt* rt, uint32_t buffer, uint32_t view_index, uint8_t* abs_pair) {
  if (!rt || !abs_pair || buffer >= rt->buf.size() || view_index >= rt->buf[buffer].abst.size()) return COH_E_ARG;
  *abs_pair = (uint8_t)rt->buf[buffer].abst[view_index];
  return COH_OK;
}

void* coh_rt_buffer_host_ptr(coh_rt* rt, uint32_t buffer) {
  return rt && buffer < rt->buf.size() ? rt->buf[buffer].host : nullptr;
}
void* coh_rt_buffer_device_ptr(coh_rt* rt, uint32_t buffer) {
  return rt && buffer < rt->buf.size() ? rt->buf[buffer].dev : nullptr;
}

int coh_rt_buffer_planes(coh_rt* rt, uint32_t buffer, uint32_t* planes_out) {
  if (!rt || !planes_out || buffer >= rt->buf.size()) return COH_E_ARG;
  const RtBuffer& b = rt->buf[buffer];
  const size_t words = (b.n_cells + 31u) / 32u;
  if (cudaMemcpy2DAsync(planes_out, words * 4, b.planes, (size_t)b.W * 4, words * 4, 2, cudaMemcpyDeviceToHost,
                        rt->stream) != cudaSuccess ||
      cudaStreamSynchronize(rt->stream) != cudaSuccess) {
    rt->ctx->err = "coh_rt_buffer_planes: copy";
    return COH_E_CUDA;
  }
  harvest(rt);
  return COH_OK;
}

int coh_rt_copy_log(const coh_rt* rt, coh_rt_copy* out, uint64_t cap, uint64_t* n) {
  if (!rt || !n || (cap && !out)) return COH_E_ARG;
  *n = rt->log.size();
  const size_t k = (size_t)std::min<uint64_t>(cap, rt->log.size());
  if (k) std::memcpy(out, rt->log.data(), sizeof(coh_rt_copy) * k);  // (out may be NULL when cap == 0)
  return COH_OK;
}

namespace {

// One whole-view or body range on plane p (0 = L, 1 = R) of buffer b, into the device
// range slot k.
coh_bitmap_range plane_range(const RtBuffer& b, uint32_t p, uint32_t lo, uint32_t hi) {
  return coh_bitmap_range{(uint64_t)p * b.W, lo, hi};
}

int upload_ranges(coh_rt* rt, RtBuffer& b, const coh_bitmap_range* r, uint32_t n) {
  // from pageable memory (the caller's locals): the copy is staged before the call returns,
  // so back-to-back uploads cannot overwrite a range a queued kernel has yet to read
  const cudaError_t e = cudaMemcpyAsync(b.d_rng, r, sizeof(coh_bitmap_range) * n, cudaMemcpyHostToDevice, rt->stream);
  if (e != cudaSuccess) {
    rt->ctx->err = std::string("view range upload: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

// first cell of [lo, hi] whose bit in plane p is 0, or kNoCell (synchronises)
int first_zero(coh_rt* rt, RtBuffer& b, uint32_t p, uint32_t lo, uint32_t hi, uint32_t* cell) {
  const coh_bitmap_range r = plane_range(b, p, lo, hi);
  int rc = upload_ranges(rt, b, &r, 1);
  if (!rc) rc = coh_bitmap_first_zero(rt->ctx, b.planes, b.d_rng, 1, b.d_first, rt->stream);
  if (rc) return rc;
  if (cudaMemcpyAsync(b.h_io, b.d_first, 4, cudaMemcpyDeviceToHost, rt->stream) != cudaSuccess ||
      cudaStreamSynchronize(rt->stream) != cudaSuccess) {
    rt->ctx->err = "view first-zero readback";
    return COH_E_CUDA;
  }
  harvest(rt);
  *cell = b.h_io[0];
  return COH_OK;
}

int set_range(coh_rt* rt, RtBuffer& b, uint32_t p, uint32_t lo, uint32_t hi, bool value) {
  const coh_bitmap_range r = plane_range(b, p, lo, hi);
  int rc = upload_ranges(rt, b, &r, 1);
  if (rc) return rc;
  return value ? coh_bitmap_range_set(rt->ctx, b.planes, b.d_rng, 1, rt->stream)
               : coh_bitmap_range_clear(rt->ctx, b.planes, b.d_rng, 1, rt->stream);
}

}  // namespace

int coh_rt_call_view(coh_rt* rt, uint32_t buffer, const coh_elem_call* call, coh_rt_fn fn, void* user) {
  if (!rt || !call || buffer >= rt->buf.size()) return COH_E_ARG;
  RtBuffer& b = rt->buf[buffer];
  const uint32_t nv = (uint32_t)b.lo.size();
  if (call->view >= nv || call->kind > COH_RW || call->site > COH_REMOTE || call->n_body > 2) {
    rt->ctx->err = "coh_rt_call_view: malformed call";
    return COH_E_CONSTRUCTION;
  }
  const uint32_t vlo = b.lo[call->view], vlen = b.hi[call->view] - vlo + 1;
  for (uint32_t k = 0; k < call->n_body; ++k) {
    const coh_elem_op& op = call->body[k];
    if (op.lo > op.hi || op.hi >= vlen || (op.effect != COH_READ && op.effect != COH_WRITE) || op.site > COH_REMOTE) {
      rt->ctx->err = "coh_rt_call_view: malformed body op";
      return COH_E_CONSTRUCTION;
    }
  }
  auto stuck = [&](const std::string& what) {
    rt->ctx->err = "stuck: " + what;
    rt->stats.stuck_calls++;
    return COH_E_DEFECT;
  };
  // infer_overlap_closure (overlap.hpp:182-230): W/RW on x adds RW@site on every
  // overlapping view, in declaration order; an R infers nothing
  struct M {
    uint32_t view, kind;
  };
  std::vector<M> modes{{call->view, call->kind}};
  if (call->kind != COH_R)
    for (uint32_t y = 0; y < nv; ++y)
      if (y != call->view && b.lo[y] <= b.hi[call->view] && b.lo[call->view] <= b.hi[y]) modes.push_back({y, COH_RW});
  const uint32_t site = call->site;
  for (const M& m : modes) {
    const uint32_t v = m.view, lo = b.lo[v], hi = b.hi[v];
    if (m.kind == COH_R || m.kind == COH_RW) {
      const bool valid = site ? (b.abst[v] >> 1) & 1u : b.abst[v] & 1u;
      if (!valid) {
        // concrete whole-view sync, Local site (ast.hpp:144): pull needs R and sets L
        // (the download before a CPU component), push needs L and sets R (the upload)
        const uint32_t sync = site ? COH_PUSH : COH_PULL;
        const uint32_t src = sync == COH_PULL ? 1u : 0u, dst = 1u - src;
        const coh_bitmap_range r[2] = {plane_range(b, src, lo, hi), plane_range(b, dst, lo, hi)};
        int rc = upload_ranges(rt, b, r, 2);
        if (!rc) rc = coh_bitmap_first_zero(rt->ctx, b.planes, b.d_rng, 1, b.d_first, rt->stream);
        if (!rc)
          rc = coh_bitmap_extract_zero_runs(rt->ctx, b.planes, b.d_rng + 1, 1, b.d_runs, b.d_runs + b.cap, b.cap,
                                            b.d_off, rt->stream);
        if (rc) return rc;
        // one readback: the first zero of the source, then the runs of the destination
        uint64_t* h_off = reinterpret_cast<uint64_t*>(b.h_io + 2);
        if (cudaMemcpyAsync(b.h_io, b.d_first, 4, cudaMemcpyDeviceToHost, rt->stream) != cudaSuccess ||
            cudaMemcpyAsync(h_off, b.d_off, 16, cudaMemcpyDeviceToHost, rt->stream) != cudaSuccess ||
            cudaStreamSynchronize(rt->stream) != cudaSuccess) {
          rt->ctx->err = "view sync readback";
          return COH_E_CUDA;
        }
        harvest(rt);
        if (b.h_io[0] != 0xFFFFFFFFu)  // atomic sync: nothing is written (semantics.hpp:155-166)
          return stuck(std::string(sync == COH_PULL ? "pull" : "push") + " view " + std::to_string(v) + " at cell " +
                       std::to_string(b.h_io[0]));
        const uint64_t n_runs = h_off[1] - h_off[0];
        uint32_t* h_runs = b.h_io + 8;
        if (n_runs) {
          if (cudaMemcpyAsync(h_runs, b.d_runs, n_runs * 4, cudaMemcpyDeviceToHost, rt->stream) != cudaSuccess ||
              cudaMemcpyAsync(h_runs + n_runs, b.d_runs + b.cap, n_runs * 4, cudaMemcpyDeviceToHost, rt->stream) !=
                  cudaSuccess ||
              cudaStreamSynchronize(rt->stream) != cudaSuccess) {
            rt->ctx->err = "view runs readback";
            return COH_E_CUDA;
          }
          harvest(rt);
        }
        for (uint64_t k = 0; k < n_runs; ++k) {  // the transfer ranges: one copy each
          const uint32_t a = h_runs[k], z = h_runs[n_runs + k];
          const size_t off = (size_t)a * b.elem_bytes, bytes = (size_t)(z - a + 1) * b.elem_bytes;
          char* hp = static_cast<char*>(b.host) + off;
          char* dp = static_cast<char*>(b.dev) + off;
          const cudaEvent_t e0 = take_event(rt), e1 = take_event(rt);
          cudaEventRecord(e0, rt->stream);
          const cudaError_t e = sync == COH_PUSH ? cudaMemcpyAsync(dp, hp, bytes, cudaMemcpyHostToDevice, rt->stream)
                                                 : cudaMemcpyAsync(hp, dp, bytes, cudaMemcpyDeviceToHost, rt->stream);
          cudaEventRecord(e1, rt->stream);
          rt->ev_open.emplace_back(e0, e1);
          if (e != cudaSuccess) {
            rt->ctx->err = std::string("view copy: ") + cudaGetErrorString(e);
            return COH_E_CUDA;
          }
          if (sync == COH_PUSH) {
            rt->stats.h2d_bytes += bytes;
            rt->stats.h2d_copies++;
          } else {
            rt->stats.d2h_bytes += bytes;
            rt->stats.d2h_copies++;
          }
          rt->log.push_back(coh_rt_copy{buffer, a, z, sync == COH_PUSH ? 1u : 0u});
        }
        if ((rc = set_range(rt, b, dst, lo, hi, true))) return rc;
        const int a = apply_pair(sync, COH_LOCAL, b.abst[v]);
        if (a < 0) return stuck(std::string(sync == COH_PULL ? "pull" : "push") + " view " + std::to_string(v) + "^");
        b.abst[v] = (uint32_t)a;
      } else {
        rt->stats.syncs_elided++;
      }
    }
    if (m.kind == COH_W || m.kind == COH_RW) b.abst[v] = (uint32_t)apply_pair(COH_WRITE, site, b.abst[v]);
  }
  // body ops in order: a READ needs the op site's plane on its range, a WRITE sets it and
  // clears the other (partial effects persist when a READ gets stuck)
  for (uint32_t k = 0; k < call->n_body; ++k) {
    const coh_elem_op& op = call->body[k];
    const uint32_t lo = vlo + op.lo, hi = vlo + op.hi, p = op.site ? 1u : 0u;
    int rc;
    if (op.effect == COH_READ) {
      uint32_t cell = 0;
      if ((rc = first_zero(rt, b, p, lo, hi, &cell))) return rc;
      if (cell != 0xFFFFFFFFu) return stuck("r at cell " + std::to_string(cell));
    } else {
      if ((rc = set_range(rt, b, p, lo, hi, true)) || (rc = set_range(rt, b, 1u - p, lo, hi, false))) return rc;
    }
  }
  if (fn) {
    if (site == COH_REMOTE) {
      fn(user, rt->stream);
    } else {
      const cudaError_t e = cudaStreamSynchronize(rt->stream);  // the downloads land first
      if (e != cudaSuccess) {
        rt->ctx->err = std::string("coh_rt_call_view sync: ") + cudaGetErrorString(e);
        return COH_E_CUDA;
      }
      harvest(rt);
      fn(user, nullptr);
    }
  }
  rt->stats.calls++;
  return COH_OK;
}

// ---- built-in components (trivial bodies: the point of C5 is the coherence traffic) ----
// user -> coh_rt_touch { rt, n, vec[8], kind[8] }: written vectors get x = x * 0.5f + 1,
// read vectors are summed into a checksum (so the reads are real).
void coh_rt_touch_cpu(void* user, void* /*stream*/) {
  coh_rt_touch* t = static_cast<coh_rt_touch*>(user);
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  for (uint32_t k = 0; k < t->n; ++k) {
    RtVector& v = t->rt->vec[t->vec[k]];
    float* x = static_cast<float*>(v.host);
    const size_t n = v.bytes / sizeof(float);
    const bool write = t->kind[k] != COH_R;
    std::vector<std::thread> pool;
    std::vector<double> part(nth, 0.0);
    for (unsigned w = 0; w < nth; ++w)
      pool.emplace_back([&, w] {
        const size_t lo = n * w / nth, hi = n * (w + 1) / nth;
        double s = 0;
        if (t->kind[k] == COH_W)
          for (size_t i = lo; i < hi; ++i) x[i] = 1.0f;
        else if (write)
          for (size_t i = lo; i < hi; ++i) x[i] = x[i] * 0.5f + 1.0f;
        else
          for (size_t i = lo; i < hi; i += 16) s += x[i];
        part[w] = s;
      });
    for (auto& th : pool) th.join();
    for (double s : part) t->checksum += s;
  }
}

}  // extern "C"
