// Coherent-container runtime (config C5): VectorPU's coherence control
// (coherent_on_{cpu,gpu}_{r,w,rw}, download/upload) rebuilt on the
// calculus.  Each vector keeps the calculus state of its whole-array variable — concrete
// pair (which copies really hold the data) and abstract pair (the flags VectorPU keeps,
// PAPER.md:1211) — and a component call executes exactly the translated block
// (modes.hpp:31-59): for every argument in order, the guard on the abstract flag decides
// whether to copy (`pull x` = cudaMemcpyAsync D2H for a CPU component, `push x` = H2D for
// a GPU component), then `w x^` for W/RW; then the component runs (CPU: on the calling
// thread after the stream drains; GPU: launched on the runtime stream); then its body
// effects (R: `r x`, W: `w x`, RW: both, at the component's site).  A step that cannot
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
};

struct coh_rt {
  coh_ctx* ctx = nullptr;
  std::vector<RtVector> vec;
  cudaStream_t stream = nullptr;
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
  if (cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking) != cudaSuccess) {
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
  harvest(rt);
  for (cudaEvent_t e : rt->ev_free) cudaEventDestroy(e);
  for (auto& v : rt->vec) {
    cudaFreeHost(v.host);
    cudaFree(v.dev);
  }
  cudaStreamDestroy(rt->stream);
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
        // the transfer: upload for a GPU component (push), download for a CPU one (pull)
        const cudaEvent_t e0 = take_event(rt), e1 = take_event(rt);
        cudaEventRecord(e0, rt->stream);
        cudaError_t e = sync == COH_PUSH
                            ? cudaMemcpyAsync(v.dev, v.host, v.bytes, cudaMemcpyHostToDevice, rt->stream)
                            : cudaMemcpyAsync(v.host, v.dev, v.bytes, cudaMemcpyDeviceToHost, rt->stream);
        cudaEventRecord(e1, rt->stream);
        rt->ev_open.emplace_back(e0, e1);
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
  if (fn) {
    if (site == COH_REMOTE) {
      fn(user, rt->stream);
    } else {
      cudaError_t e = cudaStreamSynchronize(rt->stream);  // copies (and earlier GPU work) land first
      if (e != cudaSuccess) {
        rt->ctx->err = std::string("coh_rt_call sync: ") + cudaGetErrorString(e);
        return COH_E_CUDA;
      }
      harvest(rt);
      fn(user, nullptr);
    }
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
  if (e != cudaSuccess) {
    rt->ctx->err = std::string("coh_rt_sync: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  harvest(rt);
  return COH_OK;
}

int coh_rt_get_stats(const coh_rt* rt, coh_rt_stats* out) {
  if (!rt || !out) return COH_E_ARG;
  *out = rt->stats;
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
