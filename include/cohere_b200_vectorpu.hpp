// cohere_b200_vectorpu.hpp — a header-only C++ facade restoring VectorPU's programming
// surface on top of the C ABI in cohere_b200.h:
//
//   coh::vpu::runtime rt(ctx);
//   coh::vpu::vector<float> x(rt, n), y(rt, n);
//   float* hx = coh::vpu::W(x);          // CPU write: x's host copy, no transfer
//   kernel<<<g, b, 0, rt.stream()>>>(coh::vpu::GR(x), coh::vpu::GW(y), n);   // uploads x
//   const float* hy = coh::vpu::R(y);    // CPU read: downloads y (after the kernel)
//   coh::vpu::pvector<float> v(x, 1000, 1999);   // a view of x's cells [1000, 1999]
//   float* dv = coh::vpu::GRW(v);        // uploads only v's cells the GPU lacks
//
// Each accessor is one annotated component argument (a block with one mode, modes.hpp:
// 31-59): it runs the calculus' guard — the copies the evaluator predicts, issued with
// cudaMemcpyAsync on the runtime stream — then the mode's abstract write and body effect,
// and returns the pointer the component uses (host for R/W/RW, device for GR/GW/GRW; a
// pvector's pointer is offset to its first cell).  CPU accessors return after the stream
// drained, so the host data is current.  Unlike VectorPU the containers start at the
// calculus' initial store (V,I), the state its evaluator assumes.
// Errors (a stuck step: data valid nowhere the mode needs it) throw coh::vpu::error with
// coh_last_error's text.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "cohere_b200.h"

namespace coh {
namespace vpu {

struct error : std::runtime_error {
  int code;
  error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

class runtime {
 public:
  explicit runtime(coh_ctx* ctx) : ctx_(ctx) { check(coh_rt_create(ctx, &rt_), "coh_rt_create"); }
  ~runtime() { coh_rt_destroy(rt_); }
  runtime(const runtime&) = delete;
  runtime& operator=(const runtime&) = delete;

  coh_rt* handle() const { return rt_; }
  void* stream() const { return coh_rt_stream(rt_); }
  void sync() { check(coh_rt_sync(rt_), "coh_rt_sync"); }
  coh_rt_stats stats() const {
    coh_rt_stats s{};
    coh_rt_get_stats(rt_, &s);
    return s;
  }
  void check(int rc, const char* what) const {
    if (rc != COH_OK) throw error(rc, std::string(what) + ": " + coh_last_error(ctx_));
  }

 private:
  coh_ctx* ctx_;
  coh_rt* rt_ = nullptr;
};

// A whole-array container: one calculus variable (one validity pair for all elements).
// Backed by a buffer so that pvector views of it share its element-granular validity.
template <class T>
class vector {
 public:
  vector(runtime& rt, size_t n) : rt_(&rt), n_(n) {
    rt.check(coh_rt_buffer(rt.handle(), (uint32_t)n, (uint32_t)sizeof(T), &buf_), "coh_rt_buffer");
    rt.check(coh_rt_view(rt.handle(), buf_, 0, (uint32_t)n - 1, &whole_), "coh_rt_view");
  }
  size_t size() const { return n_; }
  runtime& rt() const { return *rt_; }
  uint32_t buffer() const { return buf_; }
  uint32_t whole_view() const { return whole_; }
  T* host() const { return static_cast<T*>(coh_rt_buffer_host_ptr(rt_->handle(), buf_)); }
  T* device() const { return static_cast<T*>(coh_rt_buffer_device_ptr(rt_->handle(), buf_)); }

 private:
  runtime* rt_;
  size_t n_;
  uint32_t buf_ = 0, whole_ = 0;
};

// pvector<T>(mother, lo, hi): the mother's cells [lo, hi] (inclusive).
// Declare views before the mother is used by a component (declaration order is the
// closure's order, overlap.hpp:212-228).
template <class T>
class pvector {
 public:
  pvector(vector<T>& mother, size_t lo, size_t hi) : m_(&mother), lo_(lo), hi_(hi) {
    mother.rt().check(coh_rt_view(mother.rt().handle(), mother.buffer(), (uint32_t)lo, (uint32_t)hi, &view_),
                      "coh_rt_view");
  }
  size_t size() const { return hi_ - lo_ + 1; }
  vector<T>& mother() const { return *m_; }
  uint32_t view() const { return view_; }
  size_t lo() const { return lo_; }

 private:
  vector<T>* m_;
  size_t lo_, hi_;
  uint32_t view_ = 0;
};

namespace detail {
// one component argument: mode `kind` at `site` on view `view`, the component reads
// (R, RW) and writes (W, RW) all of the view's cells
template <class T>
T* access(vector<T>& m, uint32_t view, size_t lo, size_t len, uint32_t kind, uint32_t site) {
  runtime& rt = m.rt();
  coh_elem_call c{};
  c.view = view;
  c.kind = (uint8_t)kind;
  c.site = (uint8_t)site;
  uint32_t k = 0;
  if (kind != COH_W) c.body[k++] = coh_elem_op{(uint8_t)COH_READ, (uint8_t)site, 0, 0, (uint32_t)len - 1};
  if (kind != COH_R) c.body[k++] = coh_elem_op{(uint8_t)COH_WRITE, (uint8_t)site, 0, 0, (uint32_t)len - 1};
  c.n_body = (uint8_t)k;
  rt.check(coh_rt_call_view(rt.handle(), m.buffer(), &c, nullptr, nullptr), "component argument");
  if (site == COH_LOCAL) rt.sync();  // host data current before the CPU component runs
  return (site == COH_LOCAL ? m.host() : m.device()) + lo;
}
}  // namespace detail

// CPU modes (host pointers)
template <class T> T* R(vector<T>& x) { return detail::access(x, x.whole_view(), 0, x.size(), COH_R, COH_LOCAL); }
template <class T> T* W(vector<T>& x) { return detail::access(x, x.whole_view(), 0, x.size(), COH_W, COH_LOCAL); }
template <class T> T* RW(vector<T>& x) { return detail::access(x, x.whole_view(), 0, x.size(), COH_RW, COH_LOCAL); }
// GPU modes (device pointers; launch the component on rt.stream())
template <class T> T* GR(vector<T>& x) { return detail::access(x, x.whole_view(), 0, x.size(), COH_R, COH_REMOTE); }
template <class T> T* GW(vector<T>& x) { return detail::access(x, x.whole_view(), 0, x.size(), COH_W, COH_REMOTE); }
template <class T> T* GRW(vector<T>& x) { return detail::access(x, x.whole_view(), 0, x.size(), COH_RW, COH_REMOTE); }
// the same on views
template <class T> T* R(pvector<T>& v) { return detail::access(v.mother(), v.view(), v.lo(), v.size(), COH_R, COH_LOCAL); }
template <class T> T* W(pvector<T>& v) { return detail::access(v.mother(), v.view(), v.lo(), v.size(), COH_W, COH_LOCAL); }
template <class T> T* RW(pvector<T>& v) { return detail::access(v.mother(), v.view(), v.lo(), v.size(), COH_RW, COH_LOCAL); }
template <class T> T* GR(pvector<T>& v) { return detail::access(v.mother(), v.view(), v.lo(), v.size(), COH_R, COH_REMOTE); }
template <class T> T* GW(pvector<T>& v) { return detail::access(v.mother(), v.view(), v.lo(), v.size(), COH_W, COH_REMOTE); }
template <class T> T* GRW(pvector<T>& v) { return detail::access(v.mother(), v.view(), v.lo(), v.size(), COH_RW, COH_REMOTE); }

}  // namespace vpu
}  // namespace coh
