// VectorPU-style program through include/cohere_b200_vectorpu.hpp (built and run by
// tests/test_vpu_facade.py on the GPU box).  Prints "ok" and the copy log when every check
// passes, exits non-zero otherwise.
#include <cstdio>
#include <vector>

#include "cohere_b200_vectorpu.hpp"

__global__ void twice(float* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] *= 2.0f;
}

int main() {
  coh_ctx* ctx = nullptr;
  if (coh_ctx_create(0, &ctx) != COH_OK) return 2;
  int bad = 0;
  {
    namespace vpu = coh::vpu;
    vpu::runtime rt(ctx);
    const int n = 4096;
    vpu::vector<float> x(rt, n);
    vpu::pvector<float> v(x, 100, 199);
    float* hx = vpu::W(x);  // CPU write: no transfer
    for (int i = 0; i < n; ++i) hx[i] = (float)i;
    vpu::GR(x);  // the GPU reads all of x: one upload of every cell
    float* dv = vpu::GRW(v);  // the GPU updates v: already valid there, no transfer
    twice<<<1, 128, 0, (cudaStream_t)rt.stream()>>>(dv, (int)v.size());
    const float* hx2 = vpu::R(x);  // the CPU reads x: downloads only v's cells
    for (int i = 0; i < n; ++i) {
      const float want = (i >= 100 && i <= 199) ? 2.0f * i : (float)i;
      if (hx2[i] != want) {
        if (bad < 5) std::printf("cell %d: %f != %f\n", i, hx2[i], want);
        ++bad;
      }
    }
    coh_rt_copy log[8];
    uint64_t nlog = 0;
    coh_rt_copy_log(rt.handle(), log, 8, &nlog);
    for (uint64_t k = 0; k < nlog && k < 8; ++k)
      std::printf("copy %u..%u %s\n", log[k].first, log[k].last, log[k].h2d ? "h2d" : "d2h");
    if (nlog != 2 || log[0].first != 0 || log[0].last != n - 1 || !log[0].h2d || log[1].first != 100 ||
        log[1].last != 199 || log[1].h2d)
      ++bad;
    // a CPU write of x closes over v (shadow RW: v's cells are already valid on the
    // CPU), then a CPU read of v: nothing more to copy
    vpu::W(x);
    vpu::R(v);
    coh_rt_copy_log(rt.handle(), log, 8, &nlog);
    if (nlog != 2) ++bad;
  }
  coh_ctx_destroy(ctx);
  if (bad) return 1;
  std::printf("ok\n");
  return 0;
}
