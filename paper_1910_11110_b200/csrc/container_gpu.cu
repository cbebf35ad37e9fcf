// Built-in GPU component of the container runtime (trivial body, see coh_rt_touch).
#include <cuda_runtime.h>

#include "internal.hpp"

namespace {
__global__ void k_touch(float4* x, size_t n4, uint32_t kind, double* sum) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v;
    if (kind == COH_W) {
      v = make_float4(1.f, 1.f, 1.f, 1.f);
      x[i] = v;
    } else {
      v = x[i];
      if (kind == COH_RW) {
        v = make_float4(v.x * 0.5f + 1.f, v.y * 0.5f + 1.f, v.z * 0.5f + 1.f, v.w * 0.5f + 1.f);
        x[i] = v;
      } else {
        s += v.x;
      }
    }
  }
  if (kind == COH_R && s != 0.0) atomicAdd(sum, s);
}
}  // namespace

extern "C" void coh_rt_touch_gpu(void* user, void* stream) {
  coh_rt_touch* t = static_cast<coh_rt_touch*>(user);
  static double* d_sum = nullptr;
  if (!d_sum) cudaMalloc(&d_sum, sizeof(double));
  for (uint32_t k = 0; k < t->n; ++k) {
    float4* x = static_cast<float4*>(coh_rt_device_ptr(t->rt, t->vec[k]));
    const size_t bytes = t->bytes[k];  // float vectors, multiples of 16 bytes
    k_touch<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, bytes / 16, t->kind[k], d_sum);
  }
}
