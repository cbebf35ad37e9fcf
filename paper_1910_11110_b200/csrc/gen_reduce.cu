// Device-side synthetic record generator (records materialised in HBM)
// and the per-batch counter reduction that feeds the multi-GPU allreduce (§8(e)).
#include <cuda_runtime.h>

#include "gen_common.h"
#include "internal.hpp"

namespace cohb {

// One thread writes one 16-byte chunk (8 calls of one trace): coalesced across the warp.
__global__ void k_gen_records(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                              uint32_t n_arrays, uint32_t adv, uint4* out) {
  const uint32_t n_chunks = (n_calls + 7u) / 8u;
  const uint64_t total = (uint64_t)n_chunks * n_traces;
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(idx / n_traces);
    const uint64_t t = idx - (uint64_t)c * n_traces;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i0 = c * 8u + 2u * k, i1 = i0 + 1u;
      const uint32_t r0 = i0 < n_calls ? coh_gen_record(seed, trace0 + t, i0, n_arrays, adv) : 0u;
      const uint32_t r1 = i1 < n_calls ? coh_gen_record(seed, trace0 + t, i1, n_arrays, adv) : 0u;
      w[k] = r0 | (r1 << 16);
    }
    out[idx] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// COH_REC_CONT bits (coh_gen_cont): one thread walks one trace's calls in order, keeping the
// set of arrays of the current block.
__global__ void k_gen_blocks(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls, uint32_t cont,
                             uint16_t* rec) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_traces;
       t += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long in_block = 0ull;
    for (uint32_t i = 0; i < n_calls; ++i) {
      uint16_t* p = rec + ((uint64_t)(i >> 3) * n_traces + t) * 8u + (i & 7u);
      const uint16_t r = *p;
      const unsigned long long bit = 1ull << COH_REC_ARRAY(r);
      if (i > 0 && !(in_block & bit) && coh_gen_cont(seed, trace0 + t, i, cont)) {
        *p = (uint16_t)(r | COH_REC_CONT);
        in_block |= bit;
      } else {
        in_block = bit;
      }
    }
  }
}

// 12 bytes (8 calls of 12 bits) -> one 16-byte chunk of 16-bit records, per thread.
__global__ void k_unpack12(const uint32_t* __restrict__ src, uint4* __restrict__ dst, uint64_t total) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w0 = __ldcs(src + 3 * q), w1 = __ldcs(src + 3 * q + 1), w2 = __ldcs(src + 3 * q + 2);
    const uint64_t lo = (uint64_t)w0 | ((uint64_t)w1 << 32);
    uint32_t r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t bit = 12u * k;
      uint32_t v;
      if (bit + 12u <= 64u) v = (uint32_t)(lo >> bit) & 0xFFFu;
      else if (bit >= 64u) v = (w2 >> (bit - 64u)) & 0xFFFu;
      else v = (uint32_t)((lo >> bit) | ((uint64_t)w2 << (64u - bit))) & 0xFFFu;
      r[k] = ((v >> 6) << 8) | ((v & 63u) << 2);  // array in bits 8-13, call type in bits 2-7
    }
    __stcs(dst + q, make_uint4(r[0] | (r[1] << 16), r[2] | (r[3] << 16), r[4] | (r[5] << 16), r[6] | (r[7] << 16)));
  }
}

int launch_unpack12(const uint8_t* d_packed, uint16_t* d_records, uint64_t n_traces, uint32_t n_chunks, void* stream,
                    std::string* err) {
  const uint64_t total = (uint64_t)n_chunks * n_traces;
  if (!total) return COH_OK;
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  k_unpack12<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint32_t*>(d_packed), reinterpret_cast<uint4*>(d_records), total);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("unpack12 launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

int launch_gen_blocks(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls, uint32_t cont,
                      uint16_t* d_records, void* stream, std::string* err) {
  if (!n_traces || !n_calls || !cont) return COH_OK;
  uint64_t blocks = (n_traces + 127) / 128;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  k_gen_blocks<<<(unsigned)blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(seed, trace0, n_traces, n_calls, cont,
                                                                                d_records);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("gen_blocks launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

int launch_gen_records(uint64_t seed, uint64_t trace0, uint64_t n_traces, uint32_t n_calls,
                       uint32_t n_arrays, uint32_t adv, uint16_t* d_records, void* stream,
                       std::string* err) {
  const uint64_t total = (uint64_t)((n_calls + 7u) / 8u) * n_traces;
  if (total == 0) return COH_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (total + 255) / 256;
  const uint64_t cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  k_gen_records<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, trace0, n_traces, n_calls, n_arrays, adv, reinterpret_cast<uint4*>(d_records));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("gen_records launch: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

// Counters (include/cohere_b200.h, COH_N_COUNTERS): grid-stride accumulation, warp
// shuffle + shared-memory block reduction, then one atomic per counter per block (a
// per-warp atomic made this kernel contention-bound).
constexpr int kRedThreads = 256;
__global__ void __launch_bounds__(kRedThreads) k_reduce_counters(const coh_trace_result* __restrict__ r,
                                                                 uint64_t n, unsigned long long* __restrict__ out) {
  __shared__ uint64_t part[kRedThreads / 32][COH_N_COUNTERS];
  uint64_t c[COH_N_COUNTERS] = {0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 q2 = __ldcs(reinterpret_cast<const uint4*>(r + i) + 2);
    const uint4 q3 = __ldcs(reinterpret_cast<const uint4*>(r + i) + 3);
    const uint32_t status = q3.w & 0xFFu;
    c[0] += status == COH_RUN_STUCK;
    c[1] += status == COH_RUN_FUEL_EXHAUSTED;
    c[2] += q3.y != 0u;
    c[3] += status == COH_RUN_DEFECT;
    c[4] += q2.z;
    c[5] += q2.w;
    c[6] += (uint64_t)q2.x | ((uint64_t)q2.y << 32);
    c[7] += q3.y;
    c[8] += q3.x;
    c[9] += 1;
    c[10] += (q3.w >> 24) & COH_FLAG_UNSAFE ? 1u : 0u;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < COH_N_COUNTERS; ++k) {
    uint64_t v = c[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < COH_N_COUNTERS) {
    uint64_t v = 0;
#pragma unroll
    for (int w = 0; w < kRedThreads / 32; ++w) v += part[w][threadIdx.x];
    if (v) atomicAdd(out + threadIdx.x, (unsigned long long)v);
  }
}

int launch_reduce_counters(const coh_trace_result* d_results, uint64_t n_traces,
                           uint64_t* d_counters, void* stream, std::string* err) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_counters, 0, sizeof(uint64_t) * COH_N_COUNTERS, s);
  if (e == cudaSuccess && n_traces) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (n_traces + kRedThreads - 1) / kRedThreads;
    if (blocks > (uint64_t)sms * 4) blocks = (uint64_t)sms * 4;
    k_reduce_counters<<<(unsigned)blocks, kRedThreads, 0, s>>>(
        d_results, n_traces, reinterpret_cast<unsigned long long*>(d_counters));
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    *err = std::string("reduce_counters: ") + cudaGetErrorString(e);
    return COH_E_CUDA;
  }
  return COH_OK;
}

}  // namespace cohb
