// Counter-based synthetic call generator shared by host (C++) and device (CUDA).
// Definition: include/cohere_b200.h, "synthetic record generator".
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define COH_HD __host__ __device__ __forceinline__
#else
#define COH_HD static inline
#endif

COH_HD uint64_t coh_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

COH_HD uint16_t coh_gen_record(uint64_t seed, uint64_t trace_id, uint32_t call_idx,
                               uint32_t n_arrays, uint32_t adv_per1024) {
  const uint64_t h = coh_splitmix64(seed ^ (trace_id << 20) ^ (uint64_t)call_idx);
  const uint32_t arr = (uint32_t)(((h & 0xFFFFFFFFull) * (uint64_t)n_arrays) >> 32);
  const uint32_t kind = (uint32_t)((((h >> 32) & 0xFFFFull) * 3ull) >> 16);
  const uint32_t site = (uint32_t)((h >> 48) & 1ull);
  const uint32_t adv = ((uint32_t)((h >> 49) & 0x3FFull)) < adv_per1024;
  const uint32_t var = adv ? 1u + (uint32_t)((((h >> 59) & 0x1Full) * 7ull) >> 5) : 0u;
  return (uint16_t)((arr << 8) | (kind << 2) | (site << 4) | (var << 5));
}

// Fragmentation mask of plane word w (include/cohere_b200.h coh_frag_mask, same draws).
COH_HD uint32_t coh_frag_word(uint64_t frag_seed, uint32_t frag_log2, uint32_t w) {
  if (frag_log2 == 0) return 0u;
  uint32_t x = ((uint32_t)frag_seed ^ (w * 0x9E3779B9u)) + (uint32_t)(frag_seed >> 32);
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  if (frag_log2 > 5) {
    const uint32_t t = frag_log2 - 5;
    return (x >> (32u - t)) == ((1u << t) - 1u) ? 1u << (x & 31u) : 0u;
  }
  uint32_t m = x;
  for (uint32_t j = 1; j < frag_log2; ++j) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    m &= x;
  }
  return m;
}

// Multi-mode blocks for synthetic traces (COH_BATCH_BLOCKS): call i > 0 continues the
// current block with probability cont_per1024 / 1024 when its array is not in the block
// yet (a DeclBlock names each variable once).  Applied to a trace's records in call order.
COH_HD bool coh_gen_cont(uint64_t seed, uint64_t trace_id, uint32_t call_idx, uint32_t cont_per1024) {
  const uint64_t h = coh_splitmix64(seed ^ 0x5851F42D4C957F2Dull ^ (trace_id << 20) ^ (uint64_t)call_idx);
  return (uint32_t)(h & 0x3FFull) < cont_per1024;
}
