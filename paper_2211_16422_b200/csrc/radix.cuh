// The library's own device-wide primitives (radix.cu): stable LSD radix sort of (key, u32 value) pairs and an
// exclusive prefix sum, on the context's stream.
#pragma once

#include <cstddef>
#include <cstdint>

struct homs_b200_ctx;

namespace hb {

// bytes of device scratch radix_sort_pairs needs for n items
size_t radix_temp_bytes(uint64_t n);

// Sorts n pairs by key bits [begin_bit, end_bit), stable, ping-ponging between the a and b arrays
// (ceil((end_bit - begin_bit) / 8) passes).  *result_in_b tells where the sorted pairs ended up.
// first_vals_iota: the input values are 0, 1, 2, ... and vals_a need not be initialised.
// K = uint8_t, uint32_t or uint64_t.  Stream-ordered, no host synchronisation.
template <typename K>
int radix_sort_pairs(homs_b200_ctx* ctx, K* keys_a, K* keys_b, uint32_t* vals_a, uint32_t* vals_b, uint64_t n,
                     int begin_bit, int end_bit, void* d_temp, bool first_vals_iota, bool* result_in_b);

// The same for 64-bit keys ordered by (high 32 bits + low 32 bits), bits [0, end_bit) of that sum.
int radix_sort_pairs_by_half_sum(homs_b200_ctx* ctx, uint64_t* keys_a, uint64_t* keys_b, uint32_t* vals_a,
                                 uint32_t* vals_b, uint64_t n, int end_bit, void* d_temp, bool* result_in_b);

// Device-wide exclusive prefix sum of n entries (T = uint32_t or uint64_t; in != out), stream-ordered.
size_t exclusive_sum_temp_bytes(uint64_t n);
template <typename T>
int exclusive_sum(homs_b200_ctx* ctx, const T* d_in, T* d_out, uint64_t n, void* d_temp);

#ifdef __CUDACC__
// CTA-wide sum / exclusive prefix sum of one u32 per thread (kThreads a multiple of 32, <= 1024; every thread calls)
template <int kThreads>
__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v) {
  __shared__ uint32_t s_part[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t t = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) t += s_part[w];
  __syncthreads();
  return t;
}
template <int kThreads>
__device__ __forceinline__ uint32_t block_exclusive_sum_u32(uint32_t v) {
  __shared__ uint32_t s_part[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_part[warp] = incl;
  __syncthreads();
  uint32_t before = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w)
    if (w < warp) before += s_part[w];
  __syncthreads();
  return before + incl - v;
}
#endif

}  // namespace hb
