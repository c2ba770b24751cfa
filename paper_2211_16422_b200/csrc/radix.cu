// Stable LSD radix sort of (key, u32 value) pairs, 8 bits per pass -- the library's own, so that no
// library kernel runs on the search step (the queries are ordered by window start before every
// search, search.cu) or in build_index (the (charge, m/z, id, ordinal) entry order, library.cu).
//
// One pass = three kernels over tiles of kTile consecutive elements (one CTA per tile, one warp per
// consecutive 512-element chunk):
//   radix_hist_kernel     per-tile digit counts, stored digit-major: hist[digit][tile]
//   radix_scan_kernel     exclusive prefix sum over that array in place (one CTA; the array is
//                         256 x tiles entries: 4 K for a 64 Ki-query search, 270 K for 4.3 M rows)
//   radix_scatter_kernel  every warp recounts its chunk, a prefix over the warps of the CTA gives each
//                         warp its first output slot per digit, then the warp replays its chunk IN ORDER,
//                         32 elements per step: __match_any_sync groups the lanes of equal digit, a
//                         lane's rank inside its group is the number of lower lanes in it -- equal
//                         digits keep their input order (stable), which LSD passes rely on.
// The caller names the key bits that can differ; bits outside [begin_bit, end_bit) are ignored.
#include <algorithm>

#include "common.cuh"
#include "radix.cuh"

namespace hb {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixMaxPerLane = 16;  // a warp's chunk is 32 x per_lane consecutive elements, a CTA's tile 8 chunks

// shift_mask = shift | (digit mask << 8): the last pass of a bit range may be narrower than 8 bits.
// kSum (64-bit keys only): the pairs are ordered by (high half + low half) of the key instead of the key itself --
// the search orders its queries by window start + window end (search.cu).
template <typename K, bool kSum>
__device__ __forceinline__ uint32_t radix_digit(K key, int shift_mask) {
  if constexpr (kSum) {
    const uint64_t v = (static_cast<uint64_t>(key) >> 32) + (static_cast<uint64_t>(key) & 0xFFFFFFFFull);
    return static_cast<uint32_t>(v >> (shift_mask & 0xFF)) & static_cast<uint32_t>(shift_mask >> 8);
  }
  return static_cast<uint32_t>(key >> (shift_mask & 0xFF)) & static_cast<uint32_t>(shift_mask >> 8);
}

// counts of this warp's chunk into its private row of s_cnt (zeroed by the caller)
template <typename K, bool kSum>
__device__ __forceinline__ void radix_count_chunk(const K* __restrict__ keys, uint64_t n, uint64_t chunk0, int shift,
                                                  uint32_t* s_row, int lane, int per_lane) {
#pragma unroll 4
  for (int j = 0; j < per_lane; ++j) {
    const uint64_t i = chunk0 + uint64_t(j) * 32 + lane;
    if (i < n) atomicAdd(&s_row[radix_digit<K, kSum>(keys[i], shift)], 1u);
  }
}

template <typename K, bool kSum>
__global__ void __launch_bounds__(kRadixThreads)
radix_hist_kernel(const K* __restrict__ keys, uint64_t n, int shift, uint32_t n_tiles, uint32_t* __restrict__ hist,
                  int per_lane) {
  __shared__ uint32_t s_cnt[256];
  s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t chunk = 32ull * per_lane;
  radix_count_chunk<K, kSum>(keys, n, (uint64_t(blockIdx.x) * kRadixWarps + warp) * chunk, shift, s_cnt, lane, per_lane);
  __syncthreads();
  hist[uint64_t(threadIdx.x) * n_tiles + blockIdx.x] = s_cnt[threadIdx.x];
}

// exclusive prefix sum of `count` entries by one CTA of 1024 threads (in == out allowed); `add` is added to every
// result (multi-tile scans pass the tile's offset)
template <typename T>
__device__ __forceinline__ void scan_cta_1024(const T* in, T* out, uint64_t count, T add,
                                              T* total_out) {
  __shared__ T s_warp[32];
  __shared__ T s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = add;
  __syncthreads();
  for (uint64_t base = 0; base < count; base += 4096) {  // 4 consecutive entries per thread
    const uint64_t i0 = base + uint64_t(threadIdx.x) * 4;
    T v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = i0 + j < count ? in[i0 + j] : T(0);
    const T mine = v[0] + v[1] + v[2] + v[3];
    T incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const T w = s_warp[lane];
      T wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      s_warp[lane] = wi - w;  // exclusive over the warps
    }
    __syncthreads();
    T run = s_carry + s_warp[warp] + incl - mine;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + j < count) out[i0 + j] = run;
      run += v[j];
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = run;
    __syncthreads();
  }
  if (total_out != nullptr && threadIdx.x == 0) *total_out = s_carry - add;
}

template <typename T>
__global__ void __launch_bounds__(1024) scan_single_kernel(const T* in, T* out, uint64_t count) {
  scan_cta_1024<T>(in, out, count, T(0), nullptr);
}
__global__ void __launch_bounds__(1024) radix_scan_kernel(uint32_t* __restrict__ data, uint64_t count) {
  scan_cta_1024<uint32_t>(data, data, count, 0u, nullptr);
}

// ---- device-wide exclusive sum (three kernels: tile totals, scan of the totals, per-tile scan) ----------------
constexpr uint64_t kScanTile = 16384;  // entries per CTA

template <typename T>
__global__ void __launch_bounds__(1024) scan_tile_totals_kernel(const T* __restrict__ in, uint64_t n, T* __restrict__ totals) {
  __shared__ T s_warp[32];
  const uint64_t t0 = uint64_t(blockIdx.x) * kScanTile;
  T acc = 0;
  for (uint64_t i = t0 + threadIdx.x; i < min(n, t0 + kScanTile); i += 1024) acc += in[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    T v = s_warp[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) totals[blockIdx.x] = v;
  }
}
template <typename T>
__global__ void __launch_bounds__(1024)
scan_tiles_kernel(const T* __restrict__ in, T* __restrict__ out, uint64_t n, const T* __restrict__ tile_offs) {
  const uint64_t t0 = uint64_t(blockIdx.x) * kScanTile;
  scan_cta_1024<T>(in + t0, out + t0, min(kScanTile, n - t0), tile_offs[blockIdx.x], nullptr);
}

size_t exclusive_sum_temp_bytes(uint64_t n) { return static_cast<size_t>((n + kScanTile - 1) / kScanTile + 1) * 8; }

template <typename T>
int exclusive_sum(homs_b200_ctx* ctx, const T* d_in, T* d_out, uint64_t n, void* d_temp) {
  if (n == 0) return HOMS_B200_OK;
  if (n <= kScanTile) {
    scan_single_kernel<T><<<1, 1024, 0, ctx->stream>>>(d_in, d_out, n);
    HB_LAUNCHED(ctx);
    return HOMS_B200_OK;
  }
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  T* totals = static_cast<T*>(d_temp);
  scan_tile_totals_kernel<T><<<static_cast<unsigned>(tiles), 1024, 0, ctx->stream>>>(d_in, n, totals);
  HB_LAUNCHED(ctx);
  scan_single_kernel<T><<<1, 1024, 0, ctx->stream>>>(totals, totals, tiles);
  HB_LAUNCHED(ctx);
  scan_tiles_kernel<T><<<static_cast<unsigned>(tiles), 1024, 0, ctx->stream>>>(d_in, d_out, n, totals);
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}
template int exclusive_sum<uint32_t>(homs_b200_ctx*, const uint32_t*, uint32_t*, uint64_t, void*);
template int exclusive_sum<uint64_t>(homs_b200_ctx*, const uint64_t*, uint64_t*, uint64_t, void*);

template <typename K, bool kSum>
__global__ void __launch_bounds__(kRadixThreads)
radix_scatter_kernel(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
                     uint32_t* __restrict__ vals_out, uint64_t n, int shift, uint32_t n_tiles,
                     const uint32_t* __restrict__ offs, int per_lane) {
  __shared__ uint32_t s_cnt[kRadixWarps][256];  // counts, then the first output slot of (warp, digit)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) s_cnt[w][threadIdx.x] = 0;
  __syncthreads();
  const uint64_t chunk0 = (uint64_t(blockIdx.x) * kRadixWarps + warp) * (32ull * per_lane);
  radix_count_chunk<K, kSum>(keys_in, n, chunk0, shift, s_cnt[warp], lane, per_lane);
  __syncthreads();
  {
    uint32_t run = offs[uint64_t(threadIdx.x) * n_tiles + blockIdx.x];  // thread = digit
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t c = s_cnt[w][threadIdx.x];
      s_cnt[w][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
  uint32_t* slot = s_cnt[warp];
  for (int j = 0; j < per_lane; ++j) {
    const uint64_t i = chunk0 + uint64_t(j) * 32 + lane;
    const bool live = i < n;
    K key = 0;
    uint32_t val = 0;
    if (live) {
      key = keys_in[i];
      val = vals_in ? vals_in[i] : static_cast<uint32_t>(i);
    }
    const uint32_t d = live ? radix_digit<K, kSum>(key, shift) : 256u;  // dead lanes form their own group
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (live) {
      const uint32_t pos = slot[d] + rank;
      keys_out[pos] = key;
      vals_out[pos] = val;
    }
    __syncwarp();
    if (live && rank == 0) slot[d] += __popc(peers);  // one lane per digit group
    __syncwarp();
  }
}

// Elements per lane: long chunks (16 per lane) amortise the per-tile counters at library sizes; at query counts
// (16 K ... 64 K) they would leave a few dozen warps on the whole GPU walking their chunks serially (measured 35 us
// per pass at n = 16 000), so the chunk shrinks until every SM has a couple of CTAs.
static int radix_per_lane(const homs_b200_ctx* ctx, uint64_t n) {
  const uint64_t want = n / (uint64_t(kRadixThreads) * 2 * static_cast<uint64_t>(std::max(1, ctx->sm_count)));
  return static_cast<int>(std::min<uint64_t>(kRadixMaxPerLane, std::max<uint64_t>(1, want)));
}
size_t radix_temp_bytes(uint64_t n) {  // sized for the shortest chunks
  const uint64_t tiles = (n + kRadixThreads - 1) / kRadixThreads;
  return static_cast<size_t>(std::max<uint64_t>(1, tiles)) * 256 * sizeof(uint32_t);
}

template <typename K, bool kSum>
static int radix_sort_impl(homs_b200_ctx* ctx, K* keys_a, K* keys_b, uint32_t* vals_a, uint32_t* vals_b, uint64_t n,
                           int begin_bit, int end_bit, void* d_temp, bool first_vals_iota, bool* result_in_b) {
  *result_in_b = false;
  if (n == 0 || end_bit <= begin_bit) return HOMS_B200_OK;
  HB_REQUIRE(ctx, n <= 0xFFFFFFFFull, HOMS_B200_ERR_ARGUMENT, "radix sort: more than 2^32-1 items");
  const int per_lane = radix_per_lane(ctx, n);
  const uint64_t tile = uint64_t(kRadixThreads) * per_lane;
  const uint32_t tiles = static_cast<uint32_t>((n + tile - 1) / tile);
  auto* hist = static_cast<uint32_t*>(d_temp);
  K *kin = keys_a, *kout = keys_b;
  uint32_t *vin = vals_a, *vout = vals_b;
  bool iota = first_vals_iota;
  for (int bit = begin_bit; bit < end_bit; bit += 8) {
    const int shift = bit | (((1 << std::min(8, end_bit - bit)) - 1) << 8);
    radix_hist_kernel<K, kSum><<<tiles, kRadixThreads, 0, ctx->stream>>>(kin, n, shift, tiles, hist, per_lane);
    HB_LAUNCHED(ctx);
    radix_scan_kernel<<<1, 1024, 0, ctx->stream>>>(hist, uint64_t(tiles) * 256);
    HB_LAUNCHED(ctx);
    radix_scatter_kernel<K, kSum><<<tiles, kRadixThreads, 0, ctx->stream>>>(kin, iota ? nullptr : vin, kout, vout, n, shift,
                                                                             tiles, hist, per_lane);
    HB_LAUNCHED(ctx);
    iota = false;
    std::swap(kin, kout);
    std::swap(vin, vout);
    *result_in_b = !*result_in_b;
  }
  return HOMS_B200_OK;
}

template <typename K>
int radix_sort_pairs(homs_b200_ctx* ctx, K* keys_a, K* keys_b, uint32_t* vals_a, uint32_t* vals_b, uint64_t n,
                     int begin_bit, int end_bit, void* d_temp, bool first_vals_iota, bool* result_in_b) {
  return radix_sort_impl<K, false>(ctx, keys_a, keys_b, vals_a, vals_b, n, begin_bit, end_bit, d_temp, first_vals_iota,
                                   result_in_b);
}
int radix_sort_pairs_by_half_sum(homs_b200_ctx* ctx, uint64_t* keys_a, uint64_t* keys_b, uint32_t* vals_a,
                                 uint32_t* vals_b, uint64_t n, int end_bit, void* d_temp, bool* result_in_b) {
  return radix_sort_impl<uint64_t, true>(ctx, keys_a, keys_b, vals_a, vals_b, n, 0, end_bit, d_temp, false, result_in_b);
}
template int radix_sort_pairs<uint8_t>(homs_b200_ctx*, uint8_t*, uint8_t*, uint32_t*, uint32_t*, uint64_t, int, int,
                                       void*, bool, bool*);
template int radix_sort_pairs<uint32_t>(homs_b200_ctx*, uint32_t*, uint32_t*, uint32_t*, uint32_t*, uint64_t, int, int,
                                        void*, bool, bool*);
template int radix_sort_pairs<uint64_t>(homs_b200_ctx*, uint64_t*, uint64_t*, uint32_t*, uint32_t*, uint64_t, int, int,
                                        void*, bool, bool*);

}  // namespace hb
