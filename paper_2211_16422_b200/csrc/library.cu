// Device-resident library index: build_index (src/search.cpp:17-60) re-designed for the GPU.
//
// The reference keeps one std::map<charge, Bucket> of separately sorted arrays.  Here the whole
// library is ONE array sorted by (charge, precursor m/z, id, ordinal); a bucket is a contiguous
// row range, which turns every candidate window into a row interval of a single matrix.  The
// string comparison of ids (search.cpp:43) is replaced by the integer id_rank the host computed
// once, so the 4-level tie-break key is numeric on the device.
//
// Sharding: shard g of G keeps rows [size*g/G, size*(g+1)/G) of EVERY bucket
// (contiguous m/z slices); precursor m/z, id_rank and the rank->ordinal table are replicated so
// that window bounds are computed in full-bucket coordinates on every rank.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "common.cuh"
#include "radix.cuh"

namespace hb {

// one warp per destination row: dst[r] = src[src_index[r]] (dense W words -> padded S words)
__global__ void gather_rows_kernel(uint64_t n_rows, const uint32_t* __restrict__ src_index,
                                   const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                   uint32_t W, uint32_t S) {
  const int lane = threadIdx.x & 31;
  const uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (row >= n_rows) return;
  const uint64_t* s = src + uint64_t(src_index[row]) * W;
  uint64_t* d = dst + row * S;
  for (uint32_t w = lane; w < S; w += 32) d[w] = w < W ? s[w] : 0;
}

// ---- (charge, precursor m/z, id, ordinal) order on the device (search.cpp:37-46) ---------------
// Three stable LSD radix sorts (radix.cu) of the entry indices, least significant key first: id_rank (when ids
// are given; otherwise the initial order already is the ordinal order), the m/z bits mapped to an
// order-preserving u64, the charge.  1.2 M entries sort in well under a millisecond; the host's
// comparison sort took 0.2-0.3 s.

// IEEE double -> u64 with the same order (negative values flipped; -0.0 joins +0.0 as the reference's
// `mz[a] != mz[b]` sees them equal)
__global__ void index_mz_keys_kernel(uint64_t n, const double* __restrict__ mz, const uint32_t* __restrict__ idx,
                                     uint64_t* __restrict__ keys) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(mz[idx[i]]));
  if (b == 0x8000000000000000ull) b = 0;
  keys[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__global__ void index_charge_keys_kernel(uint64_t n, const uint8_t* __restrict__ charge,
                                         const uint32_t* __restrict__ idx, uint8_t* __restrict__ keys) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = charge[idx[i]];
}
__global__ void index_iota_kernel(uint64_t n, uint32_t* __restrict__ idx) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) idx[i] = static_cast<uint32_t>(i);
}

static int device_sort_order(homs_b200_ctx* ctx, uint64_t n, const double* mz, const uint8_t* charge,
                             const uint32_t* id_rank, uint32_t* h_order) {
  const size_t temp = (radix_temp_bytes(n) + 255) / 256 * 256;
  const size_t a8 = (n * 8 + 255) / 256 * 256, a4 = (n * 4 + 255) / 256 * 256, a1 = (n + 255) / 256 * 256;
  // layout: mz | key64 a | key64 b | idx a | idx b | rank a | rank b | charge | key8 a | key8 b | sort scratch
  HB_TRY(ensure(ctx, ctx->scratch[kScrIndexSort], 3 * a8 + 4 * a4 + 3 * a1 + temp));
  auto* base = ctx->scratch[kScrIndexSort].as<unsigned char>();
  auto* d_mz = reinterpret_cast<double*>(base);
  auto* k64a = reinterpret_cast<uint64_t*>(base + a8);
  auto* k64b = reinterpret_cast<uint64_t*>(base + 2 * a8);
  auto* idx_a = reinterpret_cast<uint32_t*>(base + 3 * a8);
  auto* idx_b = idx_a + a4 / 4;
  auto* rank_a = idx_b + a4 / 4;
  auto* rank_b = rank_a + a4 / 4;
  auto* d_charge = base + 3 * a8 + 4 * a4;
  auto* k8a = d_charge + a1;
  auto* k8b = k8a + a1;
  void* d_temp = k8b + a1;
  cudaStream_t st = ctx->stream;
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  HB_CUDA(ctx, cudaMemcpyAsync(d_mz, mz, n * 8, cudaMemcpyHostToDevice, st));
  HB_CUDA(ctx, cudaMemcpyAsync(d_charge, charge, n, cudaMemcpyHostToDevice, st));
  uint32_t* cur = idx_a;
  uint32_t* alt = idx_b;
  bool in_b = false;
  if (id_rank) {  // ranks are positions in a sort of n entries: only the low bit_width(n - 1) bits differ
    int bits = 1;
    while (bits < 32 && (uint64_t(1) << bits) < n) ++bits;
    HB_CUDA(ctx, cudaMemcpyAsync(rank_a, id_rank, n * 4, cudaMemcpyHostToDevice, st));
    HB_TRY(radix_sort_pairs<uint32_t>(ctx, rank_a, rank_b, cur, alt, n, 0, bits, d_temp, true, &in_b));
    if (in_b) std::swap(cur, alt);
  } else {
    index_iota_kernel<<<blocks, 256, 0, st>>>(n, cur);
    HB_LAUNCHED(ctx);
  }
  index_mz_keys_kernel<<<blocks, 256, 0, st>>>(n, d_mz, cur, k64a);
  HB_LAUNCHED(ctx);
  HB_TRY(radix_sort_pairs<uint64_t>(ctx, k64a, k64b, cur, alt, n, 0, 64, d_temp, false, &in_b));
  if (in_b) std::swap(cur, alt);
  index_charge_keys_kernel<<<blocks, 256, 0, st>>>(n, d_charge, cur, k8a);
  HB_LAUNCHED(ctx);
  HB_TRY(radix_sort_pairs<uint8_t>(ctx, k8a, k8b, cur, alt, n, 0, 8, d_temp, false, &in_b));
  if (in_b) std::swap(cur, alt);
  HB_CUDA(ctx, cudaMemcpyAsync(h_order, cur, n * 4, cudaMemcpyDeviceToHost, st));
  HB_CUDA(ctx, cudaStreamSynchronize(st));
  return HOMS_B200_OK;
}

int library_build(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* h_words,
                  const uint64_t* d_words_in, const double* mz, const uint8_t* charge,
                  const uint32_t* id_rank, uint32_t shard_index, uint32_t shard_count,
                  const uint32_t* row_of_entry) {
  HB_REQUIRE(ctx, n >= 1, HOMS_B200_ERR_INVARIANT, "build_index: library is empty");  // search.cpp:18
  HB_REQUIRE(ctx, dim >= 1, HOMS_B200_ERR_ARGUMENT, "build_index: dim must be positive");
  HB_REQUIRE(ctx, n <= 0x7FFFFFFFull, HOMS_B200_ERR_ARGUMENT, "build_index: more than 2^31-1 entries");
  HB_REQUIRE(ctx, mz && charge && (h_words || d_words_in), HOMS_B200_ERR_ARGUMENT,
             "build_index: null argument");
  HB_REQUIRE(ctx, shard_count >= 1 && shard_index < shard_count, HOMS_B200_ERR_ARGUMENT,
             "build_index: shard_index must be below shard_count");
  Library& lib = ctx->lib;
  lib.ready = false;
  lib.dim = dim;
  lib.W = words_for(dim);
  lib.S = stride_for(dim);
  lib.n = n;
  lib.shard_index = shard_index;
  lib.shard_count = shard_count;

  // (charge, mz, id, ordinal) order; id comparison through id_rank (search.cpp:37-46, :30-33)
  std::vector<uint32_t> order(n);
  HB_TRY(device_sort_order(ctx, n, mz, charge, id_rank, order.data()));

  lib.h_mz.resize(n);
  lib.h_ordinal = order;
  std::vector<uint32_t> rank_sorted(n), ord_of_rank(n);
  for (uint64_t r = 0; r < n; ++r) {
    lib.h_mz[r] = mz[order[r]];
    rank_sorted[r] = id_rank ? id_rank[order[r]] : order[r];
  }
  if (id_rank) {
    std::vector<uint8_t> seen(n, 0);
    for (uint64_t i = 0; i < n; ++i) {
      HB_REQUIRE(ctx, id_rank[i] < n && !seen[id_rank[i]], HOMS_B200_ERR_ARGUMENT,
                 "build_index: id_rank must be a permutation of 0..n-1");
      seen[id_rank[i]] = 1;
      ord_of_rank[id_rank[i]] = static_cast<uint32_t>(i);
    }
  } else {
    std::iota(ord_of_rank.begin(), ord_of_rank.end(), 0u);
  }

  lib.bucket_charge.clear();
  lib.buckets.clear();
  int32_t bucket_of_charge[256];
  std::fill(bucket_of_charge, bucket_of_charge + 256, -1);
  uint64_t local = 0;
  for (uint64_t r = 0; r < n;) {
    uint64_t e = r;
    const uint8_t c = charge[order[r]];
    while (e < n && charge[order[e]] == c) ++e;
    BucketDev b;
    b.begin = r;
    b.size = e - r;
    b.shard_begin = b.size * shard_index / shard_count;
    b.shard_end = b.size * (shard_index + 1) / shard_count;
    b.local_offset = local;
    local += b.shard_end - b.shard_begin;
    bucket_of_charge[c] = static_cast<int32_t>(lib.buckets.size());
    lib.bucket_charge.push_back(c);
    lib.buckets.push_back(b);
    r = e;
  }
  lib.n_local = local;

  // local (resident) rows: source ordinal, m/z and id_rank per local row
  std::vector<uint32_t> local_src(std::max<uint64_t>(local, 1));
  std::vector<double> local_mz(std::max<uint64_t>(local, 1));
  std::vector<uint32_t> local_rank(std::max<uint64_t>(local, 1));
  for (const BucketDev& b : lib.buckets)
    for (uint64_t i = b.shard_begin; i < b.shard_end; ++i) {
      const uint64_t l = b.local_offset + (i - b.shard_begin), g = b.begin + i;
      local_src[l] = row_of_entry ? row_of_entry[order[g]] : order[g];
      local_mz[l] = lib.h_mz[g];
      local_rank[l] = rank_sorted[g];
    }

  HB_TRY(ensure(ctx, lib.d_mz, n * 8));
  HB_TRY(ensure(ctx, lib.d_id_rank, n * 4));
  HB_TRY(ensure(ctx, lib.d_ord_of_rank, n * 4));
  HB_TRY(ensure(ctx, lib.d_mz_local, local * 8));
  HB_TRY(ensure(ctx, lib.d_id_rank_local, local * 4));
  HB_TRY(ensure(ctx, lib.d_words, local * lib.S * 8));
  HB_TRY(ensure(ctx, lib.d_buckets, lib.buckets.size() * sizeof(BucketDev)));
  HB_TRY(ensure(ctx, lib.d_bucket_of_charge, sizeof bucket_of_charge));
  cudaStream_t st = ctx->stream;
  HB_CUDA(ctx, cudaMemcpyAsync(lib.d_mz.p, lib.h_mz.data(), n * 8, cudaMemcpyHostToDevice, st));
  HB_CUDA(ctx, cudaMemcpyAsync(lib.d_id_rank.p, rank_sorted.data(), n * 4, cudaMemcpyHostToDevice, st));
  HB_CUDA(ctx, cudaMemcpyAsync(lib.d_ord_of_rank.p, ord_of_rank.data(), n * 4, cudaMemcpyHostToDevice, st));
  if (local) {
    HB_CUDA(ctx, cudaMemcpyAsync(lib.d_mz_local.p, local_mz.data(), local * 8, cudaMemcpyHostToDevice, st));
    HB_CUDA(ctx, cudaMemcpyAsync(lib.d_id_rank_local.p, local_rank.data(), local * 4, cudaMemcpyHostToDevice, st));
  }
  HB_CUDA(ctx, cudaMemcpyAsync(lib.d_buckets.p, lib.buckets.data(),
                               lib.buckets.size() * sizeof(BucketDev), cudaMemcpyHostToDevice, st));
  HB_CUDA(ctx, cudaMemcpyAsync(lib.d_bucket_of_charge.p, bucket_of_charge, sizeof bucket_of_charge,
                               cudaMemcpyHostToDevice, st));

  if (local) {
    if (d_words_in) {
      // rows are already on the device: permute there
      HB_TRY(ensure(ctx, ctx->scratch[kScrMisc], local * 4));
      HB_CUDA(ctx, cudaMemcpyAsync(ctx->scratch[kScrMisc].p, local_src.data(), local * 4,
                                   cudaMemcpyHostToDevice, st));
      const uint64_t threads = local * 32;
      gather_rows_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
          local, ctx->scratch[kScrMisc].as<uint32_t>(), d_words_in, lib.d_words.as<uint64_t>(),
          lib.W, lib.S);
      HB_LAUNCHED(ctx);
    } else {
      // host rows: gather the resident rows through a double-buffered pinned block
      const size_t row_bytes = size_t(lib.S) * 8;
      const uint64_t rows_per_chunk = std::max<uint64_t>(1, (32u << 20) / row_bytes);
      HB_TRY(ensure_pinned(ctx, 2 * rows_per_chunk * row_bytes));
      cudaEvent_t done[2];
      HB_CUDA(ctx, cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
      HB_CUDA(ctx, cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
      int which = 0;
      int rc = HOMS_B200_OK;
      for (uint64_t r0 = 0; r0 < local && rc == HOMS_B200_OK; r0 += rows_per_chunk, which ^= 1) {
        const uint64_t cnt = std::min(rows_per_chunk, local - r0);
        auto* stage = static_cast<uint64_t*>(ctx->pinned) + size_t(which) * rows_per_chunk * lib.S;
        if (cudaEventSynchronize(done[which]) != cudaSuccess) rc = HOMS_B200_ERR_CUDA;
        for (uint64_t r = 0; r < cnt; ++r) {
          uint64_t* d = stage + r * lib.S;
          std::memcpy(d, h_words + uint64_t(local_src[r0 + r]) * lib.W, size_t(lib.W) * 8);
          if (lib.S > lib.W) std::memset(d + lib.W, 0, size_t(lib.S - lib.W) * 8);
        }
        if (cudaMemcpyAsync(lib.d_words.as<uint64_t>() + r0 * lib.S, stage, cnt * row_bytes,
                            cudaMemcpyHostToDevice, st) != cudaSuccess)
          rc = HOMS_B200_ERR_CUDA;
        cudaEventRecord(done[which], st);
      }
      cudaStreamSynchronize(st);
      cudaEventDestroy(done[0]);
      cudaEventDestroy(done[1]);
      if (rc != HOMS_B200_OK) return set_error(ctx, rc, "build_index: host->device row upload failed");
    }
  }
  if (ctx->engine != HOMS_B200_ENGINE_POPC && ctx->engine != HOMS_B200_ENGINE_DIRECT && local) {
    HB_TRY(tc_expand_library(ctx));
  } else {
    release(lib.d_x);
    lib.x_rows = 0;
  }
  HB_CUDA(ctx, cudaStreamSynchronize(st));  // host vectors above go out of scope
  lib.ready = true;
  return HOMS_B200_OK;
}

int library_build_from_device(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* d_words,
                              const double* mz, const uint8_t* charge, const uint32_t* id_rank,
                              uint32_t shard_index, uint32_t shard_count, const uint32_t* row_of_entry) {
  return library_build_any(ctx, dim, n, nullptr, d_words, mz, charge, id_rank, shard_index, shard_count, row_of_entry);
}

}  // namespace hb

using namespace hb;

extern "C" {

int homs_b200_library_upload(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* words,
                             const double* precursor_mz, const uint8_t* charge,
                             const uint32_t* id_rank, uint32_t shard_index, uint32_t shard_count) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  return library_build_any(ctx, dim, n, words, nullptr, precursor_mz, charge, id_rank, shard_index, shard_count, nullptr);
}

int homs_b200_library_upload_dev(homs_b200_ctx* ctx, uint32_t dim, uint64_t n,
                                 const uint64_t* d_words, const double* precursor_mz,
                                 const uint8_t* charge, const uint32_t* id_rank,
                                 uint32_t shard_index, uint32_t shard_count) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  return library_build_any(ctx, dim, n, nullptr, d_words, precursor_mz, charge, id_rank, shard_index, shard_count, nullptr);
}

int homs_b200_library_bucket_count(const homs_b200_ctx* ctx, uint32_t* out_count) {
  if (!ctx || !out_count) return HOMS_B200_ERR_ARGUMENT;
  HB_REQUIRE(ctx, ctx->lib.ready, HOMS_B200_ERR_STATE, "no library uploaded");
  *out_count = static_cast<uint32_t>(ctx->lib.buckets.size());
  return HOMS_B200_OK;
}

int homs_b200_library_bucket_info(const homs_b200_ctx* ctx, uint32_t which, uint8_t* out_charge,
                                  uint64_t* out_size, uint64_t* out_shard_begin,
                                  uint64_t* out_shard_end) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  HB_REQUIRE(ctx, ctx->lib.ready, HOMS_B200_ERR_STATE, "no library uploaded");
  HB_REQUIRE(ctx, which < ctx->lib.buckets.size(), HOMS_B200_ERR_ARGUMENT, "bucket index out of range");
  const BucketDev& b = ctx->lib.buckets[which];
  if (out_charge) *out_charge = ctx->lib.bucket_charge[which];
  if (out_size) *out_size = b.size;
  // a multi-device context holds the whole bucket, spread over its members
  if (out_shard_begin) *out_shard_begin = is_group(ctx) ? 0 : b.shard_begin;
  if (out_shard_end) *out_shard_end = is_group(ctx) ? b.size : b.shard_end;
  return HOMS_B200_OK;
}

int homs_b200_library_bucket_export(homs_b200_ctx* ctx, uint32_t which, double* out_mz,
                                    uint32_t* out_ordinal, uint64_t* out_words) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  const Library& lib = ctx->lib;
  HB_REQUIRE(ctx, lib.ready, HOMS_B200_ERR_STATE, "no library uploaded");
  HB_REQUIRE(ctx, which < lib.buckets.size(), HOMS_B200_ERR_ARGUMENT, "bucket index out of range");
  const BucketDev& b = lib.buckets[which];
  if (out_mz) std::copy(lib.h_mz.begin() + b.begin, lib.h_mz.begin() + b.begin + b.size, out_mz);
  if (out_ordinal)
    std::copy(lib.h_ordinal.begin() + b.begin, lib.h_ordinal.begin() + b.begin + b.size, out_ordinal);
  if (out_words) {
    // every member holds a contiguous slice of the bucket, in member order
    const size_t n_members = std::max<size_t>(1, ctx->members.size());
    for (size_t g = 0; g < n_members; ++g) {
      homs_b200_ctx* m = g == 0 ? ctx : ctx->members[g];
      const BucketDev& mb = m->lib.buckets[which];
      cudaSetDevice(m->device);
      const int rc = download_rows(m, out_words + (mb.shard_begin - (is_group(ctx) ? 0 : b.shard_begin)) * lib.W,
                                   m->lib.d_words.as<uint64_t>() + mb.local_offset * lib.S,
                                   mb.shard_end - mb.shard_begin, lib.W, lib.S);
      if (rc != HOMS_B200_OK || cudaStreamSynchronize(m->stream) != cudaSuccess) {
        cudaSetDevice(ctx->device);
        return set_error(ctx, HOMS_B200_ERR_CUDA, "bucket_export: device -> host copy failed");
      }
    }
    cudaSetDevice(ctx->device);
  }
  return HOMS_B200_OK;
}

}  // extern "C"
