// Fused raw-spectra entry points: spectra are encoded on the device and stay there.
//
//   library_build_from_spectra == build_index(encode_spectra(spectra).encoded)
//                                 (src/pipeline.cpp:60-85 followed by src/search.cpp:17-60)
//   queries_from_spectra       == the `queries` argument of search_batch / cascade_search built by
//                                 encode_spectra (pipeline.cpp:121-122), resident for search_resident
//
// The reference round-trips every hypervector through std::vector<EncodedSpectrum> between the two
// steps; here the rows go from the encoder's output straight into the m/z-sorted index matrix (one
// gather) and only the 1-byte ok flags travel to the host, which needs them for the order-preserving
// compaction of pipeline.cpp:75-83: entry e of the index / query set is the e-th processable
// spectrum, exactly the ordinal the reference would report.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace hb {

__global__ void gather_rows_kernel(uint64_t n_rows, const uint32_t* __restrict__ src_index,
                                   const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                   uint32_t W, uint32_t S);  // library.cu

// encode n spectra into scratch (dense rows), ok flags to the host; returns the compaction map
static int encode_keep(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                       const uint64_t* offsets, const double* mz, const double* intensity,
                       uint8_t* out_ok, std::vector<uint32_t>* row_of_entry) {
  HB_REQUIRE(ctx, n < 0xFFFFFFFFull, HOMS_B200_ERR_ARGUMENT, "more than 2^32-2 spectra");
  const uint32_t W = ctx->cb.W;
  HB_TRY(ensure(ctx, ctx->scratch[kScrFusedRows], std::max<size_t>(1, n) * W * 8));
  std::vector<uint8_t> ok_local;
  if (!out_ok) {
    ok_local.resize(n);
    out_ok = ok_local.data();
  }
  HB_TRY(encode_pipeline(ctx, cfg, n, offsets, mz, intensity, ctx->scratch[kScrFusedRows].as<uint64_t>(),
                         nullptr, nullptr, out_ok));
  row_of_entry->clear();
  row_of_entry->reserve(n);
  for (uint64_t i = 0; i < n; ++i)
    if (out_ok[i]) row_of_entry->push_back(static_cast<uint32_t>(i));
  return HOMS_B200_OK;
}

// precursor m/z and charge of the kept spectra, gathered on the device
__global__ void gather_meta_kernel(uint64_t m, const uint32_t* __restrict__ idx, const double* __restrict__ src_mz,
                                   const uint8_t* __restrict__ src_charge, double* __restrict__ dst_mz,
                                   uint8_t* __restrict__ dst_charge) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m) return;
  dst_mz[e] = src_mz[idx[e]];
  dst_charge[e] = src_charge[idx[e]];
}

}  // namespace hb

using namespace hb;

extern "C" {

int homs_b200_library_build_from_spectra(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg,
                                         uint64_t n, const uint64_t* offsets, const double* mz,
                                         const double* intensity, const double* precursor_mz,
                                         const uint8_t* charge, const uint32_t* id_rank,
                                         uint32_t shard_index, uint32_t shard_count, uint8_t* out_ok,
                                         uint64_t* out_n_encoded) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->cb.ready, HOMS_B200_ERR_STATE, "encode: no codebook uploaded");
  HB_REQUIRE(ctx, n == 0 || (offsets && precursor_mz && charge), HOMS_B200_ERR_ARGUMENT,
             "library_build_from_spectra: null argument");
  std::vector<uint32_t> rows;
  HB_TRY(encode_keep(ctx, cfg, n, offsets, mz, intensity, out_ok, &rows));
  const uint64_t m = rows.size();
  if (out_n_encoded) *out_n_encoded = m;
  HB_REQUIRE(ctx, m >= 1, HOMS_B200_ERR_INVARIANT, "build_index: library is empty");  // search.cpp:18
  // metadata of the processable spectra, in order (pipeline.cpp:75-83)
  std::vector<double> mz_c(m);
  std::vector<uint8_t> ch_c(m);
  for (uint64_t e = 0; e < m; ++e) {
    mz_c[e] = precursor_mz[rows[e]];
    ch_c[e] = charge[rows[e]];
  }
  // id ranks over all n spectra -> ranks over the m survivors (relative order is all that matters)
  std::vector<uint32_t> rank_c;
  if (id_rank) {
    std::vector<uint32_t> entry_of_rank(n, kNone);
    for (uint64_t e = 0; e < m; ++e) {
      const uint32_t r = id_rank[rows[e]];
      HB_REQUIRE(ctx, r < n && entry_of_rank[r] == kNone, HOMS_B200_ERR_ARGUMENT,
                 "build_index: id_rank must be a permutation of 0..n-1");
      entry_of_rank[r] = static_cast<uint32_t>(e);
    }
    rank_c.resize(m);
    uint32_t next = 0;
    for (uint64_t r = 0; r < n; ++r)
      if (entry_of_rank[r] != kNone) rank_c[entry_of_rank[r]] = next++;
  }
  return library_build_from_device(ctx, ctx->cb.dim, m, ctx->scratch[kScrFusedRows].as<uint64_t>(), mz_c.data(),
                                   ch_c.data(), id_rank ? rank_c.data() : nullptr, shard_index, shard_count,
                                   rows.data());
}

int homs_b200_queries_from_spectra(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                                   const uint64_t* offsets, const double* mz, const double* intensity,
                                   const double* precursor_mz, const uint8_t* charge, uint8_t* out_ok,
                                   uint64_t* out_n_encoded) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->cb.ready, HOMS_B200_ERR_STATE, "encode: no codebook uploaded");
  HB_REQUIRE(ctx, n == 0 || (offsets && precursor_mz && charge), HOMS_B200_ERR_ARGUMENT,
             "queries_from_spectra: null argument");
  std::vector<uint32_t> rows;
  HB_TRY(encode_keep(ctx, cfg, n, offsets, mz, intensity, out_ok, &rows));
  const uint64_t m = rows.size();
  if (out_n_encoded) *out_n_encoded = m;
  Queries& q = ctx->q;
  q.ready = false;
  q.dim = ctx->cb.dim;
  q.nq = m;
  const uint32_t W = ctx->cb.W, S = stride_for(q.dim);
  HB_TRY(ensure(ctx, q.d_words, m * S * 8));
  HB_TRY(ensure(ctx, q.d_mz, m * 8));
  HB_TRY(ensure(ctx, q.d_charge, m));
  if (m) {
    std::vector<double> mz_c(m);
    std::vector<uint8_t> ch_c(m);
    for (uint64_t e = 0; e < m; ++e) {
      mz_c[e] = precursor_mz[rows[e]];
      ch_c[e] = charge[rows[e]];
    }
    HB_TRY(ensure(ctx, ctx->scratch[kScrFusedOk], m * 4));
    auto* d_idx = ctx->scratch[kScrFusedOk].as<uint32_t>();
    cudaStream_t st = ctx->stream;
    HB_CUDA(ctx, cudaMemcpyAsync(d_idx, rows.data(), m * 4, cudaMemcpyHostToDevice, st));
    HB_CUDA(ctx, cudaMemcpyAsync(q.d_mz.p, mz_c.data(), m * 8, cudaMemcpyHostToDevice, st));
    HB_CUDA(ctx, cudaMemcpyAsync(q.d_charge.p, ch_c.data(), m, cudaMemcpyHostToDevice, st));
    gather_rows_kernel<<<static_cast<unsigned>((m * 32 + 255) / 256), 256, 0, st>>>(
        m, d_idx, ctx->scratch[kScrFusedRows].as<uint64_t>(), q.d_words.as<uint64_t>(), W, S);
    HB_LAUNCHED(ctx);
    HB_CUDA(ctx, cudaStreamSynchronize(st));  // host vectors above go out of scope
  }
  q.ready = true;
  if (is_group(ctx)) HB_TRY(queries_replicate_locked(ctx));  // encoded on the leading device, searched on all
  return HOMS_B200_OK;
}

int homs_b200_queries_from_mgf(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint8_t* out_state,
                               uint64_t* out_n_queries) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->cb.ready, HOMS_B200_ERR_STATE, "encode: no codebook uploaded");
  HB_REQUIRE(ctx, ctx->mgf.ready, HOMS_B200_ERR_STATE, "queries_from_mgf: no parsed MGF resident (call mgf_parse first)");
  const MgfState& mg = ctx->mgf;
  const uint64_t n = mg.n_spectra;
  HB_REQUIRE(ctx, n < 0xFFFFFFFFull, HOMS_B200_ERR_ARGUMENT, "more than 2^32-2 spectra");
  const uint32_t W = ctx->cb.W;
  HB_TRY(ensure(ctx, ctx->scratch[kScrFusedRows], std::max<size_t>(1, n) * W * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrEncOk], std::max<size_t>(1, n)));
  auto* d_rows = ctx->scratch[kScrFusedRows].as<uint64_t>();
  auto* d_ok = ctx->scratch[kScrEncOk].as<uint8_t>();
  cudaStream_t st = ctx->stream;
  // encode every parsed spectrum where it lies (the CSR never left the device) ...
  HB_TRY(encode_dev_locked(ctx, cfg, n, mg.d_offsets, mg.d_mz, mg.d_int, d_rows, d_ok));
  // ... and let the host decide the order-preserving compaction from two bytes per spectrum
  std::vector<uint8_t> ok(n), charge(n);
  if (n) {
    HB_CUDA(ctx, cudaMemcpyAsync(ok.data(), d_ok, n, cudaMemcpyDeviceToHost, st));
    HB_CUDA(ctx, cudaMemcpyAsync(charge.data(), mg.d_charge, n, cudaMemcpyDeviceToHost, st));
    HB_CUDA(ctx, cudaStreamSynchronize(st));
  }
  std::vector<uint32_t> rows;
  rows.reserve(n);
  for (uint64_t i = 0; i < n; ++i) {
    uint8_t state = 0;
    if (charge[i] == 0) {
      state = 1;  // pipeline.cpp:127-134: no known charge, never encoded by the reference
    } else {
      // quantize_intensity's exception escapes the reference's encode_spectra (pipeline.cpp:67-72)
      HB_REQUIRE(ctx, ok[i] != HOMS_B200_OK_FLAG_INVARIANT, HOMS_B200_ERR_INVARIANT,
                 "quantize_intensity: intensity outside [0, 1]");
      if (!ok[i]) state = 2;
      else rows.push_back(static_cast<uint32_t>(i));
    }
    if (out_state) out_state[i] = state;
  }
  const uint64_t m = rows.size();
  if (out_n_queries) *out_n_queries = m;
  Queries& q = ctx->q;
  q.ready = false;
  q.dim = ctx->cb.dim;
  q.nq = m;
  const uint32_t S = stride_for(q.dim);
  HB_TRY(ensure(ctx, q.d_words, m * S * 8));
  HB_TRY(ensure(ctx, q.d_mz, m * 8));
  HB_TRY(ensure(ctx, q.d_charge, m));
  if (m) {
    HB_TRY(ensure(ctx, ctx->scratch[kScrFusedOk], m * 4));
    auto* d_idx = ctx->scratch[kScrFusedOk].as<uint32_t>();
    HB_CUDA(ctx, cudaMemcpyAsync(d_idx, rows.data(), m * 4, cudaMemcpyHostToDevice, st));
    gather_rows_kernel<<<static_cast<unsigned>((m * 32 + 255) / 256), 256, 0, st>>>(m, d_idx, d_rows,
                                                                                   q.d_words.as<uint64_t>(), W, S);
    HB_LAUNCHED(ctx);
    gather_meta_kernel<<<static_cast<unsigned>((m + 255) / 256), 256, 0, st>>>(
        m, d_idx, mg.d_pepmass, mg.d_charge, q.d_mz.as<double>(), q.d_charge.as<uint8_t>());
    HB_LAUNCHED(ctx);
    HB_CUDA(ctx, cudaStreamSynchronize(st));  // `rows` goes out of scope
  }
  q.ready = true;
  if (is_group(ctx)) HB_TRY(queries_replicate_locked(ctx));
  return HOMS_B200_OK;
}

}  // extern "C"
