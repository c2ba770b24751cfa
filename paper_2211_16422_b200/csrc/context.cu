// Context lifetime, device buffers, and the host-only pieces of the ABI (configuration checks,
// codebook generation, FDR curve).  Reference lines cited are under /root/reference/proj/core/.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>

#include "common.cuh"

namespace {
thread_local std::string g_global_error;
}

namespace hb {

int set_error(const homs_b200_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->error = msg;
  else g_global_error = msg;
  return code;
}

int ensure(homs_b200_ctx* ctx, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return HOMS_B200_OK;
  if (b.p) {
    // pending work may still read the old block
    HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    HB_CUDA(ctx, cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
  }
  const size_t want = (bytes + 255) / 256 * 256;
  HB_CUDA(ctx, cudaMalloc(&b.p, want));
  b.cap = want;
  return HOMS_B200_OK;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

int ensure_pinned(homs_b200_ctx* ctx, size_t bytes) {
  if (ctx->pinned_cap >= bytes) return HOMS_B200_OK;
  if (ctx->pinned) {
    HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_cap = 0;
  }
  HB_CUDA(ctx, cudaMallocHost(&ctx->pinned, bytes));
  ctx->pinned_cap = bytes;
  return HOMS_B200_OK;
}


int upload_rows(homs_b200_ctx* ctx, uint64_t* d_dst, const uint64_t* h_src, uint64_t n, uint32_t W,
                uint32_t S) {
  if (n == 0) return HOMS_B200_OK;
  if (W == S) {
    HB_CUDA(ctx, cudaMemcpyAsync(d_dst, h_src, n * W * 8, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    HB_CUDA(ctx, cudaMemsetAsync(d_dst, 0, n * S * 8, ctx->stream));
    HB_CUDA(ctx, cudaMemcpy2DAsync(d_dst, size_t(S) * 8, h_src, size_t(W) * 8, size_t(W) * 8, n,
                                   cudaMemcpyHostToDevice, ctx->stream));
  }
  return HOMS_B200_OK;
}

int download_rows(homs_b200_ctx* ctx, uint64_t* h_dst, const uint64_t* d_src, uint64_t n,
                  uint32_t W, uint32_t S) {
  if (n == 0) return HOMS_B200_OK;
  if (W == S) {
    HB_CUDA(ctx, cudaMemcpyAsync(h_dst, d_src, n * W * 8, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    HB_CUDA(ctx, cudaMemcpy2DAsync(h_dst, size_t(W) * 8, d_src, size_t(S) * 8, size_t(W) * 8, n,
                                   cudaMemcpyDeviceToHost, ctx->stream));
  }
  return HOMS_B200_OK;
}

int repack_rows_dev(homs_b200_ctx* ctx, uint64_t* d_dst, const uint64_t* d_src, uint64_t n,
                    uint32_t W, uint32_t S) {
  if (n == 0) return HOMS_B200_OK;
  if (W == S) {
    HB_CUDA(ctx, cudaMemcpyAsync(d_dst, d_src, n * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    HB_CUDA(ctx, cudaMemsetAsync(d_dst, 0, n * S * 8, ctx->stream));
    HB_CUDA(ctx, cudaMemcpy2DAsync(d_dst, size_t(S) * 8, d_src, size_t(W) * 8, size_t(W) * 8, n,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return HOMS_B200_OK;
}

static uint32_t env_u32(const char* name) {
  const char* e = getenv(name);
  return e ? static_cast<uint32_t>(std::max(1, atoi(e))) : 0u;
}

int ctx_create_single(int device, homs_b200_ctx** out) {
  if (!out) return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "ctx_create: out is null");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return set_error(nullptr, HOMS_B200_ERR_CUDA,
                     std::string("no CUDA device available (this library has no CPU fallback): ") +
                         cudaGetErrorString(e));
  if (device < 0 || device >= count)
    return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "ctx_create: device index out of range");
  e = cudaSetDevice(device);
  if (e != cudaSuccess)
    return set_error(nullptr, HOMS_B200_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  auto* ctx = new homs_b200_ctx;
  ctx->device = device;
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    delete ctx;
    return set_error(nullptr, HOMS_B200_ERR_CUDA, std::string("cudaGetDeviceProperties: ") + cudaGetErrorString(e));
  }
  ctx->sm_count = prop.multiProcessorCount;
  e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return set_error(nullptr, HOMS_B200_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
  }
  ctx->stream = ctx->own_stream;
  // planner development knobs: read here, once, never on the search path
  ctx->knobs.group_tiles = env_u32("HOMS_B200_TC_GROUP");
  ctx->knobs.items_per_sm = env_u32("HOMS_B200_TC_ITEMS_PER_SM");
  ctx->knobs.max_strip = env_u32("HOMS_B200_TC_MAX_STRIP");
  ctx->knobs.item_cap = env_u32("HOMS_B200_TC_ITEM_CAP");
  ctx->knobs.group_mb = env_u32("HOMS_B200_TC_GROUP_MB");
  ctx->knobs.ccap = env_u32("HOMS_B200_TC_CCAP");
  if (const char* e = getenv("HOMS_B200_TC_TOPK"))
    ctx->knobs.topk_lists = std::string(e) == "lists" ? 1u : (std::string(e) == "collect" ? 2u : 0u);
  if (const char* e = getenv("HOMS_B200_TC_L2_HINTS")) ctx->knobs.l2_hints = static_cast<uint32_t>(atoi(e)) & 3u;
  ctx->knobs.debug = env_u32("HOMS_B200_TC_DEBUG");
  if (const char* e = getenv("HOMS_B200_TC_ARES")) ctx->knobs.ares = atoi(e) != 0 ? 1u : 0u;
  if (const char* e = getenv("HOMS_B200_TC_PAIR")) ctx->knobs.pair = atoi(e) != 0 ? 1u : 0u;
  ctx->tc_pair_ctas = ctx->knobs.pair ? tc_query_pair_ctas(ctx) : 0;
  *out = ctx;
  return HOMS_B200_OK;
}

void ctx_free_resources(homs_b200_ctx* ctx) {
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& b : ctx->scratch) release(b);
  for (DevBuf* b : {&ctx->cb.d_pos, &ctx->cb.d_lvl, &ctx->lib.d_mz, &ctx->lib.d_id_rank,
                    &ctx->lib.d_ord_of_rank, &ctx->lib.d_mz_local, &ctx->lib.d_id_rank_local,
                    &ctx->lib.d_words, &ctx->lib.d_buckets, &ctx->lib.d_bucket_of_charge, &ctx->lib.d_x,
                    &ctx->q.d_words, &ctx->q.d_mz, &ctx->q.d_charge, &ctx->group_gather})
    release(*b);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t e : {ctx->pipe_in_ready[i], ctx->pipe_done[i], ctx->pipe_out_free[i]})
      if (e) cudaEventDestroy(e);
  for (auto& list : ctx->prof)
    for (auto& pr : list) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
  if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
  cudaStreamDestroy(ctx->own_stream);
}

}  // namespace hb

using namespace hb;

extern "C" {

int homs_b200_abi_version(void) { return HOMS_B200_ABI_VERSION; }

int homs_b200_ctx_create(int device, homs_b200_ctx** out) { return ctx_create_single(device, out); }

int homs_b200_device_count(int* out_count) {
  if (!out_count) return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "device_count: out is null");
  *out_count = 0;
  const cudaError_t e = cudaGetDeviceCount(out_count);
  if (e != cudaSuccess)
    return set_error(nullptr, HOMS_B200_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  return HOMS_B200_OK;
}

void homs_b200_ctx_destroy(homs_b200_ctx* ctx) {
  if (!ctx) return;
  group_destroy_members(ctx);  // no-op for a plain context
  ctx_free_resources(ctx);
  delete ctx;
}

const char* homs_b200_last_error(const homs_b200_ctx* ctx) {
  return ctx ? ctx->error.c_str() : g_global_error.c_str();
}

int homs_b200_ctx_set_stream(homs_b200_ctx* ctx, void* cuda_stream) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
  return HOMS_B200_OK;
}

int homs_b200_ctx_set_engine(homs_b200_ctx* ctx, int engine) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, engine >= HOMS_B200_ENGINE_AUTO && engine <= HOMS_B200_ENGINE_DIRECT,
             HOMS_B200_ERR_ARGUMENT, "set_engine: unknown engine");
  const bool tensor = engine == HOMS_B200_ENGINE_TENSOR || engine == HOMS_B200_ENGINE_TENSOR_FP4;
  HB_REQUIRE(ctx, !tensor || !ctx->lib.ready || tc_available(ctx), HOMS_B200_ERR_STATE,
             "set_engine: the resident library was uploaded without the tensor image");
  if (engine == HOMS_B200_ENGINE_TENSOR) engine = HOMS_B200_ENGINE_TENSOR_FP4;  // one tensor encoding (e2m1)
  ctx->engine = engine;
  for (size_t g = 1; g < ctx->members.size(); ++g) ctx->members[g]->engine = engine;
  return HOMS_B200_OK;
}

int homs_b200_ctx_last_engine(const homs_b200_ctx* ctx) { return ctx ? ctx->last_engine : -1; }
int homs_b200_ctx_tensor_cta_pairs(const homs_b200_ctx* ctx) { return ctx ? (hb::tc_uses_pairs(ctx) ? 1 : 0) : -1; }

int homs_b200_ctx_synchronize(homs_b200_ctx* ctx) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  return sync_all_locked(ctx);
}

uint64_t homs_b200_ctx_launch_count(const homs_b200_ctx* ctx) {
  if (!ctx) return 0;
  uint64_t total = ctx->launches;
  for (size_t g = 1; g < ctx->members.size(); ++g) total += ctx->members[g]->launches;
  return total;
}

int homs_b200_ctx_profile(homs_b200_ctx* ctx, int enable) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  ctx->profiling = enable != 0;
  for (size_t g = 1; g < ctx->members.size(); ++g) ctx->members[g]->profiling = enable != 0;
  return HOMS_B200_OK;
}

int homs_b200_ctx_kernel_time(homs_b200_ctx* ctx, int which, double* out_total_ms,
                              uint64_t* out_launches) {
  if (!ctx || which < 0 || which > 2) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  double total = 0.0;
  uint64_t count = 0;
  const size_t n_members = std::max<size_t>(1, ctx->members.size());
  for (size_t g = 0; g < n_members; ++g) {  // a group reports the sum over its members
    homs_b200_ctx* m = g == 0 ? ctx : ctx->members[g];
    cudaSetDevice(m->device);
    HB_CUDA(ctx, cudaStreamSynchronize(m->stream));
    for (auto& pr : m->prof[which]) {
      float ms = 0.f;
      HB_CUDA(ctx, cudaEventElapsedTime(&ms, pr.first, pr.second));
      total += ms;
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    count += m->prof[which].size();
    m->prof[which].clear();
  }
  cudaSetDevice(ctx->device);
  if (out_total_ms) *out_total_ms = total;
  if (out_launches) *out_launches = count;
  return HOMS_B200_OK;
}

int homs_b200_tensor_peak_probe(homs_b200_ctx* ctx, int engine, double seconds, double* out_ops_per_s,
                                double* out_kernel_ms) {
  if (!ctx || !out_ops_per_s) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, engine == HOMS_B200_ENGINE_TENSOR || engine == HOMS_B200_ENGINE_TENSOR_FP4,
             HOMS_B200_ERR_ARGUMENT, "tensor_peak_probe: engine must be TENSOR_FP4");
  HB_REQUIRE(ctx, seconds > 0.0 && seconds <= 10.0, HOMS_B200_ERR_ARGUMENT,
             "tensor_peak_probe: seconds must be in (0, 10]");
  return tc_peak_probe(ctx, seconds, out_ops_per_s, out_kernel_ms);
}

// ---- host-only configuration --------------------------------------------------------------

static constexpr double kBinEpsilon = 1e-9;  // preprocess.cpp:17

int homs_b200_preprocess_validate(const homs_b200_preprocess_config* c) {  // preprocess.cpp:21-34
  if (!c) return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "preprocess config is null");
  if (!(c->min_mz < c->max_mz))
    return set_error(nullptr, HOMS_B200_ERR_CONFIG, "preprocess: min_mz must be smaller than max_mz");
  if (!(c->bin_size > 0.0))
    return set_error(nullptr, HOMS_B200_ERR_CONFIG, "preprocess: bin_size must be positive");
  if (c->min_peaks < 1 || c->max_peaks < c->min_peaks)
    return set_error(nullptr, HOMS_B200_ERR_CONFIG, "preprocess: need max_peaks >= min_peaks >= 1");
  if (!(c->intensity_floor >= 0.0 && c->intensity_floor < 1.0))
    return set_error(nullptr, HOMS_B200_ERR_CONFIG, "preprocess: intensity_floor must lie in [0, 1)");
  return HOMS_B200_OK;
}

uint32_t homs_b200_dimension(const homs_b200_preprocess_config* c) {  // preprocess.cpp:36-39
  const double q = (c->max_mz - c->min_mz) / c->bin_size;
  return static_cast<uint32_t>(std::ceil(q - kBinEpsilon));
}

int homs_b200_encoder_validate(const homs_b200_encoder_config* c) {  // codebook.cpp:26-36
  if (!c) return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "encoder config is null");
  if (c->dim < 64 || c->dim % 64 != 0)
    return set_error(nullptr, HOMS_B200_ERR_CONFIG, "encoder dim must be a multiple of 64 and at least 64");
  if (c->step_flips < 1)
    return set_error(nullptr, HOMS_B200_ERR_CONFIG, "encoder step_flips must be at least 1");
  if (c->levels < 2)
    return set_error(nullptr, HOMS_B200_ERR_CONFIG, "encoder levels must be at least 2");
  return HOMS_B200_OK;
}

int homs_b200_quantize_intensity(double v, uint32_t levels, uint32_t* out) {  // encoder.cpp:11-17
  if (!(v >= 0.0 && v <= 1.0))
    return set_error(nullptr, HOMS_B200_ERR_INVARIANT, "quantize_intensity: intensity outside [0, 1]");
  const double level = std::round(v * static_cast<double>(levels));
  *out = std::min(static_cast<uint32_t>(level), levels);
  return HOMS_B200_OK;
}

namespace {

// rng.hpp:10-44.  std::mt19937_64 is fully specified by ISO C++, so the streams are identical to
// the reference's on every toolchain.
uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
uint64_t named_stream(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag)); }

uint64_t draw_below(std::mt19937_64& rng, uint64_t n) {  // mask rejection, rng.hpp:26-39
  uint64_t mask = n - 1;
  for (int s = 1; s < 64; s <<= 1) mask |= mask >> s;
  for (;;) {
    const uint64_t v = rng() & mask;
    if (v < n) return v;
  }
}

void fill_random(uint64_t* w, uint32_t dim, std::mt19937_64& rng) {  // codebook.cpp:17-22
  const uint32_t W = hb::words_for(dim);
  for (uint32_t i = 0; i < W; ++i) w[i] = rng();
  if (dim % 64) w[W - 1] &= (uint64_t{1} << (dim % 64)) - 1;
}

inline void toggle(uint64_t* w, uint32_t bit) { w[bit >> 6] ^= uint64_t{1} << (bit & 63); }

}  // namespace

int homs_b200_make_codebook(const homs_b200_encoder_config* c, uint32_t n_bins, uint64_t* pos,
                            uint64_t* lvl) {
  if (!c || !pos || !lvl) return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "make_codebook: null argument");
  if (c->dim == 0 || c->levels == 0)
    return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "make_codebook: dim and levels must be positive");
  const uint32_t dim = c->dim, W = hb::words_for(dim);

  // position rows: a chain, each row = predecessor with step_flips with-replacement flips
  // (codebook.cpp:38-53); stream tag "position" (:14)
  {
    std::mt19937_64 rng(named_stream(c->seed, 0x706f736974696f6eULL));
    std::vector<uint64_t> cur(W);
    fill_random(cur.data(), dim, rng);
    for (uint32_t i = 0; i < n_bins; ++i) {
      if (i > 0)
        for (uint32_t k = 0; k < c->step_flips; ++k)
          toggle(cur.data(), static_cast<uint32_t>(draw_below(rng, dim)));
      std::memcpy(pos + size_t(i) * W, cur.data(), size_t(W) * 8);
    }
  }
  // level rows: level q = level 0 with the first floor((dim/2) q / Q) entries of one partial
  // Fisher-Yates order flipped (codebook.cpp:55-85); stream tag "levelhvs" (:15)
  {
    std::mt19937_64 rng(named_stream(c->seed, 0x6c6576656c687673ULL));
    const uint32_t half = dim / 2;
    std::vector<uint64_t> cur(W);
    fill_random(cur.data(), dim, rng);
    std::vector<uint32_t> order(dim);
    std::iota(order.begin(), order.end(), 0u);
    for (uint32_t i = 0; i < half; ++i)
      std::swap(order[i], order[i + static_cast<uint32_t>(draw_below(rng, dim - i))]);
    uint64_t done = 0;
    for (uint32_t q = 0; q <= c->levels; ++q) {
      const uint64_t cut = uint64_t(half) * q / c->levels;
      for (; done < cut; ++done) toggle(cur.data(), order[done]);
      std::memcpy(lvl + size_t(q) * W, cur.data(), size_t(W) * 8);
    }
  }
  return HOMS_B200_OK;
}

int homs_b200_compute_fdr_curve(uint64_t n, const double* score, const uint8_t* is_decoy,
                                uint64_t* out_input_index, double* out_fdr, double* out_q) {
  // fdr.cpp:8-50: stable order by (score desc, decoy before target), running counts,
  // fdr = decoys / max(1, targets), q = suffix minimum.
  if (n == 0) return HOMS_B200_OK;
  if (!score || !is_decoy || !out_input_index || !out_fdr || !out_q)
    return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "compute_fdr_curve: null argument");
  std::iota(out_input_index, out_input_index + n, uint64_t{0});
  std::stable_sort(out_input_index, out_input_index + n, [&](uint64_t a, uint64_t b) {
    if (score[a] != score[b]) return score[a] > score[b];
    return (is_decoy[a] != 0) > (is_decoy[b] != 0);
  });
  uint64_t targets = 0, decoys = 0;
  for (uint64_t p = 0; p < n; ++p) {
    (is_decoy[out_input_index[p]] ? decoys : targets) += 1;
    out_fdr[p] = static_cast<double>(decoys) / static_cast<double>(std::max<uint64_t>(1, targets));
  }
  double low = out_fdr[n - 1];
  for (uint64_t p = n; p-- > 0;) {
    low = std::min(low, out_fdr[p]);
    out_q[p] = low;
  }
  return HOMS_B200_OK;
}

}  // extern "C"
