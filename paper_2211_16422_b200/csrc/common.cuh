// Internal definitions shared by the translation units of libhoms_b200.so.
// Nothing here is part of the ABI (that is include/homs_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "homs_b200.h"

namespace hb {

// Device row layout: every hypervector row is padded with zero words to a multiple of 128 bytes
// (16 u64) so that a row is a whole number of 128-byte cp.async / LDS.128 chunks groups.  Padding
// is zero in library AND query rows, so XOR+popcount over the padded row equals the reference's
// sum over W words (hypervector.hpp:70-81).
constexpr uint32_t kRowAlignWords = 16;

inline uint32_t words_for(uint32_t dim) { return (dim + 63u) / 64u; }
inline uint32_t stride_for(uint32_t dim) {
  return (words_for(dim) + kRowAlignWords - 1) / kRowAlignWords * kRowAlignWords;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct BucketDev {           // one charge bucket, device + host view
  uint64_t begin;            // offset of the bucket in the library-wide sorted order
  uint64_t size;             // rows in the full bucket
  uint64_t shard_begin;      // [shard_begin, shard_end) of the bucket is resident here ...
  uint64_t shard_end;
  uint64_t local_offset;     // ... at local rows [local_offset, local_offset + shard_end - shard_begin)
};

// One candidate of the windowed top-k, == homs_b200_candidate (16 bytes).  Lexicographic order on
// (d, ad, rk) is the reference's key (score desc, |q - r| asc, id asc, ordinal asc),
// search.cpp:133-146.
struct Cand {
  uint32_t d, rk;
  uint64_t ad;
};
static_assert(sizeof(Cand) == 16 && sizeof(homs_b200_candidate) == 16, "candidate record is 16 bytes");
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct Library {
  bool ready = false;
  uint32_t dim = 0, W = 0, S = 0;  // bits, dense words, padded stride (u64 words)
  uint64_t n = 0, n_local = 0;
  uint32_t shard_index = 0, shard_count = 1;
  std::vector<uint8_t> bucket_charge;
  std::vector<BucketDev> buckets;
  std::vector<double> h_mz;         // full library, sorted order
  std::vector<uint32_t> h_ordinal;  // full library, sorted order
  // device (owned through ctx buffers)
  DevBuf d_mz, d_id_rank, d_ord_of_rank, d_mz_local, d_id_rank_local, d_words, d_buckets,
      d_bucket_of_charge;
  // +-1 e2m1 image of the resident rows for the tensor-core engine (search_tc.cu):
  // [n_kc][x_rows][128 B], every 128-byte row pre-swizzled for a SWIZZLE_128B K-major UMMA operand
  DevBuf d_x;
  uint64_t x_rows = 0;  // n_local rounded up to the 224-row tile, plus one all-zero tile of slack
  uint32_t n_kc = 0;    // k-chunks: ceil(dim / 256)
};

struct Queries {
  bool ready = false;
  uint32_t dim = 0;
  uint64_t nq = 0;
  DevBuf d_words, d_mz, d_charge;  // words: padded stride of the query dim
};

struct MgfState {  // CSR result of the last homs_b200_mgf_parse, resident in the context's scratch
  bool ready = false;
  uint64_t n_spectra = 0, n_peaks = 0;
  const uint64_t* d_offsets = nullptr;
  const double *d_mz = nullptr, *d_int = nullptr, *d_pepmass = nullptr;
  const uint8_t* d_charge = nullptr;
  const uint32_t *d_title_off = nullptr, *d_title_len = nullptr, *d_seq_off = nullptr, *d_seq_len = nullptr;
};

struct Codebook {
  bool ready = false;
  uint32_t dim = 0, n_bins = 0, levels = 0, W = 0, S = 0;
  DevBuf d_pos, d_lvl;  // padded rows
};

struct GroupWorkers;  // group.cu: one issuing thread per non-leading member of a multi-GPU group

// development knobs of the tensor-engine planner, read from the environment ONCE per context
// (homs_b200_ctx_create), never on the search path; 0 = the built-in choice
struct TcKnobs {
  uint32_t group_tiles = 0, items_per_sm = 0, max_strip = 0, item_cap = 0, group_mb = 0;
  uint32_t l2_hints = 0;  // see TcParams::l2_hints (default: none; round 2's evict_first on library tiles stopped paying)
  uint32_t topk_lists = 0;  // top-k path: 0 / 2 = collect + select (default), 1 = register-list passes
  uint32_t ccap = 0;        // collect mode: candidate buffer entries per query (0: built-in)
  uint32_t ares = 1;        // 0: never keep the query tile's k-chunks resident in shared memory (HOMS_B200_TC_ARES)
  uint32_t debug = 0;       // 1: development statistics on stderr (HOMS_B200_TC_DEBUG)
  uint32_t pair = 2;        // tensor search on CTA pairs (cta_group::2, search_tc.cu TcShape<true>): 0 never, 1 always, 2 by dimension
};

}  // namespace hb

struct homs_b200_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  mutable std::string error;
  uint64_t launches = 0;
  hb::Codebook cb;
  hb::Library lib;
  hb::Queries q;
  hb::MgfState mgf;
  // grow-only scratch, keyed by purpose
  enum { kScratchSlots = 56 };
  hb::DevBuf scratch[kScratchSlots];
  int engine = HOMS_B200_ENGINE_AUTO;  // homs_b200_ctx_set_engine
  int last_engine = HOMS_B200_ENGINE_AUTO;  // engine the last search call ran on (never AUTO after a search)
  void* pinned = nullptr;  // small pinned staging block
  size_t pinned_cap = 0;
  // chunked host <-> device pipeline of the encoder (encode.cu:encode_pipeline): copy-in and
  // copy-out streams beside the compute stream, per-slot events, created on first use
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t pipe_in_ready[2] = {nullptr, nullptr}, pipe_done[2] = {nullptr, nullptr},
              pipe_out_free[2] = {nullptr, nullptr};
  // optional per-kernel timing (homs_b200_ctx_profile)
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof[3];
  hb::TcKnobs knobs;
  int tc_pair_ctas = 0;  // grid of the CTA-pair search kernel: 2 x co-resident 2-CTA clusters (0: unavailable)
  // ---- multi-GPU group (homs_b200_ctx_create_multi, group.cu) --------------------------------
  // members[0] == this (the leader, on devices[0]); members[g >= 1] are owned single-device contexts
  // that are only ever driven through the leader (under the leader's mutex).  Empty: a plain context.
  std::vector<homs_b200_ctx*> members;
  std::vector<uint8_t> peer_ok;      // member g's device addresses the leader's memory (same device, or P2P on)
  std::vector<cudaEvent_t> ev_join;  // member g's work of the current group call is complete (g >= 1)
  cudaEvent_t ev_fork = nullptr;     // leader's stream has reached the start of the current group call
  hb::DevBuf group_gather;           // leader: [n_members][n][k] candidate records, written by the members
  hb::GroupWorkers* workers = nullptr;
};

namespace hb {

int set_error(const homs_b200_ctx* ctx, int code, const std::string& msg);

#define HB_CUDA(ctx, expr)                                                                   \
  do {                                                                                       \
    cudaError_t e__ = (expr);                                                                \
    if (e__ != cudaSuccess)                                                                  \
      return ::hb::set_error((ctx), HOMS_B200_ERR_CUDA,                                      \
                             std::string(#expr) + ": " + cudaGetErrorString(e__));           \
  } while (0)

#define HB_TRY(expr)                      \
  do {                                    \
    int rc__ = (expr);                    \
    if (rc__ != HOMS_B200_OK) return rc__; \
  } while (0)

#define HB_REQUIRE(ctx, cond, code, msg)                     \
  do {                                                       \
    if (!(cond)) return ::hb::set_error((ctx), (code), (msg)); \
  } while (0)

// Kernel launch bookkeeping: counts the launch and checks for launch errors.
#define HB_LAUNCHED(ctx)               \
  do {                                 \
    ++(ctx)->launches;                 \
    HB_CUDA((ctx), cudaGetLastError()); \
  } while (0)

// Brackets one kernel launch with events when profiling is on.
struct KernelTimer {
  KernelTimer(homs_b200_ctx* c, int which) : ctx(c), slot(which) {
    if (!ctx->profiling) return;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, ctx->stream);
  }
  ~KernelTimer() {
    if (!e0) return;
    cudaEventRecord(e1, ctx->stream);
    ctx->prof[slot].emplace_back(e0, e1);
  }
  homs_b200_ctx* ctx;
  int slot;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

int ensure(homs_b200_ctx* ctx, DevBuf& b, size_t bytes);
int ensure_pinned(homs_b200_ctx* ctx, size_t bytes);
void release(DevBuf& b);

// scratch slot names
enum Scratch {
  kScrOffsets = 0, kScrMz, kScrInt, kScrSvBins, kScrSvLev, kScrSvCount, kScrEncOut, kScrEncOk,
  kScrQFirst, kScrQLast, kScrKeys, kScrKeysAlt, kScrVals, kScrValsAlt, kScrCub, kScrPlan,
  kScrPartial, kScrRecords, kScrSubset, kScrDecode, kScrMisc, kScrMisc2, kScrRecords2, kScrHas,
  kScrTcQx, kScrTcPlan, kScrTcPartial, kScrTcTiles, kScrTcBest, kScrFnv, kScrCacheBlock,
  kScrPipeIn0, kScrPipeIn1, kScrPipeOut0, kScrPipeOut1, kScrFusedRows, kScrFusedOk,
  kScrMgfText, kScrMgfTiles, kScrMgfLines, kScrMgfBlocks, kScrMgfPeaks, kScrMgfHard, kScrIndexSort,
  kScrTcCount, kScrTcBuf, kScrTcOverflow, kScrTcKeysFix
};

// Tensor-core engine (search_tc.cu).  expand: packed rows -> +-1 e2m1 swizzled image.
int tc_expand_library(homs_b200_ctx* ctx);
// top-k (k <= tc_max_topk()) of n sorted slots (keys/vals as produced by bounds + radix sort) -> out[slot * k_stride + j]
int tc_search_sorted(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n, const uint64_t* d_keys,
                     const uint32_t* d_vals, Cand* d_out, uint32_t k, uint32_t k_stride);
uint32_t tc_max_topk();
bool tc_available(const homs_b200_ctx* ctx);
int tc_peak_probe(homs_b200_ctx* ctx, double seconds, double* out_ops_per_s, double* out_ms);
int tc_query_pair_ctas(homs_b200_ctx* ctx);
bool tc_uses_pairs(const homs_b200_ctx* ctx);  // CTA pairs (cta_group::2) for the resident library?

// dense host rows (W words) -> padded device rows (S words), zero padded.  Async on ctx->stream.
int upload_rows(homs_b200_ctx* ctx, uint64_t* d_dst, const uint64_t* h_src, uint64_t n, uint32_t W,
                uint32_t S);
int download_rows(homs_b200_ctx* ctx, uint64_t* h_dst, const uint64_t* d_src, uint64_t n,
                  uint32_t W, uint32_t S);
// dense device rows -> padded device rows
int repack_rows_dev(homs_b200_ctx* ctx, uint64_t* d_dst, const uint64_t* d_src, uint64_t n,
                    uint32_t W, uint32_t S);

// Chunked, double-buffered encoder pipeline over HOST spectra (CSR): H2D of chunk c+1 and D2H of
// chunk c-1 overlap the kernels of chunk c.  Hypervector rows go to d_keep (dense u64[n][W] on the
// device, may be null) and/or h_words (host, may be null); ok flags likewise.
int encode_pipeline(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                    const uint64_t* offsets, const double* mz, const double* intensity, uint64_t* d_keep,
                    uint8_t* d_keep_ok, uint64_t* h_words, uint8_t* h_ok);
// refine_peaks -> vectorize -> encode of n spectra whose CSR is on the device; dense rows + ok flags out
int encode_dev_locked(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                      const uint64_t* d_off, const double* d_mz, const double* d_int, uint64_t* d_out,
                      uint8_t* d_ok);
// build_index over rows already on the device; row_of_entry (host, may be null) maps entry i of the
// metadata arrays to its row in d_words
int library_build_from_device(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* d_words,
                              const double* mz, const uint8_t* charge, const uint32_t* id_rank,
                              uint32_t shard_index, uint32_t shard_count,
                              const uint32_t* row_of_entry = nullptr);

struct Lock {
  explicit Lock(homs_b200_ctx* c) : g(c->mu) { cudaSetDevice(c->device); }
  std::lock_guard<std::mutex> g;
};

// ---- multi-GPU group (group.cu) -----------------------------------------------------------------
inline bool is_group(const homs_b200_ctx* c) { return !c->members.empty(); }
// runs fn(g) for every member: g = 0 on the calling thread, g >= 1 on that member's issuing thread
// with its device current; returns the first non-OK code (the member's message copied to the leader)
int group_for_each(homs_b200_ctx* leader, const std::function<int(uint32_t, homs_b200_ctx*)>& fn);
// leader's stream -> every member's stream (work enqueued by members after this sees the leader's
// earlier work) and back (the leader's later work sees the members')
int group_fork(homs_b200_ctx* leader);
int group_join(homs_b200_ctx* leader);
void group_destroy_members(homs_b200_ctx* leader);
int sync_all_locked(homs_b200_ctx* ctx);  // the context's stream, and every member's for a group  // no-op for a plain context

// single-context building blocks the group composes (defined in search.cu / library.cu)
int search_dev_locked(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n, const homs_b200_tolerance* tol,
                      uint32_t k, Cand* d_out, uint64_t* d_first, uint64_t* d_last, uint8_t* d_has);
int queries_set_locked(homs_b200_ctx* ctx, uint32_t dim, uint64_t nq, const uint64_t* words, const double* mz,
                       const uint8_t* charge, bool on_device);
int merge_launch(homs_b200_ctx* ctx, uint64_t n, uint32_t k, uint32_t n_parts, const Cand* d_parts, Cand* d_out);
int library_build(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* h_words, const uint64_t* d_words_in,
                  const double* mz, const uint8_t* charge, const uint32_t* id_rank, uint32_t shard_index,
                  uint32_t shard_count, const uint32_t* row_of_entry);
// the same operations on a plain context or on a group leader
int search_any_locked(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n, const homs_b200_tolerance* tol,
                      uint32_t k, Cand* d_out, uint64_t* d_first, uint64_t* d_last, uint8_t* d_has);
int queries_set_any_locked(homs_b200_ctx* ctx, uint32_t dim, uint64_t nq, const uint64_t* words, const double* mz,
                           const uint8_t* charge, bool on_device);
int queries_replicate_locked(homs_b200_ctx* leader);  // leader's resident queries -> every other member
int library_build_any(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* h_words,
                      const uint64_t* d_words_in, const double* mz, const uint8_t* charge, const uint32_t* id_rank,
                      uint32_t shard_index, uint32_t shard_count, const uint32_t* row_of_entry);
int codebook_upload_locked(homs_b200_ctx* ctx, uint32_t dim, uint32_t n_bins, uint32_t levels, const uint64_t* pos,
                           const uint64_t* lvl);
void ctx_free_resources(homs_b200_ctx* ctx);  // everything a single context owns (context.cu)
int ctx_create_single(int device, homs_b200_ctx** out);

}  // namespace hb
