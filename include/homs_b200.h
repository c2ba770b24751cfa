/* homs_b200.h -- C ABI of the B200-native HyperOMS hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch types.  The reference
 * (`homs_core`, C++20, CPU only) has no FFI layer of its own; its boundary is the public C++ API
 * of proj/core.  Each entry point below names the reference interface it
 * replaces (paths relative to /root/reference/proj/core/).  The C++ facade that keeps the
 * reference's signatures on top of this ABI is include/homs_b200/homs.hpp; INTEGRATION.md shows
 * the binding a reference maintainer would add.
 *
 * Conventions
 *   - every function returns HOMS_B200_OK (0) or an error code; homs_b200_last_error(ctx) gives
 *     the message.  HOMS_B200_ERR_CONFIG / _INVARIANT correspond to the reference's
 *     homs::ConfigError / homs::InvariantError (include/homs/errors.hpp:16-56); the C++ facade
 *     re-throws them as such.  No exception ever crosses this boundary.
 *   - hypervectors are little-endian u64 words, bit d at word d/64 bit d%64, tail bits zero,
 *     W = ceil(dim/64) words per row, rows dense (include/homs/hypervector.hpp:12-15).
 *   - spectra travel as CSR: offsets u64[n+1], mz f64[], intensity f64[]; peaks of one spectrum
 *     strictly ascending in m/z (RawSpectrum invariant, include/homs/spectrum.hpp:34-35).
 *   - the caller owns every host buffer for the duration of the call; the context owns all device
 *     memory.  Calls on one context are serialised internally; results never depend on the
 *     reference's `threads` / `batch_size` knobs (search.hpp:102-103), which therefore do not
 *     appear here.
 *   - functions with the suffix _dev take DEVICE pointers and enqueue work on the context's
 *     stream without synchronising; all others take HOST pointers and are blocking.
 *   - there is no CPU fallback: without a CUDA device homs_b200_ctx_create fails.
 */
#ifndef HOMS_B200_H
#define HOMS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOMS_B200_ABI_VERSION 2

enum {
  HOMS_B200_OK = 0,
  HOMS_B200_ERR_CONFIG = 1,    /* homs::ConfigError    */
  HOMS_B200_ERR_INVARIANT = 2, /* homs::InvariantError */
  HOMS_B200_ERR_CUDA = 3,      /* CUDA runtime failure (message carries cudaGetErrorString) */
  HOMS_B200_ERR_ARGUMENT = 4,  /* null pointer / size out of the supported range */
  HOMS_B200_ERR_STATE = 5,     /* call order (e.g. search before library upload) */
  HOMS_B200_ERR_CACHE_FORMAT = 6,  /* homs::CacheFormatError  (bad magic / version) */
  HOMS_B200_ERR_CACHE_STALE = 7,   /* homs::StaleCacheError   (profile block differs) */
  HOMS_B200_ERR_CACHE_CORRUPT = 8, /* homs::CacheCorruptError (truncated / bad string / checksum) */
  HOMS_B200_ERR_PARSE = 9          /* homs::ParseError (message: "line N: ...", errors.hpp:22-32) */
};

enum { HOMS_B200_TOL_PPM = 0, HOMS_B200_TOL_DALTON = 1 };
#define HOMS_B200_NO_HIT 0xFFFFFFFFu
#define HOMS_B200_MAX_TOPK 64u

typedef struct homs_b200_ctx homs_b200_ctx;

/* PreprocessConfig, include/homs/preprocess.hpp:13-25 */
typedef struct {
  double min_mz, max_mz, bin_size;
  uint32_t max_peaks, min_peaks;
  double intensity_floor;
  uint32_t scaling; /* IntensityScaling: 0 none, 1 sqrt (preprocess.hpp:11) */
  uint32_t reserved;
} homs_b200_preprocess_config;

/* EncoderConfig, include/homs/codebook.hpp:12-23 */
typedef struct {
  uint32_t dim, step_flips, levels, reserved;
  uint64_t seed;
} homs_b200_encoder_config;

/* Tolerance, include/homs/search.hpp:16-33 */
typedef struct {
  uint32_t kind; /* HOMS_B200_TOL_PPM | HOMS_B200_TOL_DALTON */
  uint32_t reserved;
  double value;
} homs_b200_tolerance;

/* One candidate of the windowed top-k: 16 bytes, ordered lexicographically by
 * (distance, abs_diff_bits, id_rank) == the reference's key (score desc, |q - r| asc, id asc,
 * ordinal asc) of search.cpp:133-146.  distance = dim - raw_score; abs_diff_bits is the IEEE-754
 * pattern of the non-negative double |q_mz - ref_mz| (monotone as an integer); id_rank is the
 * entry's position in the library-wide sort by (id, ordinal).  distance == 0xFFFFFFFF: empty. */
typedef struct {
  uint32_t distance;
  uint32_t id_rank;
  uint64_t abs_diff_bits;
} homs_b200_candidate;

/* ---- context ------------------------------------------------------------------------------- */

int homs_b200_abi_version(void);
/* Creates a context on CUDA device `device`.  *out is NULL on failure; the message is then
 * available through homs_b200_last_error(NULL). */
int homs_b200_ctx_create(int device, homs_b200_ctx** out);
/* CUDA devices visible to this process. */
int homs_b200_device_count(int* out_count);
/* ONE handle over n devices of this process: SURVEY.md 8(b)'s `ctx_create(device_ids[], n)`.  It takes
 * the place of the reference's only parallel construct, the thread fan-out of parallel_for
 * (include/homs/parallel.hpp:20-48, used by search_batch search.cpp:175-181 and encode_spectra
 * pipeline.cpp:66-73): every call below accepts the handle unchanged and fans out over the GPUs.
 *   - library_upload* / library_load_cache / library_build_from_spectra (pass shard 0 of 1): slice g of
 *     every charge bucket (contiguous precursor-m/z ranges) becomes resident on devices[g], metadata
 *     is replicated;
 *   - queries_* / search_batch / search_resident* / cascade_*: queries are replicated, every device
 *     searches its slice, the 16-byte candidate records are stored by each device's last kernel
 *     straight into the first device's memory (peer-mapped stores over NVLink) and merged there;
 *     results are identical to a single-device context;
 *   - codebook_upload: replicated; encode_batch: spectra split evenly over the devices;
 *   - everything else (window_bounds, preprocess_batch, encode_vectors, mgf_*, cache_write, _dev
 *     encoders) runs on devices[0].  Device pointers passed to _dev calls belong to devices[0].
 * devices may repeat (aliases of one GPU: the same code path, used by the single-GPU tests).
 * n_devices == 1 yields a plain context.  kernel_time() of a group is the sum over its devices. */
int homs_b200_ctx_create_multi(const int* devices, int n_devices, homs_b200_ctx** out);
/* Devices behind a handle (1 for homs_b200_ctx_create). */
int homs_b200_ctx_device_count(const homs_b200_ctx* ctx);
void homs_b200_ctx_destroy(homs_b200_ctx* ctx);
const char* homs_b200_last_error(const homs_b200_ctx* ctx);
/* Adopt an external cudaStream_t for all subsequent work (NULL: back to the context's own). */
int homs_b200_ctx_set_stream(homs_b200_ctx* ctx, void* cuda_stream);
int homs_b200_ctx_synchronize(homs_b200_ctx* ctx);
/* Kernels launched by this context so far (bench.py's gpu_launches). */
uint64_t homs_b200_ctx_launch_count(const homs_b200_ctx* ctx);
/* Per-kernel device timing for roofline reports: while enabled, every launch of the three hot
 * kernels is bracketed by CUDA events on the context's stream.  kernel_time() synchronises, returns
 * the summed duration and launch count since the last call, and resets the counters. */
enum { HOMS_B200_KERNEL_SEARCH = 0, HOMS_B200_KERNEL_ENCODE = 1, HOMS_B200_KERNEL_PREPROCESS = 2 };
/* Search engine: POPC (XOR + POPC on the integer pipes), DIRECT (warp per query) or TENSOR_FP4, a
 * tcgen05 tensor-core contraction of the +-1 expanded hypervectors (similarity = (dim + dot) / 2,
 * exact) with e2m1 operands and unit block scales.  AUTO = TENSOR_FP4, or DIRECT for calls with narrow
 * windows.  All engines are bit-exact.
 * Set it BEFORE library_upload: the tensor image of the library (4x the packed size) is built
 * there, and POPC / DIRECT skip it. */
enum {
  HOMS_B200_ENGINE_AUTO = 0,
  HOMS_B200_ENGINE_POPC = 1,
  HOMS_B200_ENGINE_TENSOR = 2,     /* alias of TENSOR_FP4 (the int8 operand encoding of ABI 1 was removed:
                                      twice the image, 2.3x slower, identical results) */
  HOMS_B200_ENGINE_TENSOR_FP4 = 3, /* e2m1 operands with unit block scales, fp32 accumulate (kind::mxf4) */
  HOMS_B200_ENGINE_DIRECT = 4      /* one warp per query over exactly its window rows (XOR + POPC, warp-level
                                      top-k): the engine for windows of a few dozen rows (ppm tolerances).
                                      AUTO picks it per call when the rows it would read are far fewer bytes
                                      than one pass over the tensor image; forcing it keeps only the packed
                                      rows */
};
int homs_b200_ctx_set_engine(homs_b200_ctx* ctx, int engine);
/* The engine the last search call of this context ran on (one of the non-AUTO codes; reporting aid). */
int homs_b200_ctx_last_engine(const homs_b200_ctx* ctx);
/* 1 when the tensor engine runs the resident library on CTA pairs (tcgen05 cta_group::2: two SMs per 256-query
 * tile, from D = 2048 up), 0 for one CTA per SM, -1 without a context (reporting aid). */
int homs_b200_ctx_tensor_cta_pairs(const homs_b200_ctx* ctx);
int homs_b200_ctx_profile(homs_b200_ctx* ctx, int enable);
int homs_b200_ctx_kernel_time(homs_b200_ctx* ctx, int which, double* out_total_ms,
                              uint64_t* out_launches);
/* Measurement aid (no reference counterpart): sustained issue rate of the tensor engine's MMA shape
 * on this device with every SM busy and no memory traffic -- the ceiling bench.py quotes the search
 * kernel against.  engine: HOMS_B200_ENGINE_TENSOR_FP4; runs for about `seconds`. */
int homs_b200_tensor_peak_probe(homs_b200_ctx* ctx, int engine, double seconds, double* out_ops_per_s,
                                double* out_kernel_ms);

/* ---- host-side configuration (no device work) ----------------------------------------------- */

/* PreprocessConfig::validate, src/preprocess.cpp:21-34 */
int homs_b200_preprocess_validate(const homs_b200_preprocess_config* cfg);
/* dimension(), src/preprocess.cpp:36-39 */
uint32_t homs_b200_dimension(const homs_b200_preprocess_config* cfg);
/* EncoderConfig::validate, src/codebook.cpp:26-36 */
int homs_b200_encoder_validate(const homs_b200_encoder_config* cfg);
/* quantize_intensity, src/encoder.cpp:11-17 (HOMS_B200_ERR_INVARIANT outside [0,1]) */
int homs_b200_quantize_intensity(double v, uint32_t levels, uint32_t* out_level);
/* make_codebook, src/codebook.cpp:87-94 (gen_position_hvs :38-53, gen_level_hvs :55-85).  The
 * RNG chain is inherently serial, so this runs on the host once per configuration.
 * pos: n_bins x W words, lvl: (levels+1) x W words. */
int homs_b200_make_codebook(const homs_b200_encoder_config* cfg, uint32_t n_bins, uint64_t* pos,
                            uint64_t* lvl);
/* compute_fdr_curve, src/fdr.cpp:8-50.  out_input_index[p] = input position of sorted position
 * p, out_fdr / out_q_value per sorted position. */
int homs_b200_compute_fdr_curve(uint64_t n, const double* score, const uint8_t* is_decoy,
                                uint64_t* out_input_index, double* out_fdr, double* out_q_value);

/* ---- encoding (preprocess.cpp:41-110, encoder.cpp:19-55, pipeline.cpp:60-85) --------------- */

/* Makes a codebook resident on the device (replaces the `const Codebook&` argument of
 * encode()/encode_spectra(), include/homs/codebook.hpp:29-34). */
int homs_b200_codebook_upload(homs_b200_ctx* ctx, uint32_t dim, uint32_t n_bins, uint32_t levels,
                              const uint64_t* pos, const uint64_t* lvl);

/* encode_spectra, src/pipeline.cpp:60-85: refine_peaks -> vectorize -> encode per spectrum.
 * out_ok[i] = 1 and row i of out_words holds the hypervector when spectrum i is processable,
 * else out_ok[i] = 0 and the row is zero (the reference drops such spectra; the C++ facade
 * compacts).  HOMS_B200_ERR_INVARIANT when homs_b200_dimension(cfg) != uploaded n_bins, and --
 * as quantize_intensity throws out of the reference's encode_spectra (src/encoder.cpp:12-14) --
 * when a kept peak's normalised intensity is outside [0, 1] (an infinite intensity: inf / inf).
 * The _dev form cannot fail late: it marks such a spectrum with
 * d_out_ok[i] = HOMS_B200_OK_FLAG_INVARIANT and a zero row, for the caller to act on. */
#define HOMS_B200_OK_FLAG_INVARIANT 2
int homs_b200_encode_batch(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                           const uint64_t* offsets, const double* mz, const double* intensity,
                           uint64_t* out_words, uint8_t* out_ok);
int homs_b200_encode_batch_dev(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg,
                               uint64_t n, uint64_t n_peaks_total, const uint64_t* d_offsets,
                               const double* d_mz, const double* d_intensity,
                               uint64_t* d_out_words, uint8_t* d_out_ok);

/* refine_peaks + vectorize + quantize_intensity only (preprocess.cpp:41-110, encoder.cpp:11-17):
 * per spectrum the ascending bin list and its levels.  out_bins / out_levels are
 * n x cfg->max_peaks (row i holds out_count[i] entries; out_count[i] = 0: unprocessable). */
int homs_b200_preprocess_batch(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg,
                               uint32_t levels, uint64_t n, const uint64_t* offsets,
                               const double* mz, const double* intensity, uint32_t* out_bins,
                               uint32_t* out_levels, uint32_t* out_count);

/* encode(), src/encoder.cpp:19-55, on already vectorized spectra (SpectrumVector,
 * preprocess.hpp:29-34) given as CSR (sv_offsets u64[n+1], bins u32[], intensities f64[] in
 * [0,1]).  HOMS_B200_ERR_INVARIANT on an empty vector, a bin >= n_bins or an intensity outside
 * [0,1] (encoder.cpp:20-25, :12-14). */
int homs_b200_encode_vectors(homs_b200_ctx* ctx, uint64_t n, const uint64_t* sv_offsets,
                             const uint32_t* bins, const double* intensities,
                             uint64_t* out_words);

/* hamming_similarity, include/homs/hypervector.hpp:70-81, for n row pairs. */
int homs_b200_hamming_similarity(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* a,
                                 const uint64_t* b, uint32_t* out_similarity);

/* ---- library index (build_index, src/search.cpp:17-60) ------------------------------------- */

/* Builds the charge-partitioned, precursor-m/z-sorted device index from entries in INPUT order
 * (ordinal = position in these arrays).  Sort key inside a charge bucket: (mz asc, id asc,
 * ordinal asc) == (mz asc, id_rank asc) where id_rank[i] is the position of entry i in the
 * library-wide sort by (id, ordinal); id_rank == NULL means "all ids equal" (rank = ordinal).
 * shard_index / shard_count: this context keeps hypervectors only for slice shard_index of
 * every bucket (contiguous equal-row m/z slices); metadata is replicated.  Use 0 / 1 for a
 * single GPU.  HOMS_B200_ERR_INVARIANT on n == 0 (search.cpp:18). */
int homs_b200_library_upload(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* words,
                             const double* precursor_mz, const uint8_t* charge,
                             const uint32_t* id_rank, uint32_t shard_index, uint32_t shard_count);
/* Same, hypervector rows already on the device (e.g. straight from homs_b200_encode_batch_dev);
 * the metadata arrays stay host pointers. */
int homs_b200_library_upload_dev(homs_b200_ctx* ctx, uint32_t dim, uint64_t n,
                                 const uint64_t* d_words, const double* precursor_mz,
                                 const uint8_t* charge, const uint32_t* id_rank,
                                 uint32_t shard_index, uint32_t shard_count);
int homs_b200_library_bucket_count(const homs_b200_ctx* ctx, uint32_t* out_count);
/* Bucket `which` in ascending charge order: its charge, full size, and the slice
 * [shard_begin, shard_end) of it resident on this context. */
int homs_b200_library_bucket_info(const homs_b200_ctx* ctx, uint32_t which, uint8_t* out_charge,
                                  uint64_t* out_size, uint64_t* out_shard_begin,
                                  uint64_t* out_shard_end);
/* LibraryIndex::Bucket arrays (search.hpp:41-47): precursor_mz / ordinal for the FULL bucket,
 * words for the resident slice only.  Any pointer may be NULL. */
int homs_b200_library_bucket_export(homs_b200_ctx* ctx, uint32_t which, double* out_mz,
                                    uint32_t* out_ordinal, uint64_t* out_words);

/* ---- encoded-library cache (src/cache.cpp:98-211; format include/homs/cache.hpp:48-57) ------- */

/* Where things are inside a cache image. */
typedef struct {
  uint64_t count;         /* entries */
  uint64_t hv_offset;     /* byte offset of the hypervector block */
  uint64_t hv_bytes;      /* count * ceil(dim/64) * 8 */
  uint64_t stored_digest; /* the FNV-1a-64 the file carries for that block */
  uint64_t id_bytes, peptide_bytes; /* total string bytes */
} homs_b200_cache_layout;

/* FNV-1a-64 exactly as cache.cpp:18-29 (state 1469598103934665603, prime 1099511628211), computed
 * ON THE DEVICE by a chunked parallel formulation of the serial chain (csrc/cache.cu).  _dev takes
 * device bytes, the plain form uploads host bytes first.  Blocking. */
int homs_b200_fnv1a64_dev(homs_b200_ctx* ctx, const void* d_bytes, uint64_t n_bytes, uint64_t* out_digest);
int homs_b200_fnv1a64(homs_b200_ctx* ctx, const void* bytes, uint64_t n_bytes, uint64_t* out_digest);

/* Header and per-entry metadata of read_cache (cache.cpp:158-190), host only, no checksum: checks
 * magic / version (ERR_CACHE_FORMAT), the 61-byte profile block against pre+enc (ERR_CACHE_STALE),
 * truncation and string lengths (ERR_CACHE_CORRUPT).  Output arrays are nullable; strings are
 * returned as (position, length) inside the image. */
int homs_b200_cache_parse(const void* image, uint64_t n_bytes, const homs_b200_preprocess_config* pre,
                          const homs_b200_encoder_config* enc, homs_b200_cache_layout* out_layout,
                          double* mz, uint8_t* charge, uint8_t* is_decoy, uint64_t* id_pos, uint32_t* id_len,
                          uint64_t* peptide_pos, uint32_t* peptide_len);

/* read_cache + build_index in one call (pipeline.cpp:121-122): the hypervector block of the image
 * goes straight to the device, its checksum is verified there (ERR_CACHE_CORRUPT on mismatch), ids
 * are ranked from the image, and the resident index is built as by homs_b200_library_upload_dev. */
int homs_b200_library_load_cache(homs_b200_ctx* ctx, const void* image, uint64_t n_bytes,
                                 const homs_b200_preprocess_config* pre, const homs_b200_encoder_config* enc,
                                 uint32_t shard_index, uint32_t shard_count, uint64_t* out_count);

/* write_cache (cache.cpp:122-156) into a caller buffer, byte-identical to the reference's file.
 * Strings travel as a blob + u64 offsets[n+1] (NULL: empty).  out == NULL: only *out_size is set.
 * _dev: the rows (dense u64[n][W]) are on the device, e.g. straight from encode_batch_dev. */
int homs_b200_cache_write(homs_b200_ctx* ctx, const homs_b200_preprocess_config* pre,
                          const homs_b200_encoder_config* enc, uint64_t n, const uint64_t* words, const double* mz,
                          const uint8_t* charge, const uint8_t* is_decoy, const char* id_blob,
                          const uint64_t* id_off, const char* peptide_blob, const uint64_t* peptide_off, void* out,
                          uint64_t out_cap, uint64_t* out_size);
int homs_b200_cache_write_dev(homs_b200_ctx* ctx, const homs_b200_preprocess_config* pre,
                              const homs_b200_encoder_config* enc, uint64_t n, const uint64_t* d_words,
                              const double* mz, const uint8_t* charge, const uint8_t* is_decoy, const char* id_blob,
                              const uint64_t* id_off, const char* peptide_blob, const uint64_t* peptide_off,
                              void* out, uint64_t out_cap, uint64_t* out_size);

/* ---- search (src/search.cpp:62-183) -------------------------------------------------------- */

/* select_candidates, src/search.cpp:62-89: [first,last) inside the query's charge bucket (full
 * bucket coordinates); out_has_bucket[i] = 0 when the charge is unknown (0) or has no bucket. */
int homs_b200_window_bounds(homs_b200_ctx* ctx, uint64_t nq, const double* q_mz,
                            const uint8_t* q_charge, const homs_b200_tolerance* tol,
                            uint64_t* out_first, uint64_t* out_last, uint8_t* out_has_bucket);

/* search_batch, src/search.cpp:171-183, generalised to the k best per query (k = 1 is the
 * reference's search_one; 1 <= k <= HOMS_B200_MAX_TOPK).  The tensor engine serves any k in ONE pass over the
 * library (candidates at or above a per-query floor are buffered, the k best selected exactly afterwards); the
 * direct engine keeps up to 32 candidates per query in registers and takes a second pass, bounded below by the
 * first pass's last key, for 33 <= k <= 64; the POPC engine runs k passes.  Entry j of query i: out_raw_score[i*k+j] (Hamming similarity) and
 * out_ordinal[i*k+j] (input position of the library entry; HOMS_B200_NO_HIT and score 0 when
 * fewer than j+1 candidates exist).  out_first / out_last (nullable) as in window_bounds.
 * The library must be whole behind this handle (one device, or a multi-device context); a context
 * that holds one shard of a library split across PROCESSES uses the _resident/_merge calls below.
 * HOMS_B200_ERR_INVARIANT when query_dim differs from the library's (search.cpp:107-109). */
int homs_b200_search_batch(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                           const uint64_t* q_words, const double* q_mz, const uint8_t* q_charge,
                           const homs_b200_tolerance* tol, uint32_t k, uint32_t* out_raw_score,
                           uint32_t* out_ordinal, uint64_t* out_first, uint64_t* out_last);

/* Device-resident query set: upload once, search many times (cascade stages, benchmarks). */
int homs_b200_queries_upload(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                             const uint64_t* q_words, const double* q_mz, const uint8_t* q_charge);
int homs_b200_queries_upload_dev(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                                 const uint64_t* d_q_words, const double* d_q_mz,
                                 const uint8_t* d_q_charge);
/* Searches the resident queries (all of them, or the n_subset positions listed in the DEVICE
 * array d_subset) against this context's library shard; writes n*k candidate records (16 B
 * each, see homs_b200_candidate) to the DEVICE buffer d_out.  Asynchronous. */
int homs_b200_search_resident_dev(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n_subset,
                                  const homs_b200_tolerance* tol, uint32_t k,
                                  homs_b200_candidate* d_out);
/* Lexicographic k-way merge of per-shard candidate lists: d_parts is [n_parts][n][k] (the
 * layout an all-gather produces), d_out is [n][k].  Asynchronous. */
int homs_b200_merge_candidates_dev(homs_b200_ctx* ctx, uint64_t n, uint32_t k, uint32_t n_parts,
                                   const homs_b200_candidate* d_parts, homs_b200_candidate* d_out);
/* Candidate records -> (raw_score, ordinal) on the host.  Blocking. */
int homs_b200_candidates_decode(homs_b200_ctx* ctx, uint64_t n, uint32_t k,
                                const homs_b200_candidate* d_records, uint32_t* out_raw_score,
                                uint32_t* out_ordinal);

/* ---- fused raw-spectra entry points (no single reference counterpart) -------
 * The reference composes these from its public calls and moves every hypervector through host
 * vectors in between; here the rows never leave the device.
 *
 * library_build_from_spectra == build_index(encode_spectra(spectra).encoded)
 *   (src/pipeline.cpp:60-85 then src/search.cpp:17-60; `homs encode` + index load,
 *   pipeline.cpp:97-99,121).  Unprocessable spectra are dropped in order exactly as
 *   pipeline.cpp:75-83 does, so the library ordinals a search reports count PROCESSABLE spectra
 *   only.  precursor_mz / charge / id_rank are indexed by raw spectrum; id_rank (may be NULL =
 *   input order) is a permutation of 0..n-1 over the raw list.  out_ok[n] (may be NULL) receives
 *   1 for encoded, 0 for dropped; *out_n_encoded the library size.  Fails with ERR_INVARIANT
 *   ("library is empty", search.cpp:18) when nothing survives.  The codebook must be uploaded to
 *   THIS context. */
int homs_b200_library_build_from_spectra(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg,
                                         uint64_t n, const uint64_t* offsets, const double* mz,
                                         const double* intensity, const double* precursor_mz,
                                         const uint8_t* charge, const uint32_t* id_rank,
                                         uint32_t shard_index, uint32_t shard_count, uint8_t* out_ok,
                                         uint64_t* out_n_encoded);
/* queries_from_spectra == the encode_spectra step of run_search (pipeline.cpp:121-122) with the
 * result left resident: query e of the resident set is the e-th processable spectrum. */
int homs_b200_queries_from_spectra(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                                   const uint64_t* offsets, const double* mz, const double* intensity,
                                   const double* precursor_mz, const uint8_t* charge, uint8_t* out_ok,
                                   uint64_t* out_n_encoded);
/* search_batch (search.cpp:171-183) / cascade_search (search.cpp:219-248) over the RESIDENT
 * queries (queries_upload*, queries_from_spectra); outputs as in the host-query forms, sized by
 * the resident query count. */
int homs_b200_search_resident(homs_b200_ctx* ctx, const homs_b200_tolerance* tol, uint32_t k,
                              uint32_t* out_raw_score, uint32_t* out_ordinal, uint64_t* out_first,
                              uint64_t* out_last);
int homs_b200_cascade_resident(homs_b200_ctx* ctx, const homs_b200_tolerance* narrow,
                               const homs_b200_tolerance* wide, double fdr_q, const uint8_t* lib_is_decoy,
                               uint64_t* out_query, uint32_t* out_ordinal, uint8_t* out_stage,
                               uint32_t* out_raw_score, double* out_q_value, uint64_t* out_count);

/* ---- MGF text -> CSR spectra on the device ----------------------------------
 * parse_mgf, src/mgf.cpp:93-181 (finalize_block :66-89): BEGIN IONS / END IONS blocks, KEY=VALUE
 * headers (PEPMASS required; CHARGE, TITLE, SEQ interpreted, last one wins), "mz intensity" peak
 * lines, peaks stable-sorted by m/z with exact duplicates merged by intensity sum.  Numbers are
 * std::from_chars doubles: the results are the same bits.  A grammar violation returns
 * HOMS_B200_ERR_PARSE with the reference's ParseError text ("line N: message") and the first
 * offending line in info->error_line, exactly the error the sequential parser stops at.
 * The CSR stays resident in the context (until the next mgf_parse) so it can be handed to
 * encode_batch_dev without touching the host; mgf_fetch copies any of it out.  TITLE / SEQ values
 * are returned as (offset, length) into the image; length 0 = absent (the caller synthesises
 * "spectrum_<ordinal>" ids and applies the decoy prefix as mgf.cpp:68-76 does).  charge 0 =
 * unknown (spectrum.hpp:10).  Images must be smaller than 4 GiB. */
typedef struct {
  uint64_t n_lines, n_spectra, n_peaks;
  uint64_t n_hard_numbers; /* tokens that needed the exact big-integer conversion */
  uint64_t error_line;     /* 1-based, 0 = none */
  uint32_t error_code, reserved;
} homs_b200_mgf_info;
int homs_b200_mgf_parse(homs_b200_ctx* ctx, const void* image, uint64_t n_bytes, homs_b200_mgf_info* info);
/* Same, image already in device memory. */
int homs_b200_mgf_parse_dev(homs_b200_ctx* ctx, const void* d_image, uint64_t n_bytes, homs_b200_mgf_info* info);
int homs_b200_mgf_fetch(homs_b200_ctx* ctx, uint64_t* offsets, double* mz, double* intensity,
                        double* precursor_mz, uint8_t* charge, uint32_t* title_off, uint32_t* title_len,
                        uint32_t* seq_off, uint32_t* seq_len);
int homs_b200_mgf_device_csr(homs_b200_ctx* ctx, uint64_t* out_n_spectra, uint64_t* out_n_peaks,
                             const uint64_t** d_offsets, const double** d_mz, const double** d_intensity,
                             const double** d_precursor_mz, const uint8_t** d_charge);

/* The query side of run_search (src/pipeline.cpp:119-150) with nothing but the text crossing PCIe:
 *   homs_b200_mgf_parse(image)          parse_mgf_file            (:121)
 *   homs_b200_queries_from_mgf(cfg)     known-charge filter + encode_spectra  (:127-141)
 *   homs_b200_cascade_resident(...)     cascade_search            (:146-147)
 * queries_from_mgf encodes the CSR the last mgf_parse* left resident, where it lies, and makes the
 * result the resident query set: query e is the e-th spectrum with out_state == 0.
 * out_state[i] (n_spectra entries, may be NULL): 0 = resident query, 1 = skipped, charge unknown
 * (the reference never encodes it), 2 = unprocessable (dropped by encode_spectra, :75-83). */
int homs_b200_queries_from_mgf(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint8_t* out_state,
                               uint64_t* out_n_queries);

/* cascade_search, src/search.cpp:219-248 (run_stage :188-215): narrow stage on all queries,
 * target-decoy FDR, wide stage on the not-accepted rest, FDR again.  lib_is_decoy is indexed by
 * library ordinal.  Outputs need room for nq entries; accepted matches come narrow block first,
 * then wide, each in query order.  Query hypervectors stay on the device between stages. */
int homs_b200_cascade_search(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                             const uint64_t* q_words, const double* q_mz, const uint8_t* q_charge,
                             const homs_b200_tolerance* narrow, const homs_b200_tolerance* wide,
                             double fdr_q, const uint8_t* lib_is_decoy, uint64_t* out_query,
                             uint32_t* out_ordinal, uint8_t* out_stage, uint32_t* out_raw_score,
                             double* out_q_value, uint64_t* out_count);

#ifdef __cplusplus
}
#endif
#endif /* HOMS_B200_H */
