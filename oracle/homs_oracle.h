/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference hot path.
 *
 * Never linked into, imported by or executed from the product (paper_2211_16422_b200/,
 * include/).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it,
 * and only as the checker.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks this restatement against
 *   (a) the known answers the reference's own tests hold for the path
 *       (proj/tests/test_{encoder,preprocess,search,fdr,codebook}.cpp, see tests/golden/),
 *   (b) the golden fingerprints in SURVEY.md section 8(c), and
 *   (c) the unmodified reference compiled into oracle/_ref/ (when present).
 *
 * The flat signatures below are identical to oracle/ref_shim.cpp's (prefix hr_ there, ho_ here)
 * so that oracle/binding.py drives both through one class.
 */
#ifndef HOMS_ORACLE_H
#define HOMS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double min_mz, max_mz, bin_size;
  uint32_t max_peaks, min_peaks;
  double intensity_floor;
  uint32_t scaling; /* 0 none, 1 sqrt */
  uint32_t pad_;
} ho_precfg;

typedef struct {
  uint64_t n_library, n_query;
  uint32_t peaks_per_spectrum, pad_;
  double mz_min, mz_max, fraction_modified, precursor_shift_da, fraction_peaks_shifted,
      intensity_noise, decoy_ratio;
  uint64_t seed;
} ho_synthcfg;

const char* ho_last_error(void);
uint64_t ho_fnv1a64(const void* data, uint64_t n_bytes);

long long ho_dimension(const ho_precfg* cfg);
long long ho_validate_preprocess(const ho_precfg* cfg);
long long ho_refine_vectorize(const ho_precfg* cfg, uint64_t n_peaks, const double* mz,
                              const double* inten, uint32_t levels, uint32_t* out_bins,
                              double* out_intens, uint32_t* out_levels);
long long ho_quantize_intensity(double v, uint32_t levels);

void* ho_codebook_create(uint32_t dim, uint32_t step_flips, uint32_t levels, uint64_t seed,
                         uint32_t n_bins);
void* ho_codebook_from_words(uint32_t dim, uint32_t levels, uint32_t n_bins, const uint64_t* pos,
                             const uint64_t* lvl);
void ho_codebook_export(const void* h, uint64_t* pos, uint64_t* lvl);
void ho_codebook_free(void* h);

long long ho_encode_spectra(const void* codebook, const ho_precfg* cfg, uint64_t n,
                            const uint64_t* offsets, const double* mz, const double* inten,
                            unsigned threads, uint64_t batch, uint64_t* out_words,
                            uint8_t* out_ok);
long long ho_encode_vector(const void* codebook, uint32_t n_bins_sv, const uint32_t* bins,
                           const double* intens, int unpacked, uint64_t* out_words);
long long ho_hamming_similarity(uint32_t dim, const uint64_t* a, const uint64_t* b, int bitwise);

void* ho_index_create(uint32_t dim, uint64_t n, const uint64_t* words, const double* mz,
                      const uint8_t* charge, const uint8_t* is_decoy, const char* id_blob,
                      const uint64_t* id_off);
void ho_index_free(void* h);
long long ho_index_bucket_count(const void* h);
long long ho_index_bucket_info(const void* h, uint32_t which, uint8_t* charge, uint64_t* size);
long long ho_index_bucket_export(const void* h, uint32_t which, double* mz, uint32_t* ordinal,
                                 uint64_t* words);
long long ho_select_candidates(const void* h, uint64_t nq, const double* q_mz,
                               const uint8_t* q_charge, int tol_kind, double tol_value,
                               uint64_t* out_first, uint64_t* out_last, uint8_t* out_has_bucket);
long long ho_search_batch(const void* h, uint64_t nq, const uint64_t* q_words, const double* q_mz,
                          const uint8_t* q_charge, int tol_kind, double tol_value,
                          unsigned threads, uint64_t batch, int linear, uint8_t* out_has,
                          uint32_t* out_raw_score, uint32_t* out_ordinal, double* out_mass_diff);
/* top-k generalisation: full sort of the window on the reference's key
 * (score desc, |mass diff| asc, id asc, ordinal asc); missing entries: ordinal 0xFFFFFFFF. */
long long ho_search_topk(const void* h, uint64_t nq, const uint64_t* q_words, const double* q_mz,
                         const uint8_t* q_charge, int tol_kind, double tol_value, uint32_t k,
                         uint32_t* out_raw_score, uint32_t* out_ordinal);
long long ho_cascade_search(const void* h, uint64_t nq, const uint64_t* q_words,
                            const double* q_mz, const uint8_t* q_charge, int narrow_kind,
                            double narrow_value, int wide_kind, double wide_value, double fdr_q,
                            unsigned threads, uint64_t batch, uint64_t* out_query,
                            uint32_t* out_ordinal, uint8_t* out_stage, uint32_t* out_raw_score,
                            double* out_q_value);
long long ho_compute_fdr_curve(uint64_t n, const double* score, const uint8_t* is_decoy,
                               uint64_t* out_input_index, double* out_fdr, double* out_q);

void* ho_synth_create(const ho_synthcfg* cfg);
void ho_synth_free(void* h);
void ho_synth_sizes(const void* h, int which, uint64_t* sizes);
void ho_synth_export(const void* h, int which, uint64_t* offsets, double* mz, double* inten,
                     double* precursor, uint8_t* charge, uint8_t* is_decoy, char* id_blob,
                     uint64_t* id_off);
void ho_synth_truth(const void* h, uint64_t* source_index, uint8_t* modified);

/* encoded-library cache, src/cache.cpp:98-211 (format: include/homs/cache.hpp:48-57) */
typedef struct {
  uint32_t dim, step_flips, levels, pad_;
  uint64_t seed;
} ho_enccfg;
long long ho_cache_write(const ho_precfg* pre, const ho_enccfg* enc, uint64_t n, const uint64_t* words,
                         const double* mz, const uint8_t* charge, const uint8_t* is_decoy,
                         const char* id_blob, const uint64_t* id_off, const char* pep_blob,
                         const uint64_t* pep_off, unsigned char* out, uint64_t out_cap);
long long ho_cache_read(const unsigned char* image, uint64_t n_bytes, const ho_precfg* pre,
                        const ho_enccfg* enc, uint64_t* words, double* mz, uint8_t* charge,
                        uint8_t* is_decoy, char* id_blob, uint64_t* id_off, char* pep_blob,
                        uint64_t* pep_off);

/* MGF text, src/mgf.cpp:93-181 (parse_mgf, finalize_block :66-89) and :183-208 (write_mgf).
 * parse returns a handle (NULL after a grammar violation: ho_last_error() == "ParseError: line N: ...").
 * sizes[0] = spectra, [1] = peaks, [2] = id bytes, [3] = peptide bytes. */
void* ho_mgf_parse(const char* text, uint64_t n_bytes, const char* decoy_prefix);
void ho_mgf_free(void* h);
void ho_mgf_sizes(const void* h, uint64_t* sizes);
void ho_mgf_export(const void* h, uint64_t* offsets, double* mz, double* inten, double* precursor,
                   uint8_t* charge, uint8_t* is_decoy, char* id_blob, uint64_t* id_off, char* pep_blob,
                   uint64_t* pep_off);
long long ho_mgf_write(uint64_t n, const uint64_t* offsets, const double* mz, const double* inten,
                       const double* precursor, const uint8_t* charge, const char* id_blob,
                       const uint64_t* id_off, const char* pep_blob, const uint64_t* pep_off, char* out,
                       uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif
