// TEST INFRASTRUCTURE ONLY -- never linked into, imported by or executed from the
// product path (paper_2211_16422_b200/, include/). See oracle/README.md.
//
// Flat extern "C" window onto the UNMODIFIED reference (`homs_core`, compiled by
// oracle/Makefile straight from /root/reference/proj/core/src/*.cpp into
// oracle/_ref/).  Nothing here re-implements reference arithmetic: every entry
// point marshals flat arrays into the reference's own types, calls the
// reference's own function, and marshals the answer back.  Python reaches it
// through ctypes (tests/_oracle.py); bench.py's `--impl reference` /
// `cpu_baseline` legs time hr_search_batch / hr_encode_spectra.
//
// Conventions
//   * hypervectors travel as little-endian u64 words, W = ceil(dim/64) per row
//     (reference layout: hypervector.hpp:12-15);
//   * spectra travel as CSR: offsets u64[n+1], mz f64[], intensity f64[];
//   * strings travel as a byte blob + u64 offsets[n+1] (NULL blob => empty ids);
//   * every function returns >= 0 on success and -1 after catching a reference
//     exception; hr_last_error() then names the exception class and message.
//   * to map reference results (which carry ids, not positions) back to flat
//     positions the shim tags query ids / library peptides with decimal indices.

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <iterator>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <typeinfo>
#include <vector>

#include "homs/cache.hpp"
#include "homs/codebook.hpp"
#include "homs/encoder.hpp"
#include "homs/errors.hpp"
#include "homs/fdr.hpp"
#include "homs/mgf.hpp"
#include "homs/pipeline.hpp"
#include "homs/preprocess.hpp"
#include "homs/search.hpp"
#include "homs/synth.hpp"
#include "oracles.hpp"  // /root/reference/proj/tests/oracles.hpp (independent test oracles)

namespace {

thread_local std::string g_error;

template <typename Fn>
long long guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const homs::ConfigError& e) {
    g_error = std::string("ConfigError: ") + e.what();
  } catch (const homs::InvariantError& e) {
    g_error = std::string("InvariantError: ") + e.what();
  } catch (const homs::ParseError& e) {
    g_error = std::string("ParseError: ") + e.what();
  } catch (const homs::CacheFormatError& e) {
    g_error = std::string("CacheFormatError: ") + e.what();
  } catch (const homs::StaleCacheError& e) {
    g_error = std::string("StaleCacheError: ") + e.what();
  } catch (const homs::CacheCorruptError& e) {
    g_error = std::string("CacheCorruptError: ") + e.what();
  } catch (const homs::Error& e) {
    g_error = std::string("Error: ") + e.what();
  } catch (const std::exception& e) {
    g_error = std::string("std::exception: ") + e.what();
  }
  return -1;
}

struct PreCfgPod {  // must match oracle/_pods.py and include/homs_b200.h
  double min_mz, max_mz, bin_size;
  std::uint32_t max_peaks, min_peaks;
  double intensity_floor;
  std::uint32_t scaling;
  std::uint32_t pad_;
};

homs::PreprocessConfig to_cfg(const PreCfgPod* p) {
  homs::PreprocessConfig c;
  c.min_mz = p->min_mz;
  c.max_mz = p->max_mz;
  c.bin_size = p->bin_size;
  c.max_peaks = p->max_peaks;
  c.min_peaks = p->min_peaks;
  c.intensity_floor = p->intensity_floor;
  c.scaling = p->scaling ? homs::IntensityScaling::sqrt : homs::IntensityScaling::none;
  return c;
}

homs::Hypervector hv_from(const std::uint64_t* words, std::uint32_t dim) {
  homs::Hypervector hv(dim);
  auto w = hv.words();
  std::memcpy(w.data(), words, w.size() * sizeof(std::uint64_t));
  return hv;
}

std::string str_at(const char* blob, const std::uint64_t* off, std::size_t i) {
  if (blob == nullptr || off == nullptr) return {};
  return std::string(blob + off[i], blob + off[i + 1]);
}

std::size_t parse_index(const std::string& s) {
  std::size_t v = 0;
  std::from_chars(s.data(), s.data() + s.size(), v);
  return v;
}

homs::Tolerance make_tol(int kind, double value) {
  return homs::Tolerance{kind == 0 ? homs::Tolerance::Kind::ppm : homs::Tolerance::Kind::dalton,
                         value};
}

struct IndexBox {
  std::uint32_t dim = 0;
  std::vector<homs::EncodedSpectrum> refs;  // kept for linear_search
  homs::LibraryIndex index;
};

std::vector<homs::EncodedSpectrum> make_queries(std::size_t nq, std::uint32_t dim,
                                                const std::uint64_t* words, const double* mz,
                                                const std::uint8_t* charge) {
  const std::size_t W = homs::Hypervector::words_for(dim);
  std::vector<homs::EncodedSpectrum> qs(nq);
  for (std::size_t i = 0; i < nq; ++i) {
    qs[i].meta.id = std::to_string(i);
    qs[i].meta.precursor_mz = mz[i];
    qs[i].meta.charge = charge[i];
    qs[i].hv = hv_from(words + i * W, dim);
  }
  return qs;
}

}  // namespace

extern "C" {

const char* hr_last_error() { return g_error.c_str(); }

// ---- preprocess -----------------------------------------------------------------------------

long long hr_dimension(const PreCfgPod* cfg) {
  return guarded([&]() -> long long { return homs::dimension(to_cfg(cfg)); });
}

long long hr_validate_preprocess(const PreCfgPod* cfg) {
  return guarded([&]() -> long long {
    to_cfg(cfg).validate();
    return 0;
  });
}

// refine_peaks + vectorize + quantize_intensity for ONE spectrum.
// returns n_bins (>0), 0 when refine_peaks says "unprocessable".
long long hr_refine_vectorize(const PreCfgPod* cfg, std::uint64_t n_peaks, const double* mz,
                              const double* inten, std::uint32_t levels, std::uint32_t* out_bins,
                              double* out_intens, std::uint32_t* out_levels) {
  return guarded([&]() -> long long {
    homs::RawSpectrum s;
    s.peaks.resize(n_peaks);
    for (std::uint64_t i = 0; i < n_peaks; ++i) s.peaks[i] = {mz[i], inten[i]};
    const auto c = to_cfg(cfg);
    auto refined = homs::refine_peaks(s, c);
    if (!refined) return 0;
    const auto sv = homs::vectorize(*refined, c);
    for (std::size_t k = 0; k < sv.bins.size(); ++k) {
      out_bins[k] = sv.bins[k];
      out_intens[k] = sv.intensities[k];
      if (out_levels) out_levels[k] = homs::quantize_intensity(sv.intensities[k], levels);
    }
    return static_cast<long long>(sv.bins.size());
  });
}

long long hr_quantize_intensity(double v, std::uint32_t levels) {
  return guarded([&]() -> long long { return homs::quantize_intensity(v, levels); });
}

// ---- codebook -------------------------------------------------------------------------------

void* hr_codebook_create(std::uint32_t dim, std::uint32_t step_flips, std::uint32_t levels,
                         std::uint64_t seed, std::uint32_t n_bins) {
  homs::Codebook* cb = nullptr;
  const long long rc = guarded([&]() -> long long {
    homs::EncoderConfig ec{dim, step_flips, levels, seed};
    cb = new homs::Codebook(homs::make_codebook(n_bins, ec));
    return 0;
  });
  return rc < 0 ? nullptr : cb;
}

// Hand-built codebook (reference tests construct Codebook structs directly).
void* hr_codebook_from_words(std::uint32_t dim, std::uint32_t levels, std::uint32_t n_bins,
                             const std::uint64_t* pos, const std::uint64_t* lvl) {
  auto* cb = new homs::Codebook;
  cb->config = homs::EncoderConfig{dim, 1, levels, 0};
  cb->spectrum_dims = n_bins;
  const std::size_t W = homs::Hypervector::words_for(dim);
  for (std::uint32_t i = 0; i < n_bins; ++i) cb->position.push_back(hv_from(pos + i * W, dim));
  for (std::uint32_t q = 0; q <= levels; ++q) cb->level.push_back(hv_from(lvl + q * W, dim));
  return cb;
}

void hr_codebook_export(const void* h, std::uint64_t* pos, std::uint64_t* lvl) {
  const auto* cb = static_cast<const homs::Codebook*>(h);
  const std::size_t W = homs::Hypervector::words_for(cb->config.dim);
  for (std::size_t i = 0; i < cb->position.size(); ++i)
    std::memcpy(pos + i * W, cb->position[i].words().data(), W * 8);
  for (std::size_t q = 0; q < cb->level.size(); ++q)
    std::memcpy(lvl + q * W, cb->level[q].words().data(), W * 8);
}

void hr_codebook_free(void* h) { delete static_cast<homs::Codebook*>(h); }

// ---- encode ---------------------------------------------------------------------------------

// pipeline.cpp:60-85 encode_spectra.  out_ok[i] = 1 and out_words row i filled for every
// processable input (rows of unprocessable inputs are zeroed).  Returns `unprocessable`.
long long hr_encode_spectra(const void* codebook, const PreCfgPod* cfg, std::uint64_t n,
                            const std::uint64_t* offsets, const double* mz, const double* inten,
                            unsigned threads, std::uint64_t batch, std::uint64_t* out_words,
                            std::uint8_t* out_ok) {
  return guarded([&]() -> long long {
    const auto* cb = static_cast<const homs::Codebook*>(codebook);
    const std::size_t W = homs::Hypervector::words_for(cb->config.dim);
    std::vector<homs::RawSpectrum> spectra(n);
    for (std::uint64_t i = 0; i < n; ++i) {
      spectra[i].meta.id = std::to_string(i);
      const std::uint64_t a = offsets[i], b = offsets[i + 1];
      spectra[i].peaks.resize(b - a);
      for (std::uint64_t k = a; k < b; ++k) spectra[i].peaks[k - a] = {mz[k], inten[k]};
    }
    const auto outcome = homs::encode_spectra(spectra, *cb, to_cfg(cfg), threads, batch);
    std::memset(out_ok, 0, n);
    std::memset(out_words, 0, n * W * 8);
    for (const auto& e : outcome.encoded) {
      const std::size_t i = parse_index(e.meta.id);
      out_ok[i] = 1;
      std::memcpy(out_words + i * W, e.hv.words().data(), W * 8);
    }
    return static_cast<long long>(outcome.unprocessable);
  });
}

// encoder.cpp:19-55 encode() on an already vectorized spectrum; `unpacked` != 0 switches to
// the independent accumulator oracle (tests/oracles.hpp:36-55).
long long hr_encode_vector(const void* codebook, std::uint32_t n_bins_sv, const std::uint32_t* bins,
                           const double* intens, int unpacked, std::uint64_t* out_words) {
  return guarded([&]() -> long long {
    const auto* cb = static_cast<const homs::Codebook*>(codebook);
    homs::SpectrumVector sv;
    sv.dims = cb->spectrum_dims;
    sv.bins.assign(bins, bins + n_bins_sv);
    sv.intensities.assign(intens, intens + n_bins_sv);
    const homs::Hypervector hv =
        unpacked ? oracle::encode_unpacked(sv, *cb) : homs::encode(sv, *cb);
    std::memcpy(out_words, hv.words().data(), hv.words().size() * 8);
    return 0;
  });
}

long long hr_hamming_similarity(std::uint32_t dim, const std::uint64_t* a, const std::uint64_t* b,
                                int bitwise) {
  return guarded([&]() -> long long {
    const auto x = hv_from(a, dim), y = hv_from(b, dim);
    return bitwise ? oracle::bitwise_hamming(x, y) : homs::hamming_similarity(x, y);
  });
}

// ---- index + search -------------------------------------------------------------------------

void* hr_index_create(std::uint32_t dim, std::uint64_t n, const std::uint64_t* words,
                      const double* mz, const std::uint8_t* charge, const std::uint8_t* is_decoy,
                      const char* id_blob, const std::uint64_t* id_off) {
  IndexBox* box = nullptr;
  const long long rc = guarded([&]() -> long long {
    auto b = std::make_unique<IndexBox>();
    b->dim = dim;
    const std::size_t W = homs::Hypervector::words_for(dim);
    b->refs.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) {
      auto& r = b->refs[i];
      r.meta.id = str_at(id_blob, id_off, i);
      r.meta.peptide = std::to_string(i);  // carries the ordinal through Ssm::peptide
      r.meta.precursor_mz = mz[i];
      r.meta.charge = charge[i];
      r.meta.is_decoy = is_decoy ? is_decoy[i] != 0 : false;
      r.hv = hv_from(words + i * W, dim);
    }
    b->index = homs::build_index(b->refs);
    box = b.release();
    return 0;
  });
  return rc < 0 ? nullptr : box;
}

void hr_index_free(void* h) { delete static_cast<IndexBox*>(h); }

// Bucket layout as build_index produced it (search.cpp:30-58).
long long hr_index_bucket_count(const void* h) {
  return static_cast<long long>(static_cast<const IndexBox*>(h)->index.buckets().size());
}
long long hr_index_bucket_info(const void* h, std::uint32_t which, std::uint8_t* charge,
                               std::uint64_t* size) {
  const auto& bs = static_cast<const IndexBox*>(h)->index.buckets();
  auto it = bs.begin();
  std::advance(it, which);
  *charge = it->first;
  *size = it->second.size();
  return 0;
}
long long hr_index_bucket_export(const void* h, std::uint32_t which, double* mz,
                                 std::uint32_t* ordinal, std::uint64_t* words) {
  const auto& bs = static_cast<const IndexBox*>(h)->index.buckets();
  auto it = bs.begin();
  std::advance(it, which);
  const auto& b = it->second;
  if (mz) std::copy(b.precursor_mz.begin(), b.precursor_mz.end(), mz);
  if (ordinal) std::copy(b.ordinal.begin(), b.ordinal.end(), ordinal);
  if (words) std::copy(b.words.begin(), b.words.end(), words);
  return 0;
}

// search.cpp:62-89.  out_first/out_last are positions inside the query's charge bucket;
// out_has_bucket[i] = 0 when the reference returned a null bucket.
long long hr_select_candidates(const void* h, std::uint64_t nq, const double* q_mz,
                               const std::uint8_t* q_charge, int tol_kind, double tol_value,
                               std::uint64_t* out_first, std::uint64_t* out_last,
                               std::uint8_t* out_has_bucket) {
  return guarded([&]() -> long long {
    const auto* box = static_cast<const IndexBox*>(h);
    const auto tol = make_tol(tol_kind, tol_value);
    for (std::uint64_t i = 0; i < nq; ++i) {
      homs::SpectrumMeta m;
      m.precursor_mz = q_mz[i];
      m.charge = q_charge[i];
      const auto r = homs::select_candidates(m, box->index, tol);
      out_first[i] = r.first;
      out_last[i] = r.last;
      out_has_bucket[i] = r.bucket != nullptr;
    }
    return 0;
  });
}

// search.cpp:171-183 search_batch (linear = 0) or tests/oracles.hpp:60-108 linear_search.
long long hr_search_batch(const void* h, std::uint64_t nq, const std::uint64_t* q_words,
                          const double* q_mz, const std::uint8_t* q_charge, int tol_kind,
                          double tol_value, unsigned threads, std::uint64_t batch, int linear,
                          std::uint8_t* out_has, std::uint32_t* out_raw_score,
                          std::uint32_t* out_ordinal, double* out_mass_diff) {
  return guarded([&]() -> long long {
    const auto* box = static_cast<const IndexBox*>(h);
    const auto tol = make_tol(tol_kind, tol_value);
    const auto qs = make_queries(nq, box->dim, q_words, q_mz, q_charge);
    std::vector<std::optional<homs::Ssm>> hits;
    if (linear) {
      hits.resize(nq);
      for (std::uint64_t i = 0; i < nq; ++i)
        hits[i] = oracle::linear_search(qs[i], box->refs, tol, box->dim);
    } else {
      homs::SearchOptions opt;
      opt.threads = threads;
      opt.batch_size = batch;
      hits = homs::search_batch(qs, box->index, tol, opt);
    }
    long long n_hits = 0;
    for (std::uint64_t i = 0; i < nq; ++i) {
      out_has[i] = hits[i].has_value();
      out_raw_score[i] = hits[i] ? hits[i]->raw_score : 0;
      out_ordinal[i] = hits[i] ? static_cast<std::uint32_t>(parse_index(hits[i]->peptide))
                               : 0xFFFFFFFFu;
      if (out_mass_diff) out_mass_diff[i] = hits[i] ? hits[i]->mass_diff : 0.0;
      n_hits += hits[i].has_value();
    }
    return n_hits;
  });
}

// search.cpp:219-248 cascade_search.  Output arrays need room for nq entries; returns the
// number of accepted SSMs (narrow block first, then wide, each in query order).
long long hr_cascade_search(const void* h, std::uint64_t nq, const std::uint64_t* q_words,
                            const double* q_mz, const std::uint8_t* q_charge, int narrow_kind,
                            double narrow_value, int wide_kind, double wide_value, double fdr_q,
                            unsigned threads, std::uint64_t batch, std::uint64_t* out_query,
                            std::uint32_t* out_ordinal, std::uint8_t* out_stage,
                            std::uint32_t* out_raw_score, double* out_q_value) {
  return guarded([&]() -> long long {
    const auto* box = static_cast<const IndexBox*>(h);
    const auto qs = make_queries(nq, box->dim, q_words, q_mz, q_charge);
    homs::SearchOptions opt;
    opt.threads = threads;
    opt.batch_size = batch;
    const auto acc = homs::cascade_search(qs, box->index, make_tol(narrow_kind, narrow_value),
                                          make_tol(wide_kind, wide_value), fdr_q, opt);
    for (std::size_t i = 0; i < acc.size(); ++i) {
      out_query[i] = parse_index(acc[i].query_id);
      out_ordinal[i] = static_cast<std::uint32_t>(parse_index(acc[i].peptide));
      out_stage[i] = static_cast<std::uint8_t>(acc[i].stage);
      out_raw_score[i] = acc[i].raw_score;
      out_q_value[i] = acc[i].q_value.value_or(-1.0);
    }
    return static_cast<long long>(acc.size());
  });
}

// fdr.cpp:8-50.  out_input_index[p] = input position of sorted position p; out_q[p] its q-value.
long long hr_compute_fdr_curve(std::uint64_t n, const double* score, const std::uint8_t* is_decoy,
                               std::uint64_t* out_input_index, double* out_fdr, double* out_q) {
  return guarded([&]() -> long long {
    std::vector<homs::Ssm> ssms(n);
    for (std::uint64_t i = 0; i < n; ++i) {
      ssms[i].score = score[i];
      ssms[i].is_decoy = is_decoy[i] != 0;
    }
    const auto curve = homs::compute_fdr_curve(std::move(ssms));
    for (std::size_t p = 0; p < curve.size(); ++p) {
      out_input_index[p] = curve.input_index[p];
      out_fdr[p] = curve.fdr[p];
      out_q[p] = curve.q_value[p];
    }
    return static_cast<long long>(curve.size());
  });
}

// ---- synth ----------------------------------------------------------------------------------

struct SynthPod {
  std::uint64_t n_library, n_query;
  std::uint32_t peaks_per_spectrum, pad_;
  double mz_min, mz_max, fraction_modified, precursor_shift_da, fraction_peaks_shifted,
      intensity_noise, decoy_ratio;
  std::uint64_t seed;
};

void* hr_synth_create(const SynthPod* p) {
  homs::SynthOutput* out = nullptr;
  const long long rc = guarded([&]() -> long long {
    homs::SynthConfig c;
    c.n_library = p->n_library;
    c.n_query = p->n_query;
    c.peaks_per_spectrum = p->peaks_per_spectrum;
    c.mz_min = p->mz_min;
    c.mz_max = p->mz_max;
    c.fraction_modified = p->fraction_modified;
    c.precursor_shift_da = p->precursor_shift_da;
    c.fraction_peaks_shifted = p->fraction_peaks_shifted;
    c.intensity_noise = p->intensity_noise;
    c.decoy_ratio = p->decoy_ratio;
    c.seed = p->seed;
    out = new homs::SynthOutput(homs::generate_benchmark(c));
    return 0;
  });
  return rc < 0 ? nullptr : out;
}
void hr_synth_free(void* h) { delete static_cast<homs::SynthOutput*>(h); }

static const std::vector<homs::RawSpectrum>& synth_set(const void* h, int which) {
  const auto* s = static_cast<const homs::SynthOutput*>(h);
  return which == 0 ? s->library : s->queries;
}

// which: 0 library, 1 queries.  sizes[0]=n spectra, [1]=total peaks, [2]=total id bytes
void hr_synth_sizes(const void* h, int which, std::uint64_t* sizes) {
  const auto& v = synth_set(h, which);
  sizes[0] = v.size();
  sizes[1] = sizes[2] = 0;
  for (const auto& s : v) {
    sizes[1] += s.peaks.size();
    sizes[2] += s.meta.id.size();
  }
}

void hr_synth_export(const void* h, int which, std::uint64_t* offsets, double* mz, double* inten,
                     double* precursor, std::uint8_t* charge, std::uint8_t* is_decoy,
                     char* id_blob, std::uint64_t* id_off) {
  const auto& v = synth_set(h, which);
  std::uint64_t p = 0, c = 0;
  for (std::size_t i = 0; i < v.size(); ++i) {
    offsets[i] = p;
    id_off[i] = c;
    for (const auto& pk : v[i].peaks) {
      mz[p] = pk.mz;
      inten[p] = pk.intensity;
      ++p;
    }
    std::memcpy(id_blob + c, v[i].meta.id.data(), v[i].meta.id.size());
    c += v[i].meta.id.size();
    precursor[i] = v[i].meta.precursor_mz;
    charge[i] = v[i].meta.charge;
    is_decoy[i] = v[i].meta.is_decoy;
  }
  offsets[v.size()] = p;
  id_off[v.size()] = c;
}

// truth: source library position (targets only: "LIB_%06zu" -> index) and modified flag
void hr_synth_truth(const void* h, std::uint64_t* source_index, std::uint8_t* modified) {
  const auto* s = static_cast<const homs::SynthOutput*>(h);
  for (std::size_t i = 0; i < s->truth.size(); ++i) {
    source_index[i] = parse_index(s->truth[i].source_id.substr(4)) - 1;
    modified[i] = s->truth[i].modified;
  }
}

// ---- encoded-library cache (src/cache.cpp:122-211) ---------------------------------------------

struct EncCfgPod {
  std::uint32_t dim, step_flips, levels, pad_;
  std::uint64_t seed;
};

static homs::EncodingProfile to_profile(const PreCfgPod* pre, const EncCfgPod* enc) {
  homs::EncodingProfile p;
  p.preprocess = to_cfg(pre);
  p.encoder.dim = enc->dim;
  p.encoder.step_flips = enc->step_flips;
  p.encoder.levels = enc->levels;
  p.encoder.seed = enc->seed;
  return p;
}

// write_cache into a caller buffer; returns the image size (call with out == NULL to size it)
long long hr_cache_write(const PreCfgPod* pre, const EncCfgPod* enc, std::uint64_t n,
                         const std::uint64_t* words, const double* mz, const std::uint8_t* charge,
                         const std::uint8_t* is_decoy, const char* id_blob, const std::uint64_t* id_off,
                         const char* pep_blob, const std::uint64_t* pep_off, unsigned char* out,
                         std::uint64_t out_cap) {
  return guarded([&]() -> long long {
    const homs::EncodingProfile profile = to_profile(pre, enc);
    const std::size_t W = homs::Hypervector::words_for(enc->dim);
    std::vector<homs::EncodedSpectrum> entries(n);
    for (std::size_t i = 0; i < n; ++i) {
      entries[i].meta.id = str_at(id_blob, id_off, i);
      entries[i].meta.precursor_mz = mz[i];
      entries[i].meta.charge = charge[i];
      entries[i].meta.is_decoy = is_decoy[i] != 0;
      entries[i].meta.peptide = str_at(pep_blob, pep_off, i);
      entries[i].hv = hv_from(words + i * W, enc->dim);
    }
    std::ostringstream os(std::ios::binary);
    homs::write_cache(os, entries, profile);
    const std::string image = std::move(os).str();
    if (out != nullptr) {
      if (image.size() > out_cap) throw homs::Error("hr_cache_write: buffer too small");
      std::memcpy(out, image.data(), image.size());
    }
    return static_cast<long long>(image.size());
  });
}

// read_cache from a byte image; returns the entry count.  With words == NULL only validates.
// Strings come back as blobs with offsets (capacity: the image size is always enough).
long long hr_cache_read(const unsigned char* image, std::uint64_t n_bytes, const PreCfgPod* pre,
                        const EncCfgPod* enc, std::uint64_t* words, double* mz, std::uint8_t* charge,
                        std::uint8_t* is_decoy, char* id_blob, std::uint64_t* id_off, char* pep_blob,
                        std::uint64_t* pep_off) {
  return guarded([&]() -> long long {
    std::istringstream is(std::string(reinterpret_cast<const char*>(image), n_bytes), std::ios::binary);
    const std::vector<homs::EncodedSpectrum> entries = homs::read_cache(is, to_profile(pre, enc));
    if (words != nullptr) {
      const std::size_t W = homs::Hypervector::words_for(enc->dim);
      std::uint64_t io = 0, po = 0;
      for (std::size_t i = 0; i < entries.size(); ++i) {
        const auto& e = entries[i];
        std::memcpy(words + i * W, e.hv.words().data(), W * 8);
        mz[i] = e.meta.precursor_mz;
        charge[i] = e.meta.charge;
        is_decoy[i] = e.meta.is_decoy;
        id_off[i] = io;
        std::memcpy(id_blob + io, e.meta.id.data(), e.meta.id.size());
        io += e.meta.id.size();
        pep_off[i] = po;
        std::memcpy(pep_blob + po, e.meta.peptide.data(), e.meta.peptide.size());
        po += e.meta.peptide.size();
      }
      id_off[entries.size()] = io;
      pep_off[entries.size()] = po;
    }
    return static_cast<long long>(entries.size());
  });
}

// ---- MGF text (src/mgf.cpp:93-181 parse_mgf, :183-208 write_mgf) -------------------------------

void* hr_mgf_parse(const char* text, std::uint64_t n_bytes, const char* decoy_prefix) {
  std::vector<homs::RawSpectrum>* out = nullptr;
  const long long rc = guarded([&]() -> long long {
    std::istringstream in(std::string(text, n_bytes));
    out = new std::vector<homs::RawSpectrum>(homs::parse_mgf(in, decoy_prefix ? decoy_prefix : ""));
    return 0;
  });
  return rc < 0 ? nullptr : out;
}
void hr_mgf_free(void* h) { delete static_cast<std::vector<homs::RawSpectrum>*>(h); }

// sizes[0] = spectra, [1] = peaks, [2] = id bytes, [3] = peptide bytes
void hr_mgf_sizes(const void* h, std::uint64_t* sizes) {
  const auto& v = *static_cast<const std::vector<homs::RawSpectrum>*>(h);
  sizes[0] = v.size();
  sizes[1] = sizes[2] = sizes[3] = 0;
  for (const auto& s : v) {
    sizes[1] += s.peaks.size();
    sizes[2] += s.meta.id.size();
    sizes[3] += s.meta.peptide.size();
  }
}

void hr_mgf_export(const void* h, std::uint64_t* offsets, double* mz, double* inten, double* precursor,
                   std::uint8_t* charge, std::uint8_t* is_decoy, char* id_blob, std::uint64_t* id_off,
                   char* pep_blob, std::uint64_t* pep_off) {
  const auto& v = *static_cast<const std::vector<homs::RawSpectrum>*>(h);
  std::uint64_t p = 0, c = 0, q = 0;
  for (std::size_t i = 0; i < v.size(); ++i) {
    offsets[i] = p;
    id_off[i] = c;
    pep_off[i] = q;
    for (const auto& pk : v[i].peaks) {
      mz[p] = pk.mz;
      inten[p] = pk.intensity;
      ++p;
    }
    std::memcpy(id_blob + c, v[i].meta.id.data(), v[i].meta.id.size());
    c += v[i].meta.id.size();
    std::memcpy(pep_blob + q, v[i].meta.peptide.data(), v[i].meta.peptide.size());
    q += v[i].meta.peptide.size();
    precursor[i] = v[i].meta.precursor_mz;
    charge[i] = v[i].meta.charge;
    is_decoy[i] = v[i].meta.is_decoy;
  }
  offsets[v.size()] = p;
  id_off[v.size()] = c;
  pep_off[v.size()] = q;
}

// write_mgf of the given spectra; returns the text size (copies it when it fits in cap)
long long hr_mgf_write(std::uint64_t n, const std::uint64_t* offsets, const double* mz, const double* inten,
                       const double* precursor, const std::uint8_t* charge, const char* id_blob,
                       const std::uint64_t* id_off, const char* pep_blob, const std::uint64_t* pep_off,
                       char* out, std::uint64_t cap) {
  return guarded([&]() -> long long {
    std::vector<homs::RawSpectrum> v(n);
    for (std::uint64_t i = 0; i < n; ++i) {
      v[i].meta.id.assign(id_blob + id_off[i], id_off[i + 1] - id_off[i]);
      if (pep_blob) v[i].meta.peptide.assign(pep_blob + pep_off[i], pep_off[i + 1] - pep_off[i]);
      v[i].meta.precursor_mz = precursor[i];
      v[i].meta.charge = charge[i];
      for (std::uint64_t j = offsets[i]; j < offsets[i + 1]; ++j) v[i].peaks.push_back({mz[j], inten[j]});
    }
    std::ostringstream os;
    homs::write_mgf(os, v);
    const std::string text = os.str();
    if (out && text.size() <= cap) std::memcpy(out, text.data(), text.size());
    return static_cast<long long>(text.size());
  });
}

// The query side of run_search (pipeline.cpp:119-150) on an MGF text image, against an index built by
// hr_index_build, with the codebook made elsewhere (make_codebook is not part of the timed stages):
// parse_mgf -> drop unknown charges (:127-134) -> encode_spectra (:140-141) -> cascade_search (:146-147)
// -> write_ssm_tsv (:179-195).  stage_seconds: parse, encode, cascade.  stats: total queries, skipped
// (unknown charge), unprocessable, accepted narrow, accepted wide, unidentified.  Returns the TSV size
// (copied when it fits in cap).
long long hr_query_flow(const void* index, const void* codebook, const PreCfgPod* cfg, const char* text,
                        std::uint64_t n_bytes, const char* decoy_prefix, int narrow_kind, double narrow_value,
                        int wide_kind, double wide_value, double fdr_q, unsigned threads, std::uint64_t batch,
                        double* stage_seconds, std::uint64_t* stats, char* tsv, std::uint64_t cap) {
  return guarded([&]() -> long long {
    using Clock = std::chrono::steady_clock;
    const auto* box = static_cast<const IndexBox*>(index);
    const auto* cb = static_cast<const homs::Codebook*>(codebook);
    auto t0 = Clock::now();
    std::istringstream in(std::string(text, n_bytes));
    const auto raw = homs::parse_mgf(in, decoy_prefix ? decoy_prefix : "");
    auto t1 = Clock::now();
    std::vector<homs::RawSpectrum> with_charge;
    with_charge.reserve(raw.size());
    std::size_t skipped = 0;
    for (const auto& q : raw) {
      if (q.meta.has_known_charge()) with_charge.push_back(q);
      else ++skipped;
    }
    auto encoded = homs::encode_spectra(with_charge, *cb, to_cfg(cfg), threads, batch);
    auto t2 = Clock::now();
    homs::SearchOptions opt;
    opt.threads = threads;
    opt.batch_size = batch;
    const auto accepted = homs::cascade_search(encoded.encoded, box->index, make_tol(narrow_kind, narrow_value),
                                               make_tol(wide_kind, wide_value), fdr_q, opt);
    auto t3 = Clock::now();
    if (stage_seconds) {
      stage_seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      stage_seconds[1] = std::chrono::duration<double>(t2 - t1).count();
      stage_seconds[2] = std::chrono::duration<double>(t3 - t2).count();
    }
    if (stats) {
      std::uint64_t narrow = 0;
      for (const auto& s : accepted) narrow += s.stage == homs::SearchStage::narrow;
      stats[0] = raw.size();
      stats[1] = skipped;
      stats[2] = encoded.unprocessable;
      stats[3] = narrow;
      stats[4] = accepted.size() - narrow;
      stats[5] = encoded.encoded.size() - accepted.size();
    }
    std::ostringstream os;
    homs::write_ssm_tsv(os, accepted);
    const std::string out = os.str();
    if (tsv && out.size() <= cap) std::memcpy(tsv, out.data(), out.size());
    return static_cast<long long>(out.size());
  });
}

}  // extern "C"
