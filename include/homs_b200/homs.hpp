// homs_b200/homs.hpp -- C++20 host facade over the C ABI (include/homs_b200.h).
//
// It keeps the call shapes of the reference's encoder/search API so that a caller of `homs_core`
// can switch to the GPU by changing a namespace (paths under /root/reference/proj/core/):
//
//   encode_spectra   include/homs/pipeline.hpp:45-48     src/pipeline.cpp:60-85
//   encode           include/homs/encoder.hpp:20         src/encoder.cpp:19-55
//   build_index      include/homs/search.hpp:82          src/search.cpp:17-60
//   search_one       include/homs/search.hpp:99-100      src/search.cpp:105-169
//   search_batch     include/homs/search.hpp:104-107     src/search.cpp:171-183
//   cascade_search   include/homs/search.hpp:114-117     src/search.cpp:219-248
//   parse_mgf        include/homs/mgf.hpp:20             src/mgf.cpp:93-181
//
// plus one composition the reference spells as two calls with host vectors in between:
//
//   encode_and_index == build_index(encode_spectra(spectra, ...).encoded)   (hypervectors never leave HBM)
//
// The facade is header-only and generic over the data types: instantiate it with a traits struct
// that names the caller's own types.  With the reference's headers that is
//
//   struct HomsApi {
//     using RawSpectrum = homs::RawSpectrum;   using EncodedSpectrum = homs::EncodedSpectrum; ...
//   };
//   auto out = homs_b200::encode_spectra<HomsApi>(spectra, codebook, preprocess, threads, batch);
//
// and homs_b200::types / homs_b200::DefaultApi provide structurally identical stand-alone types.
// Errors surface as the Api's ConfigError / InvariantError (include/homs/errors.hpp:16-56) with the
// library's message; everything else as Api::Error.  `threads` and `batch_size` are accepted for
// signature parity and never change results (search.hpp:102-103).  There is no CPU fallback: every
// call needs a CUDA device.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <istream>
#include <iterator>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../homs_b200.h"

namespace homs_b200 {

// ---- stand-alone mirror of the reference's boundary types -----------------------------------
namespace types {

struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : Error { using Error::Error; };
struct InvariantError : Error { using Error::Error; };
struct ParseError : Error {  // errors.hpp:22-32
  ParseError(std::size_t line, const std::string& message)
      : Error("line " + std::to_string(line) + ": " + message), line_(line) {}
  std::size_t line() const noexcept { return line_; }

 private:
  std::size_t line_;
};

struct Peak { double mz = 0.0, intensity = 0.0; };
struct SpectrumMeta {
  std::string id;
  double precursor_mz = 0.0;
  std::uint8_t charge = 0;
  bool is_decoy = false;
  std::string peptide;
};
struct RawSpectrum { SpectrumMeta meta; std::vector<Peak> peaks; };

class Hypervector {
 public:
  Hypervector() = default;
  explicit Hypervector(std::uint32_t bits) : bits_(bits), words_((std::size_t(bits) + 63) / 64, 0) {}
  std::uint32_t size_bits() const noexcept { return bits_; }
  std::span<const std::uint64_t> words() const noexcept { return words_; }
  std::span<std::uint64_t> words() noexcept { return words_; }
  friend bool operator==(const Hypervector&, const Hypervector&) = default;
 private:
  std::uint32_t bits_ = 0;
  std::vector<std::uint64_t> words_;
};

struct EncodedSpectrum { SpectrumMeta meta; Hypervector hv; };
enum class IntensityScaling : std::uint8_t { none = 0, sqrt = 1 };
struct PreprocessConfig {
  double min_mz = 101.0, max_mz = 1500.0, bin_size = 0.05;
  std::uint32_t max_peaks = 50, min_peaks = 10;
  double intensity_floor = 0.01;
  IntensityScaling scaling = IntensityScaling::none;
};
struct EncoderConfig { std::uint32_t dim = 8192, step_flips = 4096, levels = 16; std::uint64_t seed = 1; };
struct Codebook {
  EncoderConfig config;
  std::uint32_t spectrum_dims = 0;
  std::vector<Hypervector> position, level;
};
struct SpectrumVector {
  std::uint32_t dims = 0;
  std::vector<std::uint32_t> bins;
  std::vector<double> intensities;
  SpectrumMeta meta;
};
struct Tolerance {
  enum class Kind : std::uint8_t { ppm, dalton };
  Kind kind = Kind::ppm;
  double value = 20.0;
};
enum class SearchStage : std::uint8_t { narrow = 0, wide = 1 };
struct Ssm {
  std::string query_id, library_id, peptide;
  std::uint8_t charge = 0;
  double query_precursor_mz = 0.0, library_precursor_mz = 0.0, mass_diff = 0.0;
  std::uint32_t raw_score = 0;
  double score = 0.0;
  bool is_decoy = false;
  SearchStage stage = SearchStage::narrow;
  std::optional<double> q_value;
};
struct EncodeOutcome { std::vector<EncodedSpectrum> encoded; std::size_t unprocessable = 0; };
struct SearchOptions { unsigned threads = 1; std::size_t batch_size = 512; };

}  // namespace types

struct DefaultApi {
  using Error = types::Error;
  using ConfigError = types::ConfigError;
  using InvariantError = types::InvariantError;
  using ParseError = types::ParseError;
  using SpectrumMeta = types::SpectrumMeta;
  using RawSpectrum = types::RawSpectrum;
  using Hypervector = types::Hypervector;
  using EncodedSpectrum = types::EncodedSpectrum;
  using PreprocessConfig = types::PreprocessConfig;
  using Codebook = types::Codebook;
  using SpectrumVector = types::SpectrumVector;
  using Tolerance = types::Tolerance;
  using SearchStage = types::SearchStage;
  using Ssm = types::Ssm;
  using EncodeOutcome = types::EncodeOutcome;
  using SearchOptions = types::SearchOptions;
};

constexpr int kConfiguredDevices = -1;  // `device` argument: use the configured device set (set_devices)

namespace detail {

template <class Api>
[[noreturn]] inline void raise(int rc, const homs_b200_ctx* ctx) {
  const char* m = homs_b200_last_error(ctx);
  const std::string msg = (m && *m) ? m : ("homs_b200 error " + std::to_string(rc));
  if (rc == HOMS_B200_ERR_CONFIG) throw typename Api::ConfigError(msg);
  if (rc == HOMS_B200_ERR_INVARIANT) throw typename Api::InvariantError(msg);
  throw typename Api::Error(msg);
}
template <class Api>
inline void check(int rc, const homs_b200_ctx* ctx) {
  if (rc != HOMS_B200_OK) raise<Api>(rc, ctx);
}

struct CtxDeleter { void operator()(homs_b200_ctx* c) const { homs_b200_ctx_destroy(c); } };
using CtxPtr = std::unique_ptr<homs_b200_ctx, CtxDeleter>;

// The devices a call uses when its `device` argument is left at kConfiguredDevices: set_devices(), or
// the environment variable HOMS_B200_DEVICES ("0,1,2,3" or "all") read on first use, else device 0.
// More than one device makes every index / encoder a multi-device context (homs_b200_ctx_create_multi):
// build_index shards the library over them and search_batch / cascade_search / encode_spectra fan out
// with no change at the call site -- the GPU form of the reference's `threads` argument
// (parallel.hpp:20-48).

inline std::vector<int>& device_list() {
  static std::vector<int> devices = [] {
    std::vector<int> d;
    if (const char* e = std::getenv("HOMS_B200_DEVICES")) {
      const std::string v(e);
      if (v == "all") {
        int n = 0;
        if (homs_b200_device_count(&n) == HOMS_B200_OK)
          for (int i = 0; i < n; ++i) d.push_back(i);
      } else {
        std::size_t pos = 0;
        while (pos < v.size()) {
          std::size_t end = v.find(',', pos);
          if (end == std::string::npos) end = v.size();
          if (end > pos) d.push_back(std::atoi(v.substr(pos, end - pos).c_str()));
          pos = end + 1;
        }
      }
    }
    if (d.empty()) d.push_back(0);
    return d;
  }();
  return devices;
}

inline unsigned& device_generation() {
  static unsigned generation = 0;
  return generation;
}

template <class Api>
inline CtxPtr make_ctx(int device) {
  homs_b200_ctx* raw = nullptr;
  int rc;
  if (device == kConfiguredDevices) {
    const std::vector<int> devices = device_list();
    rc = homs_b200_ctx_create_multi(devices.data(), static_cast<int>(devices.size()), &raw);
  } else {
    rc = homs_b200_ctx_create(device, &raw);
  }
  if (rc != HOMS_B200_OK) raise<Api>(rc, nullptr);
  return CtxPtr(raw);
}

// 64-bit content hash of a list of hypervectors (every word; four independent multiply-xor lanes)
template <class Range>
inline std::uint64_t content_hash(const Range& rows, std::uint64_t seed) {
  std::uint64_t h[4] = {seed ^ 0x9E3779B97F4A7C15ull, seed ^ 0xC2B2AE3D27D4EB4Full, seed ^ 0x165667B19E3779F9ull,
                        seed ^ 0x27D4EB2F165667C5ull};
  for (const auto& r : rows) {
    const auto w = r.words();
    std::size_t i = 0;
    for (; i + 4 <= w.size(); i += 4)
      for (int l = 0; l < 4; ++l) h[l] = (h[l] ^ w[i + l]) * 0x100000001B3ull + (h[l] >> 29);
    for (; i < w.size(); ++i) h[0] = (h[0] ^ w[i]) * 0x100000001B3ull + (h[0] >> 29);
    h[1] += w.size();
  }
  return (h[0] ^ (h[1] << 17 | h[1] >> 47)) * 0x9E3779B97F4A7C15ull ^ (h[2] + (h[3] << 31 | h[3] >> 33));
}

template <class Cfg>
inline homs_b200_preprocess_config pod(const Cfg& c) {
  homs_b200_preprocess_config p{};
  p.min_mz = c.min_mz;
  p.max_mz = c.max_mz;
  p.bin_size = c.bin_size;
  p.max_peaks = c.max_peaks;
  p.min_peaks = c.min_peaks;
  p.intensity_floor = c.intensity_floor;
  p.scaling = static_cast<std::uint32_t>(c.scaling);
  return p;
}

template <class Tol>
inline homs_b200_tolerance pod_tol(const Tol& t) {
  homs_b200_tolerance p{};
  p.kind = t.kind == Tol::Kind::ppm ? HOMS_B200_TOL_PPM : HOMS_B200_TOL_DALTON;
  p.value = t.value;
  return p;
}

// dense row-major words of a list of hypervectors
template <class Range, class GetHv>
inline std::vector<std::uint64_t> flatten(const Range& items, std::size_t W, GetHv get) {
  std::vector<std::uint64_t> flat(items.size() * W);
  std::size_t i = 0;
  for (const auto& it : items) {
    const auto w = get(it).words();
    std::memcpy(flat.data() + i * W, w.data(), W * sizeof(std::uint64_t));
    ++i;
  }
  return flat;
}

// One context per device (slot 0: the configured device set) for encoding; remembers which codebook is
// resident by a hash of its whole content.
template <class Api>
struct Encoder {
  CtxPtr ctx;
  std::mutex mu;
  bool cb_resident = false;
  std::uint64_t cb_tag = 0;
  unsigned generation = 0;

  static Encoder& on(int device) {
    static std::mutex table_mu;
    static std::vector<std::unique_ptr<Encoder>> table;
    std::lock_guard<std::mutex> g(table_mu);
    const std::size_t slot = device == kConfiguredDevices ? 0 : static_cast<std::size_t>(device) + 1;
    if (table.size() <= slot) table.resize(slot + 1);
    if (!table[slot] || (slot == 0 && table[slot]->generation != device_generation())) {
      table[slot] = std::make_unique<Encoder>();  // (re)created after set_devices()
      table[slot]->ctx = make_ctx<Api>(device);
      table[slot]->generation = device_generation();
    }
    return *table[slot];
  }

  void ensure_codebook(const typename Api::Codebook& cb) {
    const std::uint32_t dim = cb.config.dim;
    const std::size_t W = (std::size_t(dim) + 63) / 64;
    if (cb.position.size() != cb.spectrum_dims || cb.level.size() != std::size_t(cb.config.levels) + 1)
      throw typename Api::InvariantError("encode: codebook shape does not match its configuration");
    if (dim < 1) throw typename Api::InvariantError("encode: codebook dimension must be positive");
    for (const auto& r : cb.position)
      if (r.words().size() != W) throw typename Api::InvariantError("encode: codebook shape does not match its configuration");
    for (const auto& r : cb.level)
      if (r.words().size() != W) throw typename Api::InvariantError("encode: codebook shape does not match its configuration");
    // identity of the resident codebook: a hash of EVERY position and level word (a few ms for the
    // 28.7 MB table of D = 8192 -- less than the flatten + upload it saves), never addresses or samples
    const std::uint64_t tag = content_hash(cb.position, (std::uint64_t(dim) << 32) ^ cb.spectrum_dims) ^
                              content_hash(cb.level, cb.config.levels) * 0xD6E8FEB86659FD93ull;
    if (cb_resident && cb_tag == tag) return;
    const auto pos = flatten(cb.position, W, [](const auto& h) -> const auto& { return h; });
    const auto lvl = flatten(cb.level, W, [](const auto& h) -> const auto& { return h; });
    check<Api>(homs_b200_codebook_upload(ctx.get(), dim, cb.spectrum_dims, cb.config.levels, pos.data(),
                                         lvl.data()),
               ctx.get());
    cb_resident = true;
    cb_tag = tag;
  }
};

}  // namespace detail

// Devices used by every call whose `device` argument is left at its default (see detail::device_list).
// Call it before the indexes / encoders it should apply to are created, from one thread.
inline void set_devices(std::vector<int> devices) {
  if (devices.empty()) devices.push_back(0);
  detail::device_list() = std::move(devices);
  ++detail::device_generation();
}
inline const std::vector<int>& devices() { return detail::device_list(); }

// ---- LibraryIndex (search.hpp:39-66): the device-resident index --------------------------------
// Owns a context whose library is the charge-partitioned, m/z-sorted matrix built by
// homs_b200_library_upload; keeps the metadata in input order like the reference (search.cpp:27).
template <class Api = DefaultApi>
class LibraryIndex {
 public:
  std::uint32_t dim() const noexcept { return dim_; }
  std::size_t size() const noexcept { return metas_.size(); }
  const typename Api::SpectrumMeta& meta(std::size_t ordinal) const { return metas_[ordinal]; }
  homs_b200_ctx* context() const noexcept { return ctx_.get(); }
  const std::vector<std::uint8_t>& decoy_flags() const noexcept { return decoy_; }

 private:
  template <class A>
  friend LibraryIndex<A> build_index(std::span<const typename A::EncodedSpectrum>, int);
  template <class A>
  friend LibraryIndex<A> encode_and_index(std::span<const typename A::RawSpectrum>, const typename A::Codebook&,
                                          const typename A::PreprocessConfig&, std::size_t*, int);
  std::uint32_t dim_ = 0;
  std::vector<typename Api::SpectrumMeta> metas_;
  std::vector<std::uint8_t> decoy_;
  detail::CtxPtr ctx_;
};

// ---- encode_spectra (pipeline.cpp:60-85) --------------------------------------------------------
template <class Api = DefaultApi>
typename Api::EncodeOutcome encode_spectra(std::span<const typename Api::RawSpectrum> spectra,
                                           const typename Api::Codebook& codebook,
                                           const typename Api::PreprocessConfig& preprocess,
                                           unsigned /*threads*/ = 1, std::size_t /*batch_size*/ = 0,
                                           int device = kConfiguredDevices) {
  auto& enc = detail::Encoder<Api>::on(device);
  std::lock_guard<std::mutex> g(enc.mu);
  typename Api::EncodeOutcome outcome;
  if (spectra.empty()) return outcome;
  enc.ensure_codebook(codebook);
  const std::size_t n = spectra.size();
  const std::uint32_t dim = codebook.config.dim;
  const std::size_t W = (std::size_t(dim) + 63) / 64;
  std::vector<std::uint64_t> offsets(n + 1, 0);
  for (std::size_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + spectra[i].peaks.size();
  std::vector<double> mz(offsets[n]), intensity(offsets[n]);
  for (std::size_t i = 0; i < n; ++i) {
    std::size_t o = offsets[i];
    for (const auto& p : spectra[i].peaks) {
      mz[o] = p.mz;
      intensity[o] = p.intensity;
      ++o;
    }
  }
  std::vector<std::uint64_t> words(n * W);
  std::vector<std::uint8_t> ok(n);
  const auto cfg = detail::pod(preprocess);
  detail::check<Api>(homs_b200_encode_batch(enc.ctx.get(), &cfg, n, offsets.data(), mz.data(), intensity.data(),
                                            words.data(), ok.data()),
                     enc.ctx.get());
  outcome.encoded.reserve(n);
  for (std::size_t i = 0; i < n; ++i) {  // order-preserving compaction, pipeline.cpp:75-83
    if (!ok[i]) {
      ++outcome.unprocessable;
      continue;
    }
    typename Api::EncodedSpectrum e{spectra[i].meta, typename Api::Hypervector(dim)};
    std::memcpy(e.hv.words().data(), words.data() + i * W, W * sizeof(std::uint64_t));
    outcome.encoded.push_back(std::move(e));
  }
  return outcome;
}

// ---- encode (encoder.cpp:19-55) on one vectorized spectrum --------------------------------------
template <class Api = DefaultApi>
typename Api::Hypervector encode(const typename Api::SpectrumVector& sv, const typename Api::Codebook& codebook,
                                 int device = kConfiguredDevices) {
  auto& enc = detail::Encoder<Api>::on(device);
  std::lock_guard<std::mutex> g(enc.mu);
  if (sv.dims != codebook.spectrum_dims)  // encoder.cpp:20-22
    throw typename Api::InvariantError("encode: spectrum vector dimensionality does not match codebook");
  enc.ensure_codebook(codebook);
  const std::uint64_t off[2] = {0, sv.bins.size()};
  typename Api::Hypervector hv(codebook.config.dim);
  detail::check<Api>(homs_b200_encode_vectors(enc.ctx.get(), 1, off, sv.bins.data(), sv.intensities.data(),
                                              hv.words().data()),
                     enc.ctx.get());
  return hv;
}

// ---- build_index (search.cpp:17-60) -------------------------------------------------------------
template <class Api = DefaultApi>
LibraryIndex<Api> build_index(std::span<const typename Api::EncodedSpectrum> refs, int device = kConfiguredDevices) {
  if (refs.empty()) throw typename Api::InvariantError("build_index: library is empty");  // search.cpp:18
  LibraryIndex<Api> index;
  index.dim_ = refs.front().hv.size_bits();
  const std::size_t n = refs.size(), W = (std::size_t(index.dim_) + 63) / 64;
  for (const auto& r : refs)
    if (r.hv.size_bits() != index.dim_)  // search.cpp:24-26
      throw typename Api::InvariantError("build_index: mixed hypervector dimensionalities");
  index.metas_.reserve(n);
  std::vector<double> mz(n);
  std::vector<std::uint8_t> charge(n);
  index.decoy_.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    index.metas_.push_back(refs[i].meta);
    mz[i] = refs[i].meta.precursor_mz;
    charge[i] = refs[i].meta.charge;
    index.decoy_[i] = refs[i].meta.is_decoy ? 1 : 0;
  }
  // id_rank: position in the sort by (id, ordinal) -- the integer form of search.cpp:43
  std::vector<std::uint32_t> order(n), rank(n);
  for (std::size_t i = 0; i < n; ++i) order[i] = static_cast<std::uint32_t>(i);
  std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
    return index.metas_[a].id < index.metas_[b].id;
  });
  for (std::size_t p = 0; p < n; ++p) rank[order[p]] = static_cast<std::uint32_t>(p);
  const auto words = detail::flatten(refs, W, [](const auto& r) -> const auto& { return r.hv; });
  index.ctx_ = detail::make_ctx<Api>(device);
  detail::check<Api>(homs_b200_library_upload(index.ctx_.get(), index.dim_, n, words.data(), mz.data(),
                                              charge.data(), rank.data(), 0, 1),
                     index.ctx_.get());
  return index;
}

namespace detail {

template <class Api>
typename Api::Ssm make_ssm(const typename Api::EncodedSpectrum& query, const LibraryIndex<Api>& index,
                           std::uint32_t ordinal, std::uint32_t raw_score) {  // search.cpp:155-168
  const auto& lib = index.meta(ordinal);
  typename Api::Ssm s;
  s.query_id = query.meta.id;
  s.library_id = lib.id;
  s.peptide = lib.peptide;
  s.charge = query.meta.charge;
  s.query_precursor_mz = query.meta.precursor_mz;
  s.library_precursor_mz = lib.precursor_mz;
  s.mass_diff = query.meta.precursor_mz - lib.precursor_mz;
  s.raw_score = raw_score;
  s.score = static_cast<double>(raw_score) / static_cast<double>(index.dim());
  s.is_decoy = lib.is_decoy;
  s.stage = Api::SearchStage::narrow;
  return s;
}

template <class Api>
struct FlatQueries {
  std::vector<std::uint64_t> words;
  std::vector<double> mz;
  std::vector<std::uint8_t> charge;
  std::uint32_t dim = 0;
  explicit FlatQueries(std::span<const typename Api::EncodedSpectrum> q, std::uint32_t index_dim) {
    dim = index_dim;
    for (const auto& e : q)
      if (e.hv.size_bits() != index_dim)  // search.cpp:107-109
        throw typename Api::InvariantError("search_one: query dimensionality does not match index");
    const std::size_t W = (std::size_t(dim) + 63) / 64;
    words = flatten(q, W, [](const auto& e) -> const auto& { return e.hv; });
    mz.reserve(q.size());
    charge.reserve(q.size());
    for (const auto& e : q) {
      mz.push_back(e.meta.precursor_mz);
      charge.push_back(e.meta.charge);
    }
  }
};

}  // namespace detail

// ---- search_batch / search_one (search.cpp:105-183) ---------------------------------------------
template <class Api = DefaultApi>
std::vector<std::optional<typename Api::Ssm>> search_batch(std::span<const typename Api::EncodedSpectrum> queries,
                                                           const LibraryIndex<Api>& index,
                                                           const typename Api::Tolerance& tol,
                                                           const typename Api::SearchOptions& = {}) {
  std::vector<std::optional<typename Api::Ssm>> results(queries.size());
  if (queries.empty()) return results;
  const detail::FlatQueries<Api> q(queries, index.dim());
  std::vector<std::uint32_t> score(queries.size()), ordinal(queries.size());
  const auto t = detail::pod_tol(tol);
  detail::check<Api>(homs_b200_search_batch(index.context(), q.dim, queries.size(), q.words.data(), q.mz.data(),
                                            q.charge.data(), &t, 1, score.data(), ordinal.data(), nullptr, nullptr),
                     index.context());
  for (std::size_t i = 0; i < queries.size(); ++i)
    if (ordinal[i] != HOMS_B200_NO_HIT) results[i] = detail::make_ssm<Api>(queries[i], index, ordinal[i], score[i]);
  return results;
}

template <class Api = DefaultApi>
std::optional<typename Api::Ssm> search_one(const typename Api::EncodedSpectrum& query,
                                            const LibraryIndex<Api>& index, const typename Api::Tolerance& tol) {
  return search_batch<Api>(std::span<const typename Api::EncodedSpectrum>(&query, 1), index, tol)[0];
}

// ---- cascade_search (search.cpp:219-248) ---------------------------------------------------------
template <class Api = DefaultApi>
std::vector<typename Api::Ssm> cascade_search(std::span<const typename Api::EncodedSpectrum> queries,
                                              const LibraryIndex<Api>& index,
                                              const typename Api::Tolerance& narrow,
                                              const typename Api::Tolerance& wide, double fdr_q,
                                              const typename Api::SearchOptions& = {}) {
  if (!(narrow.value > 0.0) || !(wide.value > 0.0))  // Tolerance::validate, search.cpp:13-15
    throw typename Api::ConfigError("tolerance value must be positive");
  std::vector<typename Api::Ssm> out;
  if (queries.empty()) return out;
  const detail::FlatQueries<Api> q(queries, index.dim());
  const std::size_t n = queries.size();
  std::vector<std::uint64_t> which(n);
  std::vector<std::uint32_t> ordinal(n), score(n);
  std::vector<std::uint8_t> stage(n);
  std::vector<double> qv(n);
  std::uint64_t count = 0;
  const auto tn = detail::pod_tol(narrow), tw = detail::pod_tol(wide);
  detail::check<Api>(homs_b200_cascade_search(index.context(), q.dim, n, q.words.data(), q.mz.data(),
                                              q.charge.data(), &tn, &tw, fdr_q, index.decoy_flags().data(),
                                              which.data(), ordinal.data(), stage.data(), score.data(), qv.data(),
                                              &count),
                     index.context());
  out.reserve(count);
  for (std::uint64_t m = 0; m < count; ++m) {  // narrow block, then wide, each in query order
    auto s = detail::make_ssm<Api>(queries[which[m]], index, ordinal[m], score[m]);
    s.stage = stage[m] == 0 ? Api::SearchStage::narrow : Api::SearchStage::wide;
    s.q_value = qv[m];
    out.push_back(std::move(s));
  }
  return out;
}

// ---- encode_and_index: build_index(encode_spectra(...).encoded) without the host round trip -------
// (pipeline.cpp:60-85 + search.cpp:17-60).  Library ordinals -- and index.meta(ordinal) -- count the
// processable spectra only, exactly as if the reference's two calls had been made.
template <class Api = DefaultApi>
LibraryIndex<Api> encode_and_index(std::span<const typename Api::RawSpectrum> spectra,
                                   const typename Api::Codebook& codebook,
                                   const typename Api::PreprocessConfig& preprocess,
                                   std::size_t* unprocessable = nullptr, int device = kConfiguredDevices) {
  if (spectra.empty()) throw typename Api::InvariantError("build_index: library is empty");  // search.cpp:18
  LibraryIndex<Api> index;
  index.dim_ = codebook.config.dim;
  index.ctx_ = detail::make_ctx<Api>(device);
  {
    detail::Encoder<Api> enc;  // uploads the codebook into the index's own context
    enc.ctx = std::move(index.ctx_);
    enc.ensure_codebook(codebook);
    index.ctx_ = std::move(enc.ctx);
  }
  const std::size_t n = spectra.size();
  std::vector<std::uint64_t> offsets(n + 1, 0);
  for (std::size_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + spectra[i].peaks.size();
  std::vector<double> mz(offsets[n]), intensity(offsets[n]), prec(n);
  std::vector<std::uint8_t> charge(n), ok(n);
  for (std::size_t i = 0; i < n; ++i) {
    std::size_t o = offsets[i];
    for (const auto& p : spectra[i].peaks) {
      mz[o] = p.mz;
      intensity[o] = p.intensity;
      ++o;
    }
    prec[i] = spectra[i].meta.precursor_mz;
    charge[i] = spectra[i].meta.charge;
  }
  std::vector<std::uint32_t> order(n), rank(n);  // id_rank over the raw list (search.cpp:43)
  for (std::size_t i = 0; i < n; ++i) order[i] = static_cast<std::uint32_t>(i);
  std::stable_sort(order.begin(), order.end(),
                   [&](std::uint32_t a, std::uint32_t b) { return spectra[a].meta.id < spectra[b].meta.id; });
  for (std::size_t p = 0; p < n; ++p) rank[order[p]] = static_cast<std::uint32_t>(p);
  const auto cfg = detail::pod(preprocess);
  std::uint64_t n_encoded = 0;
  detail::check<Api>(homs_b200_library_build_from_spectra(index.ctx_.get(), &cfg, n, offsets.data(), mz.data(),
                                                          intensity.data(), prec.data(), charge.data(), rank.data(),
                                                          0, 1, ok.data(), &n_encoded),
                     index.ctx_.get());
  index.metas_.reserve(n_encoded);
  index.decoy_.reserve(n_encoded);
  for (std::size_t i = 0; i < n; ++i)
    if (ok[i]) {
      index.metas_.push_back(spectra[i].meta);
      index.decoy_.push_back(spectra[i].meta.is_decoy ? 1 : 0);
    }
  if (unprocessable) *unprocessable = n - n_encoded;
  return index;
}

// ---- parse_mgf (mgf.cpp:93-181) -------------------------------------------------------------------
// Same spectra, same doubles, same first ParseError (line and message) as the reference's sequential
// parser; the text is parsed on the device.  Api::ParseError(line, message) when the traits name one.
template <class Api = DefaultApi>
std::vector<typename Api::RawSpectrum> parse_mgf(std::istream& in, const std::string& decoy_prefix, int device = kConfiguredDevices) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  auto& enc = detail::Encoder<Api>::on(device);
  std::lock_guard<std::mutex> g(enc.mu);
  homs_b200_mgf_info info{};
  const int rc = homs_b200_mgf_parse(enc.ctx.get(), text.data(), text.size(), &info);
  if (rc == HOMS_B200_ERR_PARSE) {
    std::string msg = homs_b200_last_error(enc.ctx.get());
    const auto colon = msg.find(": ");
    if (colon != std::string::npos) msg = msg.substr(colon + 2);
    if constexpr (requires { typename Api::ParseError; })
      throw typename Api::ParseError(static_cast<std::size_t>(info.error_line), msg);
    else
      throw typename Api::Error("line " + std::to_string(info.error_line) + ": " + msg);
  }
  detail::check<Api>(rc, enc.ctx.get());
  const std::size_t n = info.n_spectra;
  std::vector<std::uint64_t> offsets(n + 1);
  std::vector<double> mz(info.n_peaks), intensity(info.n_peaks), prec(n);
  std::vector<std::uint8_t> charge(n);
  std::vector<std::uint32_t> toff(n), tlen(n), soff(n), slen(n);
  detail::check<Api>(homs_b200_mgf_fetch(enc.ctx.get(), offsets.data(), mz.data(), intensity.data(), prec.data(),
                                         charge.data(), toff.data(), tlen.data(), soff.data(), slen.data()),
                     enc.ctx.get());
  std::vector<typename Api::RawSpectrum> spectra(n);
  for (std::size_t i = 0; i < n; ++i) {  // finalize_block, mgf.cpp:66-76
    auto& s = spectra[i];
    s.meta.id = tlen[i] ? text.substr(toff[i], tlen[i]) : "spectrum_" + std::to_string(i + 1);
    s.meta.precursor_mz = prec[i];
    s.meta.charge = charge[i];
    s.meta.peptide = text.substr(soff[i], slen[i]);
    s.meta.is_decoy = !decoy_prefix.empty() && (s.meta.id.compare(0, decoy_prefix.size(), decoy_prefix) == 0 ||
                                                s.meta.peptide.compare(0, decoy_prefix.size(), decoy_prefix) == 0);
    s.peaks.resize(offsets[i + 1] - offsets[i]);
    for (std::size_t k = 0; k < s.peaks.size(); ++k) {
      s.peaks[k].mz = mz[offsets[i] + k];
      s.peaks[k].intensity = intensity[offsets[i] + k];
    }
  }
  return spectra;
}

}  // namespace homs_b200
