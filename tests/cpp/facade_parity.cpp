// Parity of the C++ facade (include/homs_b200/homs.hpp) against the UNMODIFIED reference, in the
// style of the reference's own acceptance binary (proj/tests/acceptance/acceptance_main.cpp):
// plain main(), one "[PASS]/[FAIL] <check>" line per check, exit code 0 iff all pass.
//
// TEST INFRASTRUCTURE: this program links the reference objects compiled by oracle/Makefile and the
// reference headers from $(REF); it is built only where /root/reference exists (tests/cpp/Makefile)
// and the binary travels to the GPU box.  Needs a CUDA device to run.
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "homs/codebook.hpp"
#include "homs/encoder.hpp"
#include "homs/errors.hpp"
#include "homs/mgf.hpp"
#include "homs/pipeline.hpp"
#include "homs/preprocess.hpp"
#include "homs/search.hpp"
#include "homs/synth.hpp"

#include "homs_b200/homs.hpp"

// the traits a reference maintainer would write
struct HomsApi {
  using Error = homs::Error;
  using ConfigError = homs::ConfigError;
  using InvariantError = homs::InvariantError;
  using ParseError = homs::ParseError;
  using SpectrumMeta = homs::SpectrumMeta;
  using RawSpectrum = homs::RawSpectrum;
  using Hypervector = homs::Hypervector;
  using EncodedSpectrum = homs::EncodedSpectrum;
  using PreprocessConfig = homs::PreprocessConfig;
  using Codebook = homs::Codebook;
  using SpectrumVector = homs::SpectrumVector;
  using Tolerance = homs::Tolerance;
  using SearchStage = homs::SearchStage;
  using Ssm = homs::Ssm;
  using EncodeOutcome = homs::EncodeOutcome;
  using SearchOptions = homs::SearchOptions;
};
namespace gpu = homs_b200;

static int g_failed = 0;
static void report(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++g_failed;
}

static bool same_ssm(const homs::Ssm& a, const homs::Ssm& b) {
  return a.query_id == b.query_id && a.library_id == b.library_id && a.peptide == b.peptide &&
         a.charge == b.charge && a.query_precursor_mz == b.query_precursor_mz &&
         a.library_precursor_mz == b.library_precursor_mz && a.mass_diff == b.mass_diff &&
         a.raw_score == b.raw_score && a.score == b.score && a.is_decoy == b.is_decoy && a.stage == b.stage &&
         a.q_value.has_value() == b.q_value.has_value() &&
         (!a.q_value || std::memcmp(&*a.q_value, &*b.q_value, sizeof(double)) == 0);
}

int main() {
  using homs::Tolerance;
  // BASELINE config 1: 5000 targets + 5000 decoys, 1000 queries, D = 2048
  homs::SynthConfig sc;
  sc.n_library = 5000;
  sc.n_query = 1000;
  sc.fraction_modified = 0.6;
  sc.seed = 1;
  homs::SynthOutput synth = homs::generate_benchmark(sc);
  // a few unprocessable spectra and an unknown-charge query exercise the compaction / bucket rules
  synth.library[7].peaks.resize(3);
  synth.queries[11].peaks.clear();
  synth.queries[5].meta.charge = 0;

  const homs::PreprocessConfig pre;
  const homs::EncoderConfig ec{2048, 1024, 16, 1};
  const homs::Codebook cb = homs::make_codebook(homs::dimension(pre), ec);

  const auto ref_lib = homs::encode_spectra(synth.library, cb, pre, 8, 64);
  const auto gpu_lib = gpu::encode_spectra<HomsApi>(synth.library, cb, pre, 8, 64);
  report(gpu_lib.unprocessable == ref_lib.unprocessable && gpu_lib.encoded == ref_lib.encoded,
         "encode_spectra(library): identical EncodedSpectrum list, unprocessable = " +
             std::to_string(gpu_lib.unprocessable));
  const auto ref_q = homs::encode_spectra(synth.queries, cb, pre, 8, 64);
  const auto gpu_q = gpu::encode_spectra<HomsApi>(synth.queries, cb, pre, 1, 0);
  report(gpu_q.unprocessable == ref_q.unprocessable && gpu_q.encoded == ref_q.encoded,
         "encode_spectra(queries): identical, unprocessable = " + std::to_string(gpu_q.unprocessable));

  {  // encode() on one vectorized spectrum
    const auto refined = homs::refine_peaks(synth.library[0], pre);
    const homs::SpectrumVector sv = homs::vectorize(*refined, pre);
    report(gpu::encode<HomsApi>(sv, cb) == homs::encode(sv, cb), "encode(SpectrumVector): identical hypervector");
  }

  const homs::LibraryIndex ref_ix = homs::build_index(ref_lib.encoded);
  const auto gpu_ix = gpu::build_index<HomsApi>(gpu_lib.encoded);
  report(gpu_ix.dim() == ref_ix.dim() && gpu_ix.size() == ref_ix.size(), "build_index: dim and size");

  for (const Tolerance tol : {Tolerance{Tolerance::Kind::dalton, 500.0}, Tolerance{Tolerance::Kind::ppm, 20.0}}) {
    const auto want = homs::search_batch(ref_q.encoded, ref_ix, tol, homs::SearchOptions{8, 64});
    const auto got = gpu::search_batch<HomsApi>(gpu_q.encoded, gpu_ix, tol);
    bool ok = want.size() == got.size();
    std::size_t hits = 0;
    for (std::size_t i = 0; ok && i < want.size(); ++i) {
      ok = want[i].has_value() == got[i].has_value() && (!want[i] || same_ssm(*want[i], *got[i]));
      hits += want[i].has_value();
    }
    report(ok, std::string("search_batch ") + (tol.kind == Tolerance::Kind::ppm ? "20 ppm" : "500 Da") +
                   ": identical optional<Ssm> list, hits = " + std::to_string(hits));
  }
  {
    const auto one_ref = homs::search_one(ref_q.encoded[3], ref_ix, Tolerance{Tolerance::Kind::dalton, 500.0});
    const auto one_gpu = gpu::search_one<HomsApi>(gpu_q.encoded[3], gpu_ix, Tolerance{Tolerance::Kind::dalton, 500.0});
    report(one_ref.has_value() == one_gpu.has_value() && (!one_ref || same_ssm(*one_ref, *one_gpu)), "search_one");
  }
  {
    const Tolerance narrow{Tolerance::Kind::ppm, 20.0}, wide{Tolerance::Kind::dalton, 500.0};
    const auto want = homs::cascade_search(ref_q.encoded, ref_ix, narrow, wide, 0.01, homs::SearchOptions{8, 64});
    const auto got = gpu::cascade_search<HomsApi>(gpu_q.encoded, gpu_ix, narrow, wide, 0.01);
    bool ok = want.size() == got.size();
    std::size_t n_narrow = 0;
    for (std::size_t i = 0; ok && i < want.size(); ++i) {
      ok = same_ssm(want[i], got[i]);
      n_narrow += want[i].stage == homs::SearchStage::narrow;
    }
    report(ok, "cascade_search (20 ppm, 500 Da, 1% FDR): identical accepted list = " + std::to_string(want.size()) +
                   " (" + std::to_string(n_narrow) + " narrow)");
  }
  {  // encode_and_index == build_index(encode_spectra(...).encoded): same answers, no host round trip
    std::size_t dropped = 0;
    const auto fused_ix = gpu::encode_and_index<HomsApi>(synth.library, cb, pre, &dropped);
    bool ok = dropped == ref_lib.unprocessable && fused_ix.size() == ref_ix.size();
    const Tolerance wide{Tolerance::Kind::dalton, 500.0};
    const auto want = homs::search_batch(ref_q.encoded, ref_ix, wide, homs::SearchOptions{8, 64});
    const auto got = gpu::search_batch<HomsApi>(gpu_q.encoded, fused_ix, wide);
    for (std::size_t i = 0; ok && i < want.size(); ++i)
      ok = want[i].has_value() == got[i].has_value() && (!want[i] || same_ssm(*want[i], *got[i]));
    report(ok, "encode_and_index: identical search results, unprocessable = " + std::to_string(dropped));
  }
  {  // parse_mgf: write_mgf of the synthetic library (plus dirt) parsed by both
    std::ostringstream text;
    homs::write_mgf(text, std::span<const homs::RawSpectrum>(synth.library.data(), 300));
    std::string mgf = "# comment\nSEARCH=MIS\n\n" + text.str() +
                      "BEGIN IONS\nPEPMASS=1e2 7\nCHARGE=+3\nSEQ=DECOY_X\n300.5 1\n200.25\t2e0\r\n300.5 3\nEND IONS";
    std::istringstream a(mgf), b(mgf);
    const auto want = homs::parse_mgf(a, "DECOY_");
    const auto got = gpu::parse_mgf<HomsApi>(b, "DECOY_");
    bool ok = want.size() == got.size();
    for (std::size_t i = 0; ok && i < want.size(); ++i)
      ok = want[i].meta.id == got[i].meta.id && want[i].meta.peptide == got[i].meta.peptide &&
           want[i].meta.charge == got[i].meta.charge && want[i].meta.is_decoy == got[i].meta.is_decoy &&
           want[i].meta.precursor_mz == got[i].meta.precursor_mz && want[i].peaks == got[i].peaks;
    report(ok, "parse_mgf: identical RawSpectrum list, " + std::to_string(want.size()) + " spectra");
    for (const char* bad : {"BEGIN IONS\nTITLE=x\n100 1\nEND IONS\n", "BEGIN IONS\nPEPMASS=500\n100 abc\nEND IONS\n",
                            "BEGIN IONS\nPEPMASS=500\n100 1\n", "END IONS\n"}) {
      std::string ref_what, gpu_what;
      std::size_t ref_line = 0, gpu_line = 0;
      try {
        std::istringstream in(bad);
        homs::parse_mgf(in, "DECOY_");
      } catch (const homs::ParseError& e) { ref_what = e.what(); ref_line = e.line(); }
      try {
        std::istringstream in(bad);
        gpu::parse_mgf<HomsApi>(in, "DECOY_");
      } catch (const homs::ParseError& e) { gpu_what = e.what(); gpu_line = e.line(); }
      report(!ref_what.empty() && ref_what == gpu_what && ref_line == gpu_line, "parse_mgf error: " + gpu_what);
    }
  }
  {  // the resident codebook is identified by its whole content: a codebook mutated IN PLACE (same
     // storage, same seed, same sampled words) must be re-uploaded, not served from the stale copy
    homs::Codebook cb2 = cb;
    const auto before = gpu::encode_spectra<HomsApi>(std::span<const homs::RawSpectrum>(synth.queries.data(), 64), cb2, pre);
    cb2.position[12345].words()[3] ^= 0x0000100000000000ull;
    cb2.level[9].words()[17] ^= 0x4ull;
    const auto want = homs::encode_spectra(std::span<const homs::RawSpectrum>(synth.queries.data(), 64), cb2, pre, 8, 64);
    const auto got = gpu::encode_spectra<HomsApi>(std::span<const homs::RawSpectrum>(synth.queries.data(), 64), cb2, pre);
    report(got.encoded == want.encoded && before.encoded.size() == got.encoded.size(),
           "encode_spectra after an in-place codebook mutation: re-uploaded, identical to the reference");
  }
  {  // the same calls over a multi-device set (aliases of device 0 on a one-GPU box): the library is
     // sharded by m/z slices, queries replicated, candidates merged -- nothing changes at the call site
    int n_dev = 0;
    homs_b200_device_count(&n_dev);
    std::vector<int> devs;
    if (n_dev >= 2) for (int i = 0; i < n_dev; ++i) devs.push_back(i);
    else devs = {0, 0, 0};
    gpu::set_devices(devs);
    const auto lib2 = gpu::encode_spectra<HomsApi>(synth.library, cb, pre, 8, 64);
    report(lib2.unprocessable == ref_lib.unprocessable && lib2.encoded == ref_lib.encoded,
           "multi-device encode_spectra (" + std::to_string(devs.size()) + " devices): identical list");
    const auto ix2 = gpu::build_index<HomsApi>(lib2.encoded);
    report(homs_b200_ctx_device_count(ix2.context()) == static_cast<int>(devs.size()), "multi-device build_index: one handle, " +
                                                                                    std::to_string(devs.size()) + " devices");
    for (const Tolerance tol : {Tolerance{Tolerance::Kind::dalton, 500.0}, Tolerance{Tolerance::Kind::ppm, 20.0}}) {
      const auto want = homs::search_batch(ref_q.encoded, ref_ix, tol, homs::SearchOptions{8, 64});
      const auto got = gpu::search_batch<HomsApi>(gpu_q.encoded, ix2, tol);
      bool ok = want.size() == got.size();
      for (std::size_t i = 0; ok && i < want.size(); ++i)
        ok = want[i].has_value() == got[i].has_value() && (!want[i] || same_ssm(*want[i], *got[i]));
      report(ok, std::string("multi-device search_batch ") + (tol.kind == Tolerance::Kind::ppm ? "20 ppm" : "500 Da"));
    }
    const Tolerance narrow{Tolerance::Kind::ppm, 20.0}, wide{Tolerance::Kind::dalton, 500.0};
    const auto want = homs::cascade_search(ref_q.encoded, ref_ix, narrow, wide, 0.01, homs::SearchOptions{8, 64});
    const auto got = gpu::cascade_search<HomsApi>(gpu_q.encoded, ix2, narrow, wide, 0.01);
    bool ok = want.size() == got.size();
    for (std::size_t i = 0; ok && i < want.size(); ++i) ok = same_ssm(want[i], got[i]);
    report(ok, "multi-device cascade_search: identical accepted list = " + std::to_string(got.size()));
    std::size_t dropped = 0;
    const auto fused2 = gpu::encode_and_index<HomsApi>(synth.library, cb, pre, &dropped);
    const auto want_w = homs::search_batch(ref_q.encoded, ref_ix, wide, homs::SearchOptions{8, 64});
    const auto got_w = gpu::search_batch<HomsApi>(gpu_q.encoded, fused2, wide);
    ok = dropped == ref_lib.unprocessable && want_w.size() == got_w.size();
    for (std::size_t i = 0; ok && i < want_w.size(); ++i)
      ok = want_w[i].has_value() == got_w[i].has_value() && (!want_w[i] || same_ssm(*want_w[i], *got_w[i]));
    report(ok, "multi-device encode_and_index: identical search results");
    gpu::set_devices({0});
  }
  // error behaviour
  {
    bool threw = false;
    try {
      gpu::build_index<HomsApi>(std::span<const homs::EncodedSpectrum>{});
    } catch (const homs::InvariantError&) { threw = true; }
    report(threw, "build_index(empty) throws InvariantError (search.cpp:18)");
    threw = false;
    try {
      homs::EncodedSpectrum bad{ref_q.encoded[0].meta, homs::Hypervector(1024)};
      gpu::search_one<HomsApi>(bad, gpu_ix, Tolerance{});
    } catch (const homs::InvariantError&) { threw = true; }
    report(threw, "search_one(dim mismatch) throws InvariantError (search.cpp:107-109)");
    threw = false;
    try {
      gpu::cascade_search<HomsApi>(gpu_q.encoded, gpu_ix, Tolerance{Tolerance::Kind::ppm, 0.0},
                                   Tolerance{Tolerance::Kind::dalton, 500.0}, 0.01);
    } catch (const homs::ConfigError&) { threw = true; }
    report(threw, "cascade_search(zero tolerance) throws ConfigError (search.cpp:13-15)");
  }
  std::printf("%s: %d check(s) failed\n", g_failed ? "FAILED" : "OK", g_failed);
  return g_failed ? 1 : 0;
}
