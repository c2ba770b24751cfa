"""The C++ facade (include/homs_b200/homs.hpp): it compiles stand-alone with its own mirror types
(CPU), and the parity binary built against the UNMODIFIED reference passes on the GPU."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "facade_parity")

STANDALONE = r"""
#include "homs_b200/homs.hpp"
namespace g = homs_b200;
using A = g::DefaultApi;
int main() {   // instantiate every entry point with the stand-alone types; never executed on CPU
  std::vector<A::RawSpectrum> spectra(1);
  A::Codebook cb;
  A::PreprocessConfig pre;
  auto out = g::encode_spectra<>(std::span<const A::RawSpectrum>(spectra), cb, pre, 4, 64);
  A::SpectrumVector sv;
  auto hv = g::encode<>(sv, cb);
  auto ix = g::build_index<>(std::span<const A::EncodedSpectrum>(out.encoded));
  A::Tolerance tol;
  auto hits = g::search_batch<>(std::span<const A::EncodedSpectrum>(out.encoded), ix, tol);
  auto one = g::search_one<>(out.encoded[0], ix, tol);
  auto acc = g::cascade_search<>(std::span<const A::EncodedSpectrum>(out.encoded), ix, tol, tol, 0.01);
  return int(hits.size() + acc.size() + one.has_value() + hv.size_bits());
}
"""


def test_facade_compiles_and_links_standalone():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "standalone.cpp")
        with open(src, "w") as f:
            f.write(STANDALONE)
        libdir = os.path.join(ROOT, "paper_2211_16422_b200")
        subprocess.run(["g++", "-std=gnu++20", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
                        src, "-o", os.path.join(d, "standalone"), "-L" + libdir, "-l:libhoms_b200.so",
                        "-Wl,-rpath," + libdir], check=True)


@pytest.mark.gpu
def test_facade_parity_against_compiled_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/facade_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout and r.stdout.count("[PASS]") >= 10
