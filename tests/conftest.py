import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: minutes of CPU time on the reference side (whole-config parity)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Everything is built in-tree; build lazily when a fresh checkout runs the tests."""
    import __graft_entry__ as g
    lib = os.path.join(ROOT, "paper_2211_16422_b200", "libhoms_b200.so")
    port = os.path.join(ROOT, "oracle", "libhoms_oracle.so")
    if not (os.path.exists(lib) and os.path.exists(port)):
        g.build()


@pytest.fixture(scope="session")
def port():
    from oracle.binding import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import binding
    if not binding.available("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return binding.Oracle("ref")


@pytest.fixture(scope="session")
def best_oracle():
    """The compiled reference when it travelled with the repo, else the C restatement."""
    from oracle import binding
    return binding.Oracle("ref" if binding.available("ref") else "port")


@pytest.fixture(scope="session")
def hb():
    import paper_2211_16422_b200 as hb
    return hb


@pytest.fixture()
def ctx(hb):
    c = hb.Context(0)
    yield c
    c.close()
