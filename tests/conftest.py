import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def built():
    """Everything compiled: CUDA library (nvcc cross-compiles on CPU) and the oracle."""
    import __graft_entry__ as entry

    entry.build()
    return True


@pytest.fixture(scope="session")
def oracle(built):
    from oracle.oracle import Oracle

    return Oracle("port")


@pytest.fixture(scope="session")
def ref_oracle(built):
    from oracle.oracle import Oracle, REF_PATH

    if not os.path.exists(REF_PATH):
        pytest.skip("oracle/_ref/libslab_ref.so not built (reference headers absent)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def slab(built):
    import paper_2304_08232_b200 as pkg

    pkg.load_library()
    return pkg


@pytest.fixture(scope="session")
def ctx(slab):
    """One GPU context for the whole session. Fails loudly (no skip, no fallback) without a GPU."""
    return slab.Context(0)
