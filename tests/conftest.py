import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2410_04001_b200", "liblrnr_gpu.so")
    orc = os.path.join(ROOT, "oracle", "liblrnr_oracle.so")
    if not (os.path.exists(lib) and os.path.exists(orc)):
        import __graft_entry__

        __graft_entry__.build()


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def gpu():
    import paper_2410_04001_b200 as pkg

    ctx = pkg.GpuContext(0)
    yield ctx
    ctx.close()


def floor_rel(got, want, floor=1e-3):
    """The reference's rel_err with a floor (test_autodiff.cpp:15-17, acceptance.cpp:40-42)."""
    got, want = np.asarray(got, float), np.asarray(want, float)
    den = np.maximum(np.abs(want), floor * max(np.abs(want).max(), 1e-300))
    return float((np.abs(got - want) / den).max())


def normwise(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference compiled in place (oracle/_ref, built by oracle/Makefile in the build
    container; the .so travels to the GPU box). Missing -> the test FAILS: it is the strongest pin."""
    from oracle.oracle import Reference, reference_available

    assert reference_available(), "oracle/_ref/liblrnr_ref.so missing: run __graft_entry__.build() with /root/reference"
    return Reference()
