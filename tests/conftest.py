"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` runs on a B200."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

RESULT_KEYS = ("best_row", "best_col", "best_rho", "best_degenerate", "refined_row",
               "refined_col", "refined_rho", "below_threshold", "final_threshold", "centers",
               "eliminated", "retained", "ops", "elim_pct")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def res_vec(r):
    d = r.as_dict()
    return np.array([float(d[k]) for k in RESULT_KEYS])


def assert_same_result(got, want, keys=RESULT_KEYS, msg=""):
    """Bit-exact comparison of two MatchResult-like records (ints and FP64 bits)."""
    g = got.as_dict() if hasattr(got, "as_dict") else got
    w = want.as_dict() if hasattr(want, "as_dict") else want
    bad = {k: (g[k], w[k]) for k in keys if g[k] != w[k]}
    assert not bad, f"{msg} mismatches: {bad}"


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f != "config1.npz")


@pytest.fixture(scope="session")
def port():
    from oracle.binding import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import binding
    if not binding.available("ref"):
        if os.path.isdir("/root/reference/proj/src"):
            binding.build("ref")
        else:
            pytest.skip("reference build (oracle/_ref) not present on this machine")
    return binding.Oracle("ref", autobuild=False)


@pytest.fixture(scope="session")
def ctx():
    from paper_1407_3535_b200 import api
    c = api.Context(0)  # raises (no fallback) when the library or the GPU is missing
    yield c
    c.close()
