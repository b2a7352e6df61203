"""Shared test plumbing.

Markers: ``gpu`` = needs a CUDA device and the built libtccd.so (run on the
B200 box with ``-m gpu``); everything else runs on CPU.
"""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
GOLDEN_SETS = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                     if not os.path.basename(p).startswith(("ds_", "irf_")))  # dataset / IRF fixtures
FIELDS = ("status", "toi", "tol", "codom", "checks", "early", "witness", "level")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU and the built libtccd.so")


def load_golden(name):
    with np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")) as g:
        return {k: g[k] for k in g.files}


def assert_same_results(got, ref, where=""):
    """Bit-exact comparison of the 13-field result on non-error queries;
    error queries must carry the same error class (status >= 2)."""
    st_ref = np.asarray(ref["status"])
    st_got = np.asarray(got["status"])
    err = st_ref >= 2
    assert np.array_equal(st_got >= 2, err), f"{where}: error classes differ"
    ok = ~err
    for k in FIELDS:
        if k not in got:
            continue
        a, b = np.asarray(got[k])[ok], np.asarray(ref[k])[ok]
        if k == "witness":
            eq = (a.view(np.int64) == b.view(np.int64)).all(axis=1)
        elif a.dtype.kind == "f":
            eq = a.view(np.int64) == b.view(np.int64)  # bitwise, incl. +inf
        else:
            eq = a == b
        if not eq.all():
            i = int(np.flatnonzero(~eq)[0])
            raise AssertionError(f"{where}: field {k} differs on {(~eq).sum()} queries; "
                                 f"first idx {np.flatnonzero(ok)[i]}: got {a[i]} ref {b[i]}")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test needs a CUDA device")
    import paper_2009_13349_b200 as tccd  # noqa: F401
    return torch.device("cuda", 0)
