"""The oracle (oracle/tccd_oracle.c) reproduces the reference's own outputs.

tests/golden/*.npz were produced by running ccdkit's numba kernel
(pkg/src/ccdkit/_kernel.py:136) -- see tests/golden/make_golden.py.  This pins
the oracle; the GPU parity tests then compare against golden and oracle.
"""

import numpy as np
import pytest

import oracle
from conftest import GOLDEN_SETS, assert_same_results, load_golden


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_oracle_matches_reference_bit_for_bit(name):
    g = load_golden(name)
    r = oracle.solve_batch(g["points"], g["kind"], g["delta"], g["max_checks"],
                           g["separation"], g["t_max"])
    assert_same_results(r, g, name)


def test_golden_sets_cover_the_workloads():
    names = set(GOLDEN_SETS)
    for need in ("kat", "handcrafted", "c0", "c1", "c2", "c3", "c4_d1e-3", "c4_d1e-5",
                 "c0_tmax0.3", "c0_tmax0.7"):
        assert need in names


def test_kat_values_match_survey_appendix_b():
    g = load_golden("kat")
    names = list(g["names"])
    row = lambda n: names.index(n)
    i = row("vf_vertical")
    assert g["toi"][i] == 0.4999995231628418 and g["checks"][i] == 240
    i = row("vf_vertical_mI5")
    assert g["toi"][i] == 0.25 and g["checks"][i] == 5 and g["early"][i] == 1
    i = row("vf_vertical_d0.1")
    assert g["toi"][i] == 0.44921875 and g["checks"][i] == 1_000_000
    i = row("vf_offset_miss")
    assert g["status"][i] == 0 and g["checks"][i] == 1
    assert g["status"][row("vf_vertical_d2_error")] == 2


def test_single_query_entry_matches_batch():
    g = load_golden("kat")
    for i in range(len(g["kind"])):
        if g["status"][i] >= 2:
            continue
        pts = g["points"][i]
        eps = oracle_eps(pts, int(g["kind"][i]), float(g["separation"][i]))
        r = oracle.solve_kernel(pts[:4], pts[4:], int(g["kind"][i]), g["t_max"][i],
                                g["delta"][i], int(g["max_checks"][i]), g["separation"][i], *eps)
        assert r[0] == g["status"][i] and r[4] == g["checks"][i]
        assert np.float64(r[1]).view(np.int64) == np.float64(g["toi"][i]).view(np.int64)


def oracle_eps(pts, kind, sep):
    import ctypes
    out = np.zeros(3)
    p = np.ascontiguousarray(pts, dtype=np.float64)
    rc = oracle.lib().tccd_oracle_filters(p.ctypes.data_as(ctypes.c_void_p), kind, sep,
                                          out.ctypes.data_as(ctypes.c_void_p))
    assert rc == 1
    return tuple(out)


# --- IRF baseline: the C restatement vs the reference's
# own irf_solve outputs (tests/golden/make_irf_golden.py)

IRF_SETS = ("irf_kat", "irf_hc", "irf_c0", "irf_c1")


@pytest.mark.parametrize("name", IRF_SETS)
def test_oracle_irf_matches_reference(name):
    g = load_golden(name)
    got = oracle.irf_batch(g["points"], g["kind"], g["delta"], g["max_checks"], g["t_max"])
    assert_same_results(got, g, name)
