"""Build properties of libtccd.so (CPU-only: reads the cubin with cuobjdump).

The reference's rounding -- and the filter error bounds derived for it
(pkg/src/ccdkit/inclusion.py:8-15, core.py:19-23) -- assume every multiply
and add is a separate IEEE op, so the solver's SASS must contain no DFMA.
"""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2009_13349_b200", "libtccd.so")


def _sass():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    return subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout


def test_solver_is_fma_free_fp64_for_sm100a():
    sass = _sass()
    assert "arch = sm_100a" in sass
    assert "DFMA" not in sass
    assert "DADD" in sass and "DMUL" in sass


def test_every_engine_tier_and_prologue_present():
    out = subprocess.run(["cuobjdump", "-elf", LIB], capture_output=True, text=True).stdout
    assert "prologue_kernel" in out
    assert out.count("engine_kernel") >= 3
