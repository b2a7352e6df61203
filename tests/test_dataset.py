"""Appendix-A dataset files <-> batch arrays, pinned to the reference's own
files (tests/golden/ds_*.csv written by ccdkit.dataset.write_queries, with
its parse results in ds_*.npz; see tests/golden/make_dataset_golden.py)."""

import io
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from paper_2009_13349_b200 import QueryKind
from paper_2009_13349_b200.dataset import (DatasetError, LabeledBatch, concat, parse_queries,
                                           write_queries)

SETS = [("handcrafted", "vf"), ("handcrafted", "ee"), ("adv", "vf"), ("adv", "ee")]
KIND = {"vf": QueryKind.VERTEX_FACE, "ee": QueryKind.EDGE_EDGE}


@pytest.mark.parametrize("name,tag", SETS)
def test_parse_matches_reference_bitwise(name, tag):
    path = os.path.join(GOLDEN_DIR, f"ds_{name}_{tag}.csv")
    g = np.load(os.path.join(GOLDEN_DIR, f"ds_{name}_{tag}.npz"))
    b = parse_queries(path, KIND[tag])
    assert b.points.shape == g["points"].shape
    assert np.array_equal(b.points.view(np.int64), g["points"].view(np.int64))
    assert np.array_equal(b.truth, g["truth"])
    assert (b.kind == int(KIND[tag])).all()


@pytest.mark.parametrize("name,tag", SETS)
def test_rewrite_is_byte_identical(name, tag, tmp_path):
    path = os.path.join(GOLDEN_DIR, f"ds_{name}_{tag}.csv")
    b = parse_queries(path, KIND[tag], keep_rationals=True)
    out = tmp_path / "o.csv"
    write_queries(b, out)
    assert out.read_bytes() == open(path, "rb").read()
    gz = tmp_path / "o.csv.gz"
    write_queries(b, gz)
    b2 = parse_queries(gz, KIND[tag])
    assert np.array_equal(b2.points, b.points) and np.array_equal(b2.truth, b.truth)


def test_binary64_writer_round_trips():
    b = parse_queries(os.path.join(GOLDEN_DIR, "ds_adv_vf.csv"), QueryKind.VERTEX_FACE)
    buf = io.StringIO()
    write_queries(b, buf)  # exact value of each double
    b2 = parse_queries(io.StringIO(buf.getvalue()), QueryKind.VERTEX_FACE)
    assert np.array_equal(b2.points.view(np.int64), b.points.view(np.int64))


def _rows(n, truth="1", fields=7):
    row = ",".join(["1", "2"] * 3 + [truth]) if fields == 7 else "1,2,3"
    return "\n".join([row] * n) + "\n"


@pytest.mark.parametrize("text,msg", [
    ("1,2,3,4,5\n", "expected 7 fields"),
    ("1,1,1,1,1,1,maybe\n" * 8, "bad truth"),
    ("1,0,1,1,1,1,1\n" * 8, "zero denominator"),
    ("1.5,1,1,1,1,1,1\n" * 8, "malformed integer"),
    ("1,1,1,1,1,1,1\n" * 7, "not a multiple of 8"),
    ("1,1,1,1,1,1,1\n" * 7 + "1,1,1,1,1,1,0\n", "truth differs"),
    ("1" + "0" * 400 + ",1,1,1,1,1,1\n" + "1,1,1,1,1,1,1\n" * 7, "overflows"),
])
def test_malformed_input_raises_like_reference(text, msg):
    with pytest.raises(DatasetError, match=msg):
        parse_queries(io.StringIO(text), QueryKind.VERTEX_FACE)


def test_tokens_blank_lines_and_concat():
    text = "\n" + "1,2,-3,4,5,-8,TRUE\n" * 8 + "\n" + "0,1,0,1,0,1,false\n" * 8
    b = parse_queries(io.StringIO(text), QueryKind.EDGE_EDGE)
    assert b.n == 2 and list(b.truth) == [1, 0]
    assert b.points[0, 0].tolist() == [0.5, -0.75, -0.625]
    c = concat([b, b])
    assert c.n == 4 and (c.kind == 1).all()
    with pytest.raises(DatasetError):
        write_queries(LabeledBatch(b.points, b.kind, np.array([1, -1], np.int8)), io.StringIO())
