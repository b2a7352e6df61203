"""Labeled query files (the paper's Appendix-A format) <-> batch arrays.

Format (pkg/src/ccdkit/dataset.py:1-16, parse/write at :168-250): one query
is eight CSV rows, one per point -- the four points at t = 0 in query order,
then the same four at t = 1 -- with seven fields per row::

    x_num, x_den, y_num, y_den, z_num, z_den, truth

Coordinates are exact rationals of arbitrary length; truth is 0/1/false/true
(case-insensitive) and must repeat on all eight rows of a record.  No
header; ``.gz`` paths are (de)compressed transparently.  The format carries
no kind, so the caller names it.

Unlike the reference, which builds one ``LabeledQuery`` object per record,
``parse_queries`` fills the batch layout the GPU consumes directly
(``points [n,8,3]`` float64, ``kind [n]`` uint8, ``truth [n]``).  Each
coordinate is the round-to-nearest binary64 image of its rational (Python's
int / int true division is correctly rounded), i.e. exactly the value the
reference's ``float(Fraction)`` produces.  Malformed input raises
``DatasetError`` naming the 1-based row, for the same conditions as the
reference.
"""

from __future__ import annotations

import csv
import gzip
import io
import math
from dataclasses import dataclass, field
from fractions import Fraction
from pathlib import Path
from typing import Iterable, TextIO

import numpy as np

from .core import QueryKind

_TRUTH = {"0": 0, "1": 1, "false": 0, "true": 1}


class DatasetError(ValueError):
    """Malformed dataset input (the message names the offending row)."""


@dataclass
class LabeledBatch:
    """A labeled query set in batch layout.

    truth: int8 per query, 1 colliding, 0 not, -1 undecided (files always
    carry a decided label; -1 only arises from programmatic construction).
    rationals: optional exact coordinates, [n][8][3] pairs (num, den), kept
    when parsing with ``keep_rationals`` so rewriting is byte-identical.
    """

    points: np.ndarray
    kind: np.ndarray
    truth: np.ndarray
    rationals: list | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.points.shape[0])


def _open(path: Path, mode: str):
    if path.suffix == ".gz":
        return gzip.open(path, mode + "t", encoding="ascii", newline="")
    return open(path, mode, encoding="ascii", newline="")


def _to_double(num: int, den: int, row: int) -> float:
    try:
        x = num / den  # correctly rounded for Python ints
    except OverflowError:
        raise DatasetError(f"row {row}: coordinate overflows binary64") from None
    if math.isinf(x):
        raise DatasetError(f"row {row}: coordinate overflows binary64")
    return x


def parse_queries(source, kind, keep_rationals: bool = False) -> LabeledBatch:
    """Read a labeled query file (path, ``.gz`` path, or text stream)."""
    kind = QueryKind(kind)
    if isinstance(source, (str, Path)):
        with _open(Path(source), "r") as fh:
            return parse_queries(fh, kind, keep_rationals)
    coords, truths, rats = [], [], []
    for idx, row in enumerate(csv.reader(source), start=1):
        if not row:
            continue
        if len(row) != 7:
            raise DatasetError(f"row {idx}: expected 7 fields, got {len(row)}")
        fields = [f.strip() for f in row]
        token = fields[6].lower()
        if token not in _TRUTH:
            raise DatasetError(f"row {idx}: bad truth value {fields[6]!r}")
        try:
            ints = [int(f) for f in fields[:6]]
        except ValueError as exc:
            raise DatasetError(f"row {idx}: malformed integer ({exc})") from None
        xyz = []
        for ax in range(3):
            num, den = ints[2 * ax], ints[2 * ax + 1]
            if den == 0:
                raise DatasetError(f"row {idx}: zero denominator")
            xyz.append(_to_double(num, den, idx))
            if keep_rationals:
                rats.append((num, den))
        coords.append(xyz)
        truths.append((_TRUTH[token], idx))
    if len(coords) % 8 != 0:
        raise DatasetError(f"row count {len(coords)} is not a multiple of 8")
    n = len(coords) // 8
    truth = np.empty(n, np.int8)
    for q in range(n):
        t0 = truths[8 * q][0]
        for off in range(8):
            t, row = truths[8 * q + off]
            if t != t0:
                raise DatasetError(f"row {row}: truth differs within record")
        truth[q] = t0
    pts = np.asarray(coords, dtype=np.float64).reshape(n, 8, 3) if n else np.zeros((0, 8, 3))
    rationals = None
    if keep_rationals:
        rationals = [rats[24 * q:24 * (q + 1)] for q in range(n)]
    return LabeledBatch(pts, np.full(n, int(kind), np.uint8), truth, rationals,
                        dict(kind=int(kind)))


def write_queries(batch: LabeledBatch, dest) -> None:
    """Write a batch in canonical form: reduced fractions with positive
    denominators (so -0.0 becomes 0/1), truth as 0/1 on every row, bare
    newline row endings (pkg/src/ccdkit/dataset.py:227-250).  Exact
    rationals are written when the batch kept them, otherwise the exact
    value of each binary64 coordinate."""
    if isinstance(dest, (str, Path)):
        with _open(Path(dest), "w") as fh:
            write_queries(batch, fh)
        return
    if np.any(batch.truth < 0):
        raise DatasetError("undecided queries cannot be written (the format has no such label)")
    w = csv.writer(dest, lineterminator="\n")
    for q in range(batch.n):
        t = "1" if batch.truth[q] else "0"
        for p in range(8):
            row = []
            for ax in range(3):
                if batch.rationals is not None:
                    r = Fraction(*batch.rationals[q][3 * p + ax])
                else:
                    r = Fraction(float(batch.points[q, p, ax]))
                row += [str(r.numerator), str(r.denominator)]
            row.append(t)
            w.writerow(row)


def concat(batches: Iterable[LabeledBatch]) -> LabeledBatch:
    bs = list(batches)
    keep = all(b.rationals is not None for b in bs)
    return LabeledBatch(np.concatenate([b.points for b in bs]),
                        np.concatenate([b.kind for b in bs]),
                        np.concatenate([b.truth for b in bs]),
                        sum((b.rationals for b in bs), []) if keep else None)


def from_workload(w, truth=None) -> LabeledBatch:
    """A seeded synthetic workload as a labeled batch (planted roots are
    colliding by construction; other labels undecided unless given)."""
    if truth is None:
        truth = np.where(np.isnan(w.planted_t), -1, 1).astype(np.int8)
    return LabeledBatch(w.points, w.kind, np.asarray(truth, np.int8))
