"""Shared test helpers: golden-fixture loading and the parity comparator
(SURVEY.md App. C): magnitudes within a tolerance of the compared set's
largest magnitude, identical indices except ties within the tolerance."""
from __future__ import annotations

import os

import numpy as np

from paper_2403_06788_b200.model import (AmbiguitySpace, DualScaleSpace, Grid, RadarParams, RangeRoi, StepSizes)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# North-star tolerance for FP32 magnitudes (BASELINE.json): 1e-3 relative.
TOL = 1e-3


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def radar(g, prefix=""):
    r = g[prefix + "radar"]
    return RadarParams(float(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]), int(r[5]), int(r[6]),
                       int(r[7]))


def space(g, p, prefix=""):
    s = DualScaleSpace(params=p, kappa=float(g[prefix + "kappa"]),
                       roi=RangeRoi(int(g[prefix + "roi"][0]), int(g[prefix + "roi"][1])))
    for row in g[prefix + "coarse"]:
        s.coarse.append(Grid(float(row[0]), float(row[1]), int(row[2])))
    for row in g[prefix + "fine"]:
        s.fine.append(Grid(float(row[0]), float(row[1]), int(row[2])))
    st = g[prefix + "steps"]
    s.steps = StepSizes(list(map(float, st[0])), list(map(float, st[1])), list(map(float, st[2])))
    return s


def cube(g):
    return g["cube"].astype(np.complex128)


def max_rel(a, b, scale=None):
    a, b = np.asarray(a), np.asarray(b)
    scale = scale if scale is not None else max(np.abs(b).max(), 1e-300)
    return float(np.max(np.abs(np.abs(a) - np.abs(b))) / scale) if a.size else 0.0


def check_candidates(gi, gv, ri, rv, retain, tol=TOL, scale=None):
    """Candidate sets equal except cells within tol of the retention threshold."""
    gset, rset = set(gi.tolist()), set(ri.tolist())
    scale = scale or max(np.abs(rv).max() if rv.size else 1.0, 1.0)
    rmag = dict(zip(ri.tolist(), np.abs(rv).tolist()))
    gmag = dict(zip(gi.tolist(), np.abs(gv).tolist()))
    for i in rset - gset:
        assert abs(rmag[i] - retain) <= tol * max(retain, 1e-30), f"candidate {i} missing (|Y|={rmag[i]})"
    for i in gset - rset:
        assert abs(gmag[i] - retain) <= tol * max(retain, 1e-30), f"extra candidate {i} (|Y|={gmag[i]})"
    common = sorted(gset & rset)
    if common:
        gpos = {v: k for k, v in enumerate(gi.tolist())}
        rpos = {v: k for k, v in enumerate(ri.tolist())}
        ga = np.array([gv[gpos[i]] for i in common])
        ra = np.array([rv[rpos[i]] for i in common])
        err = np.abs(np.abs(ga) - np.abs(ra)) / np.maximum(np.abs(ra), 1e-30)
        assert err.max() <= tol, f"candidate magnitude rel err {err.max():.2e}"
    assert np.all(np.diff(gi.astype(np.int64)) > 0), "candidates not sorted by index"


def check_peaks(gi, gv, ri, rv, tol=TOL, value_at=None):
    """Per-row peaks: identical indices unless the oracle's value at the GPU's
    index is within tol of the oracle's peak (a tie)."""
    assert len(gi) == len(ri)
    rel = np.abs(np.abs(gv) - np.abs(rv)) / np.maximum(np.abs(rv), 1e-30)
    assert rel.max() <= tol, f"peak magnitude rel err {rel.max():.2e}"
    bad = np.nonzero(gi != ri)[0]
    for r in bad:
        if value_at is None:
            raise AssertionError(f"row {r}: peak index {gi[r]} != {ri[r]}")
        alt = abs(value_at(int(gi[r])))
        assert abs(alt - abs(rv[r])) <= tol * abs(rv[r]), f"row {r}: index {gi[r]} vs {ri[r]} is not a tie"
    return len(bad)
