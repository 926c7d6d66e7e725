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


def oracle_cell(x, params, space, idx, variant=0, amb=None):
    """FP64 oracle value of one dual-scale flat cell: the C restatement run on
    the space restricted to that cell's coarse cell and ROI row (full fine and
    Doppler axes), read at the cell's (fine, Doppler) position.  Size-independent:
    lets full BASELINE-size GPU maps be checked at sampled cells."""
    import copy

    import oracle as O
    from paper_2403_06788_b200.configs import doppler_window
    from paper_2403_06788_b200.model import AmbiguitySpace, DetectorOptions, Grid, RangeRoi
    s = space
    D = doppler_window(params, s)[1] if variant == 0 else params.M
    R = s.roi.count()
    F = int(np.prod([g.count for g in s.fine[1:]])) if s.order() > 1 else 1
    if variant == 1:
        F = s.fine[1].count
    jj = idx % D
    r = (idx // D) % R
    f = (idx // (D * R)) % F
    c = idx // (D * R * F)
    sl = copy.deepcopy(s)
    sl.roi = RangeRoi(s.roi.first + r, s.roi.first + r)
    a2 = amb
    if variant == 0:
        rem = c
        for i in reversed(range(s.order())):
            ci = rem % s.coarse[i].count
            rem //= s.coarse[i].count
            sl.coarse[i] = Grid(s.coarse[i].value(ci), s.coarse[i].step, 1)
    else:
        ci = c % s.coarse[1].count
        q = amb.q_min + c // s.coarse[1].count
        sl.coarse[1] = Grid(s.coarse[1].value(ci), s.coarse[1].step, 1)
        a2 = AmbiguitySpace(q, q)
    m = O.port_ds(x, params, sl, DetectorOptions(retain_threshold=-1.0, keep_dense=True), variant, a2)
    return complex(m.dense[f * D + jj])
