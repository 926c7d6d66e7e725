"""fd_grft, the single-scale frequency-domain GRFT.

CPU: build_single_scale and the FD branch of extract_detections against the
reference (oracle/_ref).  GPU: ltci_cuda_fd_grft against the reference's
fd_grft golden maps (tests/golden/fd.npz, tests/golden/make_golden.py) at
orders 1-3 -- counters and axes exact, dense complex maps and candidates to
TOL -- and against the reference run live on a larger instance.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import _lib
from paper_2403_06788_b200.detection import extract_detections
from paper_2403_06788_b200.model import (Bounds, DetectorOptions, Grid, RadarParams, RangeRoi, SingleScaleSpace,
                                         StepSizes, build_single_scale)

from helpers import TOL, check_candidates, load, max_rel, radar

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="reference not built (oracle/_ref)")


def single(g, p, prefix):
    s = SingleScaleSpace(params=p, roi=RangeRoi(int(g[prefix + "roi"][0]), int(g[prefix + "roi"][1])))
    for row in g[prefix + "c"]:
        s.c.append(Grid(float(row[0]), float(row[1]), int(row[2])))
    st = g[prefix + "steps"]
    s.steps = StepSizes(list(map(float, st[0])), list(map(float, st[1])), list(map(float, st[2])))
    return s


def golden_map(g, prefix, p, s):
    from paper_2403_06788_b200.model import AxisDesc, DetectionMap
    m = DetectionMap(kind=0, params=p)
    m.axes = [AxisDesc(int(a[0]), int(a[1]), int(a[2])) for a in g[prefix + "axes"]]
    m.retain_threshold = float(g["retain"])
    m.cand_index = g[prefix + "cand_index"].astype(np.uint64)
    m.cand_value = g[prefix + "cand_value"]
    m.single = s
    return m


@needs_ref
def test_build_single_scale_matches_reference():
    p = RadarParams.create(3e9, 20e6, 20e6, 1000.0, 256, 512)
    for P, b, al in ((1, [(-150.0, 150.0)], [1.0]), (2, [(-150.0, 150.0), (-5.0, 5.0)], [0.5, 0.5]),
                     (3, [(-50.0, 50.0), (-5.0, 5.0), (-1.0, 1.0)], [0.4, 0.3, 0.3])):
        ours = build_single_scale(p, P, [Bounds(*x) for x in b], al, RangeRoi(3, 400))
        ref = O.ref_single_scale(p, P, b, al, 3, 400)
        assert [(g.start, g.step, g.count) for g in ours.c] == [(g.start, g.step, g.count) for g in ref.c]
        assert ours.steps.dfm == ref.steps.dfm and ours.steps.rm == ref.steps.rm
    with pytest.raises(ValueError):
        build_single_scale(p, 2, [Bounds(-1.0, 1.0)], [0.5, 0.5], RangeRoi(0, 10))


@needs_ref
def test_extract_detections_on_fd_maps_matches_reference():
    g = load("fd.npz")
    p = radar(g)
    for k in ("1", "2", "3"):
        s = single(g, p, f"s{k}_")
        m = golden_map(g, f"m{k}_", p, s)
        for gamma in (m.retain_threshold, 1.3 * m.retain_threshold):
            dets = extract_detections(m, gamma)
            rows = O.ref_extract_single(m, gamma)
            assert len(dets) == len(rows) > 0
            for d, r in zip(dets, rows):
                assert d.flat_index == int(r[5])
                assert d.statistic == pytest.approx(r[0], rel=1e-12)
                assert d.estimate == pytest.approx(list(r[1:1 + len(d.estimate)]), rel=1e-12, abs=1e-9)


# ------------------------------------------------------------------ GPU ---
@pytest.mark.gpu
@pytest.mark.parametrize("k", ["1", "2", "3"])
def test_fd_grft_golden(k):
    from paper_2403_06788_b200 import fd_grft
    g = load("fd.npz")
    p = radar(g)
    s = single(g, p, f"s{k}_")
    retain = float(g["retain"])
    gm = fd_grft(g["cube"].astype(np.complex128), p, s, DetectorOptions(retain_threshold=retain, keep_dense=True))
    pre = f"m{k}_"
    assert gm.counters == tuple(int(c) for c in g[pre + "counters"])
    assert [[a.role, a.order, a.size] for a in gm.axes] == g[pre + "axes"].tolist()
    ref = g[pre + "dense"]
    assert gm.dense_stored and gm.dense.shape == ref.shape
    assert np.abs(gm.dense - ref).max() / np.abs(ref).max() <= TOL
    assert max_rel(gm.dense, ref) <= TOL
    check_candidates(gm.cand_index, gm.cand_value, g[pre + "cand_index"], g[pre + "cand_value"], retain)
    ref_max = abs(complex(g[pre + "argmax_value"]))
    if gm.argmax != int(g[pre + "argmax"]):  # a tie within TOL
        assert abs(abs(ref[int(gm.argmax)]) - ref_max) <= TOL * ref_max
    assert abs(abs(gm.argmax_value) - ref_max) <= TOL * ref_max


@pytest.mark.gpu
def test_fd_grft_errors():
    from paper_2403_06788_b200 import fd_grft
    g = load("fd.npz")
    p = radar(g)
    s = single(g, p, "s2_")
    x = g["cube"].astype(np.complex128)
    bad = SingleScaleSpace(params=p, steps=s.steps, c=s.c, roi=RangeRoi(0, p.K))
    with pytest.raises(ValueError, match="ROI"):
        fd_grft(x, p, bad)
    other = RadarParams.create(p.fc * 2, p.fs, p.Br, p.PRF, p.M, p.K, p.K_valid)
    with pytest.raises(ValueError, match="different radar"):
        fd_grft(x, other, s)


@pytest.mark.gpu
@needs_ref
def test_fd_grft_vs_reference_live():
    """C0 radar (512 x 256), a velocity/acceleration sub-grid, the reference run here."""
    from paper_2403_06788_b200 import fd_grft
    from paper_2403_06788_b200.configs import config
    w = config(0)
    x = w.cube()
    s = build_single_scale(w.params, 2, [Bounds(80.0, 95.0), Bounds(-5.0, 5.0)], [0.5, 0.5],
                           RangeRoi(150, 260))
    gamma = O.ref_threshold(w.params, w.sigma2, 1e-4)
    opt = DetectorOptions(retain_threshold=gamma, threads=0)
    ref = O.ref_fd(x, w.params, s, opt)
    gm = fd_grft(x, w.params, s, opt)
    assert gm.counters == ref.counters
    check_candidates(gm.cand_index, gm.cand_value, ref.cand_index, ref.cand_value, gamma)
    assert abs(abs(gm.argmax_value) - abs(ref.argmax_value)) <= TOL * abs(ref.argmax_value)
    assert gm.argmax == ref.argmax
    # end to end: the detection lists agree with the reference's own extract on its map
    ours = extract_detections(gm, gamma)
    rows = O.ref_extract_single(ref, gamma)
    assert len(ours) == len(rows) > 0
    for d, r in zip(ours[:5], rows[:5]):
        assert d.flat_index == int(r[5]) and d.statistic == pytest.approx(r[0], rel=TOL)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("K,M", [(2, 16), (4, 16), (8, 8), (16, 64), (128, 32), (512, 16), (1024, 16), (2048, 8),
                                 (4096, 8), (8192, 4)])
def test_fd_grft_all_sizes_vs_reference(K, M):
    """Dense maps against the reference at every supported K (transform radix
    plans 16 .. 16x16x16x2, rotor chains of 1 .. 32 rows per thread)."""
    from paper_2403_06788_b200 import fd_grft, scene
    p = RadarParams.create(3e9, 20e6, 18e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((M, K), complex), 1.0, K + M))
    lo = min(1, K - 1)
    s = build_single_scale(p, 2, [Bounds(-40.0, 40.0), Bounds(-8000.0, 8000.0)], [0.5, 0.5],
                           RangeRoi(lo, max(K - 2, lo)))
    s.c[0].count = min(s.c[0].count, 7)
    s.c[1].count = min(s.c[1].count, 3)
    opt = DetectorOptions(retain_threshold=0.0, keep_dense=True)
    gm = fd_grft(x, p, s, opt)
    ref = O.ref_fd(x, p, s, opt)
    assert gm.counters == ref.counters
    assert np.abs(gm.dense - ref.dense).max() / np.abs(ref.dense).max() <= TOL
    assert max_rel(gm.dense, ref.dense) <= TOL
