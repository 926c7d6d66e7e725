"""The interpolating coarse gather (K1g, csrc/gather.cuh) against the oracle
and against the transform kernel K1 (csrc/coarse.cuh) it replaces.

mgift (reference proj/src/transforms.cpp:134-173) through `LTCI_COARSE=gather`
is held to the same 2e-5 as the transform kernel; whole detector runs with
the two coarse formulations must agree on every per-range-cell peak."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import AmbiguitySpace, DetectorOptions, ds_grft, ds_kt_mfp, mgift, scene
from paper_2403_06788_b200.configs import config
from paper_2403_06788_b200.detectors import Engine, detection_threshold
from paper_2403_06788_b200.model import Bounds, RadarParams, RangeRoi, build_ambiguity, build_dual_scale

from helpers import TOL, check_candidates, check_peaks, cube, load, max_rel, radar, space

pytestmark = pytest.mark.gpu

KTOL = 2e-5


@pytest.fixture
def gather(monkeypatch):
    monkeypatch.setenv("LTCI_COARSE", "gather")


@pytest.fixture
def transform(monkeypatch):
    monkeypatch.setenv("LTCI_COARSE", "transform")


def test_mgift_gather_matches_reference_golden(gather):
    g = load("transforms.npz")
    p = radar(g)
    x = cube(g)
    d = mgift(x, p, [11.7, -4.1]) - g["mgift"]
    assert np.abs(d).max() / np.abs(g["mgift"]).max() < KTOL
    d = mgift(x, p, [2.0, 3.3], 1) - g["mgift_kt"]
    assert np.abs(d).max() / np.abs(g["mgift_kt"]).max() < KTOL


@pytest.mark.parametrize("M,K", [(32, 64), (64, 128), (128, 256), (256, 512), (512, 1024), (1024, 2048),
                                 (256, 4096), (2048, 4096), (32, 8192)])
def test_mgift_gather_all_sizes(gather, M, K):
    """White noise over the whole band (the worst case for the interpolation
    window), shifts of every size and sign, third order, the keystone variant
    with a large folding number."""
    p = RadarParams.create(3e9, 20e6, 18e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((M, K), complex), 1.0, M + K))
    for c, v in (([123.0, -7.5], 0), ([-2711.0, 95.0], 0), ([41.0, 3.0, 0.4], 0), ([0.0], 0), ([3.0, 6.5], 1),
                 ([-6.0, -11.0], 1)):
        ref = O.port_mgift(x, p, c, v)
        got = mgift(x, p, c, v)
        assert np.abs(got - ref).max() / np.abs(ref).max() < KTOL, (c, v)


def test_mgift_gather_point_target(gather):
    """A single range-compressed point (sinc profile): the gathered peak
    follows the trajectory to the same accuracy."""
    M, K = 64, 512
    p = RadarParams.create(3e9, 25e6, 20e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(scene.synthesize_cube(p, [(1.0, [200.3 * p.delta_R(), 87.0, 2.0])]))
    for c in ([87.0, 2.0], [-150.0, 5.0]):
        ref = O.port_mgift(x, p, c, 0)
        assert np.abs(mgift(x, p, c, 0) - ref).max() / np.abs(ref).max() < KTOL


def _run(w, x, gamma, keep_dense=False):
    e = Engine(w.params, w.space, w.variant, w.amb, DetectorOptions(retain_threshold=gamma, keep_dense=keep_dense))
    try:
        e.run_host(x)
        return e.coarse_path(), e.result()
    finally:
        e.close()


def test_engine_paths_agree_c0(monkeypatch):
    """configs[0] through both coarse formulations: same counters, candidates
    and per-range-cell peaks (values to 1e-4, indices identical except ties)."""
    g = load("c0.npz")
    w = config(0)
    x = cube(g)
    gamma = float(g["gamma"])
    monkeypatch.setenv("LTCI_COARSE", "transform")
    pt, mt = _run(w, x, gamma)
    monkeypatch.setenv("LTCI_COARSE", "gather")
    pg, mg = _run(w, x, gamma)
    assert (pt, pg) == ("transform", "gather")
    assert mt.counters == mg.counters
    rel = np.abs(np.abs(mg.peak_value) - np.abs(mt.peak_value)) / np.abs(mt.peak_value)
    assert rel.max() < 1e-4
    assert (mg.peak_index != mt.peak_index).sum() <= 3
    check_candidates(mg.cand_index, mg.cand_value, mt.cand_index, mt.cand_value, gamma)
    # and the golden itself
    from test_gpu_parity import _cell_value
    check_peaks(mg.peak_index, mg.peak_value, g["peak_index"], g["peak_value"],
                value_at=lambda i: _cell_value(x, w, i))


def test_default_paths():
    """AUTO: the gather whenever a table serves at least 16 coarse cells
    (configs[1], [2], [4]); the transform for configs[0] (11 cells) and
    configs[3] (4 cells per folding number)."""
    for ci, want in ((0, "transform"), (4, "gather"), (3, "transform")):
        w = config(ci)
        e = Engine(w.params, w.space, w.variant, w.amb, DetectorOptions(retain_threshold=1e9))
        try:
            assert e.coarse_path() == want, ci
        finally:
            e.close()


def test_small_goldens_gather(gather):
    """The reference's dense small-case maps (DS-GRFT and DS-KT-MFP, ROI
    subset, several folding numbers) with the gather forced."""
    g = load("small_grft.npz")
    p = radar(g)
    gm = ds_grft(cube(g), p, space(g, p), DetectorOptions(retain_threshold=float(g["retain"]), keep_dense=True))
    assert np.abs(gm.dense - g["dense"]).max() / np.abs(g["dense"]).max() <= TOL
    check_peaks(gm.peak_index, gm.peak_value, g["peak_index"], g["peak_value"], value_at=lambda i: g["dense"][i])
    g = load("small_kt.npz")
    p = radar(g)
    amb = AmbiguitySpace(int(g["amb"][0]), int(g["amb"][1]))
    gm = ds_kt_mfp(cube(g), p, amb, space(g, p), DetectorOptions(retain_threshold=float(g["retain"]), keep_dense=True))
    assert np.abs(gm.dense - g["dense"]).max() / np.abs(g["dense"]).max() <= TOL
    check_peaks(gm.peak_index, gm.peak_value, g["peak_index"], g["peak_value"], value_at=lambda i: g["dense"][i])


def test_random_spaces_gather_vs_port(gather):
    """Reference-built spaces with ROI subsets: dense maps against the port."""
    rng = np.random.default_rng(11)
    for K, M, ratio in ((64, 32, 4.0), (128, 32, 8.0), (256, 128, 16.0)):
        p = RadarParams.create(ratio * 100e6, 100e6, 50e6, 2000.0, M, K)
        s = build_dual_scale(p, 2, [Bounds(-30.0, 30.0), Bounds(-8.0, 8.0)], [0.5, 0.5],
                             RangeRoi(int(rng.integers(0, K // 4)), K - 1 - int(rng.integers(0, K // 4))))
        x = scene.to_complex64_roundtrip(
            scene.add_noise(scene.synthesize_cube(p, [(0.3, [K / 2 * p.delta_R(), 11.0, 2.5])]), 1.0 / K, K + M))
        opt = DetectorOptions(retain_threshold=0.5, keep_dense=True)
        gm = ds_grft(x, p, s, opt)
        rm = O.port_ds(x, p, s, opt)
        assert max_rel(gm.dense, rm.dense) <= TOL
        assert np.abs(gm.dense - rm.dense).max() / np.abs(rm.dense).max() <= TOL
        check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])
        amb = build_ambiguity(p, Bounds(-1.6 * p.Va(), 1.6 * p.Va()))
        gk = ds_kt_mfp(x, p, amb, s, opt)
        rk = O.port_ds(x, p, s, opt, variant=1, amb=amb)
        assert np.abs(gk.dense - rk.dense).max() / np.abs(rk.dense).max() <= TOL
        check_peaks(gk.peak_index, gk.peak_value, rk.peak_index, rk.peak_value, value_at=lambda i: rk.dense[i])


def test_gather_wide_shift_spread(gather):
    """Coarse cells 40 range-migration steps apart: the shifts of one CTA's
    cells spread past the staged halo and the taps come from global memory
    (the fallback path), with wrap-around at both ends of the range axis."""
    from paper_2403_06788_b200.configs import baseline_space
    from paper_2403_06788_b200.model import Grid
    p = RadarParams.create(3e9, 20e6, 20e6, 1000.0, 64, 256)
    s = baseline_space(p, [(-2000.0, 2000.0), (-6.0, 6.0)])
    g0, f1 = s.coarse[0], s.fine[1]
    assert g0.count >= 32
    s.coarse[0] = Grid(g0.start * 40.0, g0.step * 40.0, g0.count)
    s.fine[1] = Grid(f1.start, f1.step * 30.0, 5)
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.3, [100 * p.delta_R(), 0.0, 1.0])]), 1.0 / p.K, 3))
    opt = DetectorOptions(retain_threshold=0.5, keep_dense=True)
    gm = ds_grft(x, p, s, opt)
    rm = O.port_ds(x, p, s, opt)
    assert np.abs(gm.dense - rm.dense).max() / np.abs(rm.dense).max() <= TOL
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_engine_paths_agree_full_size(monkeypatch, cfg):
    """BASELINE shapes at full size through the two independent coarse
    formulations (K-point transform per (cell, pulse) vs interpolated
    oversampled profiles): every per-range-cell peak agrees -- magnitudes to
    1e-4, indices identical except near-ties -- and so do the candidate sets.
    configs[2] on a 2 x 1 x 1 coarse slice, configs[4] on its first CPI."""
    from paper_2403_06788_b200.configs import sliced
    w = config(cfg)
    if cfg == 2:
        w = sliced(w, 2, 1)
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    monkeypatch.setenv("LTCI_COARSE", "transform")
    pt, mt = _run(w, x, gamma)
    monkeypatch.setenv("LTCI_COARSE", "gather")
    pg, mg = _run(w, x, gamma)
    assert (pt, pg) == ("transform", "gather")
    assert mt.counters == mg.counters
    rel = np.abs(np.abs(mg.peak_value) - np.abs(mt.peak_value)) / np.abs(mt.peak_value)
    assert rel.max() < 1e-4, rel.max()
    diff = np.nonzero(mg.peak_index != mt.peak_index)[0]
    assert diff.size <= max(3, mt.peak_index.size // 200), diff.size
    check_candidates(mg.cand_index, mg.cand_value, mt.cand_index, mt.cand_value, gamma)
    assert mg.argmax == mt.argmax


def test_gather_batched_weights_bit_identical(monkeypatch):
    """Plans too large for the plan-wide weight cache compute the weights per X
    batch: with a 24 MiB X budget (several batches at configs[4]'s shape) and
    the cache disabled the map is bit-identical to the cached single-batch run."""
    w = config(4)
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    monkeypatch.setenv("LTCI_COARSE", "gather")
    _, ref = _run(w, x, gamma)
    monkeypatch.setenv("LTCI_X_BUDGET_MB", "24")
    monkeypatch.setenv("LTCI_GATHER_WCACHE_MB", "0")
    _, got = _run(w, x, gamma)
    assert np.array_equal(got.peak_index, ref.peak_index)
    assert np.array_equal(got.peak_value, ref.peak_value)
    assert np.array_equal(got.cand_index, ref.cand_index) and np.array_equal(got.cand_value, ref.cand_value)


def test_more_coarse_cells_than_one_grid_extent(monkeypatch):
    """70 000 coarse cells over a one-row ROI (X is 256 B per cell, so the X
    budget alone would put them in one batch): the engine splits at the grid's
    65 535-cell extent; both coarse formulations agree on the peak and the
    retained set."""
    from paper_2403_06788_b200.configs import baseline_space
    from paper_2403_06788_b200.model import Grid
    p = RadarParams.create(3e9, 20e6, 20e6, 1000.0, 32, 64)
    s = baseline_space(p, [(-50.0, 50.0), (-1.0, 1.0)], roi=RangeRoi(20, 20))
    s.coarse[0] = Grid(-2000.0, 4000.0 / 7000, 7000)
    s.coarse[1] = Grid(-50.0, 10.0, 10)
    s.fine[1] = Grid(0.0, 1.0, 1)
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.5, [20 * p.delta_R(), 333.0, 20.0])]), 1.0 / p.K, 5))
    w = type("W", (), {"params": p, "space": s, "variant": 0, "amb": None})()
    out = {}
    for mode in ("transform", "gather"):
        monkeypatch.setenv("LTCI_COARSE", mode)
        out[mode] = _run(w, x, 14.0)[1]
    a, b = out["transform"], out["gather"]
    assert a.counters == b.counters and a.counters[2] == 70000 * p.M
    assert a.argmax == b.argmax
    assert abs(abs(a.argmax_value) - abs(b.argmax_value)) <= 1e-4 * abs(a.argmax_value)
    check_candidates(b.cand_index, b.cand_value, a.cand_index, a.cand_value, a.retain_threshold)
