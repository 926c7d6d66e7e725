"""Batched Monte-Carlo Pd: device synthesis, the
device splitmix64 / Box-Muller noise stream, and run_pd with every trial on
the GPU, against the reference (oracle/_ref) and the reference's own
test_bench.cpp cases (proj/tests/test_bench.cpp:13-88)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import _cabi as A
from paper_2403_06788_b200 import scene
from paper_2403_06788_b200.model import Bounds, RadarParams, RangeRoi
from paper_2403_06788_b200.montecarlo import Scenario

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="reference not built (oracle/_ref)")


def tiny_scenario(**kw) -> Scenario:
    """test_bench.cpp:13-29 (fixtures::small(64, 32, 8.0, 0.5, 100e6, 2000.0))."""
    p = RadarParams.create(8.0 * 100e6, 100e6, 0.5 * 100e6, 2000.0, 32, 64)
    sc = Scenario(params=p, targets=[(1.0 + 0j, [20 * p.delta_R(), 6.0, 0.0])], snr_db=[-6.0, 0.0], trials=8,
                  pfa=1e-4, seed=31, detectors=[A.FD_GRFT, A.DS_GRFT], P=2,
                  bounds=[Bounds(-20.0, 20.0), Bounds(-10.0, 10.0)], alpha=[0.5, 0.5], roi=RangeRoi(8, 40))
    for k, v in kw.items():
        setattr(sc, k, v)
    return sc


@needs_ref
def test_reference_run_pd_binding_cpu():
    """The reference's run_pd through the shim (CPU only): reproducible, saturates."""
    a = O.ref_run_pd(tiny_scenario())
    assert a == O.ref_run_pd(tiny_scenario())
    for curve in O.ref_run_pd(tiny_scenario(snr_db=[40.0], trials=2)):
        assert all(pt[1] == 1.0 for pt in curve)


@pytest.mark.gpu
def test_device_noise_matches_the_reference_stream():
    from paper_2403_06788_b200.montecarlo import add_noise
    p = RadarParams.create(3e9, 20e6, 16e6, 1000.0, 64, 128)
    clean = scene.synthesize_cube(p, [(0.3 + 0.2j, [40 * p.delta_R(), 12.0, 1.0])])
    for sigma2, seed in ((1.0, 5), (0.25, 2**63 + 11), (1.0 / p.K, 0)):
        dev = add_noise(clean, p, sigma2, seed)
        host = scene.add_noise(clean, sigma2, seed)  # numpy port pinned to rng.cpp (test_oracle)
        assert np.abs(dev - host).max() <= 1e-14 * max(1.0, np.abs(host).max())
        if O.have_ref():
            ref = O.ref_synthesize(p, [(0.3 + 0.2j, [40 * p.delta_R(), 12.0, 1.0])], sigma2, seed)
            assert np.abs(dev - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max())


@pytest.mark.gpu
def test_device_synthesis_matches_the_reference():
    from paper_2403_06788_b200.montecarlo import synthesize
    p = RadarParams.create(3e9, 20e6, 16e6, 1000.0, 64, 128)
    tg = [(0.3 + 0.2j, [40 * p.delta_R(), 12.0, 1.0]), (1.0, [77 * p.delta_R(), -40.0, 3.0, 0.5])]
    dev = synthesize(p, tg)
    host = scene.synthesize_cube(p, tg)
    assert np.abs(dev - host).max() <= 1e-9 * np.abs(host).max()
    if O.have_ref():
        ref = O.ref_synthesize(p, tg)
        assert np.abs(dev - ref).max() <= 1e-9 * np.abs(ref).max()


@pytest.mark.gpu
def test_pd_reproducible_saturates_and_brackets():
    """test_bench.cpp:43-88 on the GPU run_pd."""
    from paper_2403_06788_b200.montecarlo import run_pd
    a, b = run_pd(tiny_scenario()), run_pd(tiny_scenario())
    assert [[p.pd for p in c.points] for c in a] == [[p.pd for p in c.points] for c in b]
    for c in run_pd(tiny_scenario(snr_db=[40.0], trials=2)):
        assert all(p.pd == 1.0 for p in c.points)
    for c in run_pd(tiny_scenario(snr_db=[-20.0, -8.0, 2.0], trials=24)):
        for i in range(1, len(c.points)):
            prev = c.points[i - 1]
            assert c.points[i].pd >= prev.pd - (prev.ci_hi - prev.ci_lo)
    for c in run_pd(tiny_scenario(snr_db=[-4.0], trials=16)):
        for p in c.points:
            assert p.ci_lo <= p.pd + 1e-12 and p.ci_hi >= p.pd - 1e-12


@pytest.mark.gpu
@needs_ref
def test_pd_matches_reference_run_pd():
    """Same seeds -> the same noisy cubes (to complex64 rounding) -> the same
    per-trial decisions, except near-threshold flips between FP32 and FP64."""
    from paper_2403_06788_b200.montecarlo import run_pd
    sc = tiny_scenario(snr_db=[-12.0, -8.0, -4.0, 0.0], trials=40,
                       detectors=[A.FD_GRFT, A.DS_GRFT, A.DS_KT_MFP])
    ours = run_pd(sc)
    ref = O.ref_run_pd(sc)
    for c, r in zip(ours, ref):
        for p, q in zip(c.points, r):
            assert p.snr_db == q[0] and p.trials == q[2]
            assert abs(p.pd - q[1]) * p.trials <= 1, (c.kind, p.snr_db, p.pd, q[1])


@pytest.mark.gpu
def test_run_pd_rejects_unbuilt_detectors():
    from paper_2403_06788_b200.montecarlo import run_pd
    with pytest.raises(ValueError, match="not built"):
        run_pd(tiny_scenario(detectors=[A.TD_GRFT]))
    with pytest.raises(ValueError, match="trials"):
        run_pd(tiny_scenario(trials=0))
