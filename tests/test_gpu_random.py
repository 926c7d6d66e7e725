"""Randomised parity sweep: seeded random radars, spaces and options through the
public API against the FP64 oracle (our C restatement, pinned to the
reference by tests/test_oracle.py).  Each case draws K, M, the order P, the
fc/fs ratio, search bounds and split fractions, a ROI, the variant (DS-GRFT /
DS-KT-MFP) and the fine-stage formulation (AUTO, CUDA-core FFT, tcgen05), then
compares the dense map (1e-3 of its maximum), the candidate set (identical
except within 1e-3 of the threshold, magnitudes 1e-3 relative), the per-row
peaks (identical except ties) and the counters (exact)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import _cabi as A
from paper_2403_06788_b200 import scene
from paper_2403_06788_b200.detectors import Engine, detection_threshold
from paper_2403_06788_b200.model import (Bounds, DetectorOptions, RadarParams, RangeRoi, build_ambiguity,
                                         build_dual_scale)

from helpers import TOL, check_candidates, check_peaks, max_rel

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    K = int(rng.choice([16, 32, 64, 128, 256]))
    M = int(rng.choice([8, 16, 32, 64, 128, 256, 512]))
    variant = int(rng.integers(0, 2))
    P = 2 if variant == 1 else int(rng.integers(1, 4))
    ratio = float(rng.uniform(2.0, min(16.0, float(M))))  # (fc/fs)/M <= 1 (build_dual_scale condition)
    p = RadarParams.create(ratio * 100e6, 100e6, float(rng.uniform(0.5, 1.0)) * 100e6, 2000.0, M, K)
    scale = [30.0, 6.0, 2.0][:P]
    bounds = [Bounds(-float(rng.uniform(0.3, 1.0)) * s_, float(rng.uniform(0.3, 1.0)) * s_) for s_ in scale]
    alpha = rng.uniform(0.2, 1.0, P)
    alpha = list(alpha / alpha.sum())
    lo = int(rng.integers(0, K // 4))
    hi = K - 1 - int(rng.integers(0, K // 4))
    s = build_dual_scale(p, P, bounds, alpha, RangeRoi(lo, hi))
    amb = build_ambiguity(p, Bounds(-1.5 * p.Va(), 1.5 * p.Va())) if variant == 1 else None
    coeffs = [float(rng.uniform(lo, hi)) * p.delta_R()] + [0.4 * b.hi for b in bounds]
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.2 + 0.1j, coeffs)]), 1.0 / K, 77 + seed))
    paths = [A.FINE_AUTO, A.FINE_FFT_CUDA_CORE] + ([A.FINE_TC_DENSE] if M >= 32 else [])
    path = int(paths[int(rng.integers(0, len(paths)))])
    return p, s, amb, variant, x, path


@pytest.mark.parametrize("seed", range(16))
def test_random_case_vs_oracle(seed):
    p, s, amb, variant, x, path = _case(seed)
    gamma = detection_threshold(p, 1.0 / p.K, 1e-3)
    opt = DetectorOptions(retain_threshold=gamma, keep_dense=True, fine_path=path)
    try:
        e = Engine(p, s, variant, amb, opt)
    except ValueError as ex:  # a shape this fine path does not take is refused loudly, as documented
        assert "M" in str(ex) or "window" in str(ex), ex
        pytest.skip(f"refused: {ex}")
    e.run_host(x)
    gm = e.result()
    e.close()
    rm = O.port_ds(x, p, s, DetectorOptions(retain_threshold=gamma, keep_dense=True), variant, amb)
    assert gm.counters == rm.counters
    assert [[a.role, a.order, a.size] for a in gm.axes] == [[a.role, a.order, a.size] for a in rm.axes]
    assert max_rel(gm.dense, rm.dense) <= TOL
    check_candidates(gm.cand_index, gm.cand_value, rm.cand_index, rm.cand_value, gamma)
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])
