"""The TMEM-resident FFT fine kernel (fine_fft_tm_kernel<32, G>, M = 256, 512,
1024) against the FP64 C restatement: orders 1, 2 and 3 (the order-3 space has
two fine axes, so the kernel's outer/inner fine loop and its per-outer chirp
seeds run), DS-GRFT and DS-KT-MFP, dense maps (the DENSE instantiation),
candidates and per-range-cell peaks."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import _cabi as A
from paper_2403_06788_b200 import scene
from paper_2403_06788_b200.detectors import Engine
from paper_2403_06788_b200.model import (Bounds, DetectorOptions, RadarParams, RangeRoi, build_ambiguity,
                                         build_dual_scale)

from helpers import TOL, check_candidates, check_peaks, max_rel

pytestmark = pytest.mark.gpu

CASES = [  # (M, P, bounds, alpha)
    (256, 1, [(-40.0, 40.0)], [1.0]),
    (256, 3, [(-30.0, 30.0), (-6.0, 6.0), (-3.0, 3.0)], [0.4, 0.3, 0.3]),
    (512, 2, [(-30.0, 30.0), (-6.0, 6.0)], [0.5, 0.5]),
    (512, 3, [(-20.0, 20.0), (-3.0, 3.0), (-0.8, 0.8)], [0.4, 0.3, 0.3]),
    (1024, 1, [(-20.0, 20.0)], [1.0]),
    (1024, 3, [(-10.0, 10.0), (-1.0, 1.0), (-0.3, 0.3)], [0.4, 0.3, 0.3]),
]


def _setup(M, P, bounds, alpha, K=64):
    p = RadarParams.create(8 * 100e6, 100e6, 50e6, 2000.0, M, K)  # fc/fs = 8: several fine cells per axis
    s = build_dual_scale(p, P, [Bounds(*b) for b in bounds], alpha, RangeRoi(2, K - 3))
    coeffs = [20 * p.delta_R()] + [0.3 * b[1] for b in bounds]
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.05, coeffs)]), 1.0 / K, M + P))
    return p, s, x


@pytest.mark.parametrize("M,P,bounds,alpha", CASES)
def test_tm_fft_dense_vs_oracle(M, P, bounds, alpha):
    p, s, x = _setup(M, P, bounds, alpha)
    retain = 0.3 * float(M)
    opt = DetectorOptions(retain_threshold=retain, keep_dense=True)
    e = Engine(p, s, opt=opt)
    assert e.fine_path()[0] == A.FINE_FFT_CUDA_CORE
    e.run_host(x)
    gm = e.result()
    e.close()
    rm = O.port_ds(x, p, s, opt)
    assert gm.counters == rm.counters
    assert max_rel(gm.dense, rm.dense) <= TOL
    assert np.abs(gm.dense - rm.dense).max() / np.abs(rm.dense).max() <= TOL
    check_candidates(gm.cand_index, gm.cand_value, rm.cand_index, rm.cand_value, retain)
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])


@pytest.mark.parametrize("M", [256, 512, 1024])
def test_tm_fft_kt_vs_oracle(M):
    p, s, x = _setup(M, 2, [(-30.0, 30.0), (-6.0, 6.0)], [0.5, 0.5])
    amb = build_ambiguity(p, Bounds(-1.6 * p.Va(), 1.6 * p.Va()))
    opt = DetectorOptions(retain_threshold=0.3 * float(M), keep_dense=True)
    e = Engine(p, s, 1, amb, opt)
    assert e.fine_path()[0] == A.FINE_FFT_CUDA_CORE
    e.run_host(x)
    gk = e.result()
    e.close()
    rk = O.port_ds(x, p, s, opt, 1, amb)
    assert gk.counters == rk.counters
    assert max_rel(gk.dense, rk.dense) <= TOL
    check_peaks(gk.peak_index, gk.peak_value, rk.peak_index, rk.peak_value, value_at=lambda i: rk.dense[i])


@pytest.mark.parametrize("path", [A.FINE_FFT_CUDA_CORE, A.FINE_TC_DENSE])
def test_order_four_both_paths_vs_oracle(path):
    """P = 4 (three fine axes: the outer fine loop spans two of them) on the
    TMEM FFT path and the tensor path."""
    M, K = 256, 64
    p = RadarParams.create(8 * 100e6, 100e6, 50e6, 2000.0, M, K)
    s = build_dual_scale(p, 4, [Bounds(-20.0, 20.0), Bounds(-4.0, 4.0), Bounds(-1.0, 1.0), Bounds(-0.3, 0.3)],
                         [0.4, 0.2, 0.2, 0.2], RangeRoi(4, K - 5))
    x = scene.to_complex64_roundtrip(scene.add_noise(
        scene.synthesize_cube(p, [(0.05, [24 * p.delta_R(), 5.0, 1.0, 0.2, 0.05])]), 1.0 / K, 44))
    opt = DetectorOptions(retain_threshold=0.3 * M, keep_dense=True, fine_path=path)
    e = Engine(p, s, opt=opt)
    assert e.fine_path()[0] == path
    e.run_host(x)
    gm = e.result()
    e.close()
    rm = O.port_ds(x, p, s, opt)
    assert gm.counters == rm.counters
    assert max_rel(gm.dense, rm.dense) <= TOL
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])


@pytest.mark.parametrize("path", [A.FINE_FFT_CUDA_CORE, A.FINE_TC_DENSE])
@pytest.mark.parametrize("roi", [(0, 0), (63, 63), (60, 63), (0, 63)])
def test_roi_edges_both_paths(path, roi):
    """One-row and edge ROIs (tile tails of the tensor path, single-row CTAs of
    the FFT path) against the oracle, with fine grids of several cells."""
    M, K = 512, 64
    p = RadarParams.create(8 * 100e6, 100e6, 50e6, 2000.0, M, K)
    s = build_dual_scale(p, 2, [Bounds(-30.0, 30.0), Bounds(-6.0, 6.0)], [0.5, 0.5], RangeRoi(*roi))
    x = scene.to_complex64_roundtrip(scene.add_noise(
        scene.synthesize_cube(p, [(0.05, [(roi[0] + 0) * p.delta_R(), 5.0, 1.0])]), 1.0 / K, 7 + roi[0]))
    opt = DetectorOptions(retain_threshold=0.2 * M, keep_dense=True, fine_path=path)
    e = Engine(p, s, opt=opt)
    e.run_host(x)
    gm = e.result()
    e.close()
    rm = O.port_ds(x, p, s, opt)
    assert gm.counters == rm.counters and gm.peak_index.size == roi[1] - roi[0] + 1
    assert max_rel(gm.dense, rm.dense) <= TOL
    check_candidates(gm.cand_index, gm.cand_value, rm.cand_index, rm.cand_value, 0.2 * M)
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])


CASES_2K = [  # M = 2048 (fine_fft_tm2k_kernel: radix-2 split onto two 1024-point halves)
    (1, [(-10.0, 10.0)], [1.0]),
    (2, [(-10.0, 10.0), (-1.0, 1.0)], [0.5, 0.5]),
    (3, [(-6.0, 6.0), (-0.6, 0.6), (-0.1, 0.1)], [0.4, 0.3, 0.3]),
]


@pytest.mark.parametrize("P,bounds,alpha", CASES_2K)
def test_tm2k_fft_dense_vs_oracle(P, bounds, alpha):
    p, s, x = _setup(2048, P, bounds, alpha)
    retain = 0.3 * 2048.0
    opt = DetectorOptions(retain_threshold=retain, keep_dense=True)
    e = Engine(p, s, opt=opt)
    assert e.fine_path()[0] == A.FINE_FFT_CUDA_CORE
    e.run_host(x)
    gm = e.result()
    e.close()
    rm = O.port_ds(x, p, s, opt)
    assert gm.counters == rm.counters
    assert max_rel(gm.dense, rm.dense) <= TOL
    check_candidates(gm.cand_index, gm.cand_value, rm.cand_index, rm.cand_value, retain)
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])


@pytest.mark.parametrize("fc_over_fs", [150.0, 800.0])
def test_tm2k_wide_window_vs_oracle(fc_over_fs):
    """Doppler windows of 77 and ~400 bins (the NB = 3 and NB = 6 pruned
    second passes over both half axes), candidates and per-cell peaks."""
    M, K = 2048, 64
    fs = 20e6
    p = RadarParams.create(fc_over_fs * fs, fs, fs, 1000.0, M, K)
    s = build_dual_scale(p, 2, [Bounds(-15.0, 15.0), Bounds(-1.0, 1.0)], [0.5, 0.5], RangeRoi(20, 27))
    x = scene.to_complex64_roundtrip(scene.add_noise(
        scene.synthesize_cube(p, [(0.02, [23 * p.delta_R(), 11.0, 0.2])]), 1.0 / K, 2048 + int(fc_over_fs)))
    retain = 0.25 * M
    opt = DetectorOptions(retain_threshold=retain)
    e = Engine(p, s, opt=opt)
    assert e.fine_path()[0] == A.FINE_FFT_CUDA_CORE
    e.run_host(x)
    gm = e.result()
    e.close()
    rm = O.port_ds(x, p, s, opt)
    assert gm.counters == rm.counters and gm.argmax == rm.argmax
    check_candidates(gm.cand_index, gm.cand_value, rm.cand_index, rm.cand_value, retain)
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value)


def test_tm2k_full_axis_path_choice():
    """DS-KT-MFP keeps the whole Doppler axis: at M = 2048 AUTO runs the tensor
    path and an explicit CUDA-core request fails at engine creation."""
    M, K = 2048, 64
    p = RadarParams.create(8 * 100e6, 100e6, 50e6, 2000.0, M, K)
    s = build_dual_scale(p, 2, [Bounds(-10.0, 10.0), Bounds(-1.0, 1.0)], [0.5, 0.5], RangeRoi(2, K - 3))
    amb = build_ambiguity(p, Bounds(-1.6 * p.Va(), 1.6 * p.Va()))
    e = Engine(p, s, 1, amb, DetectorOptions())
    assert e.fine_path()[0] == A.FINE_TC_DENSE
    e.close()
    with pytest.raises(ValueError):
        Engine(p, s, 1, amb, DetectorOptions(fine_path=A.FINE_FFT_CUDA_CORE))
