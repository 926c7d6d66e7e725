"""GPU parity of the tcgen05 fine path (K2a, fine_tc.cuh) through the C-ABI.

3-term fp16 split (LTCI_FINE_TC_DENSE): same 1e-3 contract as the FFT path
(its measured error is ~1e-7).  1-term (LTCI_FINE_TC_FAST): max-normalised
magnitude error <= 1e-3 and argmax identical or a tie within 1e-3."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import AmbiguitySpace, DetectorOptions, ds_grft, ds_kt_mfp
from paper_2403_06788_b200 import _cabi as A, scene
from paper_2403_06788_b200.configs import baseline_space, config
from paper_2403_06788_b200.model import Bounds, RadarParams, RangeRoi, build_ambiguity, build_dual_scale

from helpers import TOL, check_candidates, check_peaks, cube, load, max_rel, radar, space

pytestmark = pytest.mark.gpu

TC = A.FINE_TC_DENSE


def test_tc_small_grft_golden():
    g = load("small_grft.npz")
    p = radar(g)
    s = space(g, p)
    gm = ds_grft(cube(g), p, s, DetectorOptions(retain_threshold=float(g["retain"]), keep_dense=True, fine_path=TC))
    ref = g["dense"]
    assert max_rel(gm.dense, ref) <= 1e-5
    assert np.abs(gm.dense - ref).max() / np.abs(ref).max() <= 1e-5
    assert gm.counters == tuple(int(c) for c in g["counters"])
    assert gm.argmax == int(g["argmax"])
    check_candidates(gm.cand_index, gm.cand_value, g["cand_index"], g["cand_value"], float(g["retain"]))
    check_peaks(gm.peak_index, gm.peak_value, g["peak_index"], g["peak_value"], value_at=lambda i: ref[i])


def test_tc_small_kt_golden():
    g = load("small_kt.npz")
    p = radar(g)
    s = space(g, p)
    amb = AmbiguitySpace(int(g["amb"][0]), int(g["amb"][1]))
    gm = ds_kt_mfp(cube(g), p, amb, s,
                   DetectorOptions(retain_threshold=float(g["retain"]), keep_dense=True, fine_path=TC))
    ref = g["dense"]
    assert np.abs(gm.dense - ref).max() / np.abs(ref).max() <= 1e-5
    check_peaks(gm.peak_index, gm.peak_value, g["peak_index"], g["peak_value"], value_at=lambda i: ref[i])


def test_tc_c0_golden():
    g = load("c0.npz")
    w = config(0)
    x = cube(g)
    gamma = float(g["gamma"])
    gm = ds_grft(x, w.params, w.space, DetectorOptions(retain_threshold=gamma, fine_path=TC))
    assert gm.counters == tuple(int(c) for c in g["counters"])
    assert gm.argmax == int(g["argmax"])
    check_candidates(gm.cand_index, gm.cand_value, g["cand_index"], g["cand_value"], gamma)
    assert np.array_equal(gm.peak_index, g["peak_index"])
    rel = np.abs(np.abs(gm.peak_value) - np.abs(g["peak_value"])) / np.abs(g["peak_value"])
    assert rel.max() <= 1e-5


@pytest.mark.parametrize("K,M,ratio,order", [(64, 32, 4.0, 2), (128, 64, 8.0, 2), (256, 128, 16.0, 2),
                                             (128, 64, 8.0, 3), (64, 32, 4.0, 1)])
def test_tc_matches_fft_path_and_port(K, M, ratio, order):
    p = RadarParams.create(ratio * 100e6, 100e6, 50e6, 2000.0, M, K)
    b = [Bounds(-30.0, 30.0), Bounds(-8.0, 8.0), Bounds(-20.0, 20.0)][:order]
    al = {1: [1.0], 2: [0.5, 0.5], 3: [0.4, 0.3, 0.3]}[order]
    s = build_dual_scale(p, order, b, al, RangeRoi(3, K - 5))
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.3, [K / 2 * p.delta_R(), 11.0, 2.5, 1.0])]), 1.0 / K, K))
    opt = DetectorOptions(retain_threshold=0.5, keep_dense=True, fine_path=TC)
    gm = ds_grft(x, p, s, opt)
    rm = O.port_ds(x, p, s, opt)
    assert gm.counters == rm.counters
    assert np.abs(gm.dense - rm.dense).max() / np.abs(rm.dense).max() <= 1e-5
    check_candidates(gm.cand_index, gm.cand_value, rm.cand_index, rm.cand_value, 0.5)
    check_peaks(gm.peak_index, gm.peak_value, rm.peak_index, rm.peak_value, value_at=lambda i: rm.dense[i])


def test_tc_fast_within_contract():
    g = load("c0.npz")
    w = config(0)
    x = cube(g)
    gamma = float(g["gamma"])
    gm = ds_grft(x, w.params, w.space, DetectorOptions(retain_threshold=gamma, fine_path=A.FINE_TC_FAST))
    ref_max = abs(complex(g["argmax_value"]))
    rel = np.abs(np.abs(gm.peak_value) - np.abs(g["peak_value"])) / ref_max
    assert rel.max() <= TOL
    assert abs(abs(gm.argmax_value) - ref_max) <= TOL * ref_max


def test_fine_path_selection_is_honoured():
    """Explicit FFT / tensor requests run that path; AUTO follows the measured rule."""
    from paper_2403_06788_b200.detectors import Engine
    w = config(0)
    for req, want in ((A.FINE_FFT_CUDA_CORE, A.FINE_FFT_CUDA_CORE), (A.FINE_TC_DENSE, A.FINE_TC_DENSE),
                      (A.FINE_TC_FAST, A.FINE_TC_FAST), (A.FINE_AUTO, A.FINE_FFT_CUDA_CORE)):
        e = Engine(w.params, w.space, opt=DetectorOptions(fine_path=req))
        assert e.fine_path()[0] == want
        e.close()
    w3 = config(3)
    e = Engine(w3.params, w3.space, 1, w3.amb, DetectorOptions())
    assert e.fine_path()[0] == A.FINE_FFT_CUDA_CORE  # full Doppler axis -> FFT
    e.close()
    w1 = config(1)
    e = Engine(w1.params, w1.space, opt=DetectorOptions())
    assert e.fine_path()[0] == A.FINE_FFT_CUDA_CORE  # M = 1024: TMEM-resident FFT path
    e.close()
    w2 = config(2)
    e = Engine(w2.params, w2.space, opt=DetectorOptions())
    assert e.fine_path()[0] == A.FINE_FFT_CUDA_CORE  # M = 2048, D = 151: radix-2 split FFT path
    e.close()
