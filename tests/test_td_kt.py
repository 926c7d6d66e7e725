"""td_grft (rounded-trajectory time-domain search) and kt_mfp (single-scale
keystone matched filter): the two remaining detectors of the reference's
proj/include/ltci/detectors.hpp.

CPU: our C restatement (oracle/ds_oracle.c oracle_td_grft / oracle_kt_mfp)
against the reference's golden maps (tests/golden/td_kt.npz) and against the
reference run live, including the Error trajectory policy.  GPU: the C-ABI
(ltci_cuda_td_grft / ltci_cuda_kt_mfp) against the goldens and the oracle on
more shapes -- counters and axes exact, dense complex maps and candidates to
TOL, argmax identical except ties."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import scene
from paper_2403_06788_b200.model import (AmbiguitySpace, Bounds, DetectorOptions, RadarParams, RangeRoi,
                                         build_ambiguity, build_single_scale)

from helpers import TOL, check_candidates, load, radar
from test_fd_grft import single

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="reference not built (oracle/_ref)")

TD_CASES = [("td2_zero_", "s2_", 0), ("td2_wrap_", "s2_", 1), ("td1_zero_", "s1_", 0)]


def _check_against_golden(m, g, pre, retain, tol):
    assert m.counters == tuple(int(c) for c in g[pre + "counters"])
    assert [[a.role, a.order, a.size] for a in m.axes] == g[pre + "axes"].tolist()
    ref = g[pre + "dense"]
    assert m.dense_stored and m.dense.shape == ref.shape
    assert np.abs(m.dense - ref).max() / np.abs(ref).max() <= tol
    check_candidates(m.cand_index, m.cand_value, g[pre + "cand_index"], g[pre + "cand_value"], retain, tol=max(tol, 1e-12))
    ref_max = abs(complex(g[pre + "argmax_value"]))
    if m.argmax != int(g[pre + "argmax"]):  # a tie within tol
        assert abs(abs(ref[int(m.argmax)]) - ref_max) <= tol * ref_max
    assert abs(abs(m.argmax_value) - ref_max) <= max(tol, 1e-12) * ref_max


# ------------------------------------------------------------------ CPU ---
@pytest.mark.parametrize("pre,sp,policy", TD_CASES)
def test_oracle_td_grft_matches_reference_golden(pre, sp, policy):
    g = load("td_kt.npz")
    p = radar(g)
    s = single(g, p, sp)
    retain = float(g["td_retain"])
    m = O.port_td(g["range"].astype(np.complex128), p, s,
                  DetectorOptions(retain_threshold=retain, keep_dense=True, trajectory=policy))
    _check_against_golden(m, g, pre, retain, 1e-12)
    assert m.argmax == int(g[pre + "argmax"])


def test_oracle_kt_mfp_matches_reference_golden():
    g = load("td_kt.npz")
    p = radar(g)
    s = single(g, p, "sk_")
    amb = AmbiguitySpace(int(g["amb"][0]), int(g["amb"][1]))
    retain = float(g["kt_retain"])
    m = O.port_kt(g["freq"].astype(np.complex128), p, amb, s, DetectorOptions(retain_threshold=retain, keep_dense=True))
    _check_against_golden(m, g, "kt_", retain, 1e-12)
    assert m.argmax == int(g["kt_argmax"])


@needs_ref
def test_oracle_td_error_policy_and_live_reference():
    """TrajectoryPolicy::Error raises in both; a larger live case agrees exactly."""
    p = RadarParams.create(3e9, 20e6, 20e6, 1000.0, 64, 128)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((p.M, p.K), complex), 1.0, 17))
    s = build_single_scale(p, 2, [Bounds(-400.0, 400.0), Bounds(-30.0, 30.0)], [0.5, 0.5], RangeRoi(0, p.K - 1))
    with pytest.raises(IndexError):
        O.ref_td(x, p, s, DetectorOptions(trajectory=2))
    with pytest.raises(IndexError):
        O.port_td(x, p, s, DetectorOptions(trajectory=2))
    for pol in (0, 1):
        opt = DetectorOptions(retain_threshold=20.0, keep_dense=True, trajectory=pol)
        a, b = O.ref_td(x, p, s, opt), O.port_td(x, p, s, opt)
        assert a.counters == b.counters and a.argmax == b.argmax
        assert np.abs(a.dense - b.dense).max() <= 1e-12 * np.abs(a.dense).max()
        assert np.array_equal(a.cand_index, b.cand_index)
    # a space whose trajectories stay inside: the Error policy returns the ZeroOutside map
    inner = build_single_scale(p, 1, [Bounds(-20.0, 20.0)], [1.0], RangeRoi(40, 80))
    a = O.port_td(x, p, inner, DetectorOptions(keep_dense=True, trajectory=2))
    b = O.port_td(x, p, inner, DetectorOptions(keep_dense=True, trajectory=0))
    assert np.array_equal(a.dense, b.dense)


# ------------------------------------------------------------------ GPU ---
@pytest.mark.gpu
@pytest.mark.parametrize("pre,sp,policy", TD_CASES)
def test_td_grft_golden(pre, sp, policy):
    from paper_2403_06788_b200 import td_grft
    g = load("td_kt.npz")
    p = radar(g)
    s = single(g, p, sp)
    retain = float(g["td_retain"])
    m = td_grft(g["range"].astype(np.complex128), p, s,
                DetectorOptions(retain_threshold=retain, keep_dense=True, trajectory=policy))
    assert m.kind == 1
    _check_against_golden(m, g, pre, retain, TOL)


@pytest.mark.gpu
def test_kt_mfp_golden():
    from paper_2403_06788_b200 import kt_mfp
    g = load("td_kt.npz")
    p = radar(g)
    s = single(g, p, "sk_")
    amb = AmbiguitySpace(int(g["amb"][0]), int(g["amb"][1]))
    retain = float(g["kt_retain"])
    m = kt_mfp(g["freq"].astype(np.complex128), p, amb, s, DetectorOptions(retain_threshold=retain, keep_dense=True))
    assert m.kind == 2
    _check_against_golden(m, g, "kt_", retain, TOL)


@pytest.mark.gpu
def test_td_grft_errors_and_policies():
    from paper_2403_06788_b200 import td_grft
    p = RadarParams.create(3e9, 20e6, 20e6, 1000.0, 64, 128)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((p.M, p.K), complex), 1.0, 17))
    s = build_single_scale(p, 2, [Bounds(-400.0, 400.0), Bounds(-30.0, 30.0)], [0.5, 0.5], RangeRoi(0, p.K - 1))
    with pytest.raises(IndexError, match="trajectory leaves the cube"):
        td_grft(x, p, s, DetectorOptions(trajectory=2))
    inner = build_single_scale(p, 1, [Bounds(-20.0, 20.0)], [1.0], RangeRoi(40, 80))
    a = td_grft(x, p, inner, DetectorOptions(keep_dense=True, trajectory=2))
    b = td_grft(x, p, inner, DetectorOptions(keep_dense=True, trajectory=0))
    assert np.array_equal(a.dense, b.dense)
    other = RadarParams.create(p.fc * 2, p.fs, p.Br, p.PRF, p.M, p.K, p.K_valid)
    with pytest.raises(ValueError, match="different radar"):
        td_grft(x, other, s)
    from paper_2403_06788_b200 import kt_mfp
    with pytest.raises(ValueError, match="P = 2"):
        kt_mfp(x, p, AmbiguitySpace(0, 1), inner)


@pytest.mark.gpu
@pytest.mark.parametrize("K,M,P", [(16, 8, 1), (64, 300 // 4, 2), (128, 64, 2), (512, 256, 2), (2048, 64, 3),
                                   (8192, 16, 1)])
def test_td_grft_sizes_vs_oracle(K, M, P):
    """Every policy at several shapes (M not a multiple of the pulse tile, rows
    beyond one CTA column) against the C restatement."""
    from paper_2403_06788_b200 import td_grft
    M = 1 << (M.bit_length() - 1)
    p = RadarParams.create(3e9, 20e6, 18e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((M, K), complex), 1.0, K + M))
    T = p.T()
    b = [Bounds(-6 * p.delta_R() / T, 6 * p.delta_R() / T), Bounds(-2 * p.delta_R() / T ** 2, 2 * p.delta_R() / T ** 2),
         Bounds(-p.delta_R() / T ** 3, p.delta_R() / T ** 3)][:P]
    s = build_single_scale(p, P, b, [1.0 / P] * P, RangeRoi(min(2, K - 1), K - 1))
    # keep the single-threaded oracle in seconds: thin every axis to a few cells over the same span
    from paper_2403_06788_b200.model import Grid
    for q, want in enumerate((25, 9, 5)[:P]):
        gq = s.c[q]
        k = max(1, gq.count // want)
        s.c[q] = Grid(gq.start, gq.step * k, -(-gq.count // k))
    assert int(np.prod([gr.count for gr in s.c])) <= 4000
    for pol in (0, 1):
        opt = DetectorOptions(retain_threshold=1.5 * np.sqrt(M), keep_dense=True, trajectory=pol)
        ref = O.port_td(x, p, s, opt)
        got = td_grft(x, p, s, opt)
        assert got.counters == ref.counters
        assert np.abs(got.dense - ref.dense).max() / np.abs(ref.dense).max() <= TOL
        check_candidates(got.cand_index, got.cand_value, ref.cand_index, ref.cand_value, opt.retain_threshold)
        if got.argmax != ref.argmax:
            assert abs(abs(ref.dense[got.argmax]) - abs(ref.argmax_value)) <= TOL * abs(ref.argmax_value)


@pytest.mark.gpu
@pytest.mark.parametrize("K,M", [(64, 32), (256, 128), (1024, 256)])
def test_kt_mfp_sizes_vs_oracle(K, M):
    from paper_2403_06788_b200 import kt_mfp
    p = RadarParams.create(3e9, 25e6, 20e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.4, [K / 3 * p.delta_R(), 61.0, 2.5])]), 1.0 / K, K + M))
    T = p.T()
    s = build_single_scale(p, 2, [Bounds(-10.0, 10.0), Bounds(-3 * p.delta_R() / T ** 2, 3 * p.delta_R() / T ** 2)],
                           [0.5, 0.5], RangeRoi(K // 4, K // 4 + 23))
    if s.c[1].count > 12:
        from paper_2403_06788_b200.model import Grid
        g1 = s.c[1]
        k = -(-g1.count // 12)
        s.c[1] = Grid(g1.start, g1.step * k, max(1, g1.count // k))
    amb = build_ambiguity(p, Bounds(-1.2 * p.Va(), 1.2 * p.Va()))
    opt = DetectorOptions(retain_threshold=0.6 * M, keep_dense=True)
    ref = O.port_kt(x, p, amb, s, opt)
    got = kt_mfp(x, p, amb, s, opt)
    assert got.counters == ref.counters
    assert [[a.role, a.order, a.size] for a in got.axes] == [[a.role, a.order, a.size] for a in ref.axes]
    assert np.abs(got.dense - ref.dense).max() / np.abs(ref.dense).max() <= TOL
    check_candidates(got.cand_index, got.cand_value, ref.cand_index, ref.cand_value, opt.retain_threshold)
    if got.argmax != ref.argmax:
        assert abs(abs(ref.dense[got.argmax]) - abs(ref.argmax_value)) <= TOL * abs(ref.argmax_value)
