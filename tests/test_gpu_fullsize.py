"""Parity at BASELINE full sizes through size-independent properties.

Every config is run end to end on the GPU at its BASELINE shape (C2 on a
1x1 coarse slice, as in bench.py: one full C2 step is ~1.5 h of tensor work)
and checked by properties that do not need a full-size CPU run (K1, the
coarse stage, is also checked against the oracle at every row and pulse):
  * the two independent fine-stage formulations (tcgen05 3-term contraction,
    CUDA-core chirp + FFT) agree: per-range-cell peaks (indices identical
    except ties), candidates (identical except near-threshold), argmax;
  * at sampled range cells the GPU peak equals the FP64 oracle evaluated at
    that cell (helpers.oracle_cell) within the contract (1e-3);
  * the strongest injected target is detected at its true cell.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2403_06788_b200 import _cabi as A
from paper_2403_06788_b200 import scene
from paper_2403_06788_b200.configs import config, sliced
from paper_2403_06788_b200.detection import extract_detections
from paper_2403_06788_b200.detectors import Engine, detection_threshold
from paper_2403_06788_b200.model import DetectorOptions

from helpers import TOL, check_candidates, oracle_cell

pytestmark = pytest.mark.gpu


def _run(w, x, gamma, path):
    e = Engine(w.params, w.space, w.variant, w.amb, DetectorOptions(retain_threshold=gamma, fine_path=path))
    e.run_host(x)
    m = e.result()
    e.close()
    return m


def _cross_and_oracle(w, x, gamma, samples=8, seed=0):
    tc = _run(w, x, gamma, A.FINE_TC_DENSE)
    ff = _run(w, x, gamma, A.FINE_FFT_CUDA_CORE)
    assert tc.counters == ff.counters
    # peaks: identical except ties between the two formulations
    rel = np.abs(np.abs(tc.peak_value) - np.abs(ff.peak_value)) / np.abs(ff.peak_value)
    assert rel.max() <= 1e-4
    differ = np.nonzero(tc.peak_index != ff.peak_index)[0]
    assert differ.size <= max(3, tc.peak_index.size // 200)
    check_candidates(tc.cand_index, tc.cand_value, ff.cand_index, ff.cand_value, gamma, tol=1e-4)
    # oracle at sampled range cells (and at every row where the paths disagree)
    rng = np.random.default_rng(seed)
    rows = sorted(set(rng.choice(tc.peak_index.size, size=samples, replace=False).tolist()) | set(differ[:4].tolist()))
    for r in rows:
        for m in (tc, ff):
            ref = oracle_cell(x, w.params, w.space, int(m.peak_index[r]), w.variant, w.amb)
            assert abs(abs(m.peak_value[r]) - abs(ref)) <= TOL * abs(ref), (r, m.peak_index[r])
    ref = oracle_cell(x, w.params, w.space, int(tc.argmax), w.variant, w.amb)
    assert abs(abs(tc.argmax_value) - abs(ref)) <= TOL * abs(ref)
    return tc


def _strongest_target_found(w, m, gamma):
    amp, coeffs = max(w.targets, key=lambda t: abs(t[0]))
    dets = extract_detections(m, gamma)
    p = w.params
    ok = [d for d in dets if abs(d.estimate[0] - coeffs[0]) <= 1.01 * p.delta_R()
          and abs(d.estimate[1] - coeffs[1]) <= 2.01 * p.Va() / p.M]
    assert ok, (coeffs, [d.estimate[:3] for d in dets[:5]])


def test_c1_full_size():
    w = config(1)
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    tc = _cross_and_oracle(w, x, gamma, samples=10, seed=1)
    _strongest_target_found(w, tc, gamma)


def test_c2_full_size_coarse_slice():
    w = sliced(config(2), 1, 1)
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    # M = 2048: the tcgen05 contraction and the radix-2-split CUDA-core FFT
    # (fine_fft_tm2k_kernel) against each other and the oracle
    _cross_and_oracle(w, x, gamma, samples=8, seed=2)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_coarse_stage_every_row_full_shapes(cfg):
    """K1 alone at every BASELINE shape (K = 1024, 2048, 4096; GRFT and KT
    ramps): the mgift output of two coarse cells -- the grid's first and a
    middle one -- against the FP64 oracle at EVERY range bin and pulse, so a
    K1 defect cannot hide between the sampled rows of the end-to-end checks."""
    import oracle as O
    from paper_2403_06788_b200 import mgift
    w = config(cfg)
    p, s = w.params, w.space
    x = scene.to_complex64_roundtrip(w.cube())
    if w.variant == 0:
        mids = [[g.value(0) for g in s.coarse], [g.value(g.count // 2) for g in s.coarse]]
    else:
        g2 = s.coarse[1]
        mids = [[float(w.amb.q_min), g2.value(0)], [float((w.amb.q_min + w.amb.q_max) // 2), g2.value(g2.count // 2)]]
    for ct in mids:
        got = mgift(x, p, ct, w.variant)
        ref = O.port_mgift(x, p, ct, w.variant)
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err < 2e-5, (ct, err)


def test_c3_full_size_kt():
    w = config(3)
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    _cross_and_oracle(w, x, gamma, samples=6, seed=3)


def test_c4_one_cpi_full_size():
    w = config(4)
    x = scene.to_complex64_roundtrip(w.cube(cpi=5))
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    _cross_and_oracle(w, x, gamma, samples=6, seed=4)


@pytest.mark.parametrize("cfg", [1, 0])
def test_range_shards_merge_bit_exactly(cfg):
    """C1 (and C0, whose small grid splits the inner fine axis across CTAs) on
    the TMEM-resident FFT path split into 3 uneven range-cell shards (the
    multi-GPU partition, one engine per GPU) merges to the 1-GPU map
    bit-exactly; parallel.merge_rank_maps is the merge the NCCL gather feeds."""
    from paper_2403_06788_b200.parallel import merge_rank_maps, shard_rows
    w = config(cfg)
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    opt = DetectorOptions(retain_threshold=gamma)
    full = Engine(w.params, w.space, opt=opt)
    assert full.fine_path()[0] == A.FINE_FFT_CUDA_CORE
    full.run_host(x)
    a = full.result()
    full.close()
    R = w.space.roi.count()
    maps = []
    for rank in range(3):
        lo, hi = shard_rows(R, 3, rank)
        e = Engine(w.params, w.space, opt=opt, row_begin=lo, row_end=hi)
        e.run_host(x)
        maps.append(e.result())
        e.close()
    m = merge_rank_maps(maps)
    assert np.array_equal(m.peak_index, a.peak_index) and np.array_equal(m.peak_value, a.peak_value)
    assert np.array_equal(m.cand_index, a.cand_index) and np.array_equal(m.cand_value, a.cand_value)
    assert m.argmax == a.argmax


@pytest.mark.parametrize("cfg", [1, 0])
def test_coarse_shards_merge_bit_exactly(cfg):
    """The coarse-cell partition (what bench.py runs for N > 1): 3 engines over
    disjoint coarse-cell slices, every ROI row; their raw peak slots merged on
    the device (ltci_cuda_merge_peaks) equal the 1-GPU slots bit for bit, the
    candidate union equals the 1-GPU candidates, the host merge agrees.
    Both run the TMEM FFT path (C0 with its fine-axis split)."""
    import ctypes as C

    import torch
    from paper_2403_06788_b200 import _lib
    from paper_2403_06788_b200.parallel import merge_coarse_maps, shard_coarse
    w = config(cfg)
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = detection_threshold(w.params, w.sigma2, 1e-6)
    opt = DetectorOptions(retain_threshold=gamma)
    full = Engine(w.params, w.space, opt=opt)
    full.run_host(x)
    a = full.result()
    ptr, n = full.peaks_device()
    ref_slots = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    from bench import _CAI  # __cuda_array_interface__ view of a device pointer
    ref_slots.copy_(torch.as_tensor(_CAI(ptr, (n, 4), "<i4"), device="cuda"))
    cells = int(np.prod([g.count for g in w.space.coarse]))
    world = 3
    slots = torch.empty((world, n, 4), dtype=torch.int32, device="cuda")
    maps = []
    for rank in range(world):
        lo, hi = shard_coarse(cells, world, rank)
        e = Engine(w.params, w.space, opt=opt, coarse_begin=lo, coarse_end=hi)
        e.run_host(x)
        maps.append(e.result())
        p2, n2 = e.peaks_device()
        assert n2 == n
        slots[rank].copy_(torch.as_tensor(_CAI(p2, (n, 4), "<i4"), device="cuda"))
        torch.cuda.synchronize()
        e.close()
    merged = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    lib = _lib.load()
    _lib.raise_for(lib.ltci_cuda_merge_peaks(C.c_void_p(slots.data_ptr()), world, n, C.c_void_p(merged.data_ptr()),
                                             None), lib)
    torch.cuda.synchronize()
    assert torch.equal(merged, ref_slots)
    m = merge_coarse_maps(maps, a.counters)
    assert np.array_equal(m.cand_index, a.cand_index) and np.array_equal(m.cand_value, a.cand_value)
    assert np.array_equal(m.peak_index, a.peak_index) and m.argmax == a.argmax
    full.close()
