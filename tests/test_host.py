"""CPU: host-side plan logic and the C-ABI boundary (no GPU compute)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2403_06788_b200 import _lib, configs
from paper_2403_06788_b200.model import (Bounds, ConditionViolated, RadarParams, RangeRoi, build_ambiguity,
                                         build_dual_scale, split_velocity, step_sizes)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def mmwave():
    return RadarParams.create(28e9, 491.52e6, 400e6, 1905.0, 512, 2048)


def test_step_size_kats():
    # proj/tests/test_search_space.cpp:10-65
    p = mmwave()
    s1 = step_sizes(p, 1, [1.0])
    assert abs(s1.rm[0] - 1.1355) < 1.1355e-4
    assert abs(s1.dfm[0] - 0.019933) < 0.019933e-4
    ds = build_dual_scale(p, 2, [Bounds(-50.0, 50.0), Bounds(-30.0, 30.0)], [0.5, 0.5], RangeRoi.full(p))
    assert abs(ds.kappa - 0.992857) < 1e-5
    small = RadarParams.create(28e9, 491.52e6, 400e6, 1905.0, 32, 2048)
    with pytest.raises(ConditionViolated):
        build_dual_scale(small, 2, [Bounds(-50.0, 50.0), Bounds(-30.0, 30.0)], [0.5, 0.5], RangeRoi.full(small))
    with pytest.raises(ValueError):
        step_sizes(p, 2, [0.5, 0.4])


def test_velocity_split_and_ambiguity():
    p = mmwave()
    q, base = split_velocity(20.0, p)
    assert q == 2 and abs(base + 0.4107) < 1e-3
    a = build_ambiguity(p, Bounds(10.0, 30.0))
    assert (a.q_min, a.q_max) == (1, 3)


@pytest.mark.parametrize("i,coarse,fine,D,H", [
    (0, [11, 1], [151, 151], 151, 128415232),
    (1, [83, 4], [151, 151], 151, 15503220736),
    (2, [165, 12, 2], [151, 151, 451], 151, 166795976540160),
    (4, [35, 2], [151, 151], 151, 1634375680),
])
def test_baseline_configs_match_survey_appendix_b(i, coarse, fine, D, H):
    w = configs.config(i)
    assert [g.count for g in w.space.coarse] == coarse
    assert [g.count for g in w.space.fine] == fine
    assert configs.doppler_window(w.params, w.space)[1] == D
    assert w.hypotheses() == H


def test_c3_keystone_config():
    w = configs.config(3)
    assert w.params.K_valid == 1638 and w.amb.count() == 13
    assert w.space.coarse[1].count == 4 and w.space.fine[1].count == 121
    assert w.hypotheses() == 13195280384


def test_cabi_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "ltci_cuda.h")).read()
    declared = set(re.findall(r"\b(ltci_(?:cuda|engine)_[a-z_0-9]+)\s*\(", header))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    lib = _lib.load()  # loads without a GPU
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.ltci_cuda_version() >= 100


def test_dropin_exports_reference_mangled_symbols():
    nm = os.popen(f"nm -D {_lib.DROPIN_PATH}").read()
    # proj/include/ltci/detectors.hpp:42-48 mangled names
    assert "_ZN4ltci7ds_grftERKNS_13FreqPulseCubeERKNS_14DualScaleSpaceERKNS_15DetectorOptionsE" in nm
    assert ("_ZN4ltci9ds_kt_mfpERKNS_13FreqPulseCubeERKNS_14AmbiguitySpaceERKNS_14DualScaleSpaceE"
            "RKNS_15DetectorOptionsE") in nm


def test_no_device_fails_loudly():
    """Without a GPU the product raises instead of falling back to a CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_06788_b200 import ds_grft
    w = configs.config(0)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        ds_grft(np.zeros((w.params.M, w.params.K), complex), w.params, w.space)


def test_threshold_host_arithmetic():
    from paper_2403_06788_b200 import detection_threshold
    p = RadarParams.create(28e9, 491.52e6, 400e6, 1905.0, 512, 1024)
    assert abs(detection_threshold(p, 1.0, 1e-4) - 2197.3) < 2197.3 * 2e-4
    with pytest.raises(ValueError):
        detection_threshold(p, 1.0, 0.0)
