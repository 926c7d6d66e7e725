"""Batched Monte-Carlo detection probability.

Mirrors ltci::Scenario / PdPoint / PdCurve / run_pd (proj/include/ltci/bench.hpp:12-55,
proj/src/bench.cpp:72-124) and the signal-model entry points synthesize_cube /
add_noise (proj/src/signal_model.cpp:32-60).  All of it runs in the library:
synthesis and the splitmix64 / Box-Muller noise stream on the device, every
trial's search on the device, the success test and Wilson intervals in C++.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import _cabi as A
from . import _lib
from .model import Bounds, RadarParams, RangeRoi, cube_as_f64

Target = Tuple[complex, Sequence[float]]  # (amplitude, motion coefficients c0..cP)


@dataclass
class Scenario:
    params: RadarParams
    targets: List[Target]
    snr_db: List[float]
    trials: int = 200
    pfa: float = 1e-4
    sigma2: float = 1.0
    seed: int = 0
    detectors: List[int] = field(default_factory=lambda: [A.DS_GRFT])
    P: int = 2
    bounds: List[Bounds] = field(default_factory=list)
    alpha: List[float] = field(default_factory=list)
    roi: RangeRoi = field(default_factory=RangeRoi)
    keystone_taps: int = 8
    device: int = 0

    def to_c(self) -> A.CScenario:
        s = A.CScenario()
        s.radar = self.params.to_c()
        if not 1 <= len(self.targets) <= A.MAX_TARGETS:
            raise ValueError("run_pd: scenario needs a target")
        s.n_targets = len(self.targets)
        for i, t in enumerate(self.targets):
            s.targets[i] = _target(t)
        if len(self.snr_db) > A.MAX_SNR:
            raise ValueError("run_pd: at most 64 SNR points")
        s.n_snr = len(self.snr_db)
        for i, v in enumerate(self.snr_db):
            s.snr_db[i] = v
        s.trials, s.pfa, s.sigma2, s.seed = self.trials, self.pfa, self.sigma2, self.seed
        s.n_detectors = len(self.detectors)
        for i, d in enumerate(self.detectors):
            s.detectors[i] = d
        s.P = self.P
        for p in range(self.P):
            s.bound_lo[p], s.bound_hi[p] = self.bounds[p].lo, self.bounds[p].hi
            s.alpha[p] = self.alpha[p]
        s.roi_first, s.roi_last = self.roi.first, self.roi.last
        s.keystone_taps, s.device = self.keystone_taps, self.device
        return s


@dataclass
class PdPoint:
    snr_db: float
    pd: float
    trials: int
    ci_lo: float
    ci_hi: float


@dataclass
class PdCurve:
    kind: int
    points: List[PdPoint]


def _target(t: Target) -> A.CTarget:
    amp, coeffs = t
    c = A.CTarget()
    c.amp[0], c.amp[1] = complex(amp).real, complex(amp).imag
    if not 1 <= len(coeffs) <= A.MAX_ORDER + 1:
        raise ValueError("target: 1..5 motion coefficients")
    c.order = len(coeffs) - 1
    for i, v in enumerate(coeffs):
        c.c[i] = v
    return c


def synthesize(params: RadarParams, targets: Sequence[Target]) -> np.ndarray:
    """synthesize_cube on the device (FP64); complex (M, K)."""
    lib = _lib.load()
    arr = (A.CTarget * max(1, len(targets)))(*[_target(t) for t in targets])
    out = np.empty((params.M, params.K), np.complex128)
    r = params.to_c()
    _lib.raise_for(lib.ltci_cuda_synthesize(C.byref(r), len(targets), arr, out.ctypes.data_as(C.c_void_p)), lib)
    return out


def add_noise(cube: np.ndarray, params: RadarParams, sigma2: float, seed: int) -> np.ndarray:
    """add_noise on the device: the reference's GaussianRng stream, counter-based."""
    lib = _lib.load()
    data = cube_as_f64(cube, params)
    out = np.empty_like(data)
    r = params.to_c()
    _lib.raise_for(lib.ltci_cuda_add_noise(data.ctypes.data_as(C.c_void_p), C.byref(r), sigma2, seed,
                                           out.ctypes.data_as(C.c_void_p)), lib)
    return out


def run_pd(sc: Scenario) -> List[PdCurve]:
    """run_pd (proj/src/bench.cpp:72-124) with every trial on the GPU."""
    lib = _lib.load()
    c = sc.to_c()
    out = (A.CPdPoint * (max(1, len(sc.detectors) * len(sc.snr_db))))()
    _lib.raise_for(lib.ltci_cuda_run_pd(C.byref(c), out), lib)
    n = len(sc.snr_db)
    return [PdCurve(d, [PdPoint(o.snr_db, o.pd, o.trials, o.ci_lo, o.ci_hi) for o in out[i * n:(i + 1) * n]])
            for i, d in enumerate(sc.detectors)]
