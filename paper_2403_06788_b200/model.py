"""Host-side domain model and search-space plan (Python mirror of the
reference types that cross the detector API).

Mirrors, with the same names and conventions:
  RadarParams        proj/include/ltci/radar_params.hpp:15-54, proj/src/radar_params.cpp:10-45
  Grid/Bounds/RangeRoi/StepSizes/DualScaleSpace/AmbiguitySpace
                     proj/include/ltci/search_space.hpp:11-90, proj/src/search_space.cpp:9-157
  DetectorOptions    proj/include/ltci/detectors.hpp:14-20
  DetectionMap       proj/include/ltci/detection.hpp:47-73, proj/src/detection.cpp:28-53
These are plan inputs and result containers; all arithmetic on the hot path
runs in the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _cabi as A

SPEED_OF_LIGHT = 3.0e8


def lround(x: float) -> int:
    """std::lround: nearest integer, halves away from zero."""
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


def is_power_of_two(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


class ConditionViolated(RuntimeError):
    """ltci::ConditionViolated (proj/include/ltci/common.hpp:17-20)."""


@dataclass
class RadarParams:
    fc: float = 0.0
    fs: float = 0.0
    Br: float = 0.0
    delta_f: float = 0.0
    PRF: float = 0.0
    M: int = 0
    K: int = 0
    K_valid: int = 0

    @property
    def lam(self) -> float:
        return SPEED_OF_LIGHT / self.fc

    def lambda_(self) -> float:
        return self.lam

    def T(self) -> float:
        return self.M / self.PRF

    def Va(self) -> float:
        return self.lam * self.PRF / 2.0

    def delta_R(self) -> float:
        return SPEED_OF_LIGHT / (2.0 * self.fs)

    def slow_time(self, m):
        return (np.asarray(m) + 1.0) / self.PRF

    def n0(self) -> int:
        return self.K

    def freq_of_row(self, r):
        r = np.asarray(r)
        return self.delta_f * np.where(r < self.K // 2, r, r - self.K)

    def row_of_index(self, g: int) -> int:
        return g if g >= 0 else g + self.K

    @staticmethod
    def create(fc, fs, br_nominal, prf, pulses, freq_bins, k_valid=0) -> "RadarParams":
        # RadarParams::create (proj/src/radar_params.cpp:10-28)
        p = RadarParams(fc=fc, fs=fs, PRF=prf, M=pulses, K=freq_bins)
        p.delta_f = fs / freq_bins
        if k_valid == 0:
            k_valid = lround(br_nominal / p.delta_f)
            if k_valid % 2:
                k_valid -= 1
            k_valid = max(k_valid, 2)
            k_valid = min(k_valid, freq_bins)
        p.K_valid = k_valid
        p.Br = p.delta_f * k_valid
        p.validate()
        return p

    def validate(self) -> None:
        # RadarParams::validate (proj/src/radar_params.cpp:30-45)
        if not (self.fc > 0 and self.fs > 0 and self.Br > 0 and self.PRF > 0 and self.M > 0 and self.K > 0):
            raise ValueError("RadarParams: fc, fs, Br, PRF, M, K must be positive")
        if not (is_power_of_two(self.M) and is_power_of_two(self.K)):
            raise ValueError("RadarParams: M and K must be powers of two")
        if self.fs < self.Br:
            raise ValueError("RadarParams: fs must be >= Br (Nyquist)")
        if self.K_valid <= 0 or self.K_valid > self.K or self.K_valid % 2:
            raise ValueError("RadarParams: K_valid must be even and in (0, K]")

    def to_c(self) -> A.CRadar:
        return A.CRadar(self.fc, self.fs, self.Br, self.delta_f, self.PRF, self.M, self.K, self.K_valid)

    @staticmethod
    def from_c(c: A.CRadar) -> "RadarParams":
        return RadarParams(c.fc, c.fs, c.Br, c.delta_f, c.PRF, c.M, c.K, c.K_valid)


@dataclass
class Grid:
    start: float = 0.0
    step: float = 0.0
    count: int = 0

    def value(self, i):
        return self.start + self.step * np.asarray(i, dtype=np.float64)

    def back(self) -> float:
        return float(self.value(self.count - 1))

    def nearest_index(self, x: float) -> int:
        if self.count <= 1:
            return 0
        return min(max(lround((x - self.start) / self.step), 0), self.count - 1)


@dataclass
class Bounds:
    lo: float = 0.0
    hi: float = 0.0


@dataclass
class RangeRoi:
    first: int = 0
    last: int = 0

    def count(self) -> int:
        return self.last - self.first + 1

    @staticmethod
    def full(p: RadarParams) -> "RangeRoi":
        return RangeRoi(0, p.K - 1)


@dataclass
class StepSizes:
    rm: List[float] = field(default_factory=list)
    dfm: List[float] = field(default_factory=list)
    alpha: List[float] = field(default_factory=list)

    def order(self) -> int:
        return len(self.rm)


def step_sizes(params: RadarParams, P: int, alpha: Sequence[float]) -> StepSizes:
    """step_sizes (proj/src/search_space.cpp:15-40)."""
    params.validate()
    if P < 1:
        raise ValueError("step_sizes: P must be >= 1")
    if len(alpha) != P:
        raise ValueError("step_sizes: alpha must have P entries")
    if any(not (a > 0.0) or a > 1.0 for a in alpha):
        raise ValueError("step_sizes: each alpha_p must be in (0, 1]")
    if abs(sum(alpha) - 1.0) > 1e-12:
        raise ValueError("step_sizes: alpha weights must sum to 1")
    s = StepSizes(alpha=list(alpha))
    tp = 1.0
    for p in range(1, P + 1):
        tp *= params.T()
        s.rm.append(alpha[p - 1] * SPEED_OF_LIGHT / (2.0 * params.fs * tp))
        s.dfm.append(alpha[p - 1] * SPEED_OF_LIGHT / (2.0 * params.fc * tp))
    return s


def span_grid(b: Bounds, step: float, cover: bool) -> Grid:
    """span_grid (proj/src/search_space.cpp:51-65)."""
    if not (b.hi >= b.lo):
        raise ValueError("grid bounds: min must be <= max")
    if not (step > 0):
        raise ValueError("grid step must be positive")
    span = b.hi - b.lo
    if cover:
        count = max(0, int(math.ceil(span / step - 0.5 - 1e-9))) + 1
    else:
        count = int(math.floor(span / step + 1e-9)) + 1
    if count < 1:
        raise ValueError("grid is empty")
    return Grid(b.lo, step, count)


def fine_grid(rm: float, dfm: float) -> Grid:
    """Fine grid spanning one coarse step (proj/src/search_space.cpp:97-106)."""
    half = int(math.floor(rm / dfm / 2.0 + 1e-9))
    return Grid(-dfm * half, dfm, 2 * half + 1)


@dataclass
class DualScaleSpace:
    params: RadarParams = field(default_factory=RadarParams)
    steps: StepSizes = field(default_factory=StepSizes)
    coarse: List[Grid] = field(default_factory=list)
    fine: List[Grid] = field(default_factory=list)
    kappa: float = 1.0
    roi: RangeRoi = field(default_factory=RangeRoi)

    def order(self) -> int:
        return len(self.coarse)

    def to_c(self) -> A.CDualSpace:
        c = A.CDualSpace()
        c.radar = self.params.to_c()
        c.order = self.order()
        if not 1 <= c.order <= A.MAX_ORDER:
            raise ValueError("dual-scale space: order must be in 1..4")
        for p in range(c.order):
            g, f = self.coarse[p], self.fine[p]
            c.coarse[p] = A.CGrid(g.start, g.step, g.count)
            c.fine[p] = A.CGrid(f.start, f.step, f.count)
            c.rm_step[p] = self.steps.rm[p] if p < len(self.steps.rm) else 0.0
            c.dfm_step[p] = self.steps.dfm[p] if p < len(self.steps.dfm) else 0.0
            c.alpha[p] = self.steps.alpha[p] if p < len(self.steps.alpha) else 0.0
        c.kappa = self.kappa
        c.roi_first, c.roi_last = self.roi.first, self.roi.last
        return c

    @staticmethod
    def from_c(c: A.CDualSpace) -> "DualScaleSpace":
        s = DualScaleSpace(params=RadarParams.from_c(c.radar), kappa=c.kappa, roi=RangeRoi(c.roi_first, c.roi_last))
        for p in range(c.order):
            s.coarse.append(Grid(c.coarse[p].start, c.coarse[p].step, c.coarse[p].count))
            s.fine.append(Grid(c.fine[p].start, c.fine[p].step, c.fine[p].count))
            s.steps.rm.append(c.rm_step[p])
            s.steps.dfm.append(c.dfm_step[p])
            s.steps.alpha.append(c.alpha[p])
        return s


def build_dual_scale(params: RadarParams, P: int, bounds: Sequence[Bounds], alpha: Sequence[float],
                     roi: RangeRoi) -> DualScaleSpace:
    """build_dual_scale (proj/src/search_space.cpp:82-109)."""
    if len(bounds) != P:
        raise ValueError("build_dual_scale: bounds must have P entries")
    ratio = (params.fc / params.fs) / params.M
    if ratio > 1.0:
        raise ConditionViolated(f"dual-scale space requires (fc/fs)/M <= 1, got {ratio:f}")
    s = DualScaleSpace(params=params, steps=step_sizes(params, P, alpha), roi=roi)
    s.kappa = 1.0 - params.Br / (2.0 * params.fc)
    for p in range(P):
        s.coarse.append(span_grid(bounds[p], s.steps.rm[p], True))
        s.fine.append(fine_grid(s.steps.rm[p], s.steps.dfm[p]))
    return s


@dataclass
class SingleScaleSpace:
    """SingleScaleSpace (proj/include/ltci/search_space.hpp:50-58)."""
    params: RadarParams = field(default_factory=RadarParams)
    steps: StepSizes = field(default_factory=StepSizes)
    c: List[Grid] = field(default_factory=list)
    roi: RangeRoi = field(default_factory=RangeRoi)

    def order(self) -> int:
        return len(self.c)

    def cells(self) -> int:
        n = 1
        for g in self.c:
            n *= g.count
        return n

    def to_c(self) -> A.CSingleSpace:
        c = A.CSingleSpace()
        c.radar = self.params.to_c()
        c.order = self.order()
        if not 1 <= c.order <= A.MAX_ORDER:
            raise ValueError("single-scale space: order must be in 1..4")
        for p in range(c.order):
            g = self.c[p]
            c.c[p] = A.CGrid(g.start, g.step, g.count)
            c.rm_step[p] = self.steps.rm[p] if p < len(self.steps.rm) else 0.0
            c.dfm_step[p] = self.steps.dfm[p] if p < len(self.steps.dfm) else 0.0
            c.alpha[p] = self.steps.alpha[p] if p < len(self.steps.alpha) else 0.0
        c.roi_first, c.roi_last = self.roi.first, self.roi.last
        return c

    @staticmethod
    def from_c(c: A.CSingleSpace) -> "SingleScaleSpace":
        s = SingleScaleSpace(params=RadarParams.from_c(c.radar), roi=RangeRoi(c.roi_first, c.roi_last))
        for p in range(c.order):
            s.c.append(Grid(c.c[p].start, c.c[p].step, c.c[p].count))
            s.steps.rm.append(c.rm_step[p])
            s.steps.dfm.append(c.dfm_step[p])
            s.steps.alpha.append(c.alpha[p])
        return s


def build_single_scale(params: RadarParams, P: int, bounds: Sequence[Bounds], alpha: Sequence[float],
                       roi: RangeRoi) -> SingleScaleSpace:
    """build_single_scale (proj/src/search_space.cpp:69-79): every order at its DFM step."""
    if len(bounds) != P:
        raise ValueError("build_single_scale: bounds must have P entries")
    s = SingleScaleSpace(params=params, steps=step_sizes(params, P, alpha), roi=roi)
    for p in range(P):
        s.c.append(span_grid(bounds[p], s.steps.dfm[p], False))
    return s


@dataclass
class AmbiguitySpace:
    q_min: int = 0
    q_max: int = 0

    def count(self) -> int:
        return self.q_max - self.q_min + 1

    def q_of(self, i: int) -> int:
        return self.q_min + i

    def to_c(self) -> A.CAmbiguity:
        return A.CAmbiguity(self.q_min, self.q_max)


def split_velocity(c1: float, params: RadarParams):
    """split_velocity (proj/src/search_space.cpp:147-155): (q, base)."""
    va = params.Va()
    q = int(math.floor(c1 / va + 0.5))
    return q, c1 - q * va


def build_ambiguity(params: RadarParams, velocity: Bounds) -> AmbiguitySpace:
    """build_ambiguity (proj/src/search_space.cpp:111-116)."""
    return AmbiguitySpace(split_velocity(velocity.lo, params)[0], split_velocity(velocity.hi, params)[0])


@dataclass
class DetectorOptions:
    retain_threshold: float = 0.0
    keep_dense: bool = False
    threads: int = 1
    keystone_taps: int = 8
    trajectory: int = 0
    # extensions
    fine_path: int = A.FINE_AUTO
    device: int = 0

    def to_c(self) -> A.COptions:
        return A.COptions(self.retain_threshold, int(self.keep_dense), self.threads, self.keystone_taps,
                          self.trajectory, self.fine_path, self.device)


@dataclass
class AxisDesc:
    role: int
    order: int
    size: int


DS_GRFT, DS_KT_MFP = A.DS_GRFT, A.DS_KT_MFP


@dataclass
class DetectionMap:
    """Statistic surface of one detector run (proj/include/ltci/detection.hpp:47-73).

    candidates: (index u64 array sorted ascending, complex128 values);
    peak_index / peak_value: per ROI range cell best (extension).
    """
    kind: int = DS_GRFT
    params: RadarParams = field(default_factory=RadarParams)
    axes: List[AxisDesc] = field(default_factory=list)
    counters: tuple = (0, 0, 0, 0)  # kt, mf, ifft, fft
    retain_threshold: float = 0.0
    cand_index: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    cand_value: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))
    dense_stored: bool = False
    dense: Optional[np.ndarray] = None
    argmax: int = 0
    argmax_value: complex = 0j
    dual: Optional[DualScaleSpace] = None
    amb: Optional[AmbiguitySpace] = None
    single: Optional[SingleScaleSpace] = None
    doppler_first: int = 0
    peak_index: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    peak_value: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))

    def cell_count(self) -> int:
        n = 1
        for a in self.axes:
            n *= a.size
        return n

    def decode(self, idx: int) -> List[int]:
        cell = [0] * len(self.axes)
        idx = int(idx)
        for i in range(len(self.axes) - 1, -1, -1):
            cell[i] = idx % self.axes[i].size
            idx //= self.axes[i].size
        return cell

    def encode(self, cell: Sequence[int]) -> int:
        idx = 0
        for a, c in zip(self.axes, cell):
            idx = idx * a.size + int(c)
        return idx

    def dense_at(self, cell: Sequence[int]) -> complex:
        if not self.dense_stored:
            raise RuntimeError("DetectionMap: dense storage not kept")
        return complex(self.dense[self.encode(cell)])

    @property
    def candidates(self):
        return list(zip(self.cand_index.tolist(), self.cand_value.tolist()))


def map_from_c(m: A.CDetectionMap, params: RadarParams) -> DetectionMap:
    """Copy a library-owned ltci_detection_map into Python-owned arrays."""
    out = DetectionMap(kind=m.kind, params=params, retain_threshold=m.retain_threshold,
                       doppler_first=m.doppler_first, argmax=int(m.argmax),
                       argmax_value=complex(m.argmax_value[0], m.argmax_value[1]))
    out.axes = [AxisDesc(m.axes[i].role, m.axes[i].order, m.axes[i].size) for i in range(m.n_axes)]
    out.counters = tuple(int(m.counters[i]) for i in range(4))
    n = int(m.n_candidates)
    if n:
        out.cand_index = np.ctypeslib.as_array(m.cand_index, shape=(n,)).copy()
        out.cand_value = np.ctypeslib.as_array(m.cand_value, shape=(2 * n,)).copy().view(np.complex128)
    out.dense_stored = bool(m.dense_stored)
    if out.dense_stored and m.dense_count:
        out.dense = np.ctypeslib.as_array(m.dense, shape=(2 * int(m.dense_count),)).copy().view(np.complex128)
    if m.n_rows and bool(m.peak_index):
        out.peak_index = np.ctypeslib.as_array(m.peak_index, shape=(m.n_rows,)).copy()
        out.peak_value = np.ctypeslib.as_array(m.peak_value, shape=(2 * m.n_rows,)).copy().view(np.complex128)
    return out


def cube_as_f64(cube: np.ndarray, params: RadarParams) -> np.ndarray:
    """Cube in the reference layout: complex (M, K) array, sample (k, m) at
    [m, k] == data[k + K*m] (proj/include/ltci/cube.hpp:10-11)."""
    a = np.ascontiguousarray(cube, dtype=np.complex128)
    if a.size != params.K * params.M:
        raise ValueError("detector: cube data size does not match K*M")
    return a.reshape(params.M, params.K)
