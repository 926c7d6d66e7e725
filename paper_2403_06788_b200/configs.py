"""BASELINE.json workloads (configs[0..4]) realised in reference terms.

BASELINE's step rules (coarse v rho/T, coarse a 2 rho/T^2, coarse jerk
6 rho/T^3; fine v lambda/(2T), fine a lambda/T^2, fine jerk lambda/T^3)
imply alpha_p = 1 for every order, which the reference's step_sizes rejects
(it requires sum alpha = 1, proj/src/search_space.cpp:21-28).  The
DualScaleSpace is therefore hand-built with the
reference's own grid rules: coarse grids span_grid(cover=true) on c-unit
bounds (c2 = a/2, c3 = jerk/6), fine grids of +-half a coarse step
(proj/src/search_space.cpp:51-65,97-106), kappa = 1 - Br/(2 fc), ROI = all
range cells.  Inputs are seeded synthetic echoes (no public dataset exists
for this path): sigma^2 = 1/K per frequency bin so the range-compressed noise
is CN(0,1), |A1| from the per-pulse post-compression SNR
(proj/src/bench.cpp:25-27).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .model import (AmbiguitySpace, Bounds, DualScaleSpace, RadarParams, RangeRoi, StepSizes, build_ambiguity,
                    fine_grid, span_grid)
from . import scene

FC, PRF = 3.0e9, 1000.0


@dataclass
class Workload:
    name: str
    params: RadarParams
    space: DualScaleSpace
    variant: int = 0  # 0 ds_grft, 1 ds_kt_mfp
    amb: Optional[AmbiguitySpace] = None
    targets: List[Tuple[complex, List[float]]] = field(default_factory=list)
    sigma2: float = 0.0
    seed: int = 0
    cpis: int = 1
    description: str = ""

    def cube(self, cpi: int = 0, noise: bool = True) -> np.ndarray:
        seed = self.seed if self.cpis == 1 else scene.derive_seed(self.seed, cpi)
        tg = self.targets if self.cpis == 1 else cpi_targets(self, cpi)
        c = scene.synthesize_cube(self.params, tg)
        if noise and self.sigma2 > 0:
            c = scene.add_noise(c, self.sigma2, seed)
        return c

    def hypotheses(self) -> int:
        return hypotheses(self.params, self.space, self.variant, self.amb)

    def integrations(self) -> int:
        return self.hypotheses() * self.params.M


def doppler_window(params: RadarParams, space: DualScaleSpace) -> Tuple[int, int]:
    """(dop_first, dop_count) of ds_grft (proj/src/detectors.cpp:420-432)."""
    import math
    keep = int(math.ceil(space.kappa * space.steps.rm[0] / 2.0 / (params.Va() / params.M) - 1e-9))
    keep = min(keep, params.M // 2 - 1)
    return params.M // 2 - keep, 2 * keep + 1


def hypotheses(params: RadarParams, space: DualScaleSpace, variant: int = 0,
               amb: Optional[AmbiguitySpace] = None) -> int:
    R = space.roi.count()
    if variant == 0:
        coarse = int(np.prod([g.count for g in space.coarse]))
        fine = int(np.prod([g.count for g in space.fine[1:]])) if space.order() > 1 else 1
        return coarse * fine * R * doppler_window(params, space)[1]
    return amb.count() * space.coarse[1].count * space.fine[1].count * R * params.M


def baseline_space(params: RadarParams, bounds_c: Sequence[Tuple[float, float]],
                   roi: Optional[RangeRoi] = None) -> DualScaleSpace:
    """Hand-built space with BASELINE steps; bounds in reference c-units."""
    T, dR, lam = params.T(), params.delta_R(), params.lam
    P = len(bounds_c)
    fact = [1.0, 2.0, 6.0]
    rm = [dR / T ** p for p in range(1, P + 1)]
    dfm = [lam / (2.0 * T)] + [lam / (fact[p - 1] * T ** p) for p in range(2, P + 1)]
    s = DualScaleSpace(params=params, steps=StepSizes(rm=rm, dfm=dfm, alpha=[1.0] * P),
                       roi=roi or RangeRoi.full(params))
    s.kappa = 1.0 - params.Br / (2.0 * params.fc)
    for p in range(P):
        s.coarse.append(span_grid(Bounds(*bounds_c[p]), rm[p], True))
        s.fine.append(fine_grid(rm[p], dfm[p]))
    return s


def _draw_targets(params, seed, snrs, vmax, amax, jmax=0.0, sigma2=1.0):
    rng = scene.uniform01(seed, 4 * len(snrs) + 4)
    tg = []
    for i, snr in enumerate(snrs):
        u = rng[4 * i:4 * i + 4]
        cell = 64 + int(u[0] * (params.K - 128))
        v = (u[1] - 0.5) * 2 * vmax
        a = (u[2] - 0.5) * 2 * amax
        coeffs = [cell * params.delta_R(), v, a / 2.0]
        if jmax:
            coeffs.append((u[3] - 0.5) * 2 * jmax / 6.0)
        amp = scene.a1_for_snr(sigma2, snr, params.K_valid)
        tg.append((complex(amp, 0.0), coeffs))
    return tg


def cpi_targets(w: "Workload", cpi: int):
    """C4: 0-3 seeded targets per CPI, SNR -16..-8 dB, v +-250, a +-15."""
    s = scene.derive_seed(w.seed + 1, cpi)
    u = scene.uniform01(s, 1)[0]
    n = int(u * 4) % 4
    snrs = list(-16.0 + 8.0 * scene.uniform01(s ^ 0x5A5A, max(n, 1))[:n])
    return _draw_targets(w.params, s ^ 0xA5A5, snrs, 250.0, 15.0, sigma2=w.sigma2)


def config(i: int) -> Workload:
    if i == 0:
        p = RadarParams.create(FC, 20e6, 20e6, PRF, 256, 512)
        s = baseline_space(p, [(-150.0, 150.0), (-5.0, 5.0)])
        sig = 1.0 / p.K
        amp = scene.a1_for_snr(sig, -12.0, p.K_valid)
        return Workload("C0 ds-grft 2nd order 512x256", p, s, 0, None,
                        [(complex(amp, 0.0), [200 * p.delta_R(), 87.0, 2.0])], sig, 12345,
                        description="DS-GRFT (r0,v,a), M=256 x N=512, 1 target cell 200 v=87 a=4 -12 dB")
    if i == 1:
        p = RadarParams.create(FC, 20e6, 20e6, PRF, 1024, 2048)
        s = baseline_space(p, [(-300.0, 300.0), (-10.0, 10.0)])
        sig = 1.0 / p.K
        return Workload("C1 ds-grft 2nd order 2048x1024", p, s, 0, None,
                        _draw_targets(p, 1001, [-18.0, -14.0, -10.0], 300.0, 20.0, sigma2=sig), sig, 1001,
                        description="DS-GRFT (r0,v,a), M=1024 x N=2048, 3 targets -18/-14/-10 dB")
    if i == 2:
        p = RadarParams.create(FC, 20e6, 20e6, PRF, 2048, 4096)
        s = baseline_space(p, [(-300.0, 300.0), (-10.0, 10.0), (-2.0 / 6.0, 2.0 / 6.0)])
        sig = 1.0 / p.K
        return Workload("C2 ds-grft 3rd order 4096x2048", p, s, 0, None,
                        _draw_targets(p, 2002, [-20.0, -17.0, -15.0, -12.0], 300.0, 20.0, 2.0, sigma2=sig), sig,
                        2002, description="DS-GRFT (r0,v,a,j), M=2048 x N=4096, 4 targets -20..-12 dB")
    if i == 3:
        p = RadarParams.create(FC, 25e6, 20e6, PRF, 1024, 2048)
        s = baseline_space(p, [(-300.0, 300.0), (-10.0, 10.0)])
        amb = build_ambiguity(p, Bounds(-300.0, 300.0))
        sig = 1.0 / p.K
        return Workload("C3 ds-kt-mfp 2048x1024", p, s, 1, amb,
                        _draw_targets(p, 3003, [-15.0, -15.0], 300.0, 20.0, sigma2=sig), sig, 3003,
                        description="DS-KT-MFP, M=1024 x 2048, fs=25 MHz, 2 targets -15 dB, 8-tap keystone")
    if i == 4:
        p = RadarParams.create(FC, 20e6, 20e6, PRF, 512, 1024)
        s = baseline_space(p, [(-250.0, 250.0), (-7.5, 7.5)])
        sig = 1.0 / p.K
        return Workload("C4 ds-grft 64 CPIs 1024x512", p, s, 0, None, [], sig, 4004, cpis=64,
                        description="64 CPIs of M=512 x N=1024, 0-3 targets per CPI, DS-GRFT")
    raise ValueError(f"no BASELINE config {i}")


def sliced(w: Workload, coarse_v: int, coarse_rest: int = 0) -> Workload:
    """Same workload restricted to the first ``coarse_v`` cells of the leading
    coarse axis (and, if ``coarse_rest``, of every other coarse axis) -- bounded
    samples for rate measurements; every coarse cell costs the same."""
    import copy
    w2 = copy.deepcopy(w)
    axis = 0 if w.variant == 0 else 1
    g = w2.space.coarse[axis]
    g.count = min(g.count, coarse_v)
    if coarse_rest:
        for i, gg in enumerate(w2.space.coarse):
            if i != axis:
                gg.count = min(gg.count, coarse_rest)
    w2.name = f"{w.name} [coarse slice {coarse_v}" + (f"x{coarse_rest}" if coarse_rest else "") + "]"
    return w2
