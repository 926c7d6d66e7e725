"""Seeded synthetic echoes with the reference's signal model (harness input).

numpy port of
  GaussianRng        proj/src/rng.cpp:8-48 (splitmix64 + Box-Muller, spare kept)
  synthesize_cube    proj/src/signal_model.cpp:37-56
  add_noise          proj/src/signal_model.cpp:58-65
so that bench.py and the tests can build the BASELINE workloads on any box
without the reference.  tests/test_oracle.py::test_scene_generator_matches_reference
pins it to the reference's own generator (oracle/_ref) sample by sample.
"""
from __future__ import annotations

from typing import Iterable, Sequence, Tuple

import numpy as np

from .model import SPEED_OF_LIGHT, RadarParams

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix_block(state: int, n: int) -> np.ndarray:
    """The n outputs of successive next_u64() calls starting from ``state``."""
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        s = np.uint64(state & _MASK) + k * np.uint64(_GOLDEN)
        return _mix(s)


def derive_seed(seed: int, index: int) -> int:
    """GaussianRng::derive_seed (proj/src/rng.cpp:45-48)."""
    s = (seed ^ ((0x632BE59BD9B4E019 * (index + 1)) & _MASK)) & _MASK
    with np.errstate(over="ignore"):
        return int(_mix(np.array([(s + _GOLDEN) & _MASK], dtype=np.uint64))[0])


def uniform01(state: int, n: int) -> np.ndarray:
    u = splitmix_block(state, n)
    return ((u >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53


def circular_normal(seed: int, variance: float, n: int) -> np.ndarray:
    """n draws of GaussianRng(seed).circular_normal(variance) from a fresh generator."""
    u = uniform01(seed, 2 * n)
    r = np.sqrt(-2.0 * np.log(u[0::2]))
    a = 2.0 * np.pi * u[1::2]
    s = np.sqrt(variance / 2.0)
    return s * (r * np.cos(a)) + 1j * (s * (r * np.sin(a)))


Target = Tuple[complex, Sequence[float]]  # (amplitude A1, motion coefficients c0..cP)


def synthesize_cube(params: RadarParams, targets: Iterable[Target]) -> np.ndarray:
    """y(f_k, t_m) = sum_l A1_l exp(-j 4pi/c (f_k + fc) R_l(t_m)) on the occupied
    band, zero on guard bins.  Returns complex (M, K): [m, k] = data[k + K*m]."""
    params.validate()
    M, K = params.M, params.K
    cube = np.zeros((M, K), np.complex128)
    g = np.arange(-params.K_valid // 2, params.K_valid // 2)
    rows = np.where(g >= 0, g, g + K)
    fk = params.delta_f * g.astype(np.float64)
    tm = (np.arange(M) + 1.0) / params.PRF
    c4pi = -4.0 * np.pi / SPEED_OF_LIGHT
    for amp, coeffs in targets:
        rng = np.zeros(M)
        for c in reversed(list(coeffs)):  # Horner, MotionParams::slant_range
            rng = rng * tm + c
        phase = c4pi * (fk[None, :] + params.fc) * rng[:, None]
        cube[:, rows] += complex(amp) * (np.cos(phase) + 1j * np.sin(phase))
    return cube


def add_noise(cube: np.ndarray, sigma2: float, seed: int) -> np.ndarray:
    if sigma2 < 0:
        raise ValueError("add_noise: sigma2 must be >= 0")
    if sigma2 == 0:
        return cube.copy()
    return cube + circular_normal(seed, sigma2, cube.size).reshape(cube.shape)


def a1_for_snr(sigma2: float, snr_db: float, k_valid: int) -> float:
    """Per-pulse post-compression SNR -> |A1| (proj/src/bench.cpp:25-27)."""
    return float(np.sqrt(sigma2 * 10.0 ** (snr_db / 10.0) / k_valid))


def to_complex64_roundtrip(cube: np.ndarray) -> np.ndarray:
    """The cube as the GPU sees it (complex64), upcast back for the oracle."""
    return cube.astype(np.complex64).astype(np.complex128)
