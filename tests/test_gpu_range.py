"""K0 range FFT (the configs[3] front end, ltci::range_fft,
proj/src/signal_model.cpp:97-107) and K4 keystone on the device.

* K0 against the reference's golden output and against the oracle port at
  every supported K; at full C3 size through the round-trip property
  range_fft(range_ifft(x)) == K x (proj/include/ltci/signal_model.hpp:36);
* the engine's range-domain entry (K0 -> keystone -> coarse -> fine) against
  the freq-domain run on the same scene;
* K4 through the device entry point used for back-to-back timing, against the
  oracle, including its exact-copy rows and clamped edges.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import _lib, keystone, range_fft, scene
from paper_2403_06788_b200.configs import config
from paper_2403_06788_b200.detectors import Engine, detection_threshold
from paper_2403_06788_b200.model import AmbiguitySpace, DetectorOptions, RadarParams

from helpers import TOL, cube, load, radar, space

pytestmark = pytest.mark.gpu
KTOL = 2e-5  # kernel-level transforms (FP32 FFT accuracy), as test_gpu_parity


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_range_fft_matches_reference_golden():
    g = load("range_fft.npz")
    p = radar(g)
    assert _rel(range_fft(g["noise"], p), g["noise_fft"]) < KTOL
    assert _rel(range_fft(g["scene_range"], p), g["scene_fft"]) < KTOL


@pytest.mark.parametrize("M,K", [(4, 16), (64, 32), (16, 64), (32, 128), (8, 256), (16, 512), (4, 1024),
                                 (16, 2048), (2, 4096), (2, 8192), (1024, 16)])
def test_range_fft_all_sizes(M, K):
    p = RadarParams.create(3e9, 20e6, 18e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((M, K), complex), 1.0, 3 * M + K))
    assert _rel(range_fft(x, p), O.port_range_fft(x, p)) < KTOL


def test_range_fft_round_trip_full_c3():
    """At the full C3 shape (2048 x 1024): K0 of the range-domain echo returns K x."""
    import torch
    w = config(3)
    p = w.params
    x = scene.to_complex64_roundtrip(w.cube())
    rc = np.fft.ifft(x, axis=1) * p.K  # dft_plus per pulse (range_ifft), FP64
    d_in = torch.from_numpy(np.ascontiguousarray(rc.astype(np.complex64))).cuda()
    d_out = torch.empty_like(d_in)
    lib = _lib.load()
    r = p.to_c()
    _lib.raise_for(lib.ltci_cuda_range_fft_device(C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()),
                                                  C.byref(r), None), lib)
    torch.cuda.synchronize()
    back = d_out.cpu().numpy() / p.K
    assert _rel(back, x) < KTOL


@pytest.mark.parametrize("name,variant", [("small_kt.npz", 1), ("small_grft.npz", 0)])
def test_engine_range_entry_equals_freq_entry(name, variant):
    """run_range_host(range_ifft(x) / K) searches the same scene as run_host(x):
    per-row peaks within 1e-4 of the map maximum, indices identical except
    ties, same argmax."""
    g = load(name)
    p = radar(g)
    s = space(g, p)
    amb = AmbiguitySpace(int(g["amb"][0]), int(g["amb"][1])) if variant else None
    x = cube(g)
    rc = np.fft.ifft(x, axis=1)  # range_ifft(x) / K, so that K0 returns x itself
    opt = DetectorOptions(retain_threshold=float(g["retain"]))
    e = Engine(p, s, variant, amb, opt)
    e.run_host(x)
    a = e.result()
    e.run_range_host(rc)
    b = e.result()
    e.close()
    scale = np.abs(a.peak_value).max()
    assert np.abs(np.abs(a.peak_value) - np.abs(b.peak_value)).max() <= 1e-4 * scale
    va, vb = np.abs(a.peak_value), np.abs(b.peak_value)
    for r in np.nonzero(a.peak_index != b.peak_index)[0]:
        assert abs(va[r] - vb[r]) <= TOL * scale, f"row {r}: index differs beyond a tie"
    assert a.argmax == b.argmax
    assert a.counters == b.counters


@pytest.mark.parametrize("taps", [8, 4, 6, 16, 3, 2, 20])
def test_keystone_kernels_match_oracle(taps):
    """K4 (tiled for taps <= 16, per-element beyond) against the oracle port; the
    C3 radar has exact-copy rows (f_k = 0) and clamped taps at both pulse ends."""
    p = RadarParams.create(3e9, 25e6, 20e6, 1000.0, 64, 256)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((p.M, p.K), complex), 1.0, 17 + taps))
    ref = O.port_keystone(x, p, taps)
    assert _rel(keystone(x, p, taps), ref) < KTOL


def test_keystone_device_entry_full_c3():
    import torch
    w = config(3)
    p = w.params
    x = scene.to_complex64_roundtrip(w.cube())
    d_in = torch.from_numpy(np.ascontiguousarray(x.astype(np.complex64))).cuda()
    d_out = torch.empty_like(d_in)
    lib = _lib.load()
    r = p.to_c()
    _lib.raise_for(lib.ltci_cuda_keystone_device(C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()),
                                                 C.byref(r), 8, None), lib)
    torch.cuda.synchronize()
    assert _rel(d_out.cpu().numpy(), O.port_keystone(x, p, 8)) < KTOL
