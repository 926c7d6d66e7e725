"""Python face of the B200 detectors, mirroring the reference detector API.

  ds_grft(cube, space, opt)            proj/include/ltci/detectors.hpp:42-43
  ds_kt_mfp(cube, amb, space, opt)     proj/include/ltci/detectors.hpp:47-48
  detection_threshold(params, ...)     proj/include/ltci/detectors.hpp:55
  keystone / mgift / gft               proj/include/ltci/transforms.hpp:40,52-53,74-75
Everything goes through the C-ABI of lib/libltci_cuda.so (include/ltci_cuda.h);
errors come back as the Python counterparts of the reference exceptions
(ValueError <- std::invalid_argument, ConditionViolated, MemoryError <-
std::bad_alloc).  ``Engine`` keeps a plan resident on one GPU for streaming
cubes (device-resident input or host input), optionally over a slice of the
ROI rows for range-cell sharding.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _cabi as A
from . import _lib
from .model import (AmbiguitySpace, DetectionMap, DetectorOptions, DualScaleSpace, RadarParams, SingleScaleSpace,
                    cube_as_f64, map_from_c)


def _f64_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _take_map(lib, pm: A.PMap, params: RadarParams) -> DetectionMap:
    try:
        return map_from_c(pm.contents, params)
    finally:
        lib.ltci_cuda_free_map(pm)


def ds_grft(cube: np.ndarray, params: RadarParams, space: DualScaleSpace,
            opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """Dual-scale GRFT on the GPU. ``cube`` is complex (M, K): data[k + K*m]."""
    lib = _lib.load()
    opt = opt or DetectorOptions()
    data = cube_as_f64(cube, params)
    r, s, o = params.to_c(), space.to_c(), opt.to_c()
    pm = A.PMap()
    _lib.raise_for(lib.ltci_cuda_ds_grft(_f64_ptr(data), C.byref(r), C.byref(s), C.byref(o), C.byref(pm)), lib)
    m = _take_map(lib, pm, params)
    m.dual = space
    return m


def ds_kt_mfp(cube: np.ndarray, params: RadarParams, amb: AmbiguitySpace, space: DualScaleSpace,
              opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """Dual-scale keystone matched-filter processing on the GPU."""
    lib = _lib.load()
    opt = opt or DetectorOptions()
    data = cube_as_f64(cube, params)
    r, a, s, o = params.to_c(), amb.to_c(), space.to_c(), opt.to_c()
    pm = A.PMap()
    _lib.raise_for(lib.ltci_cuda_ds_kt_mfp(_f64_ptr(data), C.byref(r), C.byref(a), C.byref(s), C.byref(o),
                                           C.byref(pm)), lib)
    m = _take_map(lib, pm, params)
    m.dual, m.amb = space, amb
    return m


def fd_grft(cube: np.ndarray, params: RadarParams, space: SingleScaleSpace,
            opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """Single-scale frequency-domain GRFT on the GPU (ltci::fd_grft,
    proj/src/detectors.cpp:105-197)."""
    lib = _lib.load()
    opt = opt or DetectorOptions()
    data = cube_as_f64(cube, params)
    r, s, o = params.to_c(), space.to_c(), opt.to_c()
    pm = A.PMap()
    _lib.raise_for(lib.ltci_cuda_fd_grft(_f64_ptr(data), C.byref(r), C.byref(s), C.byref(o), C.byref(pm)), lib)
    m = _take_map(lib, pm, params)
    m.single = space
    return m


def td_grft(range_cube: np.ndarray, params: RadarParams, space: SingleScaleSpace,
            opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """Single-scale time-domain GRFT on the GPU (ltci::td_grft,
    proj/src/detectors.cpp:199-264): nearest-bin sums along rounded
    trajectories of a RANGE-pulse cube.  ``opt.trajectory``: 0 zero outside,
    1 wrap, 2 raise IndexError (std::out_of_range) when a trajectory leaves
    the cube."""
    lib = _lib.load()
    opt = opt or DetectorOptions()
    data = cube_as_f64(range_cube, params)
    r, s, o = params.to_c(), space.to_c(), opt.to_c()
    pm = A.PMap()
    _lib.raise_for(lib.ltci_cuda_td_grft(_f64_ptr(data), C.byref(r), C.byref(s), C.byref(o), C.byref(pm)), lib)
    m = _take_map(lib, pm, params)
    m.single = space
    return m


def kt_mfp(cube: np.ndarray, params: RadarParams, amb: AmbiguitySpace, space: SingleScaleSpace,
           opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """Single-scale keystone matched-filter processing on the GPU (ltci::kt_mfp,
    proj/src/detectors.cpp:266-326): keystone once, then (folding number,
    acceleration) cells over the full Doppler axis; ``space`` must have order 2."""
    lib = _lib.load()
    opt = opt or DetectorOptions()
    data = cube_as_f64(cube, params)
    r, s, o, a = params.to_c(), space.to_c(), opt.to_c(), amb.to_c()
    pm = A.PMap()
    _lib.raise_for(lib.ltci_cuda_kt_mfp(_f64_ptr(data), C.byref(r), C.byref(a), C.byref(s), C.byref(o),
                                        C.byref(pm)), lib)
    m = _take_map(lib, pm, params)
    m.single, m.amb = space, amb
    return m


def detection_threshold(params: RadarParams, sigma2: float, pfa: float, bins: int = 0) -> float:
    lib = _lib.load()
    st = C.c_int(0)
    r = params.to_c()
    g = lib.ltci_cuda_detection_threshold(C.byref(r), sigma2, pfa, bins, C.byref(st))
    _lib.raise_for(st.value, lib)
    return g


def keystone(cube: np.ndarray, params: RadarParams, taps: int = 8) -> np.ndarray:
    lib = _lib.load()
    data = cube_as_f64(cube, params)
    out = np.zeros_like(data)
    r = params.to_c()
    _lib.raise_for(lib.ltci_cuda_keystone(_f64_ptr(data), C.byref(r), taps, _f64_ptr(out)), lib)
    return out


def range_fft(range_cube: np.ndarray, params: RadarParams) -> np.ndarray:
    """ltci::range_fft (proj/src/signal_model.cpp:97-107): per pulse the
    unnormalised forward K-point DFT of a range-pulse cube (M, K) -> the
    freq-pulse cube the detectors take (K0 on the device, complex64-exact)."""
    lib = _lib.load()
    data = np.ascontiguousarray(range_cube, dtype=np.complex128)
    out = np.zeros_like(data)
    r = params.to_c()
    _lib.raise_for(lib.ltci_cuda_range_fft(_f64_ptr(data), C.byref(r), _f64_ptr(out)), lib)
    return out


def mgift(cube: np.ndarray, params: RadarParams, ctilde: Sequence[float], variant: int = A.VARIANT_GRFT) -> np.ndarray:
    """Returns the RangePulseCube as complex (M, K): [m, n]."""
    lib = _lib.load()
    data = cube_as_f64(cube, params)
    out = np.zeros_like(data)
    r = params.to_c()
    arr = (C.c_double * len(ctilde))(*ctilde)
    _lib.raise_for(lib.ltci_cuda_mgift(_f64_ptr(data), C.byref(r), arr, len(ctilde), variant, _f64_ptr(out)), lib)
    return out


def gft(rows: np.ndarray, params: RadarParams, fine_higher: Sequence[float], roi_first: int, roi_last: int) -> np.ndarray:
    """Returns the RangeDopplerMap as complex (M, R): [j, r] == data[r + R*j]."""
    lib = _lib.load()
    data = cube_as_f64(rows, params)
    R = roi_last - roi_first + 1
    out = np.zeros((params.M, max(R, 0)), np.complex128)
    r = params.to_c()
    arr = (C.c_double * max(len(fine_higher), 1))(*fine_higher)
    _lib.raise_for(lib.ltci_cuda_gft(_f64_ptr(data), C.byref(r), arr, len(fine_higher), roi_first, roi_last,
                                     _f64_ptr(out)), lib)
    return out


class Engine:
    """Device-resident plan for repeated runs (streaming CPIs, benchmarking,
    range-cell shards).  ``variant`` 0 = ds_grft, 1 = ds_kt_mfp."""

    def __init__(self, params: RadarParams, space: DualScaleSpace, variant: int = A.VARIANT_GRFT,
                 amb: Optional[AmbiguitySpace] = None, opt: Optional[DetectorOptions] = None,
                 row_begin: int = 0, row_end: int = -1, coarse_begin: int = 0, coarse_end: int = -1):
        self._lib = _lib.load()
        self.params, self.space, self.variant, self.amb = params, space, variant, amb
        self.opt = opt or DetectorOptions()
        r, s, o = params.to_c(), space.to_c(), self.opt.to_c()
        a = amb.to_c() if amb is not None else None
        h = C.c_void_p()
        rc = self._lib.ltci_engine_create(C.byref(r), C.byref(s), C.byref(a) if a is not None else None, variant,
                                          C.byref(o), row_begin, row_end, C.byref(h))
        _lib.raise_for(rc, self._lib)
        self._h = h
        if coarse_begin != 0 or coarse_end != -1:
            self.set_coarse_slice(coarse_begin, coarse_end)

    def set_coarse_slice(self, c_begin: int, c_end: int):
        """Search only coarse cells [c_begin, c_end) (coarse-cell sharding; flat indices stay global)."""
        _lib.raise_for(self._lib.ltci_engine_set_coarse_slice(self._h, c_begin, c_end if c_end >= 0 else (1 << 64) - 1),
                       self._lib)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ltci_engine_destroy(self._h)
            self._h = None

    __del__ = close

    def set_timing(self, on: bool = True):
        _lib.raise_for(self._lib.ltci_engine_set_timing(self._h, int(on)), self._lib)

    def run_device(self, d_cube_ptr: int, stream: int = 0):
        """Run on a device complex64 cube (K*M float2, column-major)."""
        _lib.raise_for(self._lib.ltci_engine_run_device(self._h, C.c_void_p(d_cube_ptr), C.c_void_p(stream)),
                       self._lib)

    def run_host(self, cube: np.ndarray, stream: int = 0):
        data = cube if (cube.dtype == np.complex128 and cube.flags.c_contiguous) else cube_as_f64(cube, self.params)
        _lib.raise_for(self._lib.ltci_engine_run_host(self._h, _f64_ptr(data), C.c_void_p(stream)), self._lib)

    def run_range_device(self, d_range_ptr: int, stream: int = 0):
        """configs[3] front end: K0 range FFT of a device complex64 RANGE-pulse cube, then the cascade."""
        _lib.raise_for(self._lib.ltci_engine_run_range_device(self._h, C.c_void_p(d_range_ptr), C.c_void_p(stream)),
                       self._lib)

    def run_range_host(self, range_cube: np.ndarray, stream: int = 0):
        """K0 + cascade from a host RANGE-pulse cube (M, K) complex."""
        data = np.ascontiguousarray(range_cube, dtype=np.complex128)
        _lib.raise_for(self._lib.ltci_engine_run_range_host(self._h, _f64_ptr(data), C.c_void_p(stream)), self._lib)

    def run_range_host_ptr(self, host_ptr: int, stream: int = 0):
        """K0 + cascade from a (pinned) host float64 interleaved RANGE-pulse buffer given by address."""
        _lib.raise_for(self._lib.ltci_engine_run_range_host(self._h, C.c_void_p(host_ptr), C.c_void_p(stream)),
                       self._lib)

    def run_host_ptr(self, host_ptr: int, stream: int = 0):
        """Run from a (pinned) host float64 interleaved buffer given by address."""
        _lib.raise_for(self._lib.ltci_engine_run_host(self._h, C.c_void_p(host_ptr), C.c_void_p(stream)),
                       self._lib)

    def run_file(self, path: str, stream: int = 0):
        """Stream an "LTCI" freq-pulse cube file into the device and run (the wire path)."""
        _lib.raise_for(self._lib.ltci_engine_run_file(self._h, str(path).encode(), C.c_void_p(stream)), self._lib)

    def result(self, stream: int = 0) -> DetectionMap:
        pm = A.PMap()
        _lib.raise_for(self._lib.ltci_engine_result(self._h, C.c_void_p(stream), C.byref(pm)), self._lib)
        m = _take_map(self._lib, pm, self.params)
        m.dual, m.amb = self.space, self.amb
        return m

    def peaks_device(self):
        """(device pointer, n_rows) of the per-row peak records {f32 re, f32 im, u64 idx}."""
        p, n = C.c_void_p(), C.c_int32()
        _lib.raise_for(self._lib.ltci_engine_peaks_device(self._h, C.byref(p), C.byref(n)), self._lib)
        return p.value, n.value

    def stats(self):
        n, f, c, k = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        _lib.raise_for(self._lib.ltci_engine_stats(self._h, C.byref(n), C.byref(f), C.byref(c), C.byref(k)),
                       self._lib)
        return {"launches": n.value, "fine_ms": f.value, "coarse_ms": c.value, "keystone_ms": k.value}

    def fine_path(self):
        """(path, terms): the fine-stage formulation this engine runs."""
        pth, t = C.c_int32(), C.c_int32()
        _lib.raise_for(self._lib.ltci_engine_fine_path(self._h, C.byref(pth), C.byref(t)), self._lib)
        return pth.value, t.value

    def coarse_path(self) -> str:
        """'gather' (interpolated oversampled profiles, csrc/gather.cuh) or 'transform' (csrc/coarse.cuh)."""
        pth = C.c_int32()
        _lib.raise_for(self._lib.ltci_engine_coarse_path(self._h, C.byref(pth)), self._lib)
        return "gather" if pth.value == 1 else "transform"

    def work(self):
        h, i = C.c_uint64(), C.c_uint64()
        _lib.raise_for(self._lib.ltci_engine_work(self._h, C.byref(h), C.byref(i)), self._lib)
        return h.value, i.value
