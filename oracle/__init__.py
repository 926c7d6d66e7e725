"""TEST INFRASTRUCTURE -- the parity checkers.  Never imported by the product.

Two checkers with the same calling convention (POD plan structs of
include/ltci_cuda.h, complex (M, K) numpy cubes):

  port  liboracle.so          our plain-C FP64 restatement (ds_oracle.c);
                              travels to the GPU box, no reference needed
  ref   _ref/libltci_ref.so   the reference library itself, compiled read-only
                              from /root/reference/proj/src (oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from paper_2403_06788_b200 import _cabi as A
from paper_2403_06788_b200.model import (AmbiguitySpace, DetectionMap, DetectorOptions, DualScaleSpace,  # noqa: F401
                                         RadarParams, SingleScaleSpace, map_from_c)

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libltci_ref.so")

_port = None
_ref = None


def _vp(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c128(cube: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(cube, dtype=np.complex128)


def have_port() -> bool:
    return os.path.exists(PORT_PATH)


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


def port():
    global _port
    if _port is None:
        lib = C.CDLL(PORT_PATH)
        P = C.POINTER
        lib.oracle_ds.argtypes = [C.c_void_p, P(A.CRadar), P(A.CAmbiguity), P(A.CDualSpace), P(A.COptions),
                                  C.c_int, C.c_int, P(A.PMap)]
        lib.oracle_free_map.argtypes = [A.PMap]
        lib.oracle_free_map.restype = None
        lib.oracle_mgift.argtypes = [C.c_void_p, P(A.CRadar), P(C.c_double), C.c_int, C.c_int, C.c_void_p]
        lib.oracle_gft.argtypes = [C.c_void_p, P(A.CRadar), P(C.c_double), C.c_int, C.c_int, C.c_int, C.c_void_p]
        lib.oracle_keystone.argtypes = [C.c_void_p, P(A.CRadar), C.c_int, C.c_void_p]
        lib.oracle_range_fft.argtypes = [C.c_void_p, P(A.CRadar), C.c_void_p]
        lib.oracle_td_grft.argtypes = [C.c_void_p, P(A.CRadar), P(A.CSingleSpace), P(A.COptions), P(A.PMap)]
        lib.oracle_kt_mfp.argtypes = [C.c_void_p, P(A.CRadar), P(A.CAmbiguity), P(A.CSingleSpace), P(A.COptions),
                                      P(A.PMap)]
        _port = lib
    return _port


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_PATH)
        P = C.POINTER
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_free_map.argtypes = [A.PMap]
        lib.ref_free_map.restype = None
        lib.ref_radar_create.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                         P(A.CRadar)]
        lib.ref_build_dual_scale.argtypes = [P(A.CRadar), C.c_int, P(C.c_double), P(C.c_double), P(C.c_double),
                                             C.c_int, C.c_int, P(A.CDualSpace)]
        lib.ref_build_ambiguity.argtypes = [P(A.CRadar), C.c_double, C.c_double, P(A.CAmbiguity)]
        lib.ref_synthesize.argtypes = [P(A.CRadar), C.c_int, P(C.c_double), P(C.c_double), C.c_int, C.c_double,
                                       C.c_uint64, vp]
        lib.ref_rng_circular.argtypes = [C.c_uint64, C.c_double, C.c_int, vp]
        lib.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_derive_seed.restype = C.c_uint64
        lib.ref_ds_grft.argtypes = [vp, P(A.CRadar), P(A.CDualSpace), P(A.COptions), P(A.PMap)]
        lib.ref_ds_kt_mfp.argtypes = [vp, P(A.CRadar), P(A.CAmbiguity), P(A.CDualSpace), P(A.COptions), P(A.PMap)]
        lib.ref_keystone.argtypes = [vp, P(A.CRadar), C.c_int, vp]
        lib.ref_range_fft.argtypes = [vp, P(A.CRadar), vp]
        lib.ref_range_ifft.argtypes = [vp, P(A.CRadar), vp]
        lib.ref_mgift.argtypes = [vp, P(A.CRadar), P(C.c_double), C.c_int, C.c_int, vp]
        lib.ref_gft.argtypes = [vp, P(A.CRadar), P(C.c_double), C.c_int, C.c_int, C.c_int, vp]
        lib.ref_fd_grft_point.argtypes = [vp, P(A.CRadar), P(C.c_double), C.c_int, C.c_int, vp]
        lib.ref_kt_mfp_point.argtypes = [vp, P(A.CRadar), C.c_int, C.c_double, C.c_int, C.c_int, vp]
        lib.ref_detection_threshold.argtypes = [P(A.CRadar), C.c_double, C.c_double, C.c_int, P(C.c_double)]
        lib.ref_peak_map.argtypes = [vp, P(A.CRadar), P(A.CAmbiguity), P(A.CDualSpace), C.c_int, C.c_int, C.c_int,
                                     vp, vp]
        lib.ref_extract_ds.argtypes = [P(A.CDetectionMap), P(A.CDualSpace), P(A.CAmbiguity), C.c_double, C.c_int,
                                       vp, P(C.c_int)]
        lib.ref_resolve_threads.argtypes = [C.c_int]
        lib.ref_write_cube_file.argtypes = [C.c_char_p, P(A.CCubeHeader), vp]
        lib.ref_run_pd.argtypes = [P(A.CScenario), C.c_int, P(A.CPdPoint)]
        lib.ref_build_single_scale.argtypes = [P(A.CRadar), C.c_int, P(C.c_double), P(C.c_double), P(C.c_double),
                                               C.c_int, C.c_int, P(A.CSingleSpace)]
        lib.ref_fd_grft.argtypes = [vp, P(A.CRadar), P(A.CSingleSpace), P(A.COptions), P(A.PMap)]
        lib.ref_td_grft.argtypes = [vp, P(A.CRadar), P(A.CSingleSpace), P(A.COptions), P(A.PMap)]
        lib.ref_kt_mfp.argtypes = [vp, P(A.CRadar), P(A.CAmbiguity), P(A.CSingleSpace), P(A.COptions), P(A.PMap)]
        lib.ref_extract_single.argtypes = [P(A.CDetectionMap), P(A.CSingleSpace), C.c_double, C.c_int, vp,
                                           P(C.c_int)]
        lib.ref_read_cube_file.argtypes = [C.c_char_p, P(A.CCubeHeader), vp, C.c_uint64]
        _ref = lib
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int, lib=None):
    if rc != A.OK:
        msg = lib.ref_last_error().decode() if lib is not None and hasattr(lib, "ref_last_error") else ""
        raise OracleError(rc, msg)


def _map(lib, pm, params, free) -> DetectionMap:
    try:
        return map_from_c(pm.contents, params)
    finally:
        free(pm)


# ------------------------------------------------------------ port (C) ---
def port_ds(cube, params: RadarParams, space: DualScaleSpace, opt: Optional[DetectorOptions] = None,
            variant: int = 0, amb: Optional[AmbiguitySpace] = None, threads: int = 0) -> DetectionMap:
    lib = port()
    opt = opt or DetectorOptions()
    data = _c128(cube)
    r, s, o = params.to_c(), space.to_c(), opt.to_c()
    a = amb.to_c() if amb is not None else None
    pm = A.PMap()
    threads = threads or os.cpu_count() or 1
    _check(lib.oracle_ds(_vp(data), C.byref(r), C.byref(a) if a is not None else None, C.byref(s), C.byref(o),
                         variant, threads, C.byref(pm)))
    m = _map(lib, pm, params, lib.oracle_free_map)
    m.dual, m.amb = space, amb
    return m


def port_mgift(cube, params, ctilde, variant=0):
    lib = port()
    data = _c128(cube)
    out = np.zeros_like(data)
    arr = (C.c_double * len(ctilde))(*ctilde)
    r = params.to_c()
    _check(lib.oracle_mgift(_vp(data), C.byref(r), arr, len(ctilde), variant, _vp(out)))
    return out


def port_gft(rows, params, fine, roi_first, roi_last):
    lib = port()
    data = _c128(rows)
    out = np.zeros((params.M, roi_last - roi_first + 1), np.complex128)
    arr = (C.c_double * max(1, len(fine)))(*fine)
    r = params.to_c()
    _check(lib.oracle_gft(_vp(data), C.byref(r), arr, len(fine), roi_first, roi_last, _vp(out)))
    return out


def port_keystone(cube, params, taps=8):
    lib = port()
    data = _c128(cube)
    out = np.zeros_like(data)
    r = params.to_c()
    _check(lib.oracle_keystone(_vp(data), C.byref(r), taps, _vp(out)))
    return out


def port_range_fft(cube, params):
    """range_fft (proj/src/signal_model.cpp:97-107) restated in C: per pulse dft_minus."""
    lib = port()
    data = _c128(cube)
    out = np.zeros_like(data)
    r = params.to_c()
    _check(lib.oracle_range_fft(_vp(data), C.byref(r), _vp(out)))
    return out


# ------------------------------------------------------- reference (C++) ---
def ref_radar(fc, fs, br, prf, M, K, k_valid=0) -> RadarParams:
    lib = ref()
    r = A.CRadar()
    _check(lib.ref_radar_create(fc, fs, br, prf, M, K, k_valid, C.byref(r)), lib)
    return RadarParams.from_c(r)


def ref_dual_scale(params, P, bounds, alpha, roi_first, roi_last) -> DualScaleSpace:
    lib = ref()
    lo = (C.c_double * P)(*[b[0] for b in bounds])
    hi = (C.c_double * P)(*[b[1] for b in bounds])
    al = (C.c_double * P)(*alpha)
    r, s = params.to_c(), A.CDualSpace()
    _check(lib.ref_build_dual_scale(C.byref(r), P, lo, hi, al, roi_first, roi_last, C.byref(s)), lib)
    return DualScaleSpace.from_c(s)


def ref_ambiguity(params, vlo, vhi) -> AmbiguitySpace:
    lib = ref()
    r, a = params.to_c(), A.CAmbiguity()
    _check(lib.ref_build_ambiguity(C.byref(r), vlo, vhi, C.byref(a)), lib)
    return AmbiguitySpace(a.q_min, a.q_max)


def ref_synthesize(params, targets, sigma2=0.0, seed=0):
    lib = ref()
    n_coef = max(len(c) for _, c in targets) if targets else 1
    amp = np.array([[complex(a).real, complex(a).imag] for a, _ in targets] or [[0, 0]], np.float64).ravel()
    co = np.zeros((max(len(targets), 1), n_coef))
    for i, (_, c) in enumerate(targets):
        co[i, :len(c)] = c
    out = np.zeros((params.M, params.K), np.complex128)
    r = params.to_c()
    _check(lib.ref_synthesize(C.byref(r), len(targets), amp.ctypes.data_as(C.POINTER(C.c_double)),
                              co.ctypes.data_as(C.POINTER(C.c_double)), n_coef, sigma2, seed, _vp(out)), lib)
    return out


def ref_rng_circular(seed, variance, n):
    lib = ref()
    out = np.zeros(n, np.complex128)
    _check(lib.ref_rng_circular(seed, variance, n, _vp(out)), lib)
    return out


def ref_ds(cube, params, space, opt=None, variant=0, amb=None) -> DetectionMap:
    lib = ref()
    opt = opt or DetectorOptions()
    data = _c128(cube)
    r, s, o = params.to_c(), space.to_c(), opt.to_c()
    pm = A.PMap()
    if variant == 0:
        _check(lib.ref_ds_grft(_vp(data), C.byref(r), C.byref(s), C.byref(o), C.byref(pm)), lib)
    else:
        a = amb.to_c()
        _check(lib.ref_ds_kt_mfp(_vp(data), C.byref(r), C.byref(a), C.byref(s), C.byref(o), C.byref(pm)), lib)
    m = _map(lib, pm, params, lib.ref_free_map)
    m.dual, m.amb = space, amb
    return m


def ref_peak_map(cube, params, space, variant=0, amb=None, taps=8, threads=0):
    lib = ref()
    data = _c128(cube)
    R = space.roi.count()
    idx = np.zeros(R, np.uint64)
    val = np.zeros(R, np.complex128)
    r, s = params.to_c(), space.to_c()
    a = amb.to_c() if amb is not None else A.CAmbiguity()
    _check(lib.ref_peak_map(_vp(data), C.byref(r), C.byref(a), C.byref(s), variant, taps,
                            threads or os.cpu_count() or 1, _vp(idx), _vp(val)), lib)
    return idx, val


def ref_mgift(cube, params, ctilde, variant=0):
    lib = ref()
    data = _c128(cube)
    out = np.zeros_like(data)
    arr = (C.c_double * len(ctilde))(*ctilde)
    r = params.to_c()
    _check(lib.ref_mgift(_vp(data), C.byref(r), arr, len(ctilde), variant, _vp(out)), lib)
    return out


def ref_gft(rows, params, fine, roi_first, roi_last):
    lib = ref()
    data = _c128(rows)
    out = np.zeros((params.M, roi_last - roi_first + 1), np.complex128)
    arr = (C.c_double * max(1, len(fine)))(*fine)
    r = params.to_c()
    _check(lib.ref_gft(_vp(data), C.byref(r), arr, len(fine), roi_first, roi_last, _vp(out)), lib)
    return out


def ref_keystone(cube, params, taps=8):
    lib = ref()
    data = _c128(cube)
    out = np.zeros_like(data)
    r = params.to_c()
    _check(lib.ref_keystone(_vp(data), C.byref(r), taps, _vp(out)), lib)
    return out


def ref_range_fft(cube, params):
    lib = ref()
    data = _c128(cube)
    out = np.zeros_like(data)
    r = params.to_c()
    _check(lib.ref_range_fft(_vp(data), C.byref(r), _vp(out)), lib)
    return out


def ref_range_ifft(cube, params):
    lib = ref()
    data = _c128(cube)
    out = np.zeros_like(data)
    r = params.to_c()
    _check(lib.ref_range_ifft(_vp(data), C.byref(r), _vp(out)), lib)
    return out


def ref_threshold(params, sigma2, pfa, bins=0):
    lib = ref()
    r, out = params.to_c(), C.c_double()
    _check(lib.ref_detection_threshold(C.byref(r), sigma2, pfa, bins, C.byref(out)), lib)
    return out.value


def ref_point(cube, params, ctilde, range_bin):
    lib = ref()
    data = _c128(cube)
    out = np.zeros(2)
    arr = (C.c_double * len(ctilde))(*ctilde)
    r = params.to_c()
    _check(lib.ref_fd_grft_point(_vp(data), C.byref(r), arr, len(ctilde), range_bin, _vp(out)), lib)
    return complex(out[0], out[1])


# ------------------------------------------------- cube file (reference) ---
def ref_write_cube_file(path, params, cube, sigma2=0.0, domain=0):
    lib = ref()
    data = _c128(cube)
    h = A.CCubeHeader(domain, params.to_c(), sigma2)
    _check(lib.ref_write_cube_file(str(path).encode(), C.byref(h), _vp(data)), lib)


def ref_read_cube_file(path, max_samples=1 << 24):
    """(domain, params, sigma2, complex (M, K) data) via ltci::read_cube_file."""
    lib = ref()
    out = np.empty(max_samples, np.complex128)
    h = A.CCubeHeader()
    _check(lib.ref_read_cube_file(str(path).encode(), C.byref(h), _vp(out), 2 * out.size), lib)
    p = RadarParams.from_c(h.radar)
    return int(h.domain), p, float(h.sigma2), out[: p.K * p.M].reshape(p.M, p.K).copy()


# ----------------------------------------------- fd_grft (reference, C++) ---
def ref_single_scale(params, P, bounds, alpha, roi_first, roi_last) -> SingleScaleSpace:
    lib = ref()
    lo = (C.c_double * P)(*[b[0] for b in bounds])
    hi = (C.c_double * P)(*[b[1] for b in bounds])
    al = (C.c_double * P)(*alpha)
    r, s = params.to_c(), A.CSingleSpace()
    _check(lib.ref_build_single_scale(C.byref(r), P, lo, hi, al, roi_first, roi_last, C.byref(s)), lib)
    return SingleScaleSpace.from_c(s)


def ref_fd(cube, params, space: SingleScaleSpace, opt: Optional[DetectorOptions] = None) -> DetectionMap:
    lib = ref()
    opt = opt or DetectorOptions()
    data = _c128(cube)
    r, s, o = params.to_c(), space.to_c(), opt.to_c()
    pm = A.PMap()
    _check(lib.ref_fd_grft(_vp(data), C.byref(r), C.byref(s), C.byref(o), C.byref(pm)), lib)
    m = _map(lib, pm, params, lib.ref_free_map)
    m.single = space
    return m


def _single_call(fn, lib, free, cube, params, space, opt, amb=None) -> DetectionMap:
    opt = opt or DetectorOptions()
    data = _c128(cube)
    r, s, o = params.to_c(), space.to_c(), opt.to_c()
    pm = A.PMap()
    if amb is None:
        rc = fn(_vp(data), C.byref(r), C.byref(s), C.byref(o), C.byref(pm))
    else:
        a = amb.to_c()
        rc = fn(_vp(data), C.byref(r), C.byref(a), C.byref(s), C.byref(o), C.byref(pm))
    if rc == 7:  # LTCI_OUT_OF_RANGE: td_grft under TrajectoryPolicy::Error
        raise IndexError("td_grft: trajectory leaves the cube")
    _check(rc, lib)
    m = _map(lib, pm, params, free)
    m.single, m.amb = space, amb
    return m


def ref_td(range_cube, params, space: SingleScaleSpace, opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """The reference's td_grft (proj/src/detectors.cpp:199-264) on a range-pulse cube."""
    lib = ref()
    return _single_call(lib.ref_td_grft, lib, lib.ref_free_map, range_cube, params, space, opt)


def ref_kt(cube, params, amb: AmbiguitySpace, space: SingleScaleSpace,
           opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """The reference's kt_mfp (proj/src/detectors.cpp:266-326)."""
    lib = ref()
    return _single_call(lib.ref_kt_mfp, lib, lib.ref_free_map, cube, params, space, opt, amb)


def port_td(range_cube, params, space: SingleScaleSpace, opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """Our C restatement of td_grft (oracle/ds_oracle.c oracle_td_grft)."""
    lib = port()
    return _single_call(lib.oracle_td_grft, lib, lib.oracle_free_map, range_cube, params, space, opt)


def port_kt(cube, params, amb: AmbiguitySpace, space: SingleScaleSpace,
            opt: Optional[DetectorOptions] = None) -> DetectionMap:
    """Our C restatement of kt_mfp (oracle/ds_oracle.c oracle_kt_mfp)."""
    lib = port()
    return _single_call(lib.oracle_kt_mfp, lib, lib.oracle_free_map, cube, params, space, opt, amb)


def ref_extract_single(m: DetectionMap, gamma: float, max_out: int = 4096) -> np.ndarray:
    """(statistic, c0..c3, flat) rows of the reference's extract_detections on an FD map."""
    from paper_2403_06788_b200.detection import _to_c
    lib = ref()
    cm, keep = _to_c(m)
    s = m.single.to_c()
    rows = np.zeros((max_out, 6))
    n = C.c_int(0)
    _check(lib.ref_extract_single(C.byref(cm), C.byref(s), gamma, max_out, _vp(rows), C.byref(n)), lib)
    return rows[: n.value]


# ------------------------------------------------- run_pd (reference, C++) ---
def ref_run_pd(sc, threads: int = 0):
    """ltci::run_pd on a montecarlo.Scenario; list of (snr, pd, trials, lo, hi) per detector."""
    lib = ref()
    c = sc.to_c()
    out = (A.CPdPoint * (max(1, len(sc.detectors) * len(sc.snr_db))))()
    _check(lib.ref_run_pd(C.byref(c), threads or os.cpu_count() or 1, out), lib)
    n = len(sc.snr_db)
    return [[(o.snr_db, o.pd, o.trials, o.ci_lo, o.ci_hi) for o in out[i * n:(i + 1) * n]]
            for i in range(len(sc.detectors))]
