"""ctypes mirrors of the POD structs in include/ltci_cuda.h.

Shared by the product loader (_lib.py) and by the test-only oracle wrappers,
which take the same plan structs.
"""
from __future__ import annotations

import ctypes as C

MAX_ORDER = 4
MAX_AXES = 12

OK, INVALID_ARGUMENT, CONDITION_VIOLATED, RUNTIME_ERROR, BAD_ALLOC, NO_DEVICE, IO_ERROR, OUT_OF_RANGE = range(8)
FD_GRFT, TD_GRFT, KT_MFP, DS_GRFT, DS_KT_MFP = range(5)
AXIS_RANGE, AXIS_VELOCITY, AXIS_HIGHER, AXIS_DOPPLER, AXIS_COARSE, AXIS_FINE, AXIS_FOLDING = range(7)
VARIANT_GRFT, VARIANT_KTMFP = 0, 1
FINE_AUTO, FINE_FFT_CUDA_CORE, FINE_TC_DENSE, FINE_TC_FAST = 0, 1, 2, 3


class CRadar(C.Structure):
    _fields_ = [("fc", C.c_double), ("fs", C.c_double), ("Br", C.c_double), ("delta_f", C.c_double),
                ("PRF", C.c_double), ("M", C.c_int32), ("K", C.c_int32), ("K_valid", C.c_int32)]


class CGrid(C.Structure):
    _fields_ = [("start", C.c_double), ("step", C.c_double), ("count", C.c_int32)]


class CDualSpace(C.Structure):
    _fields_ = [("radar", CRadar), ("order", C.c_int32),
                ("coarse", CGrid * MAX_ORDER), ("fine", CGrid * MAX_ORDER),
                ("rm_step", C.c_double * MAX_ORDER), ("dfm_step", C.c_double * MAX_ORDER),
                ("alpha", C.c_double * MAX_ORDER), ("kappa", C.c_double),
                ("roi_first", C.c_int32), ("roi_last", C.c_int32)]


class CSingleSpace(C.Structure):
    _fields_ = [("radar", CRadar), ("order", C.c_int32), ("c", CGrid * MAX_ORDER),
                ("rm_step", C.c_double * MAX_ORDER), ("dfm_step", C.c_double * MAX_ORDER),
                ("alpha", C.c_double * MAX_ORDER), ("roi_first", C.c_int32), ("roi_last", C.c_int32)]


class CAmbiguity(C.Structure):
    _fields_ = [("q_min", C.c_int32), ("q_max", C.c_int32)]


class COptions(C.Structure):
    _fields_ = [("retain_threshold", C.c_double), ("keep_dense", C.c_int32), ("threads", C.c_int32),
                ("keystone_taps", C.c_int32), ("trajectory", C.c_int32), ("fine_path", C.c_int32),
                ("device", C.c_int32)]


class CAxis(C.Structure):
    _fields_ = [("role", C.c_int32), ("order", C.c_int32), ("size", C.c_int32)]


class CDetectionMap(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_axes", C.c_int32), ("axes", CAxis * MAX_AXES),
                ("counters", C.c_uint64 * 4), ("retain_threshold", C.c_double),
                ("doppler_first", C.c_int32), ("argmax", C.c_uint64), ("argmax_value", C.c_double * 2),
                ("n_candidates", C.c_uint64), ("cand_index", C.POINTER(C.c_uint64)),
                ("cand_value", C.POINTER(C.c_double)), ("dense_stored", C.c_int32),
                ("dense_count", C.c_uint64), ("dense", C.POINTER(C.c_double)),
                ("n_rows", C.c_int32), ("peak_index", C.POINTER(C.c_uint64)),
                ("peak_value", C.POINTER(C.c_double))]


PMap = C.POINTER(CDetectionMap)


class CDetection(C.Structure):
    _fields_ = [("statistic", C.c_double), ("c", C.c_double * (MAX_ORDER + 1)), ("n_coef", C.c_int32),
                ("has_q", C.c_int32), ("q", C.c_int32), ("baseband_velocity", C.c_double),
                ("flat_index", C.c_uint64)]


class CCubeHeader(C.Structure):
    _fields_ = [("domain", C.c_int32), ("radar", CRadar), ("sigma2", C.c_double)]


MAX_TARGETS = 8
MAX_SNR = 64


class CTarget(C.Structure):
    _fields_ = [("amp", C.c_double * 2), ("order", C.c_int32), ("c", C.c_double * (MAX_ORDER + 1))]


class CScenario(C.Structure):
    _fields_ = [("radar", CRadar), ("n_targets", C.c_int32), ("targets", CTarget * MAX_TARGETS),
                ("n_snr", C.c_int32), ("snr_db", C.c_double * MAX_SNR), ("trials", C.c_int32),
                ("pfa", C.c_double), ("sigma2", C.c_double), ("seed", C.c_uint64),
                ("n_detectors", C.c_int32), ("detectors", C.c_int32 * 5), ("P", C.c_int32),
                ("bound_lo", C.c_double * MAX_ORDER), ("bound_hi", C.c_double * MAX_ORDER),
                ("alpha", C.c_double * MAX_ORDER), ("roi_first", C.c_int32), ("roi_last", C.c_int32),
                ("keystone_taps", C.c_int32), ("device", C.c_int32)]


class CPdPoint(C.Structure):
    _fields_ = [("snr_db", C.c_double), ("pd", C.c_double), ("trials", C.c_int32), ("ci_lo", C.c_double),
                ("ci_hi", C.c_double)]
