"""Loader for the in-tree CUDA library (lib/libltci_cuda.so).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, calls raise.  Build with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2403_06788_b200/csrc all``.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _cabi as A

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.environ.get("LTCI_LIB_PATH") or os.path.join(LIB_DIR, "libltci_cuda.so")  # override: experiments
DROPIN_PATH = os.path.join(LIB_DIR, "libltci_b200.so")

# Every symbol include/ltci_cuda.h declares.
EXPORTS = (
    "ltci_cuda_ds_grft", "ltci_cuda_ds_kt_mfp", "ltci_cuda_free_map", "ltci_cuda_keystone", "ltci_cuda_keystone_device", "ltci_cuda_range_fft", "ltci_cuda_range_fft_device", "ltci_engine_run_range_device", "ltci_engine_run_range_host",
    "ltci_cuda_mgift", "ltci_cuda_gft", "ltci_cuda_detection_threshold", "ltci_engine_create",
    "ltci_engine_destroy", "ltci_engine_run_device", "ltci_engine_run_host", "ltci_engine_result",
    "ltci_engine_peaks_device", "ltci_engine_stats", "ltci_engine_set_timing", "ltci_engine_fine_path", "ltci_engine_coarse_path",
    "ltci_engine_work", "ltci_engine_run_file", "ltci_engine_set_coarse_slice", "ltci_cuda_merge_peaks", "ltci_cuda_fd_grft", "ltci_cuda_td_grft", "ltci_cuda_kt_mfp", "ltci_cuda_extract_detections_single",
    "ltci_cuda_extract_detections", "ltci_cuda_cube_file_info", "ltci_cuda_cube_file_read",
    "ltci_cuda_cube_file_write", "ltci_cuda_synthesize", "ltci_cuda_add_noise", "ltci_cuda_run_pd", "ltci_cuda_measure_fp32_peak", "ltci_cuda_pool_idle", "ltci_cuda_last_error", "ltci_cuda_version",
)

_lib = None


class LtciError(RuntimeError):
    pass


class ConditionViolated(LtciError):
    """Mirror of ltci::ConditionViolated (proj/include/ltci/common.hpp:17-20)."""


class IoError(LtciError):
    """Mirror of ltci::IoError (proj/include/ltci/common.hpp:36-39)."""


def raise_for(rc: int, lib) -> None:
    if rc == A.OK:
        return
    msg = lib.ltci_cuda_last_error().decode(errors="replace")
    if rc == A.INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == A.CONDITION_VIOLATED:
        raise ConditionViolated(msg)
    if rc == A.BAD_ALLOC:
        raise MemoryError(msg)  # std::bad_alloc
    if rc == A.IO_ERROR:
        raise IoError(msg)
    if rc == A.OUT_OF_RANGE:
        raise IndexError(msg)  # std::out_of_range
    raise LtciError(msg)


def load():
    """Load libltci_cuda.so (raises OSError when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built; run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    if os.environ.get("LTCI_LIB_PATH"):
        # A/B experiments may load an older build: bind what it exports
        class _Tolerant:
            def __init__(self, real):
                object.__setattr__(self, "_real", real)

            def __getattr__(self, name):
                try:
                    return getattr(self._real, name)
                except AttributeError:
                    return C.CFUNCTYPE(C.c_int)()  # placeholder; calling it is an error

            def __setattr__(self, name, value):
                setattr(self._real, name, value)
        lib = _Tolerant(lib)
    P = C.POINTER
    vp = C.c_void_p
    lib.ltci_cuda_ds_grft.argtypes = [vp, P(A.CRadar), P(A.CDualSpace), P(A.COptions), P(A.PMap)]
    lib.ltci_cuda_ds_kt_mfp.argtypes = [vp, P(A.CRadar), P(A.CAmbiguity), P(A.CDualSpace), P(A.COptions),
                                        P(A.PMap)]
    lib.ltci_cuda_free_map.argtypes = [A.PMap]
    lib.ltci_cuda_free_map.restype = None
    lib.ltci_cuda_keystone.argtypes = [vp, P(A.CRadar), C.c_int, vp]
    lib.ltci_cuda_keystone_device.argtypes = [vp, vp, P(A.CRadar), C.c_int, vp]
    lib.ltci_cuda_range_fft.argtypes = [vp, P(A.CRadar), vp]
    lib.ltci_cuda_range_fft_device.argtypes = [vp, vp, P(A.CRadar), vp]
    lib.ltci_engine_run_range_device.argtypes = [vp, vp, vp]
    lib.ltci_engine_run_range_host.argtypes = [vp, vp, vp]
    lib.ltci_cuda_mgift.argtypes = [vp, P(A.CRadar), P(C.c_double), C.c_int, C.c_int, vp]
    lib.ltci_cuda_gft.argtypes = [vp, P(A.CRadar), P(C.c_double), C.c_int, C.c_int, C.c_int, vp]
    lib.ltci_cuda_detection_threshold.argtypes = [P(A.CRadar), C.c_double, C.c_double, C.c_int, P(C.c_int)]
    lib.ltci_cuda_detection_threshold.restype = C.c_double
    lib.ltci_engine_create.argtypes = [P(A.CRadar), P(A.CDualSpace), P(A.CAmbiguity), C.c_int, P(A.COptions),
                                       C.c_int, C.c_int, P(vp)]
    lib.ltci_engine_destroy.argtypes = [vp]
    lib.ltci_engine_destroy.restype = None
    lib.ltci_engine_run_device.argtypes = [vp, vp, vp]
    lib.ltci_engine_run_host.argtypes = [vp, vp, vp]
    lib.ltci_engine_result.argtypes = [vp, vp, P(A.PMap)]
    lib.ltci_engine_peaks_device.argtypes = [vp, P(vp), P(C.c_int32)]
    lib.ltci_engine_stats.argtypes = [vp, P(C.c_int64), P(C.c_double), P(C.c_double), P(C.c_double)]
    lib.ltci_engine_set_timing.argtypes = [vp, C.c_int]
    lib.ltci_engine_work.argtypes = [vp, P(C.c_uint64), P(C.c_uint64)]
    lib.ltci_engine_fine_path.argtypes = [vp, P(C.c_int32), P(C.c_int32)]
    lib.ltci_engine_coarse_path.argtypes = [vp, P(C.c_int32)]
    lib.ltci_cuda_measure_fp32_peak.argtypes = [C.c_int, P(C.c_double)]
    lib.ltci_cuda_pool_idle.argtypes = [C.c_int, P(C.c_int64), P(C.c_int64)]
    lib.ltci_cuda_extract_detections.argtypes = [P(A.CDetectionMap), P(A.CDualSpace), P(A.CAmbiguity), C.c_double,
                                                 P(A.CDetection), C.c_int, P(C.c_int)]
    lib.ltci_cuda_cube_file_info.argtypes = [C.c_char_p, P(A.CCubeHeader)]
    lib.ltci_cuda_cube_file_read.argtypes = [C.c_char_p, P(A.CCubeHeader), vp, C.c_uint64]
    lib.ltci_cuda_cube_file_write.argtypes = [C.c_char_p, P(A.CCubeHeader), vp]
    lib.ltci_engine_run_file.argtypes = [vp, C.c_char_p, vp]
    lib.ltci_engine_set_coarse_slice.argtypes = [vp, C.c_uint64, C.c_uint64]
    lib.ltci_cuda_merge_peaks.argtypes = [vp, C.c_int, C.c_int, vp, vp]
    lib.ltci_cuda_synthesize.argtypes = [P(A.CRadar), C.c_int, P(A.CTarget), vp]
    lib.ltci_cuda_add_noise.argtypes = [vp, P(A.CRadar), C.c_double, C.c_uint64, vp]
    lib.ltci_cuda_run_pd.argtypes = [P(A.CScenario), P(A.CPdPoint)]
    lib.ltci_cuda_fd_grft.argtypes = [vp, P(A.CRadar), P(A.CSingleSpace), P(A.COptions), P(A.PMap)]
    lib.ltci_cuda_td_grft.argtypes = [vp, P(A.CRadar), P(A.CSingleSpace), P(A.COptions), P(A.PMap)]
    lib.ltci_cuda_kt_mfp.argtypes = [vp, P(A.CRadar), P(A.CAmbiguity), P(A.CSingleSpace), P(A.COptions), P(A.PMap)]
    lib.ltci_cuda_extract_detections_single.argtypes = [P(A.CDetectionMap), P(A.CSingleSpace), C.c_double,
                                                        P(A.CDetection), C.c_int, P(C.c_int)]
    lib.ltci_cuda_last_error.restype = C.c_char_p
    lib.ltci_cuda_version.restype = C.c_int
    _lib = lib
    return lib
