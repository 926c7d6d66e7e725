"""Detections from a dual-scale map.

``extract_detections(map, gamma)`` mirrors ltci::extract_detections
(proj/src/detection.cpp:158-244) and returns ``Detection`` records with the
motion estimate of ltci::detection_from_cell (proj/src/detection.cpp:124-153).
The work runs in the library's C++ (csrc/detection.cpp) over the candidate
list the GPU returned.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _cabi as A
from . import _lib
from .model import DetectionMap


@dataclass
class Detection:
    estimate: List[float] = field(default_factory=list)  # c0 (range) .. cP
    statistic: float = 0.0
    flat_index: int = 0
    q: Optional[int] = None
    baseband_velocity: Optional[float] = None


def _to_c(m: DetectionMap):
    """Borrowed C view of a Python map (arrays kept alive by the returned tuple)."""
    c = A.CDetectionMap()
    c.kind = m.kind
    c.n_axes = len(m.axes)
    for i, ax in enumerate(m.axes):
        c.axes[i] = A.CAxis(ax.role, ax.order, ax.size)
    c.retain_threshold = m.retain_threshold
    c.doppler_first = m.doppler_first
    idx = np.ascontiguousarray(m.cand_index, dtype=np.uint64)
    val = np.ascontiguousarray(m.cand_value, dtype=np.complex128)
    c.n_candidates = idx.size
    c.cand_index = idx.ctypes.data_as(C.POINTER(C.c_uint64))
    c.cand_value = val.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))
    return c, (idx, val)


def extract_detections(m: DetectionMap, gamma: float) -> List[Detection]:
    lib = _lib.load()
    cm, keep = _to_c(m)
    cap = max(16, min(int(m.cand_index.size), 1 << 20))
    n = C.c_int(0)
    if m.kind == A.FD_GRFT:
        ss = m.single.to_c()

        def call(buf, k):
            return lib.ltci_cuda_extract_detections_single(C.byref(cm), C.byref(ss), gamma, buf, k, C.byref(n))
    else:
        s = m.dual.to_c()
        a = m.amb.to_c() if m.amb is not None else None

        def call(buf, k):
            return lib.ltci_cuda_extract_detections(C.byref(cm), C.byref(s), C.byref(a) if a is not None else None,
                                                    gamma, buf, k, C.byref(n))
    out = (A.CDetection * cap)()
    _lib.raise_for(call(out, cap), lib)
    if n.value > cap:
        out = (A.CDetection * n.value)()
        _lib.raise_for(call(out, n.value), lib)
    del keep
    res = []
    for i in range(n.value):
        d = out[i]
        res.append(Detection(estimate=[d.c[k] for k in range(d.n_coef)], statistic=d.statistic,
                             flat_index=int(d.flat_index), q=int(d.q) if d.has_q else None,
                             baseband_velocity=float(d.baseband_velocity) if d.has_q else None))
    return res
