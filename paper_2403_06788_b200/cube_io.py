"""The reference's "LTCI" cube container.

Mirrors ltci::CubeFile / read_cube_file / write_cube_file
(proj/include/ltci/cube_io.hpp:9-32, proj/src/cube_io.cpp:38-179); the bytes
are parsed and written by the library's C++ (csrc/cube_io.cpp).  The wire path
``Engine.run_file`` streams a file straight into device memory through pinned
staging blocks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _cabi as A
from . import _lib
from .model import RadarParams, cube_as_f64

FREQ_PULSE, RANGE_PULSE = 0, 1


@dataclass
class CubeFile:
    domain: int = FREQ_PULSE
    params: RadarParams = field(default_factory=RadarParams)
    sigma2: float = 0.0
    data: np.ndarray = None  # complex128 (M, K): sample (k, m) at [m, k]

    def to_freq_cube(self) -> np.ndarray:
        # CubeFile::to_freq_cube (proj/src/cube_io.cpp:48-52)
        if self.domain != FREQ_PULSE:
            raise _lib.ConditionViolated("cube file holds range-pulse data, not freq-pulse")
        return self.data

    def to_range_cube(self) -> np.ndarray:
        if self.domain != RANGE_PULSE:
            raise _lib.ConditionViolated("cube file holds freq-pulse data, not range-pulse")
        return self.data

    @staticmethod
    def from_cube(cube: np.ndarray, params: RadarParams, sigma2: float = 0.0, domain: int = FREQ_PULSE):
        return CubeFile(domain, params, sigma2, cube_as_f64(cube, params))


def _header(h: A.CCubeHeader) -> tuple:
    return int(h.domain), RadarParams.from_c(h.radar), float(h.sigma2)


def cube_file_info(path: str):
    """(domain, params, sigma2) after every header/length check of read_cube_file."""
    lib = _lib.load()
    h = A.CCubeHeader()
    _lib.raise_for(lib.ltci_cuda_cube_file_info(str(path).encode(), C.byref(h)), lib)
    return _header(h)


def read_cube_file(path: str) -> CubeFile:
    lib = _lib.load()
    domain, params, _ = cube_file_info(path)
    out = np.empty((params.M, params.K), np.complex128)
    h = A.CCubeHeader()
    _lib.raise_for(lib.ltci_cuda_cube_file_read(str(path).encode(), C.byref(h), out.ctypes.data_as(C.c_void_p),
                                                2 * out.size), lib)
    domain, params, sigma2 = _header(h)
    return CubeFile(domain, params, sigma2, out)


def write_cube_file(path: str, cube: CubeFile) -> None:
    lib = _lib.load()
    data = cube_as_f64(cube.data, cube.params)
    h = A.CCubeHeader(cube.domain, cube.params.to_c(), cube.sigma2)
    _lib.raise_for(lib.ltci_cuda_cube_file_write(str(path).encode(), C.byref(h), data.ctypes.data_as(C.c_void_p)),
                   lib)
