"""B200-native dual-scale GRFT / DS-KT-MFP detectors (arXiv 2403.06788).

The hot path -- coarse range-migration correction, fine Doppler-migration
correction and the fused statistic reduction -- runs as hand-written sm_100a
CUDA kernels behind the C-ABI in include/ltci_cuda.h (lib/libltci_cuda.so),
with the reference's C++ detector API as the drop-in (lib/libltci_b200.so).
"""
from .model import (AmbiguitySpace, Bounds, DetectionMap, DetectorOptions, DualScaleSpace, Grid, RadarParams,
                    RangeRoi, SingleScaleSpace, StepSizes, build_ambiguity, build_dual_scale, build_single_scale, step_sizes,
                    split_velocity)
from .detectors import (Engine, detection_threshold, ds_grft, ds_kt_mfp, fd_grft, gft, keystone, kt_mfp, mgift,
                        range_fft, td_grft)
from .detection import Detection, extract_detections
from .cube_io import CubeFile, cube_file_info, read_cube_file, write_cube_file

__all__ = [
    "AmbiguitySpace", "Bounds", "DetectionMap", "DetectorOptions", "DualScaleSpace", "Grid", "RadarParams",
    "RangeRoi", "StepSizes", "build_ambiguity", "build_dual_scale", "step_sizes", "split_velocity", "Engine",
    "detection_threshold", "ds_grft", "ds_kt_mfp", "fd_grft", "td_grft", "kt_mfp", "gft", "keystone", "mgift", "range_fft", "SingleScaleSpace",
    "build_single_scale", "Detection", "extract_detections",
    "CubeFile", "cube_file_info", "read_cube_file", "write_cube_file",
]
