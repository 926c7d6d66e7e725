"""One fd_grft call on the bench_fd workload (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_06788_b200 import Bounds, DetectorOptions, RangeRoi, build_single_scale, fd_grft  # noqa: E402
from paper_2403_06788_b200.configs import config  # noqa: E402
from paper_2403_06788_b200.detectors import detection_threshold  # noqa: E402

w = config(0)
s = build_single_scale(w.params, 2, [Bounds(-150.0, 150.0), Bounds(-5.0, 5.0)], [0.5, 0.5], RangeRoi.full(w.params))
m = fd_grft(w.cube(), w.params, s, DetectorOptions(retain_threshold=detection_threshold(w.params, w.sigma2, 1e-6)))
print("cells", s.cells(), "argmax", m.argmax, abs(m.argmax_value), "candidates", m.cand_index.size)
