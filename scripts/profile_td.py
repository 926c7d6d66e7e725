"""One td_grft call on the C0 radar's full single-scale grid (for ncu)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_06788_b200 import Bounds, DetectorOptions, RangeRoi, build_single_scale, td_grft
from paper_2403_06788_b200.configs import config
from paper_2403_06788_b200.detectors import detection_threshold
w = config(0)
p = w.params
xr = np.fft.ifft(w.cube(), axis=1) * p.K
s = build_single_scale(p, 2, [Bounds(-150.0, 150.0), Bounds(-5.0, 5.0)], [0.5, 0.5], RangeRoi.full(p))
m = td_grft(xr, p, s, DetectorOptions(retain_threshold=detection_threshold(p, w.sigma2, 1e-6)))
print("td_grft argmax", m.argmax, abs(m.argmax_value), "candidates", m.cand_index.size)
