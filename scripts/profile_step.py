"""One engine pass over a BASELINE workload (for ncu / compute-sanitizer runs)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_06788_b200 import _cabi as A, configs, scene  # noqa: E402
from paper_2403_06788_b200.detectors import Engine, detection_threshold  # noqa: E402
from paper_2403_06788_b200.model import DetectorOptions  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--fine-path", default="auto", choices=["auto", "fft", "tc", "tcfast"])
ap.add_argument("--coarse-v", type=int, default=0, help="slice the coarse velocity axis")
ap.add_argument("--coarse-rest", type=int, default=0, help="with --coarse-v: also slice the other coarse axes")
ap.add_argument("--front-end", default="auto", choices=["auto", "range", "freq"],
                help="range: feed the range-pulse echo through K0 (auto: range for configs[3], as bench.py)")
a = ap.parse_args()
w = configs.config(a.config)
if a.coarse_v:
    w = configs.sliced(w, a.coarse_v, a.coarse_rest)
fp = {"auto": A.FINE_AUTO, "fft": A.FINE_FFT_CUDA_CORE, "tc": A.FINE_TC_DENSE, "tcfast": A.FINE_TC_FAST}[a.fine_path]
opt = DetectorOptions(retain_threshold=detection_threshold(w.params, w.sigma2, 1e-6), fine_path=fp)
e = Engine(w.params, w.space, w.variant, w.amb, opt)
x = scene.to_complex64_roundtrip(w.cube())
front = a.front_end if a.front_end != "auto" else ("range" if a.config == 3 else "freq")
if front == "range":
    x = scene.to_complex64_roundtrip(np.fft.ifft(x, axis=1))  # range_ifft(y) / K: K0 returns y (same threshold)
for _ in range(a.runs):
    (e.run_range_host if front == "range" else e.run_host)(x)
m = e.result()
print(w.name, "argmax", m.argmax, abs(m.argmax_value), "candidates", m.cand_index.size, e.stats())
