"""Per-call latency of the one-shot C-ABI detectors at the reference's desk
scale: repeated ds_grft / ds_kt_mfp calls (acceptance criterion 7's
wall-clock scenario, proj/tests/acceptance/acceptance.cpp:429-447) and the
noise-only fd_grft trials of criterion 6 (100 000 calls inside 60 s,
proj/tests/acceptance/acceptance.cpp:361-386).  Prints one JSON line per
scenario with the median / mean per-call latency."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2403_06788_b200 import DetectorOptions, ds_grft, ds_kt_mfp, fd_grft
from paper_2403_06788_b200.model import (Bounds, RadarParams, RangeRoi, build_dual_scale, build_ambiguity,
                                         build_single_scale)
from paper_2403_06788_b200 import scene


def timed(name, fn, n):
    fn()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    ts = np.array(ts) * 1e3
    print(json.dumps({"scenario": name, "calls": n, "median_ms": float(np.median(ts)), "mean_ms": float(ts.mean()),
                      "p90_ms": float(np.percentile(ts, 90))}), flush=True)


p = RadarParams.create(1.6e9, 100e6, 95.5e6, 320.0, 128, 256)
bin_ = p.Va() / p.M
s = build_dual_scale(p, 2, [Bounds(0.0, 104 * bin_), Bounds(-1.9, 1.9)], [0.75, 0.25], RangeRoi(185, 235))
cube = scene.synthesize_cube(p, [(1.0, [200 * p.delta_R(), 81 * bin_, -1.25])])
opt = DetectorOptions()
timed("ds_grft criterion-7 desk scale", lambda: ds_grft(cube, p, s, opt), 50)
amb = build_ambiguity(p, Bounds(0.0, 104 * bin_))
timed("ds_kt_mfp criterion-7 desk scale", lambda: ds_kt_mfp(cube, p, amb, s, opt), 50)

# criterion 6: 16 x 32 noise cube, one velocity cell, dense map
p6 = RadarParams.create(4.0 * 100e6, 100e6, 50e6, 2000.0, 16, 32)
s6 = build_single_scale(p6, 1, [Bounds(0.0, 0.0)], [1.0], RangeRoi(0, p6.K - 1))
c6 = scene.add_noise(np.zeros((p6.M, p6.K), dtype=np.complex128), 1.7, 60000)
o6 = DetectorOptions(keep_dense=True)
timed("fd_grft criterion-6 noise trial", lambda: fd_grft(c6, p6, s6, o6), 2000)
