"""Per-call latency of the one-shot C-ABI detectors at the reference's desk
scale (acceptance criterion 7's wall-clock scenario, proj/tests/acceptance/
acceptance.cpp:429-447): repeated ds_grft / ds_kt_mfp calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_06788_b200 import DetectorOptions, ds_grft, ds_kt_mfp
from paper_2403_06788_b200.model import Bounds, RadarParams, RangeRoi, build_dual_scale, build_ambiguity
from paper_2403_06788_b200 import scene

p = RadarParams.create(1.6e9, 100e6, 95.5e6, 320.0, 128, 256)
bin_ = p.Va() / p.M
s = build_dual_scale(p, 2, [Bounds(0.0, 104 * bin_), Bounds(-1.9, 1.9)], [0.75, 0.25], RangeRoi(185, 235))
cube = scene.synthesize_cube(p, [(1.0, [200 * p.delta_R(), 81 * bin_, -1.25])])
opt = DetectorOptions()
for i in range(6):
    t = time.perf_counter(); ds_grft(cube, p, s, opt); dt = time.perf_counter() - t
    print(f"ds_grft call {i}: {dt*1e3:.2f} ms", flush=True)
amb = build_ambiguity(p, Bounds(0.0, 104 * bin_))
for i in range(4):
    t = time.perf_counter(); ds_kt_mfp(cube, p, amb, s, opt); dt = time.perf_counter() - t
    print(f"ds_kt_mfp call {i}: {dt*1e3:.2f} ms", flush=True)
