"""td_grft / kt_mfp measurement: the two single-scale baselines of the paper on the BASELINE
configs[0] radar (512 x 256), through the public API (host cube in, map out), with the
reference's own td_grft / kt_mfp timed on a bounded slice of the same grids (all host threads).

One JSON line: GPU wall time per call, trajectory integrations/s (cells x R x M for td_grft;
cells x R x M x M hypothesis x pulse for kt_mfp), and the CPU rates.

    python scripts/bench_td.py [--reps 5] [--cpu-seconds 10]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_06788_b200 import (Bounds, DetectorOptions, RangeRoi, build_ambiguity, build_single_scale, kt_mfp,  # noqa
                                   td_grft)
from paper_2403_06788_b200.configs import config  # noqa: E402
from paper_2403_06788_b200.detectors import detection_threshold  # noqa: E402
from paper_2403_06788_b200.model import Grid  # noqa: E402


def best_of(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    a = ap.parse_args()
    w = config(0)
    p = w.params
    xf = w.cube()
    xr = np.fft.ifft(xf, axis=1) * p.K  # range_ifft (unnormalised dft_plus per pulse): the range-pulse cube
    s = build_single_scale(p, 2, [Bounds(-150.0, 150.0), Bounds(-5.0, 5.0)], [0.5, 0.5], RangeRoi.full(p))
    gamma = detection_threshold(p, w.sigma2, 1e-6)
    opt = DetectorOptions(retain_threshold=gamma, threads=0)
    R = s.roi.count()
    td_cells = s.cells()
    td_integ = td_cells * R * p.M
    td_grft(xr, p, s, opt)
    t_td, t_td_med = best_of(lambda: td_grft(xr, p, s, opt), a.reps)
    amb = build_ambiguity(p, Bounds(-150.0, 150.0))
    kt_cells = amb.count() * s.c[1].count
    kt_integ = kt_cells * R * p.M * p.M
    kt_mfp(xf, p, amb, s, opt)
    t_kt, t_kt_med = best_of(lambda: kt_mfp(xf, p, amb, s, opt), a.reps)
    out = {"workload": "C0 radar 512x256, single-scale grid v +-150 (x%d) c2 +-5 (x%d), full range; kt_mfp: %d folding "
                       "numbers x %d accelerations" % (s.c[0].count, s.c[1].count, amb.count(), s.c[1].count),
           "td_grft": {"cells": td_cells, "integrations": td_integ, "gpu_ms": 1e3 * t_td, "gpu_ms_median": 1e3 * t_td_med,
                       "gpu_G_per_s": td_integ / t_td / 1e9},
           "kt_mfp": {"cells": kt_cells, "integrations": kt_integ, "gpu_ms": 1e3 * t_kt, "gpu_ms_median": 1e3 * t_kt_med,
                      "gpu_G_per_s": kt_integ / t_kt / 1e9},
           "note": "public API wall time: host f64 cube in, sorted map out"}
    try:
        import oracle as O
        if O.have_ref():
            threads = os.cpu_count() or 1
            # bounded samples: a velocity slice of the td grid, an acceleration slice of the kt grid
            g0 = s.c[0]
            nv = max(threads, 16)
            while True:
                sl = build_single_scale(p, 2, [Bounds(-150.0, 150.0), Bounds(-5.0, 5.0)], [0.5, 0.5], RangeRoi.full(p))
                sl.c[0] = Grid(g0.start, g0.step, nv)
                t0 = time.perf_counter()
                O.ref_td(xr, p, sl, opt)
                dt = time.perf_counter() - t0
                if dt > a.cpu_seconds / 4 or nv >= g0.count:
                    break
                nv = min(g0.count, nv * 4)
            integ = sl.cells() * R * p.M
            out["td_grft"]["cpu_reference"] = {"G_per_s": integ / dt / 1e9, "seconds": dt, "threads": threads,
                                               "sample": "%d of %d velocity cells" % (nv, g0.count)}
            out["td_grft"]["speedup"] = out["td_grft"]["gpu_G_per_s"] / (integ / dt / 1e9)
            sk = build_single_scale(p, 2, [Bounds(-150.0, 150.0), Bounds(-5.0, 5.0)], [0.5, 0.5], RangeRoi.full(p))
            g1 = s.c[1]
            na = min(g1.count, max(1, threads // amb.count()) * 2)
            sk.c[1] = Grid(g1.start, g1.step, na)
            t0 = time.perf_counter()
            O.ref_kt(xf, p, amb, sk, opt)
            dt = time.perf_counter() - t0
            integ = amb.count() * na * R * p.M * p.M
            out["kt_mfp"]["cpu_reference"] = {"G_per_s": integ / dt / 1e9, "seconds": dt, "threads": threads,
                                              "sample": "%d of %d accelerations" % (na, g1.count)}
            out["kt_mfp"]["speedup"] = out["kt_mfp"]["gpu_G_per_s"] / (integ / dt / 1e9)
    except Exception as e:  # reported, not fatal
        out["cpu_reference_error"] = str(e)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
