"""fd_grft measurement: the single-scale FD-GRFT
search on the BASELINE configs[0] radar (512 x 256), full single-scale grid
(build_single_scale at the DFM steps, alpha 1/2, 1/2, bounds v +-150, c2 +-5,
every range cell), through the public API (host cube in, map out).

Prints one JSON line: GPU fd_grft time and matched-filter integrations/s
(cells x K x M), the same for the reference's fd_grft on a bounded slice of
the grid (all host threads), and DS-GRFT on the same radar for the paper's
FD-vs-DS comparison (PAPER Table IV: 174x on a CPU).

    python scripts/bench_fd.py [--reps 5] [--cpu-seconds 15]
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

from paper_2403_06788_b200 import Bounds, DetectorOptions, RangeRoi, build_single_scale, ds_grft, fd_grft  # noqa
from paper_2403_06788_b200.configs import config  # noqa: E402
from paper_2403_06788_b200.detectors import detection_threshold  # noqa: E402


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
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    a = ap.parse_args()
    w = config(0)
    p = w.params
    x = w.cube()
    bounds = [Bounds(-150.0, 150.0), Bounds(-5.0, 5.0)]
    s = build_single_scale(p, 2, bounds, [0.5, 0.5], RangeRoi.full(p))
    gamma = detection_threshold(p, w.sigma2, 1e-6)
    opt = DetectorOptions(retain_threshold=gamma, threads=0)
    cells = s.cells()
    mf = cells * p.K * p.M
    fd_grft(x, p, s, opt)  # warm-up (module load, workspace)
    t_fd, t_fd_med = best_of(lambda: fd_grft(x, p, s, opt), a.reps)
    ds_grft(x, p, w.space, opt)
    t_ds, t_ds_med = best_of(lambda: ds_grft(x, p, w.space, opt), a.reps)
    m = fd_grft(x, p, s, opt)
    out = {"workload": "fd_grft, C0 radar 512x256, single-scale grid v +-150 (x%d) c2 +-5 (x%d), full range"
                       % (s.c[0].count, s.c[1].count),
           "cells": cells, "mf_integrations": mf, "candidates": int(m.cand_index.size),
           "gpu": {"fd_ms": 1e3 * t_fd, "fd_ms_median": 1e3 * t_fd_med,
                   "fd_mf_integrations_per_s_G": mf / t_fd / 1e9,
                   "ds_grft_ms_same_radar": 1e3 * t_ds, "ds_over_fd_speedup": t_fd / t_ds,
                   "note": "public API wall time: host f64 cube in, sorted map out"}}
    try:
        import oracle as O
        if O.have_ref():
            # bounded sample: a velocity slice of the same grid, every other axis whole
            threads = os.cpu_count() or 1
            per_v = p.K * p.M * s.c[1].count
            nv = int(max(threads, min(s.c[0].count, a.cpu_seconds * 1.5e9 * threads / 8 / per_v)))
            sl = build_single_scale(p, 2, bounds, [0.5, 0.5], RangeRoi.full(p))
            sl.c[0].count = nv
            t0 = time.perf_counter()
            O.ref_fd(x, p, sl, DetectorOptions(retain_threshold=gamma, threads=threads))
            dt = time.perf_counter() - t0
            rate = sl.cells() * p.K * p.M / dt
            out["cpu_reference"] = {"fd_mf_integrations_per_s_G": rate / 1e9, "cores": threads,
                                    "sample": f"{sl.cells()} of {cells} cells (velocity slice {nv}) in {dt:.2f} s",
                                    "fd_full_grid_s_extrapolated": mf / rate}
            out["gpu_over_cpu_fd"] = (mf / t_fd) / rate
    except Exception as e:  # the reference build is optional on the box
        out["cpu_reference"] = f"unavailable: {e}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
