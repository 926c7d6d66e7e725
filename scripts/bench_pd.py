"""Monte-Carlo Pd measurement: a Fig. 7(a)-style Pd
sweep on the BASELINE configs[0] radar (512 x 256, one target at cell 200,
v = 87 m/s, c2 = 2), DS-GRFT, every trial's cube generated and searched on the
GPU (ltci_cuda_run_pd), against the reference's run_pd on the host cores on a
bounded sample (fewer trials, one SNR point).  Rate = trials/s.

    python scripts/bench_pd.py [--trials 100] [--cpu-trials 16]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_06788_b200 import _cabi as A  # noqa: E402
from paper_2403_06788_b200.configs import config  # noqa: E402
from paper_2403_06788_b200.model import Bounds, RangeRoi  # noqa: E402
from paper_2403_06788_b200.montecarlo import Scenario, run_pd  # noqa: E402


def scenario(snr, trials, detectors):
    w = config(0)
    p = w.params
    return Scenario(params=p, targets=[(1.0 + 0j, [200 * p.delta_R(), 87.0, 2.0])], snr_db=snr, trials=trials,
                    pfa=1e-6, sigma2=1.0 / p.K, seed=2024, detectors=detectors, P=2,
                    bounds=[Bounds(-150.0, 150.0), Bounds(-5.0, 5.0)], alpha=[0.5, 0.5], roi=RangeRoi.full(p))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=100)
    ap.add_argument("--cpu-trials", type=int, default=16)
    a = ap.parse_args()
    snr = [-22.0, -20.0, -18.0, -16.0, -14.0, -12.0]
    det = [A.DS_GRFT]
    run_pd(scenario([-10.0], 2, det))  # warm-up
    t0 = time.perf_counter()
    curves = run_pd(scenario(snr, a.trials, det))
    dt = time.perf_counter() - t0
    n = a.trials * len(snr)
    out = {"workload": "run_pd, C0 radar 512x256, DS-GRFT, target cell 200 v 87 c2 2, pfa 1e-6, "
                       f"{len(snr)} SNR points x {a.trials} trials",
           "gpu": {"seconds": dt, "trials_per_s": n / dt,
                   "curve": [(p.snr_db, p.pd, p.ci_lo, p.ci_hi) for p in curves[0].points]}}
    try:
        import oracle as O
        if O.have_ref():
            threads = os.cpu_count() or 1
            t0 = time.perf_counter()
            ref = O.ref_run_pd(scenario([-16.0], a.cpu_trials, det), threads)
            dt_c = time.perf_counter() - t0
            out["cpu_reference"] = {"trials_per_s": a.cpu_trials / dt_c, "cores": threads,
                                    "sample": f"{a.cpu_trials} trials at -16 dB in {dt_c:.1f} s", "pd": ref[0][0][1]}
            out["gpu_over_cpu"] = (n / dt) / (a.cpu_trials / dt_c)
    except Exception as e:  # the reference build is optional on the box
        out["cpu_reference"] = f"unavailable: {e}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
