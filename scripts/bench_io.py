"""Wire-path measurement: "LTCI" cube file -> device.

Times, on the C1 cube (2048 x 1024, 33.6 MB f64 payload, page-cached):
  read_host     library read_cube_file into a host buffer (GB/s of payload)
  run_file      Engine.run_file: chunked fread into pinned staging overlapped
                with async H2D + f64->c64 + the full detector step
  run_host      Engine.run_host from a pageable host array (same step)
  ref_read      the reference's read_cube_file (oracle/_ref), when present
Prints one JSON line.  Usage: python scripts/bench_io.py [--config 1] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_06788_b200 import DetectorOptions  # noqa: E402
from paper_2403_06788_b200.configs import config  # noqa: E402
from paper_2403_06788_b200.cube_io import CubeFile, read_cube_file, write_cube_file  # noqa: E402
from paper_2403_06788_b200.detectors import Engine  # noqa: E402


def _best(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    w = config(a.config)
    x = w.cube(noise=True)
    gamma = float(np.sqrt(-w.params.M * w.params.K * w.sigma2 * np.log(1e-6)))
    payload = 16 * x.size
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "cpi.bin")
        write_cube_file(path, CubeFile.from_cube(x, w.params, w.sigma2))
        read_host = _best(lambda: read_cube_file(path), a.reps)
        eng = Engine(w.params, w.space, w.variant, w.amb, DetectorOptions(retain_threshold=gamma))
        for _ in range(2):
            eng.run_file(path)
            eng.run_host(x)
        torch.cuda.synchronize()

        def step_file():
            eng.run_file(path)
            torch.cuda.synchronize()

        def step_host():
            eng.run_host(x)
            torch.cuda.synchronize()

        run_file = _best(step_file, a.reps)
        run_host = _best(step_host, a.reps)
        out = {"workload": w.name, "payload_bytes": payload,
               "read_host_GBps": payload / read_host[0] / 1e9,
               "run_file_ms": {"best": 1e3 * run_file[0], "median": 1e3 * run_file[1]},
               "run_host_ms": {"best": 1e3 * run_host[0], "median": 1e3 * run_host[1]},
               "file_overhead_ms": 1e3 * (run_file[1] - run_host[1])}
        try:
            import oracle as O
            if O.have_ref():
                ref = _best(lambda: O.ref_read_cube_file(path, x.size), a.reps)
                out["ref_read_GBps"] = payload / ref[0] / 1e9
        except Exception as e:  # the reference build is optional on the box
            out["ref_read"] = f"unavailable: {e}"
        eng.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
