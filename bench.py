#!/usr/bin/env python3
"""Benchmark of the DS-GRFT / DS-KT-MFP hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--impl b200|reference]

A step is one full dual-scale cascade (coarse RM gather -> fine DFM stage ->
fused threshold/argmax reduction) over one synthetic echo of the BASELINE
workload (default configs[1]: DS-GRFT 2nd order, 2048 x 1024, single B200).
Metric: hypothesis x pulse integrations per second (G/s), whole job.

value  device-timed (CUDA events on the launch stream, L2 flushed between
       steps), cube resident in HBM; with N > 1 ranks each rank owns a
       contiguous slice of range start cells and the per-cell peak map is
       all-gathered with NCCL (max-over-ranks timing).
e2e    the same metric through the public engine API from pinned host memory:
       H2D of the float64 cube, run, D2H of the reduced results, per step.
cpu_baseline  (rank 0, N = 1) the reference's own ds_grft/ds_kt_mfp compiled
       from its sources (oracle/_ref) on a bounded coarse-cell slice with all
       host threads.  --impl reference times that path alone.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


_T0 = time.perf_counter()


def log(msg):
    """Stage marker on stderr (stdout carries only the JSON line)."""
    print(f"[bench {time.perf_counter() - _T0:8.1f}s] {msg}", file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--fine-path", default="auto", choices=["auto", "fft", "tc", "tcfast"])
    ap.add_argument("--pfa", type=float, default=0.0,
                    help="per-cell false-alarm rate of the retention threshold; 0 = min(1e-6, 1e5 / hypotheses), "
                         "i.e. 1e-6 unless that would retain more than ~1e5 noise cells per CPI (C2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lanes", type=int, default=3, help="engine lanes for a CPI stream (configs[4])")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU sample length")
    ap.add_argument("--coarse-slice", type=int, default=0,
                    help="restrict the coarse-velocity axis (rate measurement of configs too large for one step)")
    ap.add_argument("--coarse-rest", type=int, default=0, help="with --coarse-slice: restrict the other coarse axes")
    ap.add_argument("--front-end", default="auto", choices=["auto", "range", "freq"],
                    help="input domain: range-pulse echo through K0 (range FFT) first, or the freq-pulse cube; "
                         "auto = range for configs[3] (its pipeline starts with the range FFT), freq otherwise")
    ap.add_argument("--shard", default="auto", choices=["auto", "rows", "coarse"],
                    help="one-CPI partition across ranks: coarse cells (no replicated work; default when every "
                         "rank gets one) or range cells")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.perf_counter()  # sampling is live before the timed region starts
            while not self.lines and time.perf_counter() - t0 < 3.0:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def count(self):
        return len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def fft_flops_per_row_cell(M: int, D: int) -> float:
    """Algorithmic flops of the CUDA-core fine path per (row, fine cell):
    chirp recurrence (1 complex multiply = 6 flop per sample) + M-point FFT
    (5 M log2 M) + |Y|^2 of the D window bins (3 flop each)."""
    import math
    return 6.0 * M + 5.0 * M * math.log2(M) + 3.0 * D


def metric_of(w):
    """(metric, unit) of a workload -- ONE definition for both arms, so the
    driver can divide them (BASELINE.json metric: G/s, CPIs/s for a stream)."""
    name = "DS-GRFT" if w.variant == 0 else "DS-KT-MFP"
    if w.cpis > 1:
        return f"{name} CPIs/s ({w.cpis}-CPI stream)", "CPI/s"
    return f"{name} motion-hypothesis x pulse integrations/s", "G/s"


def in_unit(w, gps: float) -> float:
    """A G/s rate in the workload's metric unit (CPI/s for a CPI stream)."""
    return gps * 1e9 / w.integrations() if w.cpis > 1 else gps


def n_coarse_cells(w) -> int:
    s = w.space
    return int(np.prod([g.count for g in s.coarse])) if w.variant == 0 else w.amb.count() * s.coarse[1].count


# coarse-stage (K1, plus K0/K4 for configs[3]) time relative to the fine stage,
# coarse / fine stage time on one B200 (profiles/r02_bench_c*.json): the transform kernel K1
# (C0 0.065, C3 0.022) and the interpolating gather K1g (C1 0.009, C4 0.013)
COARSE_OVER_FINE = {"transform": 0.03, "gather": 0.01}
# share of the coarse stage a range-cell shard repeats on every rank: all of it with K1 (the
# K-point transforms are needed whatever rows are kept), only the per-pulse tables with K1g
# (22 us of 0.92 ms at C1)
COARSE_REPEATED = {"transform": 1.0, "gather": 0.03}


def coarse_path_of(w) -> str:
    """The engine's AUTO rule (csrc/engine.cu gather_selected) for the FP32 fine path."""
    forced = os.environ.get("LTCI_COARSE")
    if forced in ("transform", "gather"):
        return forced
    p = w.params
    per_table = n_coarse_cells(w) // (w.amb.count() if w.variant == 1 else 1)
    return "gather" if p.K >= 64 and 256 <= p.M and per_table >= 16 else "transform"


def plan_shard(w, ws: int, requested: str) -> str:
    """The job's partition across ``ws`` ranks (the same answer in both arms).
    auto: the partition with the smaller busiest-rank time -- coarse-cell
    shards pay ceil(C / ws) whole cells on the busiest rank; range-cell shards
    (BASELINE's partition) split the fine stage and the gather evenly and
    repeat, on every rank, the part of the coarse stage that does not depend
    on the rows kept."""
    if w.cpis > 1:
        return "cpis"
    if requested != "auto":
        return requested
    C, R = n_coarse_cells(w), w.space.roi.count()
    if ws == 1 or C < ws:
        return "coarse" if C >= ws else "rows"
    path = coarse_path_of(w)
    cof, rep = COARSE_OVER_FINE[path], COARSE_REPEATED[path]
    coarse_cost = (1.0 + cof) * (-(-C // ws)) / C
    rows_cost = (1.0 + cof * (1.0 - rep)) * (-(-R // ws)) / R + cof * rep
    return "coarse" if coarse_cost <= rows_cost else "rows"


def front_of(args) -> str:
    """Input domain of a step: "range" = range-pulse echo through K0 (range FFT) first."""
    return args.front_end if args.front_end != "auto" else ("range" if args.config == 3 else "freq")


def job_config(w, args, ws: int) -> dict:
    """``config`` of the JSON line: the workload and its partition, identical in both arms."""
    p = w.params
    shard = plan_shard(w, ws, args.shard)
    return {"workload": w.name, "config_index": args.config, "K": p.K, "M": p.M, "cpis": w.cpis,
            "front_end": ("range-pulse echo: range FFT (ltci::range_fft) in every step" if front_of(args) == "range"
                          else "freq-pulse cube (the reference detectors' input)"),
            "hypotheses_per_cpi": w.hypotheses(), "integrations_per_step": w.integrations() * w.cpis,
            "parallelism": {"cpis": "CPI shards", "coarse": "coarse-cell shards",
                            "rows": "range-cell shards"}[shard] + f" x{ws}",
            "l2": "GPU arm: flushed between steps (512 MiB write, untimed); X stream >> L2"}


def cpu_reference_rate(w, seconds_target: float, threads: int, full=None, front="freq"):
    """Time the reference's own detector (oracle/_ref, compiled from the
    reference sources) on a coarse-cell slice sized to ~seconds_target.
    ``full``: the unsliced workload when ``w`` is itself a coarse slice, so the
    sample can still give every host thread a coarse cell (every coarse cell
    costs the same, so the per-integration rate is the slice's)."""
    unit_w = w
    if full is not None:
        w = full
    import oracle as O
    from paper_2403_06788_b200 import configs, scene
    from paper_2403_06788_b200.model import DetectorOptions
    if not O.have_ref():
        return None
    x = scene.to_complex64_roundtrip(w.cube())
    gamma = float(np.sqrt(-w.params.M * w.params.K * w.sigma2 * np.log(1e-6)))
    opt = DetectorOptions(retain_threshold=gamma, threads=threads)
    axis_cells = w.space.coarse[1].count if w.variant == 1 else int(np.prod([g.count for g in w.space.coarse[1:]]))
    per_v = axis_cells * (w.amb.count() if w.variant == 1 else 1)
    # one coarse unit per thread is the reference's parallel grain (detectors.cpp:356-358)
    nv = max(1, -(-threads // per_v))
    g0 = w.space.coarse[1 if w.variant == 1 else 0]
    if w.variant == 1:
        nv = min(nv, g0.count)
        sl = configs.sliced(w, nv)
    else:
        sl = configs.sliced(w, min(nv, g0.count))
    # bound the sample to ~seconds_target: the reference spends the same time per
    # (coarse cell, ROI row) at any row count (the per-cell mgift is < 1 % of it),
    # so large configs keep every coarse/fine cell of the slice but fewer rows
    per_row = sl.integrations() / sl.space.roi.count()
    # at least 4 rows: the reference builds each (coarse, fine) DFM filter once per
    # row set, so a 1-row sample would mostly time filter construction
    rows = int(max(min(4, sl.space.roi.count()), min(sl.space.roi.count(), seconds_target * 4e9 * threads / per_row)))
    if rows <= 4 and w.variant == 0 and g0.count >= threads:
        # huge per-row work (C2): exactly one coarse cell per thread, and enough rows
        # that the reference's per-(coarse, fine) DFM filter build stays amortised
        sl = configs.sliced(w, threads, 1)
        per_row = sl.integrations() / sl.space.roi.count()
        rows = int(max(4, min(sl.space.roi.count(), seconds_target * 4e9 * threads / per_row)))
    if rows < sl.space.roi.count():
        from paper_2403_06788_b200.model import RangeRoi
        sl.space.roi = RangeRoi(sl.space.roi.first, sl.space.roi.first + rows - 1)
        sl.name += f" [{rows} ROI rows]"
    t0 = time.perf_counter()
    O.ref_ds(x, sl.params, sl.space, opt, sl.variant, sl.amb)
    dt = time.perf_counter() - t0
    integ = sl.integrations()
    fe = ""
    if front == "range":
        # the job's range FFT (reference range_fft on the whole echo), charged to the
        # sample in proportion to its share of the job's integrations
        rc = np.fft.ifft(x, axis=1) * w.params.K
        t1 = time.perf_counter()
        O.ref_range_fft(rc, w.params)
        t_fft = time.perf_counter() - t1
        dt += t_fft * integ / w.integrations()
        fe = f" + range_fft share ({t_fft:.3f} s per echo)"
    # the reference parallelises over coarse cells (detectors.cpp:356-358): a
    # sample with fewer cells than host threads only keeps that many busy
    cells = (sl.amb.count() * sl.space.coarse[1].count if sl.variant == 1
             else int(np.prod([g.count for g in sl.space.coarse])))
    used = max(1, min(threads, cells))
    return {"value": in_unit(unit_w, integ / dt / 1e9), "unit": metric_of(unit_w)[1], "cores": used,
            "kind": "reference",
            "sample": f"{sl.name}: {integ:.3e} integrations in {dt:.2f} s{fe} (oracle/_ref, -O3, threads={threads})"}


def run_reference(args, w, ws, rank, w_full=None):
    if rank != 0:
        return
    import oracle as O
    threads = os.cpu_count() or 1
    metric, unit = metric_of(w)
    line = {"impl": "reference", "metric": metric, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "config": job_config(w, args, ws), "data": "synthetic (seeded reference signal model)"}
    if not O.have_ref():
        line["unavailable"] = "reference library oracle/_ref/libltci_ref.so not built"
        print(json.dumps(line))
        return
    for _ in range(args.warmup):
        cpu_reference_rate(w, args.cpu_seconds, threads, w_full, front_of(args))
    vals, samples = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = cpu_reference_rate(w, args.cpu_seconds, threads, w_full, front_of(args))
        vals.append(r["value"])
        samples.append(r["sample"])
    total = time.perf_counter() - t0
    v = float(np.mean(vals))
    line.update({"value": v, "ms_per_step": total / args.steps * 1e3, "dtype": "f64",
                 "cpu_baseline": {"value": v, "unit": unit, "cores": threads, "kind": "reference",
                                  "sample": samples[-1]},
                 "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line))


class _CAI:
    """Zero-copy torch view of a device buffer owned by the engine."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 2}


def _ncu_traffic(config_index, kernel, stage="fine"):
    """DRAM bytes per launch of the fine (or coarse) kernel from the committed ncu --set full
    captures of this round (profiles/r02_ncu_traffic.json, from profiles/r02_ncu_c*.txt)."""
    path = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if kernel.startswith("fine_tc") or not os.path.exists(path):
        if kernel.startswith("fine_tc") and config_index == 1:
            old = os.path.join(ROOT, "profiles", "r01_ncu_c1.json")
            if os.path.exists(old):
                return json.load(open(old)).get(kernel, {}).get("traffic_bytes_per_launch")
        return None
    ent = json.load(open(path)).get(str(config_index), {})
    if stage == "coarse":
        ent = ent.get("coarse", {})
    return ent.get("traffic_bytes_per_launch")


def main():
    args = parse()
    ws, rank, local = dist_env()
    if ws > 1 or os.environ.get("LTCI_BENCH_FORCE_DIST") == "1":
        # communicator lines (nRanks, transport) stay on stderr as the run's evidence: INFO is a
        # superset of the VERSION level the GPU boxes preset (which prints the version line only)
        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    from paper_2403_06788_b200 import configs
    w = w_full = configs.config(args.config)
    if args.coarse_slice:
        w = configs.sliced(w, args.coarse_slice, args.coarse_rest)
        # a coarse-cell slice is a rate sample of the full job: it runs the coarse kernel the full
        # job's AUTO rule picks (K1g from 16 coarse cells per table; the slice alone may be below
        # that), and pays the full job's once-per-CPI table build on its few cells (pessimistic)
        if "LTCI_COARSE" not in os.environ and w_full.variant == 0 and \
                int(np.prod([g.count for g in w_full.space.coarse])) >= 16:
            os.environ["LTCI_COARSE"] = "gather"
    if args.impl == "reference":
        run_reference(args, w, ws, rank, w_full)
        return

    import torch
    import torch.distributed as dist
    from paper_2403_06788_b200 import _cabi as A
    from paper_2403_06788_b200 import _lib, scene
    from paper_2403_06788_b200.detectors import Engine, detection_threshold
    from paper_2403_06788_b200.model import DetectorOptions

    # LTCI_BENCH_SHARED_GPU=1: functional check of the N-rank path on a 1-GPU box
    # (every rank on cuda:0, gloo over host copies); its timings mean nothing
    shared_gpu = ws > 1 and os.environ.get("LTCI_BENCH_SHARED_GPU") == "1"
    # LTCI_BENCH_FORCE_DIST=1 (under torchrun): run the N-rank code path -- NCCL communicator,
    # barriers, peak-map gather and device merge, max-over-ranks reduction -- whatever the world
    # size, so a 1-GPU box executes it over real NCCL with a world of one rank
    multi = ws > 1 or (os.environ.get("LTCI_BENCH_FORCE_DIST") == "1" and "RANK" in os.environ)
    if shared_gpu:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if multi:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2403_06788_b200.parallel import PeakGather, RankComm
    comm = RankComm(ws, host_staged=shared_gpu)
    dev = torch.device("cuda", local)
    p, s = w.params, w.space
    fine_path = {"auto": A.FINE_AUTO, "fft": A.FINE_FFT_CUDA_CORE, "tc": A.FINE_TC_DENSE,
                 "tcfast": A.FINE_TC_FAST}[args.fine_path]
    if args.pfa <= 0:
        args.pfa = min(1e-6, 1e5 / float(w.hypotheses()))
    # range front end: the echo is the range-compressed cube range_ifft(y) (CN(0,1) noise);
    # K0 returns range_fft(range_ifft(y)) = K y, i.e. a freq cube with K^2 times the variance
    sigma2_eff = w.sigma2 * (p.K ** 2 if front_of(args) == "range" else 1)
    gamma = detection_threshold(p, sigma2_eff, args.pfa)
    opt = DetectorOptions(retain_threshold=gamma, fine_path=fine_path, device=local)
    R = s.roi.count()
    cpis = w.cpis
    if w.variant == 0:
        n_coarse = int(np.prod([g.count for g in s.coarse]))
    else:
        n_coarse = w.amb.count() * s.coarse[1].count
    shard = plan_shard(w, ws, args.shard)
    c_lo, c_hi = 0, -1
    if cpis > 1:
        # CPI-level data parallelism (configs[4]): each rank streams its CPIs, full ROI
        lo, hi = 0, R
        my_cpis = list(range(rank * cpis // ws, (rank + 1) * cpis // ws))
    elif shard == "coarse":
        # one CPI sharded over coarse cells (SURVEY.md 8(e) alternative): every rank
        # searches its coarse cells over every ROI row, nothing replicated
        from paper_2403_06788_b200.parallel import shard_coarse
        lo, hi = 0, R
        c_lo, c_hi = shard_coarse(n_coarse, ws, rank)
        my_cpis = [0]
    else:
        # one CPI sharded over range start cells
        lo, hi = rank * R // ws, (rank + 1) * R // ws
        my_cpis = [0]
    log("engine")
    eng = Engine(p, s, w.variant, w.amb, opt, row_begin=lo, row_end=hi, coarse_begin=c_lo, coarse_end=c_hi)
    # a CPI stream runs on --lanes engine lanes (own buffers and stream each), so one
    # CPI's last fine wave overlaps the next CPI's coarse stage and first waves
    n_lanes = max(1, min(args.lanes, len(my_cpis)))
    lane_engs = [eng] + [Engine(p, s, w.variant, w.amb, opt, row_begin=lo, row_end=hi, coarse_begin=c_lo,
                                coarse_end=c_hi) for _ in range(n_lanes - 1)]
    log("synthesising cubes")
    hyp, integ = eng.work()

    cubes = [scene.to_complex64_roundtrip(w.cube(cpi=c)) for c in my_cpis]  # (M, K): column-major K x M
    front = front_of(args)
    if front == "range":
        # the echo as range-compressed fast-time samples (range_ifft, proj/src/signal_model.cpp:85-95);
        # every step starts with K0 (range_fft) on the device
        cubes = [scene.to_complex64_roundtrip(np.fft.ifft(c, axis=1) * p.K) for c in cubes]
        run_dev, run_hptr = Engine.run_range_device, Engine.run_range_host_ptr
    else:
        run_dev, run_hptr = Engine.run_device, Engine.run_host_ptr
    d_cubes = [torch.from_numpy(c.astype(np.complex64)).to(dev) for c in cubes]
    cube = cubes[0]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    peak_ptr, n_rows = eng.peaks_device()
    peaks = torch.as_tensor(_CAI(peak_ptr, (n_rows, 4), "<u4"), device=dev)
    per_cpi_peaks = torch.empty((len(my_cpis), n_rows, 4), dtype=torch.int32, device=dev)
    lib = _lib.load()
    gather = None
    if multi and cpis == 1:
        def merge_on_device(gathered, merged):
            _lib.raise_for(lib.ltci_cuda_merge_peaks(ctypes.c_void_p(gathered.data_ptr()), ws, R,
                                                     ctypes.c_void_p(merged.data_ptr()), ctypes.c_void_p(sptr)),
                           lib)
        # coarse shards: NCCL all-gather of the 16-byte records, then the per-row max on
        # the device with the kernels' tie-break; row shards: padded all-gather
        gather = PeakGather(comm, shard, R, peaks, merge=merge_on_device)

    def gather_peaks():
        if gather is not None:
            gather(peaks.view(torch.int32))

    lane_streams = [stream] + [torch.cuda.Stream(dev) for _ in range(n_lanes - 1)]
    lane_peaks = [peaks] + [torch.as_tensor(_CAI(e.peaks_device()[0], (n_rows, 4), "<u4"), device=dev)
                            for e in lane_engs[1:]]

    def step_local():
        if n_lanes == 1:
            for i, dc in enumerate(d_cubes):
                run_dev(eng, dc.data_ptr(), sptr)
                if cpis > 1:
                    per_cpi_peaks[i].copy_(peaks.view(torch.int32))  # keep each CPI's peak map
            return
        for ls in lane_streams[1:]:
            ls.wait_stream(stream)
        for i, dc in enumerate(d_cubes):
            ln = i % n_lanes
            ls = lane_streams[ln]
            run_dev(lane_engs[ln], dc.data_ptr(), ls.cuda_stream)
            with torch.cuda.stream(ls):
                per_cpi_peaks[i].copy_(lane_peaks[ln].view(torch.int32))
        for ls in lane_streams[1:]:
            stream.wait_stream(ls)

    def step():
        step_local()
        gather_peaks()

    log("warmup")
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)

    log("timed steps")
    # ---- value: device-timed, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if multi:
        dist.barrier()
    torch.cuda.synchronize(dev)
    wall0 = time.perf_counter()
    extra_steps = 0
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - wall0
        # a timed region shorter than the sampling period (C0: ms) gets its clocks
        # from untimed repeats of the same step, stated in the JSON line
        t1 = time.perf_counter()
        # (collective-free: ranks may repeat a different number of times)
        while clk.proc and clk.count() < 3 and time.perf_counter() - t1 < 3.0:
            step_local()
            torch.cuda.synchronize(dev)
            extra_steps += 1
    if multi:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if multi:
        comm.all_reduce_max(t)
    ms_max = float(t.item())
    total_integ = w.integrations() * cpis  # all ranks together cover every hypothesis of every CPI once
    value = total_integ * args.steps / (ms_max * 1e-3) / 1e9
    cpi_rate = cpis * args.steps / (ms_max * 1e-3)

    log("kernel split")
    # ---- kernel split (timed pass) for the roofline
    eng.set_timing(True)
    flush.zero_()
    run_dev(eng, d_cubes[0].data_ptr(), sptr)
    st = eng.stats()
    eng.set_timing(False)
    launches = st["launches"] * len(my_cpis) + (1 if multi and shard == "coarse" and cpis == 1 else 0)  # + peak merge

    log("e2e")
    # ---- e2e: public API from pinned host memory, results back to host
    hosts = [torch.from_numpy(c.view(np.float64).reshape(-1)).pin_memory() for c in cubes]
    e2e_ms = []
    d2h = 0
    # result() D2H: count + R peak slots (16 B) + 24 B per retained candidate (u64 index, complex128)
    res_bytes = lambda m: 8 + 16 * n_rows + 24 * int(m.cand_index.size)  # noqa: E731
    e2e_lanes = n_lanes
    e2e_steps = args.steps
    if not multi:
        # one process streams the job's CPIs step after step through the public API; the
        # lanes keep two in flight (CPI i+1 uploads and runs while CPI i's result drains),
        # so the timed region holds every step's H2D, run and D2H, overlapped as a
        # streaming receiver would
        e2e_lanes = max(n_lanes, min(2, args.lanes))
        while len(lane_engs) < e2e_lanes:
            lane_engs.append(Engine(p, s, w.variant, w.amb, opt, row_begin=lo, row_end=hi, coarse_begin=c_lo,
                                    coarse_end=c_hi))
            lane_streams.append(torch.cuda.Stream(dev))
        # at least ~0.25 s of steps (C0's 0.3 ms steps would otherwise time 1.5 ms of host
        # calls, at the mercy of scheduler jitter); the line reports per-step averages
        step_s = ms_max / args.steps * 1e-3
        e2e_steps = int(min(2000, max(args.steps, np.ceil(0.25 / max(step_s, 1e-6)))))
        items = [(i, k) for i in range(args.warmup + e2e_steps) for k in range(len(hosts))]
        pending = [None] * e2e_lanes
        t0 = None
        for j, (i, k) in enumerate(items):
            if t0 is None and i == args.warmup:
                for ln in range(e2e_lanes):  # drain the warm-up items, then start the clock
                    if pending[ln] is not None:
                        lane_engs[ln].result(lane_streams[ln].cuda_stream)
                        pending[ln] = None
                torch.cuda.synchronize(dev)
                d2h = 0
                t0 = time.perf_counter()
            ln = j % e2e_lanes
            ls = lane_streams[ln].cuda_stream
            if pending[ln] is not None:
                d2h += res_bytes(lane_engs[ln].result(ls))
            run_hptr(lane_engs[ln], hosts[k].data_ptr(), ls)
            pending[ln] = k
        for ln in range(e2e_lanes):
            if pending[ln] is not None:
                d2h += res_bytes(lane_engs[ln].result(lane_streams[ln].cuda_stream))
        e2e_ms.append((time.perf_counter() - t0) * 1e3 * args.steps / e2e_steps)  # scaled to args.steps steps
        d2h //= e2e_steps
    else:
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            d2h = 0
            pending = [None] * n_lanes  # pipeline over the lanes: later CPIs upload and run while earlier ones drain
            for k, hst in enumerate(hosts):
                ln = k % n_lanes
                ls = lane_streams[ln].cuda_stream
                if pending[ln] is not None:
                    d2h += res_bytes(lane_engs[ln].result(ls))
                run_hptr(lane_engs[ln], hst.data_ptr(), ls)
                pending[ln] = k
            for ln in range(n_lanes):
                if pending[ln] is not None:
                    d2h += res_bytes(lane_engs[ln].result(lane_streams[ln].cuda_stream))
            gather_peaks()
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            if i >= args.warmup:
                e2e_ms.append((t1 - t0) * 1e3)
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if multi:
        comm.all_reduce_max(e2e_t)
    e2e_value = total_integ * args.steps / (float(e2e_t.item()) * 1e-3) / 1e9

    if rank == 0:
        lib = _lib.load()
        import ctypes as C
        fp32 = C.c_double(0)
        _lib.raise_for(lib.ltci_cuda_measure_fp32_peak(local, C.byref(fp32)), lib)
        peaks_json = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        from paper_2403_06788_b200.configs import doppler_window
        D = doppler_window(p, s)[1] if w.variant == 0 else p.M
        if w.variant == 0:
            coarse = int(np.prod([g.count for g in s.coarse]))
            fine_cells = int(np.prod([g.count for g in s.fine[1:]])) if s.order() > 1 else 1
        else:
            coarse = w.amb.count() * s.coarse[1].count
            fine_cells = s.fine[1].count
        rows_here = (hi - lo)
        if shard == "coarse" and ws > 1:
            coarse = c_hi - c_lo  # this rank's coarse cells (every row)
        hbm = peaks_json.get("hbm_gbs", 6650.0)
        x_bytes = 8.0 * coarse * rows_here * p.M + 8.0 * p.K * p.M
        coarse_fft_flops = coarse * p.M * (5.0 * p.K * np.log2(p.K) + 8.0 * p.K)
        coarse_gbs = x_bytes / (st["coarse_ms"] * 1e-3) / 1e9 if st["coarse_ms"] > 0 else None
        path_id, terms = eng.fine_path()  # what the engine actually runs
        use_tc = path_id in (A.FINE_TC_DENSE, A.FINE_TC_FAST)
        fine_s = st["fine_ms"] * 1e-3
        if use_tc:
            peak_tc = peaks_json.get("bf16_tflops", 1649.5)
            peak_sus = peaks_json.get("bf16_tflops_sustained", 1394.2)
            achieved = 8.0 * integ / fine_s / 1e12  # algorithmic: 8 flop per integration
            roof = {"bound": "tensor", "kernel": f"fine_tc2_kernel<{terms}> (K2a+K3, tcgen05 cta_group::2)",
                    "achieved": achieved, "peak": peak_tc, "unit": "TFLOP/s", "frac": achieved / peak_tc,
                    "traffic": _ncu_traffic(args.config, "fine_tc2_kernel<3>") if terms == 3 else None,
                    "traffic_source": "profiles/r01_ncu_c1.json (ncu --set full, bytes per launch)",
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst, the conservative denominator: the SM "
                                   "clock drops to the power cap under this kernel, 1.29-1.43 GHz in ncu); "
                                   "frac_vs_sustained uses bf16_tflops_sustained",
                    "frac_vs_sustained": achieved / peak_sus,
                    "algorithmic": "8 flop per hypothesis x pulse integration (complex MAC)",
                    "executed_tflops": terms * achieved, "executed_frac": terms * achieved / peak_tc,
                    "split_terms": terms}
        else:
            per_launch_flops = coarse * rows_here * fine_cells * fft_flops_per_row_cell(p.M, D)
            achieved = per_launch_flops / fine_s / 1e12
            tm = p.M == 1024
            kname = ("fine_fft_tm_kernel (K2b+K3, CUDA cores, TMEM-resident rows)" if 256 <= p.M <= 1024 else
                     "fine_fft_tm2k_kernel (K2b+K3, CUDA cores, radix-2 split onto two TMEM 1024-point halves)"
                     if p.M == 2048 else "fine_fft_kernel (K2b+K3, CUDA cores)")
            roof = {"bound": "fp32",
                    "kernel": kname,
                    "achieved": achieved, "peak": fp32.value, "unit": "TFLOP/s",
                    "frac": achieved / fp32.value if fp32.value else None,
                    "traffic": _ncu_traffic(args.config, "fine_fft_tm_kernel<0>")
                    if 256 <= p.M <= 2048 and (args.config != 2 or (args.coarse_slice == 1 and args.coarse_rest == 1))
                    else None,
                    "traffic_source": "profiles/r02_ncu_traffic.json"
                    + " (ncu --set full, DRAM bytes per launch)",
                    "peak_source": "measured in-run FFMA chain microbenchmark (ltci_cuda_measure_fp32_peak)",
                    "algorithmic": "per (row, fine cell): 6M chirp + 5M log2M FFT + 3D |Y|^2 flop",
                    "dense_equiv_tflops": 8.0 * integ / fine_s / 1e12}
        roof.update({"fine_ms": st["fine_ms"], "coarse_ms": st["coarse_ms"], "keystone_ms": st["keystone_ms"],
                     "fine_share": st["fine_ms"] / max(1e-9, st["fine_ms"] + st["coarse_ms"] + st["keystone_ms"]),
                     "coarse_stage": {"bound": "hbm", "achieved": coarse_gbs, "peak": hbm, "unit": "GB/s",
                                      "frac": coarse_gbs / hbm if coarse_gbs else None,
                                      "algorithmic": "8 B x (K M echo + coarse x R x M X write)",
                                      "fp32_tflops": coarse_fft_flops / (st["coarse_ms"] * 1e-3) / 1e12
                                      if st["coarse_ms"] > 0 else None,
                                      "fp32_algorithmic": "per (coarse cell, pulse): 5 K log2 K FFT + 8 K ramp",
                                      "path": eng.coarse_path(),
                                      "traffic": _ncu_traffic(args.config, "coarse", stage="coarse")
                                      if not args.coarse_slice and ws == 1 else None,
                                      "note": ("K1g (gather.cuh): 8-tap interpolation of 2x-oversampled range "
                                               "profiles tabulated once per pulse (type-2 NUFFT, 1.3e-7 of the "
                                               "profile maximum); table build + weights + gather are all inside "
                                               "coarse_ms; fp32_tflops is what the replaced transforms would "
                                               "have cost, not work done" if eng.coarse_path() == "gather" else
                                               "K1 (coarse.cuh): one K-point transform per (coarse cell, pulse); "
                                               "issue-bound, see profiles/r01_ncu_c1.json")}})
        if w.variant == 1:
            # K4 keystone timed over back-to-back calls (one call is ~5 us of
            # traffic, launch latency would dominate a single timing)
            kt_calls, kt_ring = 200, 8  # 8 (in, out) pairs = 269 MB at C3 > L2: every call streams from HBM
            kt_in = [torch.from_numpy(scene.to_complex64_roundtrip(w.cube()).astype(np.complex64)).to(dev)
                     for _ in range(kt_ring)]
            kt_out = [torch.empty_like(d_cubes[0]) for _ in range(kt_ring)]
            cr = p.to_c()

            def kt_call(i):
                _lib.raise_for(lib.ltci_cuda_keystone_device(
                    ctypes.c_void_p(kt_in[i % kt_ring].data_ptr()), ctypes.c_void_p(kt_out[i % kt_ring].data_ptr()),
                    ctypes.byref(cr), opt.keystone_taps, ctypes.c_void_p(sptr)), lib)
            for i in range(16):
                kt_call(i)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(stream)
            for i in range(kt_calls):
                kt_call(i)
            k1.record(stream)
            torch.cuda.synchronize(dev)
            kt_ms = k0.elapsed_time(k1) / kt_calls
            kt_bytes = 16.0 * p.K * p.M
            roof["keystone_stage"] = {"bound": "hbm", "achieved": kt_bytes / (kt_ms * 1e-3) / 1e9, "peak": hbm,
                                      "unit": "GB/s", "frac": kt_bytes / (kt_ms * 1e-3) / 1e9 / hbm,
                                      "ms_per_call": kt_ms, "calls": kt_calls, "taps": opt.keystone_taps,
                                      "algorithmic": "16 B per (row, pulse): complex64 read + write",
                                      "kernel": "keystone_tiled_kernel<taps/2> (K4)",
                                      "note": "back-to-back ltci_cuda_keystone_device calls on one stream over a "
                                              "ring of 8 (in, out) cube pairs larger than L2"}
        metric, unit = metric_of(w)
        if cpis > 1:
            val, e2e_val = cpi_rate, cpis * args.steps / (float(e2e_t.item()) * 1e-3)
        else:
            val, e2e_val = value, e2e_value
        line = {
            "metric": metric, "value": val, "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,  # the same job at every N, split across ranks
            "dtype": "c64 / fp32" if not use_tc else ("fp16x3 split (FP32 class)" if terms == 3 else "fp16"),
            "data": "synthetic (seeded reference signal model: CN(0,1) range noise + targets)",
            "config": job_config(w, args, ws),
            "run": {"integrations_per_s_G": value, "retain_threshold": gamma, "pfa": args.pfa,
                    "fine_path": args.fine_path + (" -> tcgen05" if use_tc else " -> cuda-core fft"),
                    "lanes": n_lanes},
            "roofline": roof,
            "e2e": {"value": e2e_val, "unit": unit, "h2d_bytes_per_step": int(cube.size * 16 * len(cubes)),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": float(e2e_t.item()) / args.steps,
                    "lanes": e2e_lanes, "steps": e2e_steps if not multi else args.steps,
                    "pipeline": "public API (Engine.run_host_ptr from pinned f64 + result()), CPIs streamed over "
                                f"{e2e_lanes} engine lanes" if not multi else "per step: upload, run, result, gather"},
            "gpu_launches": int(launches) * args.steps,
            "clocks": dict(clk.summary(), **({"untimed_repeat_steps_sampled": extra_steps} if extra_steps else {})),
            "wall_s_timed_region": wall,
        }
        if ws == 1 and not args.no_cpu_baseline:
            try:
                log("cpu baseline")
                cb = cpu_reference_rate(w, args.cpu_seconds, os.cpu_count() or 1, w_full, front)
            except Exception as e:  # reported, not fatal
                cb = {"error": str(e)}
            line["cpu_baseline"] = cb
        if shared_gpu:
            line["shared_gpu_functional_check"] = True  # N ranks on one GPU: timings are not a measurement
        if multi and ws == 1:
            line["n_rank_path_forced"] = "LTCI_BENCH_FORCE_DIST=1: the N-rank path (NCCL) with a world of one rank"
        dump = os.environ.get("LTCI_BENCH_DUMP_PEAKS")
        if dump and cpis == 1:
            # the job's per-row peak map (R x {idx lo, idx hi, re, im}) after the rank
            # merge of the last e2e step (collectives already done on every rank)
            torch.cuda.synchronize(dev)
            full = peaks.view(torch.int32) if not multi else gather.full_map()
            np.save(dump, full.cpu().numpy())
        print(json.dumps(line))
    if multi:
        dist.destroy_process_group()
    for e in lane_engs:
        e.close()


if __name__ == "__main__":
    main()
