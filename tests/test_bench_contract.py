"""CPU: bench.py's JSON contract.  The driver divides the two arms' lines only
when metric, unit and config agree (round 1's null ratio came from two metric
strings), so the reference arm is run here -- the reference's own C++ from
oracle/_ref on a tiny sample -- and its line compared with what the B200 arm
prints for the same arguments (bench.job_config / bench.metric_of, the single
definitions both arms use)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _args(config, front="auto"):
    import argparse
    return argparse.Namespace(config=config, shard="auto", front_end=front)


@pytest.mark.parametrize("config", [0, 1, 2, 3, 4])
def test_one_config_and_metric_per_workload(config):
    import bench
    from paper_2403_06788_b200 import configs
    w = configs.config(config)
    cfg = bench.job_config(w, _args(config), 1)
    assert cfg["config_index"] == config and cfg["K"] == w.params.K and cfg["M"] == w.params.M
    assert cfg["integrations_per_step"] == w.integrations() * w.cpis
    assert ("range FFT" in cfg["front_end"]) == (config == 3)  # configs[3]'s pipeline starts with it
    metric, unit = bench.metric_of(w)
    assert unit == ("CPI/s" if w.cpis > 1 else "G/s")
    # the CPU rate reported in G/s converts into the line's own unit
    assert bench.in_unit(w, 1.0) == (1e9 / w.integrations() if w.cpis > 1 else 1.0)


@pytest.mark.skipif(not O.have_ref(), reason="reference not built (oracle/_ref)")
def test_reference_arm_line_matches_b200_arm_contract():
    import bench
    from paper_2403_06788_b200 import configs
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    w = configs.config(0)
    metric, unit = bench.metric_of(w)
    assert line["impl"] == "reference"
    assert (line["metric"], line["unit"]) == (metric, unit)
    assert line["config"] == bench.job_config(w, _args(0), 1)
    assert line["higher_is_better"] is True and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["unit"] == unit and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_bench_coarse_path_and_partition_model():
    """bench.py mirrors the engine's AUTO rule for the coarse stage (csrc/engine.cu
    gather_selected) when it plans the N-rank partition: K1g for configs[1], [2], [4];
    K1 for configs[0] (11 cells) and configs[3] (4 cells per folding number); with K1g
    a range-cell shard repeats only the per-pulse tables, so C1 takes BASELINE's
    range-cell partition at N = 8."""
    import importlib
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    bench = importlib.import_module("bench")
    from paper_2403_06788_b200 import configs
    old = os.environ.pop("LTCI_COARSE", None)
    try:
        want = {0: "transform", 1: "gather", 2: "gather", 3: "transform", 4: "gather"}
        for ci, path in want.items():
            assert bench.coarse_path_of(configs.config(ci)) == path, ci
        assert bench.plan_shard(configs.config(1), 8, "auto") == "rows"
        assert bench.plan_shard(configs.config(1), 2, "auto") == "coarse"
        assert bench.plan_shard(configs.config(0), 8, "auto") == "rows"
        assert bench.plan_shard(configs.config(4), 8, "auto") == "cpis"
        assert bench.plan_shard(configs.config(3), 8, "rows") == "rows"
    finally:
        if old is not None:
            os.environ["LTCI_COARSE"] = old
