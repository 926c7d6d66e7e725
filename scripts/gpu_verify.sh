# Verification run after a kernel/build change: GPU suite + the five bench lines (no CPU baselines).
set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
for c in 1 0 3 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; done
