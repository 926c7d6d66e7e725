set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python scripts/time_calls.py > gpurun_out/time_calls.log 2>&1
python bench.py --config 3 > gpurun_out/bench_c3.log 2>&1
python bench.py --config 0 --no-cpu-baseline > gpurun_out/bench_c0.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_step.py --config 3 > gpurun_out/ncu_launch_c3.log 2>&1
