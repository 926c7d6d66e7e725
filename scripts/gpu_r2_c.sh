set -x
timeout 900 python -m pytest tests/test_gpu_range.py -q > gpurun_out/range_tests.log 2>&1
LTCI_TRACE=1 timeout 300 python scripts/time_calls.py > gpurun_out/time_calls_trace.log 2>&1
python bench.py --config 3 > gpurun_out/bench_c3.log 2>&1
python bench.py --config 0 --no-cpu-baseline > gpurun_out/bench_c0.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_step.py --config 3 > gpurun_out/ncu_launch_c3.log 2>&1
