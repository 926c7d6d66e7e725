set -x
timeout 1200 python -m pytest tests/test_gpu_tm.py tests/test_gpu_parity.py -x -q > gpurun_out/q_tests.log 2>&1
python bench.py --no-cpu-baseline --config 3 > gpurun_out/q_c3.log 2>&1
python bench.py --no-cpu-baseline --config 0 > gpurun_out/q_c0.log 2>&1
