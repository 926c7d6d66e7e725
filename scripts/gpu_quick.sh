set -x
timeout 1200 python -m pytest tests/test_gpu_tm.py -x -q > gpurun_out/q_tests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/q_c1.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/q_c1b.log 2>&1
