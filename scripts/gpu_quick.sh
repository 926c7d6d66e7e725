set -x
timeout 1500 python -m pytest tests/test_gpu_tm.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/q_tests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/q_c1.log 2>&1
python bench.py --no-cpu-baseline --config 3 > gpurun_out/q_c3.log 2>&1
python bench.py --no-cpu-baseline --config 4 > gpurun_out/q_c4.log 2>&1
python bench.py --no-cpu-baseline --config 0 > gpurun_out/q_c0.log 2>&1
python bench.py --no-cpu-baseline --config 2 --coarse-slice 1 --coarse-rest 1 --steps 2 > gpurun_out/q_c2.log 2>&1
