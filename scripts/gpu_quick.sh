set -x
timeout 1200 python -m pytest tests/test_gpu_tm.py tests/test_gpu_fullsize.py -x -q -k "2k or c2" > gpurun_out/q_tests.log 2>&1
python bench.py --no-cpu-baseline --config 2 --coarse-slice 1 --coarse-rest 1 --steps 2 > gpurun_out/q_c2.log 2>&1
