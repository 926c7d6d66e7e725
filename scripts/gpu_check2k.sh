set -x
timeout 1200 python -m pytest tests/test_gpu_tm.py tests/test_gpu_tc.py tests/test_gpu_fullsize.py -x -q > gpurun_out/k2_tests.log 2>&1
python bench.py --no-cpu-baseline --config 2 --coarse-slice 1 --coarse-rest 1 --steps 2 > gpurun_out/k2_c2_auto.log 2>&1
python bench.py --no-cpu-baseline --config 2 --coarse-slice 1 --coarse-rest 1 --steps 2 --fine-path tc > gpurun_out/k2_c2_tc.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/k2_c1.log 2>&1
