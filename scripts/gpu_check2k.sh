set -x
timeout 1200 python -m pytest tests/test_gpu_tm.py tests/test_gpu_fullsize.py -x -q -k "2k or c2" > gpurun_out/k2_tests.log 2>&1
python bench.py --no-cpu-baseline --config 2 --coarse-slice 1 --coarse-rest 1 --steps 2 > gpurun_out/k2_c2_auto.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tm2k -c 1 -o gpurun_out/k2_ncu python scripts/profile_step.py --config 2 --coarse-v 1 --coarse-rest 1 > gpurun_out/k2_ncu.log 2>&1
