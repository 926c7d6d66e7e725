set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py tests/test_gpu_fullsize.py tests/test_gpu_engine_hazards.py -q -x > gpurun_out/tests_e.log 2>&1
python scripts/bench_coarse.py > gpurun_out/coarse_ab.log 2>&1
LTCI_COARSE_GENERIC=1 python scripts/bench_coarse.py >> gpurun_out/coarse_ab.log 2>&1
LTCI_LIB_PATH=$PWD/paper_2403_06788_b200/lib/ab/libltci_cuda_ng4.so python scripts/bench_coarse.py >> gpurun_out/coarse_ab.log 2>&1
LTCI_LIB_PATH=$PWD/paper_2403_06788_b200/lib/ab/libltci_cuda_ng16.so python scripts/bench_coarse.py >> gpurun_out/coarse_ab.log 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python bench.py --config 1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"coarse2k|keystone_tiled" -c 2 -o gpurun_out/ncu_c2k python scripts/profile_step.py --config 3 > gpurun_out/ncu_c2k.log 2>&1
