set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py tests/test_gpu_fullsize.py -q -x > gpurun_out/tests_f.log 2>&1
python scripts/bench_coarse.py > gpurun_out/coarse_ab.log 2>&1
LTCI_COARSE_GENERIC=1 python scripts/bench_coarse.py >> gpurun_out/coarse_ab.log 2>&1
LTCI_LIB_PATH=$PWD/paper_2403_06788_b200/lib/ab/libltci_cuda_ng4.so python scripts/bench_coarse.py >> gpurun_out/coarse_ab.log 2>&1
LTCI_LIB_PATH=$PWD/paper_2403_06788_b200/lib/ab/libltci_cuda_ng16.so python scripts/bench_coarse.py >> gpurun_out/coarse_ab.log 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python bench.py --config 0 --no-cpu-baseline > gpurun_out/bench_c0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"coarse2k|keystone_tiled|fine_fft_tm" -c 3 -o gpurun_out/ncu_f python scripts/profile_step.py --config 3 > gpurun_out/ncu_f.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fine_fft_tm" -c 1 -o gpurun_out/ncu_c0 python scripts/profile_step.py --config 0 > gpurun_out/ncu_c0.log 2>&1
