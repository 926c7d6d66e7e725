set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tm.py tests/test_gpu_fullsize.py -q > gpurun_out/tests_h.log 2>&1
python bench.py --config 0 --no-cpu-baseline > gpurun_out/bench_c0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fine_fft_tm" -c 1 -o gpurun_out/ncu_c0 python scripts/profile_step.py --config 0 > gpurun_out/ncu_c0.log 2>&1
