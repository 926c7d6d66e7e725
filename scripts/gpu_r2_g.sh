set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python bench.py --config 0 --no-cpu-baseline > gpurun_out/bench_c0.log 2>&1
python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fine_fft_tm" -c 1 -o gpurun_out/ncu_c0 python scripts/profile_step.py --config 0 > gpurun_out/ncu_c0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"keystone_tiled" -c 1 -o gpurun_out/ncu_kt python scripts/profile_step.py --config 3 > gpurun_out/ncu_kt.log 2>&1
