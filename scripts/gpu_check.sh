# quick GPU check after a kernel change: parity subsets + bench lines (+ optional ncu of one kernel)
set -x
timeout 900 python -m pytest tests/test_gpu_tm.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_fd_grft.py tests/test_gpu_tc.py -x -q > gpurun_out/chk_tests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/chk_c1.log 2>&1
python bench.py --no-cpu-baseline --config 4 > gpurun_out/chk_c4.log 2>&1
python bench.py --no-cpu-baseline --config 3 > gpurun_out/chk_c3.log 2>&1
python bench.py --no-cpu-baseline --config 0 > gpurun_out/chk_c0.log 2>&1
[ -x scripts/micro/ffma2_rate ] && scripts/micro/ffma2_rate > gpurun_out/ffma2_rate.log 2>&1
if [ -n "$NCU_K" ]; then
  ncu --set full --import-source on --clock-control none -k regex:"$NCU_K" -c ${NCU_C:-1} -o gpurun_out/chk_ncu python scripts/profile_step.py --config 1 > gpurun_out/chk_ncu.log 2>&1
fi
