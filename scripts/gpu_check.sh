# quick GPU check after a kernel change: parity subsets + bench lines (+ optional ncu of one kernel)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1
python bench.py --no-cpu-baseline --config 0 > gpurun_out/chk_c0.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/chk_c1.log 2>&1
python bench.py --no-cpu-baseline --config 4 > gpurun_out/chk_c4.log 2>&1
if [ -n "$NCU_K" ]; then
  ncu --set full --import-source on --clock-control none -k regex:"$NCU_K" -c ${NCU_C:-1} -o gpurun_out/chk_ncu python scripts/profile_step.py --config ${NCU_CFG:-1} > gpurun_out/chk_ncu.log 2>&1
fi
