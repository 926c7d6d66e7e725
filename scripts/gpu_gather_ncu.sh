# ncu of the K1g kernels at C1 (launch list + full capture of the gather and table kernels)
set -x
mkdir -p /tmp/ncu
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gather_launches_c1.csv python scripts/profile_step.py --config 1 > gpurun_out/gather_ncu_launch.log 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:"gather_interp" -c 1 -o /tmp/ncu/gather_c1 python scripts/profile_step.py --config 1 > gpurun_out/gather_ncu_full.log 2>&1
python scripts/ncu_brief.py /tmp/ncu/gather_c1.ncu-rep > gpurun_out/gather_ncu_c1_brief.txt 2>&1
cat gpurun_out/gather_ncu_c1_brief.txt
grep -v fine_fft gpurun_out/gather_launches_c1.csv | tail -12
