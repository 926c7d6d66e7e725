set -x
python scripts/time_calls.py > gpurun_out/time_calls.log 2>&1
for i in 1 2; do oracle/_ref/acceptance_dropin 7; done > gpurun_out/c7.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python bench.py > gpurun_out/r01_bench_c1.json.log 2>&1
for c in 0 3 4; do python bench.py --config $c > gpurun_out/r01_bench_c$c.json.log 2>&1; done
python bench.py --impl reference > gpurun_out/r01_bench_ref_c1.json.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/profile_step.py --config 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fine_fft_tm -c 1 -o gpurun_out/fine_tm_nb3 python scripts/profile_step.py --config 1 > gpurun_out/ncu_full.log 2>&1
