# Round measurement on one B200: smoke, full GPU suite, bench lines for every config (+ reference arm),
# side benchmarks (fd_grft, run_pd, cube-file wire path, one-shot call latency), the C1 launch list and
# ncu --set full captures of the top kernels.  Outputs land in gpurun_out/ (copied to profiles/ by hand).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python bench.py > gpurun_out/bench_c1.log 2>&1
python bench.py --config 0 > gpurun_out/bench_c0.log 2>&1
python bench.py --config 3 > gpurun_out/bench_c3.log 2>&1
python bench.py --config 4 > gpurun_out/bench_c4.log 2>&1
python bench.py --config 2 --coarse-slice 8 --coarse-rest 1 --steps 2 > gpurun_out/bench_c2.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref_c1.log 2>&1
python scripts/bench_fd.py > gpurun_out/side_fd.log 2>&1
python scripts/bench_pd.py > gpurun_out/side_pd.log 2>&1
python scripts/bench_io.py > gpurun_out/side_io.log 2>&1
python scripts/time_calls.py > gpurun_out/side_calls.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/profile_step.py --config 1 > gpurun_out/ncu_launch_c1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_step.py --config 3 > gpurun_out/ncu_launch_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fine_fft_tm|coarse_rm" -c 2 -o gpurun_out/ncu_c1 python scripts/profile_step.py --config 1 > gpurun_out/ncu_c1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"range_fft|keystone_tiled|fine_fft_tm" -c 3 -o gpurun_out/ncu_c3 python scripts/profile_step.py --config 3 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fine_fft_tm" -c 1 -o gpurun_out/ncu_c0 python scripts/profile_step.py --config 0 > gpurun_out/ncu_c0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fine_fft_tm" -c 1 -o gpurun_out/ncu_c4 python scripts/profile_step.py --config 4 > gpurun_out/ncu_c4.log 2>&1
