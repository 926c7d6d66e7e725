# Round measurement on one B200: smoke, full GPU suite, bench lines for every config (+ reference arm),
# side benchmarks (fd_grft, run_pd, cube-file wire path, one-shot call latency), launch lists and
# ncu --set full captures of the top kernels.  ncu reports stay in /tmp/ncu on the box (gpurun copies
# back at most 64 MiB); their headline metrics and per-opcode stall attribution come back as text.
set -x
mkdir -p /tmp/ncu
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
python scripts/bench_td.py > gpurun_out/side_td.log 2>&1
python scripts/bench_io.py > gpurun_out/side_io.log 2>&1
python scripts/time_calls.py > gpurun_out/side_calls.log 2>&1
python scripts/gather_accuracy.py > gpurun_out/gather_accuracy.jsonl 2> gpurun_out/gather_accuracy.err
bash scripts/gpu_nccl_one_rank.sh > gpurun_out/nccl_one_rank.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/profile_step.py --config 1 > gpurun_out/ncu_launch_c1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_step.py --config 3 > gpurun_out/ncu_launch_c3.log 2>&1
for spec in "c1:1:fine_fft_tm|gather_interp|coarse_rm:3" "c3:3:range_fft|keystone_tiled|fine_fft_tm|coarse:4" "c0:0:fine_fft_tm:1" "c4:4:fine_fft_tm|gather_interp:2"; do
  IFS=: read name cfg regex count <<< "$spec"
  ncu -f --set full --import-source on --clock-control none -k regex:"$regex" -c $count -o /tmp/ncu/$name \
      python scripts/profile_step.py --config $cfg > gpurun_out/ncu_$name.log 2>&1
  python scripts/ncu_brief.py /tmp/ncu/$name.ncu-rep > gpurun_out/ncu_${name}_brief.txt 2>&1
done
