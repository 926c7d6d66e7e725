# A/B of the result path (round-1 library vs current) on result()-latency-bound workloads
set -x
R1=$PWD/paper_2403_06788_b200/lib/ab/libltci_cuda_r1.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "extreme or c0 or zero" > gpurun_out/tests_x.log 2>&1
python scripts/bench_pd.py > gpurun_out/pd_new.log 2>&1
LTCI_LIB_PATH=$R1 python scripts/bench_pd.py > gpurun_out/pd_r1.log 2>&1
python scripts/e2e_breakdown.py 0 > gpurun_out/e2e_new.log 2>&1
LTCI_LIB_PATH=$R1 python scripts/e2e_breakdown.py 0 > gpurun_out/e2e_r1.log 2>&1
python bench.py --config 0 --no-cpu-baseline > gpurun_out/bench_c0.log 2>&1
