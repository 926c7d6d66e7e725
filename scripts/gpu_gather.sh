# K1g (interpolating coarse gather) check: its parity tests, then the coarse-stage A/B on C1/C3/C0/C4
set -x
timeout 900 python -m pytest tests/test_gpu_gather.py -x -q > gpurun_out/gather_tests.log 2>&1
tail -15 gpurun_out/gather_tests.log
for mode in transform gather; do
  LTCI_COARSE=$mode timeout 600 python scripts/bench_coarse.py --configs 1,3,0,4 --runs 5 --tag $mode >> gpurun_out/gather_ab.jsonl 2>> gpurun_out/gather_ab.err
done
LTCI_X_BUDGET_MB=6144 timeout 600 python scripts/bench_coarse.py --configs 1 --runs 5 --tag auto_6g >> gpurun_out/gather_ab.jsonl 2>> gpurun_out/gather_ab.err
cat gpurun_out/gather_ab.jsonl
