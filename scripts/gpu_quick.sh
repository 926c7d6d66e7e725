set -x
for i in 1 2 3; do LTCI_TRACE=1 oracle/_ref/acceptance_dropin 7; done > gpurun_out/q_c7.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_parity.py tests/test_montecarlo.py tests/test_gpu_tm.py tests/test_detections.py tests/test_gpu_tc.py -x -q > gpurun_out/q_tests.log 2>&1
python scripts/time_calls.py > gpurun_out/q_time_calls.log 2>&1
