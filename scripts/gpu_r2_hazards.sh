set -x
python scripts/time_calls.py > gpurun_out/time_calls.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engine_hazards.py -q > gpurun_out/hazards.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
