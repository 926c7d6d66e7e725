# Round-2 first check: smoke, GPU suite, C1/C0 bench lines and the reference arm on the current tree.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
python bench.py > gpurun_out/bench_c1.log 2>&1
python bench.py --config 0 > gpurun_out/bench_c0.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref_c1.log 2>&1
nvidia-smi -q | grep -iE "product name|clocks" -A3 | head -30 > gpurun_out/smi.log 2>&1
