# A/B of the fp32 coarse kernel's CTA size (LTCI_COARSE_NT32), pass-1 ILP (LTCI_COARSE_H32) and
# CTAs/SM (LTCI_COARSE_MINB32): rebuilds the library on the box per variant, runs the coarse parity
# tests and reads coarse_ms from short C1/C3 benches.  Usage: bash scripts/gpu_coarse_ab.sh "NT H MINB" ...
set -x
for v in "$@"; do
  set -- $v
  tag=$1_$2_$3
  touch paper_2403_06788_b200/csrc/engine.cu
  make -s -C paper_2403_06788_b200/csrc EXTRA="-DLTCI_COARSE_NT32=$1 -DLTCI_COARSE_H32=$2 -DLTCI_COARSE_MINB32=$3" \
    > gpurun_out/ab_build_$tag.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab_tests_$tag.log 2>&1
  for c in 1 3 4; do
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c${c}_$tag.log 2>&1
  done
done
