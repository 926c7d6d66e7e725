# A/B of the fp32 coarse kernel's pass-1 ILP (LTCI_COARSE_H32) and CTAs/SM (LTCI_COARSE_MINB32):
# rebuilds the library on the box per variant and reads coarse_ms from a short C1 bench.
set -x
for v in "1 3" "2 2" "2 3"; do
  set -- $v
  touch paper_2403_06788_b200/csrc/engine.cu
  make -s -C paper_2403_06788_b200/csrc EXTRA="-DLTCI_COARSE_H32=$1 -DLTCI_COARSE_MINB32=$2" > gpurun_out/ab_build_$1_$2.log 2>&1
  for c in 1 3; do
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c${c}_$1_$2.log 2>&1
  done
done
