# Functional check of bench.py's N-rank paths on a 1-GPU box: N ranks share cuda:0
# over gloo (LTCI_BENCH_SHARED_GPU=1); the merged per-row peak map must equal the
# 1-rank map bit for bit.  Timings printed by the N-rank runs are not measurements.
set -x
A="--config 0 --steps 3 --warmup 3 --no-cpu-baseline"
LTCI_BENCH_DUMP_PEAKS=gpurun_out/peaks_n1.npy python bench.py $A > gpurun_out/sr_n1.log 2>&1
for SH in coarse rows; do
  for N in 2 3; do
    LTCI_BENCH_SHARED_GPU=1 LTCI_BENCH_DUMP_PEAKS=gpurun_out/peaks_${SH}_n$N.npy timeout 600 \
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 \
      bench.py $A --gpus $N --shard $SH > gpurun_out/sr_${SH}_n$N.log 2>&1
  done
done
# the same with the interpolating coarse gather forced (configs[0] alone would take the transform)
LTCI_COARSE=gather LTCI_BENCH_DUMP_PEAKS=gpurun_out/gpeaks_n1.npy python bench.py $A > gpurun_out/sr_g_n1.log 2>&1
for SH in coarse rows; do
  for N in 2 3; do
    LTCI_COARSE=gather LTCI_BENCH_SHARED_GPU=1 LTCI_BENCH_DUMP_PEAKS=gpurun_out/gpeaks_${SH}_n$N.npy timeout 600 \
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 \
      bench.py $A --gpus $N --shard $SH > gpurun_out/sr_g_${SH}_n$N.log 2>&1
  done
done
LTCI_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29612 bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --gpus 2 > gpurun_out/sr_c4_n2.log 2>&1
python - <<'PY' > gpurun_out/sr_compare.log 2>&1
import numpy as np, glob
ref = np.load("gpurun_out/peaks_n1.npy")
for f in sorted(glob.glob("gpurun_out/peaks_*_n*.npy")):
    a = np.load(f)
    print(f, a.shape, "identical" if a.shape == ref.shape and (a == ref).all() else "DIFFERENT")
gref = np.load("gpurun_out/gpeaks_n1.npy")
for f in sorted(glob.glob("gpurun_out/gpeaks_*_n*.npy")):
    a = np.load(f)
    print(f, "(LTCI_COARSE=gather)", a.shape, "identical" if a.shape == gref.shape and (a == gref).all() else "DIFFERENT")
PY
