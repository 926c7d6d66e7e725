A="--config 1 --steps 2 --warmup 3 --no-cpu-baseline"
LTCI_BENCH_DUMP_PEAKS=gpurun_out/c1peaks_n1.npy python bench.py $A > gpurun_out/c1sr_n1.log 2>&1
for spec in "rows 2" "rows 8" "coarse 3"; do
  set -- $spec
  LTCI_BENCH_SHARED_GPU=1 LTCI_BENCH_DUMP_PEAKS=gpurun_out/c1peaks_$1_n$2.npy timeout 900 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 29651 \
    bench.py $A --gpus $2 --shard $1 > gpurun_out/c1sr_$1_n$2.log 2>&1
  echo "$spec rc=$?"
done
python - <<'PY'
import numpy as np, glob
ref = np.load("gpurun_out/c1peaks_n1.npy")
for f in sorted(glob.glob("gpurun_out/c1peaks_*_n*.npy")):
    a = np.load(f)
    print(f, a.shape, "identical" if a.shape == ref.shape and (a == ref).all() else "DIFFERENT")
PY
