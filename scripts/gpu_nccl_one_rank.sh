# bench.py's N-rank code path over REAL NCCL on a 1-GPU box: torchrun with one rank and
# LTCI_BENCH_FORCE_DIST=1 (NCCL communicator, barriers, peak all-gather + device merge, max-over-ranks
# all_reduce).  The gathered peak map must equal the plain 1-process map bit for bit.
set -x
A="--config 1 --steps 3 --warmup 3 --no-cpu-baseline"
LTCI_BENCH_DUMP_PEAKS=gpurun_out/n1_plain.npy python bench.py $A > gpurun_out/nccl1_plain.log 2>&1
for SH in coarse rows; do
  LTCI_BENCH_FORCE_DIST=1 LTCI_BENCH_DUMP_PEAKS=gpurun_out/n1_nccl_$SH.npy timeout 600 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29621 \
    bench.py $A --gpus 1 --shard $SH > gpurun_out/nccl1_$SH.log 2>&1
done
python - <<'PY' > gpurun_out/nccl1_compare.log 2>&1
import numpy as np, json
ref = np.load("gpurun_out/n1_plain.npy")
for sh in ("coarse", "rows"):
    a = np.load(f"gpurun_out/n1_nccl_{sh}.npy")
    line = [l for l in open(f"gpurun_out/nccl1_{sh}.log") if l.startswith("{")][-1]
    d = json.loads(line)
    nccl = [l.strip() for l in open(f"gpurun_out/nccl1_{sh}.log") if "NCCL INFO" in l and ("nranks" in l.lower() or "Init COMPLETE" in l or "NCCL version" in l)][:5]
    print(sh, a.shape, "identical to the plain 1-process map" if a.shape == ref.shape and (a == ref).all() else "DIFFERENT",
          "| value", round(d["value"], 1), d["unit"], "| e2e", round(d["e2e"]["value"], 1), "|", d["config"]["parallelism"], "|", d.get("n_rank_path_forced"))
    for l in nccl:
        print("   ", l[:220])
PY
cat gpurun_out/nccl1_compare.log
