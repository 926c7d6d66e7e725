# A/B of K1g build variants (paper_2403_06788_b200/lib/ab/libltci_cuda_<name>.so): coarse-stage time at C1 and C4
for so in paper_2403_06788_b200/lib/ab/libltci_cuda_*.so; do
  name=$(basename $so .so); name=${name#libltci_cuda_}
  LTCI_LIB_PATH=$PWD/$so LTCI_COARSE=gather timeout 300 python scripts/bench_coarse.py --configs 1,4 --runs 7 --tag $name >> gpurun_out/gather_variants.jsonl 2>> gpurun_out/gather_variants.err
done
cat gpurun_out/gather_variants.jsonl
