# A/B builds of the K1g translation unit only (gather_launch.cu; the other objects are compiled once into /tmp/abobj):
#   bash scripts/build_gather_ab.sh NAME -DLTCI_GATHER_ROWS=64 -DLTCI_GATHER_MINB=3 ...  -> lib/ab/libltci_cuda_NAME.so
# (variants measured in profiles/r02_gather_variants.jsonl; run with scripts/gpu_gather_ab.sh)
# fast A/B: only gather_launch.cu differs; link against objects of the other TUs
set -e
SRC=/root/repo/paper_2403_06788_b200/csrc
OUT=/root/repo/paper_2403_06788_b200/lib/ab
mkdir -p $OUT /tmp/abobj
cd $SRC
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
if [ ! -f /tmp/abobj/engine.o ] || [ engine.cu -nt /tmp/abobj/engine.o ]; then
  for f in engine fine_launch pd; do nvcc $FLAGS -c $f.cu -o /tmp/abobj/$f.o & done
  for f in detection cube_io; do nvcc $FLAGS -x cu -c $f.cpp -o /tmp/abobj/$f.o & done
  wait
fi
name=$1; shift
nvcc $FLAGS "$@" -c gather_launch.cu -o /tmp/abobj/gather_$name.o
nvcc -shared -o $OUT/libltci_cuda_$name.so /tmp/abobj/engine.o /tmp/abobj/fine_launch.o /tmp/abobj/pd.o /tmp/abobj/detection.o /tmp/abobj/cube_io.o /tmp/abobj/gather_$name.o
echo built $name
