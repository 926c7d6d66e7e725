# A/B builds of libltci_cuda.so with compile-time variants, into paper_2403_06788_b200/lib/ab/
# (select one at run time with LTCI_LIB_PATH=...).  usage: bash scripts/build_ab.sh NAME "-DMACRO=VAL ..."
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
SRC=$HERE/paper_2403_06788_b200/csrc
OUT=$HERE/paper_2403_06788_b200/lib/ab
mkdir -p "$OUT"
cd "$SRC"
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  --expt-relaxed-constexpr $2 -shared -o "$OUT/libltci_cuda_$1.so" engine.cu fine_launch.cu gather_launch.cu detection.cpp cube_io.cpp pd.cu
echo "built $OUT/libltci_cuda_$1.so"
