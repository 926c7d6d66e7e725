// gather_launch.cu -- launchers of K1g (gather.cuh): the deapodisation table,
// the oversampled range profiles (K1's transform passes, TAB instantiation)
// and the per-batch weights + gather.  Replaces mgift for the FP32 fine path
// (reference proj/src/transforms.cpp:134-173).
#include "coarse.cuh"
#include "gather.cuh"
#include "gather_launch.hpp"
#include "launch_util.hpp"

namespace ltcib {
namespace {

__global__ void gather_module_anchor_kernel() {}

template <int K>
void launch_tables_k(const CoarseArgs& a, cudaStream_t st) {
    auto kern = coarse_rm_kernel<K, 0, 1>;
    CoarseArgs b = a;
    b.pg = coarse_pg_launch(K, a.M, 0, a.c_count);
    const size_t smem = coarse_smem_bytes(K, a.M, 0, b.pg);
    ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    kern<<<dim3(a.M / b.pg, a.c_count), coarse_threads<0>(), smem, st>>>(b);
    cuda_check(cudaGetLastError(), "gather table launch");
}

}  // namespace

const void* gather_module_anchor() { return reinterpret_cast<const void*>(gather_module_anchor_kernel); }

void launch_gather_deap(float* deap, int K, cudaStream_t st) {
    gather_deap_kernel<<<(K / 2 + 1 + 31) / 32, 32, 0, st>>>(deap, K);
    cuda_check(cudaGetLastError(), "gather deap launch");
}

void launch_gather_tables(const CoarseArgs& a, cudaStream_t st) {
    switch (a.K) {
        case 64: launch_tables_k<64>(a, st); break;
        case 128: launch_tables_k<128>(a, st); break;
        case 256: launch_tables_k<256>(a, st); break;
        case 512: launch_tables_k<512>(a, st); break;
        case 1024: launch_tables_k<1024>(a, st); break;
        case 2048: launch_tables_k<2048>(a, st); break;
        case 4096: launch_tables_k<4096>(a, st); break;
        case 8192: launch_tables_k<8192>(a, st); break;
        default: throw CubeError(LTCI_INVALID_ARGUMENT, "ltci_cuda: unsupported K for the gather tables");
    }
}

void launch_gather_weights(const GatherArgs& a, cudaStream_t st) {
    const size_t total = static_cast<size_t>(a.c_count) * a.M;
    gather_weights_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(a);
    cuda_check(cudaGetLastError(), "gather weights launch");
}

void launch_gather_cells(const GatherArgs& a, cudaStream_t st) {
    const int rows_cap = kGatherRows + kGatherHalo;
    const size_t smem = gather_smem_bytes(rows_cap);
    ensure_smem_attr(reinterpret_cast<const void*>(gather_interp_kernel), static_cast<int>(smem));
    const unsigned long long cpt = a.cells_per_table;
    const unsigned long long gpt = (cpt + kGatherCells - 1) / kGatherCells;
    const unsigned long long t0 = a.c_begin / cpt, t1 = (a.c_begin + a.c_count - 1) / cpt;
    const unsigned long long gz = (t1 - t0 + 1) * gpt;
    if (gz > 65535) throw CubeError(LTCI_INVALID_ARGUMENT, "ltci_cuda: gather batch exceeds the grid");
    const dim3 grid(a.M / 32, static_cast<unsigned>(gz), (a.R_slice + kGatherRows - 1) / kGatherRows);
    gather_interp_kernel<<<grid, kGatherThreads, smem, st>>>(a, rows_cap);
    cuda_check(cudaGetLastError(), "gather launch");
}

}  // namespace ltcib
