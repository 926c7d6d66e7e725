// fine_launch.cu -- launchers of the CUDA-core fine stage (K2b + K3: chirp +
// FFT with TMEM-resident rows, window-pruned second pass, fused |Y|^2 /
// threshold / per-row argmax; fine_fft.cuh), in their own translation unit.
// Kernels and the algorithm: fine_fft.cuh; replaces gft + build_mf(DFM) +
// UnitScan (reference proj/src/transforms.cpp:180-214, proj/src/detectors.cpp:23-31).
#include <cstdlib>

#include "fine_fft.cuh"
#include "fine_launch.hpp"
#include "launch_util.hpp"

namespace ltcib {
namespace {

__global__ void fine_module_anchor_kernel() {}

// Doppler-window blocks: the smallest NB in {3, 6} with every needed bin in the
// first or last NB 32-bin blocks, else 0 (any window, e.g. DS-KT-MFP's full axis)
inline int fine_window_nb(const FineArgs& a, int Q, int G) {
    const int nbp = a.kA >= 0 ? a.kA / Q + 1 : 0;
    const int nbn = a.kB <= Q * G - 1 ? G - a.kB / Q : 0;
    const int nb = std::max(nbp, nbn);
    if (std::getenv("LTCI_FINE_NOPRUNE")) return 0;
    return nb <= 3 ? 3 : nb <= 6 ? 6 : 0;
}

template <int Q, int G, bool DENSE, int NB>
void launch_fine_tm_nb(const FineArgs& a, cudaStream_t st) {
    const size_t smem = fine_tm_smem_floats2<Q, G>() * sizeof(float2);
    auto kern = fine_fft_tm_kernel<Q, G, DENSE, NB>;
    ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    constexpr int rows_per_block = fine_tm_warps<Q, G>() * (32 / G);
    const int blocks = (a.rows + rows_per_block - 1) / rows_per_block;
    kern<<<dim3(blocks, a.n_split), fine_tm_warps<Q, G>() * 32, smem, st>>>(a);
    cuda_check(cudaGetLastError(), "fine kernel launch");
}

template <int Q, int G, bool DENSE>
void launch_fine_tm(const FineArgs& a, cudaStream_t st) {
    if constexpr (G >= 8) {
        const int nb = 2 * fine_window_nb(a, Q, G) <= G ? fine_window_nb(a, Q, G) : 0;
        if (nb == 3) return launch_fine_tm_nb<Q, G, DENSE, 3>(a, st);
        if (nb == 6) return launch_fine_tm_nb<Q, G, DENSE, 6>(a, st);
    }
    launch_fine_tm_nb<Q, G, DENSE, 0>(a, st);
}

template <int Q, int G, bool DENSE>
void launch_fine_qg(const FineArgs& a, cudaStream_t st) {
    if constexpr (Q == 32 && (G == 32 || G == 16 || G == 8)) {
        if (!std::getenv("LTCI_FINE_TM_OFF")) {  // TMEM-resident row variant (M = 1024, 512, 256)
            launch_fine_tm<Q, G, DENSE>(a, st);
            return;
        }
    }
    if (a.n_split != 1) throw CubeError(LTCI_RUNTIME_ERROR, "ltci_cuda: fine-axis split on a kernel without it");
    constexpr int rows_per_block = (kFineThreads / 32) * (32 / G);
    const size_t smem = fine_smem_floats2<Q, G>() * sizeof(float2);
    auto kern = fine_fft_kernel<Q, G, DENSE>;
    ensure_smem_attr(reinterpret_cast<const void*>(kern), 200 * 1024);
    const int blocks = (a.rows + rows_per_block - 1) / rows_per_block;
    kern<<<blocks, kFineThreads, smem, st>>>(a);
    cuda_check(cudaGetLastError(), "fine kernel launch");
}

template <bool DENSE, int NB>
void launch_fine_tm2k_nb(const FineArgs& a, cudaStream_t st) {
    auto kern = fine_fft_tm2k_kernel<DENSE, NB>;
    const int smem = fine_tm2k_smem_bytes();
    ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
    const int blocks = (a.rows + kTm2kWarps - 1) / kTm2kWarps;
    kern<<<blocks, kTm2kWarps * 32, smem, st>>>(a);
    cuda_check(cudaGetLastError(), "fine kernel launch");
}

template <bool DENSE>
void launch_fine_m_t(const FineArgs& a, int M, cudaStream_t st) {
    if (M == 2048) {
        const int nb = tm2k_nb(a.kA, a.kB);
        if (nb == 3) return launch_fine_tm2k_nb<DENSE, 3>(a, st);
        if (nb == 6) return launch_fine_tm2k_nb<DENSE, 6>(a, st);
        throw CubeError(LTCI_INVALID_ARGUMENT, "ltci_cuda: CUDA-core fine path at M = 2048 needs a Doppler window of "
                                               "at most 12 x 64 bins (use the tcgen05 path)");
    }
    switch (M) {
        case 4: launch_fine_qg<4, 1, DENSE>(a, st); break;
        case 8: launch_fine_qg<8, 1, DENSE>(a, st); break;
        case 16: launch_fine_qg<16, 1, DENSE>(a, st); break;
        case 32: launch_fine_qg<32, 1, DENSE>(a, st); break;
        case 64: launch_fine_qg<32, 2, DENSE>(a, st); break;
        case 128: launch_fine_qg<32, 4, DENSE>(a, st); break;
        case 256: launch_fine_qg<32, 8, DENSE>(a, st); break;
        case 512: launch_fine_qg<32, 16, DENSE>(a, st); break;
        case 1024: launch_fine_qg<32, 32, DENSE>(a, st); break;
        default: throw CubeError(LTCI_INVALID_ARGUMENT, "ltci_cuda: unsupported M");
    }
}

}  // namespace

void launch_fine_m(const FineArgs& a, int M, bool dense, cudaStream_t st) {
    if (dense)
        launch_fine_m_t<true>(a, M, st);
    else
        launch_fine_m_t<false>(a, M, st);
}

const void* fine_module_anchor() { return reinterpret_cast<const void*>(fine_module_anchor_kernel); }

}  // namespace ltcib
