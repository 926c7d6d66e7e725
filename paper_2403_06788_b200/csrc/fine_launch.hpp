// fine_launch.hpp -- the CUDA-core fine stage (K2b + K3) launchers, compiled in
// their own translation unit (fine_launch.cu): alone, ptxas allocates the
// TMEM-row kernels without the spills it produced when they shared engine.cu
// with the coarse, tcgen05 and fd_grft kernels.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>

namespace ltcib {

struct FineArgs;

// fine_fft_tm_kernel / fine_fft_tm2k_kernel / fine_fft_kernel for M = 4..2048;
// throws CubeError (LTCI_INVALID_ARGUMENT) for a shape the CUDA-core path does not take
void launch_fine_m(const FineArgs& a, int M, bool dense, cudaStream_t st);

// a kernel of fine_launch.cu's module (the engine preloads every function of it)
const void* fine_module_anchor();

// M = 2048 (fine_fft_tm2k_kernel): NB over the half-length (1024-bin) axes of
// the even and odd output bins; 0 = window too wide for the kernel
inline int tm2k_nb(int kA, int kB) {
    const int nbp = kA >= 0 ? (kA / 2) / 32 + 1 : 0;
    const int nbn = kB <= 2047 ? 32 - ((kB - 1) / 2) / 32 : 0;
    const int nb = std::max(nbp, nbn);
    return nb <= 3 ? 3 : nb <= 6 ? 6 : 0;
}

}  // namespace ltcib
