// fine_tc.cuh -- K2a: fine stage as a dense complex contraction on tcgen05
// tensor cores.  Selection helper + launcher.
#pragma once

#include "fine_fft.cuh"

namespace ltcib {

// AUTO keeps the CUDA-core FFT path until the tensor path is built.
inline bool tc_fine_selected(int fine_path, int M, int D, bool keep_dense) {
    (void)M;
    (void)D;
    (void)keep_dense;
    if (fine_path == 2 /* LTCI_FINE_TC_DENSE */)
        throw std::runtime_error("ltci_cuda: tcgen05 fine path not available in this build");
    return false;
}

inline int tc_fine_launch(const FineArgs&, int, cudaStream_t) { return 0; }

}  // namespace ltcib
