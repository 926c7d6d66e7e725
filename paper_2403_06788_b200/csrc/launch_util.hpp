// launch_util.hpp -- host helpers shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "../../include/ltci_cuda.h"
#include "cube_io.hpp"  // CubeError: a status-carrying error every C-ABI entry maps back

namespace ltcib {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CubeError(e == cudaErrorMemoryAllocation ? LTCI_BAD_ALLOC : LTCI_RUNTIME_ERROR,
                        std::string(what) + ": " + cudaGetErrorString(e));
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: raised
// per (kernel, device) whenever a launch needs more than was set before (a
// plan with a larger shared footprint -- e.g. K = 16 at M = 2048 on the fp16
// coarse path -- must not inherit a smaller earlier setting), so one process
// may drive engines of any shape on several GPUs
inline void ensure_smem_attr(const void* kern, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> set_to;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    auto it = set_to.find({kern, dev});
    if (it != set_to.end() && it->second >= bytes) return;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
               "cudaFuncSetAttribute");
    set_to[{kern, dev}] = bytes;
}

}  // namespace ltcib
