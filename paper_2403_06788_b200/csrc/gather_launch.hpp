// gather_launch.hpp -- launchers of the interpolating coarse gather (K1g,
// gather.cuh), compiled in their own translation unit (gather_launch.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace ltcib {

struct CoarseArgs;

struct GatherArgs {
    const float2* U;         // [tables][2][K][M]: even / odd fine samples of each pulse
    float4* W;               // [3][w_plane]: even-stream taps, odd-stream taps, (pre.x, pre.y, L, -);
                             // cell c, pulse m at (c - w_first) * M + m of each plane
    size_t w_plane;
    unsigned long long w_first;
    const double* cparams;   // [coarse][4]: GRFT c1..cP ; KT (q, c2)
    float2* X;               // [c_count * R_slice][M]
    unsigned long long c_begin;
    unsigned long long cells_per_table;  // GRFT: every cell reads table 0; KT: one table per folding number
    int c_count;
    int K, M, P, variant;
    int n_base, R_slice;
    double inv_prf, inv_dR, two_over_lambda, Va;
};

// shapes K1g takes (otherwise the transform kernel K1 runs)
inline bool gather_supported(int K, int M) { return K >= 64 && M >= 32; }

// bytes of the per-batch weight scratch: 3 float4 per (cell, pulse)
inline size_t gather_weight_bytes(unsigned long long cells, int M) {
    return static_cast<size_t>(cells) * static_cast<size_t>(M) * 48;
}

// deap[k], k < K: the reciprocal transform of the interpolation window per frequency row
void launch_gather_deap(float* deap, int K, cudaStream_t st);

// the oversampled profiles: a.cparams = [2 * tables][4] (delta in range cells, q, -, -),
// a.X = U [2 * tables][K][M], a.deap set, a.c_count = 2 * tables, full range axis
void launch_gather_tables(const CoarseArgs& a, cudaStream_t st);

// the (cell, pulse) weights of cells [a.c_begin, a.c_begin + a.c_count)
void launch_gather_weights(const GatherArgs& a, cudaStream_t st);

// gather of one batch of coarse cells (weights already in a.W)
void launch_gather_cells(const GatherArgs& a, cudaStream_t st);

const void* gather_module_anchor();

}  // namespace ltcib
