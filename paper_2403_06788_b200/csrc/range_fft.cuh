// range_fft.cuh -- K0: per-pulse range FFT, range-pulse cube -> freq-pulse cube.
//
// Replaces ltci::range_fft (reference proj/src/signal_model.cpp:97-107,
// declared proj/include/ltci/signal_model.hpp:33-37): per pulse m the
// unnormalised forward transform Y[k] = sum_n x[n] e^{-j 2 pi k n / K}
// (Fft::dft_minus, proj/src/fft.cpp:30-51), column-major k + K m in and out.
// It is the front end of the configs[3] DS-KT-MFP pipeline (range FFT ->
// keystone -> coarse residual RM -> fine DFM): the echo arrives as
// range-compressed fast-time samples and the keystone works per frequency row.
//
// The transform is K1's machinery with the sign flipped by conjugation,
// dft_minus(x) = conj(dft_plus(conj(x))): a CTA transforms PG = 8192 / K
// pulses in shared memory -- radix-16 DIF pass fused with the global loads
// (the f64 -> c64 conversion of a host cube folded in when IN64), middle
// radix-16 passes in place, the last radix pass fused with the store.  The
// last pass maps consecutive threads to consecutive output bins of one pulse,
// so every store is a coalesced run along k.  Bound: HBM (16 B per (row,
// pulse): read + write complex64; 24 B from an f64 input).
#pragma once

#include "coarse.cuh"

namespace ltcib {

constexpr int kRangeFftThreads = 256;

__host__ __device__ constexpr int range_fft_pg(int K, int M) {
    return (8192 / K) < M ? (8192 / K) : M;
}

template <int K>
__host__ __device__ constexpr bool range_fft_swizzled() { return K == 2048; }

inline size_t range_fft_smem_bytes(int K, int M) {
    const int PG = range_fft_pg(K, M);
    const int kp = K == 2048 ? CLayout<2048, true>::kp : coarse_kp(K);
    return static_cast<size_t>(PG) * kp * sizeof(float2);
}

__device__ __forceinline__ float2 conjf2(float2 v) { return make_float2(v.x, -v.y); }

template <int IN64>
__device__ __forceinline__ float2 load_sample(const void* __restrict__ in, size_t i) {
    if constexpr (IN64) {
        const double2 v = __ldg(static_cast<const double2*>(in) + i);
        return make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
    } else {
        return __ldg(static_cast<const float2*>(in) + i);
    }
}

// grid: ceil(M / PG) CTAs of kRangeFftThreads; dynamic smem = range_fft_smem_bytes
template <int K, int IN64>
__global__ void __launch_bounds__(kRangeFftThreads) range_fft_kernel(const void* __restrict__ in,
                                                                     float2* __restrict__ out, int M) {
    constexpr int NT = kRangeFftThreads;
    constexpr bool SW = range_fft_swizzled<K>();
    constexpr int Kp = CLayout<K, SW>::kp;
    extern __shared__ float2 smem[];
    float2* buf = smem;
    const int PG = range_fft_pg(K, M);
    const int m0 = blockIdx.x * PG;
    const int tid = threadIdx.x;

    // pass 1: radix 16 over span S = K / 16, straight from global (conjugated)
    {
        constexpr int S = K / 16;
        for (int i = tid; i < PG * S; i += NT) {
            const int p = i / S;
            const int j = i - p * S;
            const size_t base = static_cast<size_t>(m0 + p) * K + j;
            float2 v[16];
            const bool live = m0 + p < M;  // a partial last pulse group computes on zeros, stores nothing
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = live ? conjf2(load_sample<IN64>(in, base + r * S)) : make_float2(0.f, 0.f);
            dft_reg<16>(v);
            if constexpr (S > 1) twiddle_pow<16>(v, j, K);
            float2* dst = buf + p * Kp;
#pragma unroll
            for (int r = 0; r < 16; ++r) dst[CLayout<K, SW>::idx(j + r * S)] = v[r];
        }
        __syncthreads();
    }
    coarse_middle_passes<K, K / 16, NT, SW>(buf, PG, tid);

    // last pass: thread (p, kl) owns bins kl + G t of pulse p; kl fastest -> coalesced stores
    constexpr int R = K == 16 ? 1 : coarse_last_radix(K);
    constexpr int G = K / R;
    constexpr int NREV = R == 1 ? coarse_npass(K) : coarse_npass(K) - 1;
    for (int idx = tid; idx < PG * G; idx += NT) {
        const int p = idx / G;
        const int kl = idx - p * G;
        if (m0 + p >= M) break;  // idx only grows: every later p is past M too
        const int pos0 = coarse_digit_rev<K, NREV>(kl);
        const float2* src = buf + p * Kp;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[CLayout<K, SW>::idx(pos0 + r)];
        dft_reg<R>(v);
        float2* dst = out + static_cast<size_t>(m0 + p) * K + kl;
#pragma unroll
        for (int t = 0; t < R; ++t) dst[t * G] = conjf2(v[t]);
    }
}

}  // namespace ltcib
