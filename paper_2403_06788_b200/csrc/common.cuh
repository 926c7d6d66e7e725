// common.cuh -- complex helpers and in-register power-of-two DFTs (sign +1,
// the reference's dft_plus kernel exp(+j 2 pi k n / N), proj/src/fft.cpp:30-51).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ltcib {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(__fmaf_rn(a.x, b.x, -__fmul_rn(a.y, b.y)), __fmaf_rn(a.x, b.y, __fmul_rn(a.y, b.x)));
}
// |v|^2 evaluated the same way everywhere (device kernels, CAS comparisons and
// the host merge), so magnitude ties compare identically.
__host__ __device__ __forceinline__ float mag2f(float re, float im) {
#ifdef __CUDA_ARCH__
    return __fmaf_rn(re, re, __fmul_rn(im, im));
#else
    return fmaf(re, re, im * im);
#endif
}

// exp(+j 2 pi k / 64), k = 0..63, rounded to float.
__device__ __constant__ float2 kTw64[64] = {
    {1.000000000e+00f, 0.000000000e+00f},   {9.951847267e-01f, 9.801714033e-02f},
    {9.807852804e-01f, 1.950903220e-01f},   {9.569403357e-01f, 2.902846773e-01f},
    {9.238795325e-01f, 3.826834324e-01f},   {8.819212643e-01f, 4.713967368e-01f},
    {8.314696123e-01f, 5.555702330e-01f},   {7.730104534e-01f, 6.343932842e-01f},
    {7.071067812e-01f, 7.071067812e-01f},   {6.343932842e-01f, 7.730104534e-01f},
    {5.555702330e-01f, 8.314696123e-01f},   {4.713967368e-01f, 8.819212643e-01f},
    {3.826834324e-01f, 9.238795325e-01f},   {2.902846773e-01f, 9.569403357e-01f},
    {1.950903220e-01f, 9.807852804e-01f},   {9.801714033e-02f, 9.951847267e-01f},
    {6.123233996e-17f, 1.000000000e+00f},   {-9.801714033e-02f, 9.951847267e-01f},
    {-1.950903220e-01f, 9.807852804e-01f},  {-2.902846773e-01f, 9.569403357e-01f},
    {-3.826834324e-01f, 9.238795325e-01f},  {-4.713967368e-01f, 8.819212643e-01f},
    {-5.555702330e-01f, 8.314696123e-01f},  {-6.343932842e-01f, 7.730104534e-01f},
    {-7.071067812e-01f, 7.071067812e-01f},  {-7.730104534e-01f, 6.343932842e-01f},
    {-8.314696123e-01f, 5.555702330e-01f},  {-8.819212643e-01f, 4.713967368e-01f},
    {-9.238795325e-01f, 3.826834324e-01f},  {-9.569403357e-01f, 2.902846773e-01f},
    {-9.807852804e-01f, 1.950903220e-01f},  {-9.951847267e-01f, 9.801714033e-02f},
    {-1.000000000e+00f, 1.224646799e-16f},  {-9.951847267e-01f, -9.801714033e-02f},
    {-9.807852804e-01f, -1.950903220e-01f}, {-9.569403357e-01f, -2.902846773e-01f},
    {-9.238795325e-01f, -3.826834324e-01f}, {-8.819212643e-01f, -4.713967368e-01f},
    {-8.314696123e-01f, -5.555702330e-01f}, {-7.730104534e-01f, -6.343932842e-01f},
    {-7.071067812e-01f, -7.071067812e-01f}, {-6.343932842e-01f, -7.730104534e-01f},
    {-5.555702330e-01f, -8.314696123e-01f}, {-4.713967368e-01f, -8.819212643e-01f},
    {-3.826834324e-01f, -9.238795325e-01f}, {-2.902846773e-01f, -9.569403357e-01f},
    {-1.950903220e-01f, -9.807852804e-01f}, {-9.801714033e-02f, -9.951847267e-01f},
    {-1.836970199e-16f, -1.000000000e+00f}, {9.801714033e-02f, -9.951847267e-01f},
    {1.950903220e-01f, -9.807852804e-01f},  {2.902846773e-01f, -9.569403357e-01f},
    {3.826834324e-01f, -9.238795325e-01f},  {4.713967368e-01f, -8.819212643e-01f},
    {5.555702330e-01f, -8.314696123e-01f},  {6.343932842e-01f, -7.730104534e-01f},
    {7.071067812e-01f, -7.071067812e-01f},  {7.730104534e-01f, -6.343932842e-01f},
    {8.314696123e-01f, -5.555702330e-01f},  {8.819212643e-01f, -4.713967368e-01f},
    {9.238795325e-01f, -3.826834324e-01f},  {9.569403357e-01f, -2.902846773e-01f},
    {9.807852804e-01f, -1.950903220e-01f},  {9.951847267e-01f, -9.801714033e-02f},
};

constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }
constexpr int bitrev(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b)
        if (i & (1 << b)) r |= 1 << (bits - 1 - b);
    return r;
}

// Multiply by exp(+j 2 pi k / len) for compile-time k, len (k < len/2),
// skipping the trivial rotations.
template <int K, int LEN>
__device__ __forceinline__ float2 twiddle_mul(float2 b) {
    constexpr float kS = 0.70710678118654752f;
    if constexpr (K == 0) {
        return b;
    } else if constexpr (4 * K == LEN) {  // +j
        return make_float2(-b.y, b.x);
    } else if constexpr (8 * K == LEN) {  // (1+j)/sqrt2
        return make_float2((b.x - b.y) * kS, (b.x + b.y) * kS);
    } else if constexpr (8 * K == 3 * LEN) {  // (-1+j)/sqrt2
        return make_float2(-(b.x + b.y) * kS, (b.x - b.y) * kS);
    } else {
        static_assert(LEN <= 64, "twiddle table covers radices up to 64");
        return cmul(b, kTw64[K * (64 / LEN)]);
    }
}

template <int LEN, int HALF, int K, int R>
__device__ __forceinline__ void dit_stage_inner(float2 (&v)[R], int base) {
    if constexpr (K < HALF) {
        float2 a = v[base + K];
        float2 b = twiddle_mul<K, LEN>(v[base + K + HALF]);
        v[base + K] = cadd(a, b);
        v[base + K + HALF] = csub(a, b);
        dit_stage_inner<LEN, HALF, K + 1, R>(v, base);
    }
}

template <int LEN, int R>
__device__ __forceinline__ void dit_stage(float2 (&v)[R]) {
    if constexpr (LEN <= R) {
#pragma unroll
        for (int base = 0; base < R; base += LEN) dit_stage_inner<LEN, LEN / 2, 0, R>(v, base);
        dit_stage<LEN * 2, R>(v);
    }
}

template <int I, int R>
__device__ __forceinline__ void bitrev_perm(float2 (&v)[R]) {
    if constexpr (I < R) {
        constexpr int J = bitrev(I, ilog2c(R));
        if constexpr (J > I) {
            float2 t = v[I];
            v[I] = v[J];
            v[J] = t;
        }
        bitrev_perm<I + 1, R>(v);
    }
}

// In-place, unnormalised, natural-order output: v[k] <- sum_n v[n] e^{+j2pi kn/R}.
template <int R>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
    if constexpr (R > 1) {
        bitrev_perm<0, R>(v);
        dit_stage<2, R>(v);
    }
}

}  // namespace ltcib
