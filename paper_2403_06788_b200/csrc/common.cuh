// common.cuh -- complex helpers and in-register power-of-two DFTs (sign +1,
// the reference's dft_plus kernel exp(+j 2 pi k n / N), proj/src/fft.cpp:30-51).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ltcib {

// Complex arithmetic on packed FP32 pairs: sm_100 executes add/sub/mul/fma
// .f32x2 as one instruction (FADD2/FMUL2/FFMA2) whose operands may be swapped,
// partially negated or broadcast for free, so a complex add is 1 issue slot
// instead of 2 and a complex multiply 2 instead of 4 (the DFT networks below
// are issue-bound).  Rounding is per component, as for scalar add.rn/fma.rn.
__device__ __forceinline__ unsigned long long f2_pack(float2 v) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
    return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return sub2(a, b); }
// a b = a (b.x, b.x) + (-a.y, a.x) (b.y, b.y)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return fma2(make_float2(-a.y, a.x), make_float2(b.y, b.y), mul2(a, make_float2(b.x, b.x)));
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

// Factored twiddles for the FMA butterfly: w = e^{+j 2 pi k/64}, k = 0..31,
// as w = f (1 + j r) (k <= 8 or k > 24, |cos| >= |sin|) or w = f (r + j)
// otherwise, |r| <= 1, both rounded to float.
__device__ __constant__ float2 kTwF64[32] = {
    {1.000000000e+00f, 0.000000000e+00f}, {9.951847196e-01f, 9.849140048e-02f},
    {9.807852507e-01f, 1.989123672e-01f}, {9.569403529e-01f, 3.033466935e-01f},
    {9.238795042e-01f, 4.142135680e-01f}, {8.819212914e-01f, 5.345111489e-01f},
    {8.314695954e-01f, 6.681786180e-01f}, {7.730104327e-01f, 8.206787705e-01f},
    {7.071067691e-01f, 1.000000000e+00f}, {7.730104327e-01f, 8.206787705e-01f},
    {8.314695954e-01f, 6.681786180e-01f}, {8.819212914e-01f, 5.345111489e-01f},
    {9.238795042e-01f, 4.142135680e-01f}, {9.569403529e-01f, 3.033466935e-01f},
    {9.807852507e-01f, 1.989123672e-01f}, {9.951847196e-01f, 9.849140048e-02f},
    {1.000000000e+00f, 6.123234263e-17f}, {9.951847196e-01f, -9.849140048e-02f},
    {9.807852507e-01f, -1.989123672e-01f}, {9.569403529e-01f, -3.033466935e-01f},
    {9.238795042e-01f, -4.142135680e-01f}, {8.819212914e-01f, -5.345111489e-01f},
    {8.314695954e-01f, -6.681786180e-01f}, {7.730104327e-01f, -8.206787705e-01f},
    {7.071067691e-01f, -1.000000000e+00f}, {-7.730104327e-01f, -8.206787705e-01f},
    {-8.314695954e-01f, -6.681786180e-01f}, {-8.819212914e-01f, -5.345111489e-01f},
    {-9.238795042e-01f, -4.142135680e-01f}, {-9.569403529e-01f, -3.033466935e-01f},
    {-9.807852507e-01f, -1.989123672e-01f}, {-9.951847196e-01f, -9.849140048e-02f}
};

// (a + b w, a - b w) for w = e^{+j 2 pi K/LEN}: the trivial rotations by
// add/sub/swap, the others as u = b (1 + j r) then a +- f u: three packed
// FFMA2 instead of a complex multiply plus two complex adds.
// LO / HI select which of the two outputs are produced.
template <int K, int LEN, bool LO = true, bool HI = true>
__device__ __forceinline__ void butterfly_tw(const float2 a, const float2 b, float2& lo, float2& hi) {
    if constexpr (K == 0 || 4 * K == LEN) {
        const float2 t = twiddle_mul<K, LEN>(b);
        if constexpr (LO) lo = cadd(a, t);
        if constexpr (HI) hi = csub(a, t);
    } else {
        static_assert(LEN <= 64 && 2 * K < LEN, "twiddle table covers radices up to 64");
        constexpr int k64 = K * (64 / LEN);
        const float f = kTwF64[k64].x, r = kTwF64[k64].y;
        float2 u;
        if constexpr (k64 <= 8 || k64 > 24) {
            u = fma2(make_float2(-b.y, b.x), make_float2(r, r), b);                  // b (1 + j r)
        } else {
            u = fma2(b, make_float2(r, r), make_float2(-b.y, b.x));                  // b (r + j)
        }
        if constexpr (LO) lo = fma2(u, make_float2(f, f), a);
        if constexpr (HI) hi = fma2(u, make_float2(-f, -f), a);
    }
}

template <int LEN, int HALF, int K, int R>
__device__ __forceinline__ void dit_stage_inner(float2 (&v)[R], int base) {
    if constexpr (K < HALF) {
        const float2 a = v[base + K], b = v[base + K + HALF];
        butterfly_tw<K, LEN>(a, b, v[base + K], v[base + K + HALF]);
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

// ---- output-pruned DFT ------------------------------------------------------
// Same transform, but only the outputs k with bit k of NEED set are produced
// (the others are left undefined).  In a radix-2 DIT network the stage of
// length LEN feeds output k only through its own output (k mod LEN), so every
// butterfly whose two outputs are both unused at its stage is dropped, and a
// butterfly with one used output computes only that half.
template <int LEN, int R, unsigned long long NEED>
constexpr unsigned long long dit_stage_mask() {
    unsigned long long m = 0;
    for (int k = 0; k < R; ++k)
        if ((NEED >> k) & 1ull) m |= 1ull << (k % LEN);
    return m;
}

template <int LEN, int HALF, int K, int R, unsigned long long MASK>
__device__ __forceinline__ void dit_stage_inner_p(float2 (&v)[R], int base) {
    if constexpr (K < HALF) {
        constexpr bool kLo = (MASK >> K) & 1ull, kHi = (MASK >> (K + HALF)) & 1ull;
        if constexpr (kLo || kHi) {
            const float2 a = v[base + K], b = v[base + K + HALF];
            butterfly_tw<K, LEN, kLo, kHi>(a, b, v[base + K], v[base + K + HALF]);
        }
        dit_stage_inner_p<LEN, HALF, K + 1, R, MASK>(v, base);
    }
}

template <int LEN, int R, unsigned long long NEED>
__device__ __forceinline__ void dit_stage_p(float2 (&v)[R]) {
    if constexpr (LEN <= R) {
        constexpr unsigned long long kMask = dit_stage_mask<LEN, R, NEED>();
#pragma unroll
        for (int base = 0; base < R; base += LEN) dit_stage_inner_p<LEN, LEN / 2, 0, R, kMask>(v, base);
        dit_stage_p<LEN * 2, R, NEED>(v);
    }
}

template <int R, unsigned long long NEED>
__device__ __forceinline__ void dft_reg_pruned(float2 (&v)[R]) {
    static_assert(R <= 64, "mask is 64 bits");
    if constexpr (R > 1) {
        bitrev_perm<0, R>(v);
        dit_stage_p<2, R, NEED>(v);
    }
}

// outputs {0..NB-1} and {R-NB..R-1}: a Doppler window centred on d = 0
template <int R, int NB>
constexpr unsigned long long window_need_mask() {
    unsigned long long m = 0;
    for (int k = 0; k < NB; ++k) m |= (1ull << k) | (1ull << (R - 1 - k));
    return m;
}

}  // namespace ltcib
