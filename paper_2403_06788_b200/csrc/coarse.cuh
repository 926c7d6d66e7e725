// coarse.cuh -- K1 coarse range-migration correction ("gather") and K4 keystone.
//
// K1 replaces mgift = gift + compensated_ifft + build_mf(RM|KtRm, PreDfm)
// (reference proj/src/transforms.cpp:32-94,134-173).  Per coarse cell c and
// pulse m the reference forms y(:,m) .* H_RM(:,m), takes the unnormalised
// K-point dft_plus and multiplies by preDFM(m).  Mathematically that is an
// exact band-limited fractional-delay gather of the range profile along the
// coarse trajectory:
//   X_c[n,m] = preDFM_c(m) * IFFT_K( y(:,m) .* e^{j 2pi g frac/K + j b g^2} )[(n + s) mod K]
// where delta = S_c(t_m)/dR = s + frac (s integer, |frac| <= 1/2) and b is the
// keystone-variant f_r^2 term.  The integer part of the shift is applied as an
// index offset at store time, so every phase argument handed to FP32 sincos is
// bounded by pi/2 + |b| g^2 and the per-(c,m) scalars are evaluated in FP64.
// Only the ROI rows of the caller's slice are stored, pulse-contiguous
// (X[row][m]), which is the K-major layout the fine stage streams.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"

namespace ltcib {

struct CoarseArgs {
    const float2* cube;      // K x M complex64, column-major (k + K*m)
    const double* cparams;   // [coarse][4]: GRFT c1..cP ; KT (q, c2)
    float2* X;               // [c_count * R_slice][M]          (OUT16 = 0)
    uint32_t* Xh;            // [c_count * R_slice][M] half2 hi  (OUT16 = 1, tcgen05 path)
    uint32_t* Xl;            // [c_count * R_slice][M] half2 lo
    const unsigned* maxbits; // max |y|^2 for the fp16 prescale (OUT16 = 1)
    unsigned long long c_begin;
    int c_count;
    int K, M, P, variant;
    int n_base;              // first range bin stored (roi.first + row_begin)
    int R_slice;
    double inv_prf, inv_dR, two_over_lambda, Va;
    double kt_b;             // -(4 pi / c) * delta_f^2 / fc  (times q Va t)
    int npass;
    int radix[8];
};

__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }

template <int R>
__device__ __forceinline__ void stockham_pass(const float2* __restrict__ in, float2* __restrict__ out,
                                              int N, int Ns, int nfft, int stride, int tid,
                                              int nthr) {
    const int NR = N / R;
    for (int idx = tid; idx < nfft * NR; idx += nthr) {
        const int p = idx / NR;
        const int j = idx - p * NR;
        const float2* a = in + p * stride;
        float2* b = out + p * stride;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = a[padi(j + r * NR)];
        const int k = j & (Ns - 1);
        if (Ns > 1) {
            float s, c;
            __sincosf(6.28318530717958647692f * static_cast<float>(k) / static_cast<float>(Ns * R), &s, &c);
            const float2 w1 = make_float2(c, s);
            float2 w = w1;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                v[r] = cmul(v[r], w);
                w = cmul(w, w1);
            }
        }
        dft_reg<R>(v);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) b[padi(base + r * Ns)] = v[r];
    }
}

// Power-of-two prescale mapping the worst-case |X| <= K max|y| near 2^15
// (fp16 hi/lo operands of the tensor-core fine path).
__device__ __forceinline__ float fp16_prescale(const unsigned* maxbits, int K) {
    const float m2 = __uint_as_float(*maxbits);
    if (!(m2 > 0.f)) return 1.0f;
    const float bound = static_cast<float>(K) * sqrtf(m2);
    const int e = static_cast<int>(floorf(log2f(30000.0f / bound)));
    return ldexpf(1.0f, max(-60, min(60, e)));
}

// grid: (M / PG, c_count); block 256
template <int PG, int OUT16>
__global__ void __launch_bounds__(256) coarse_rm_kernel(CoarseArgs a) {
    extern __shared__ float2 smem[];
    const int K = a.K;
    const int Kp = K + (K >> 4);
    float2* bufA = smem;
    float2* bufB = smem + PG * Kp;
    __shared__ int s_shift[PG];
    __shared__ float s_ra[PG], s_rb[PG];
    __shared__ float2 s_pre[PG];

    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * PG;
    const int c_local = blockIdx.y;
    const unsigned long long c = a.c_begin + c_local;

    if (tid < PG) {
        const int m = m0 + tid;
        const double t = static_cast<double>(m + 1) * a.inv_prf;
        const double* cp = a.cparams + 4 * c;
        double s_rm, s_predfm, b = 0.0;
        if (a.variant == 0) {
            // poly_from(c, t, 1): sum_p c_p t^p (transforms.cpp:12-22)
            double tp = 1.0, acc = 0.0;
            for (int p = 0; p < a.P; ++p) {
                tp *= t;
                acc += cp[p] * tp;
            }
            s_rm = acc;
            s_predfm = acc;
        } else {
            // KtRm phase (transforms.cpp:53-70): f_r (fbar q Va t - c2 t^2)
            const double qva = cp[0] * a.Va;
            s_rm = qva * t - cp[1] * t * t;
            s_predfm = cp[1] * t * t;
            b = a.kt_b * qva * t;
        }
        const double delta = s_rm * a.inv_dR;
        const double sh = floor(delta + 0.5);
        const double frac = delta - sh;
        long long shl = static_cast<long long>(sh) % K;
        if (shl < 0) shl += K;
        s_shift[tid] = static_cast<int>(shl);
        s_ra[tid] = static_cast<float>(6.283185307179586 * frac / K);
        s_rb[tid] = static_cast<float>(b);
        const double cyc = s_predfm * a.two_over_lambda;  // 4pi/lambda * S = 2pi * (2S/lambda)
        const double fr = cyc - rint(cyc);
        double ps, pc;
        sincospi(2.0 * fr, &ps, &pc);
        s_pre[tid] = make_float2(static_cast<float>(pc), static_cast<float>(ps));
    }
    __syncthreads();

    // load + fractional ramp
    for (int idx = tid; idx < PG * K; idx += blockDim.x) {
        const int p = idx / K;
        const int k = idx - p * K;
        const float2 y = a.cube[static_cast<size_t>(m0 + p) * K + k];
        const float g = static_cast<float>(k < K / 2 ? k : k - K);
        float s, co;
        __sincosf(fmaf(s_rb[p] * g, g, s_ra[p] * g), &s, &co);
        bufA[p * Kp + padi(k)] = cmul(y, make_float2(co, s));
    }
    __syncthreads();

    float2* in = bufA;
    float2* out = bufB;
    int Ns = 1;
    for (int ps = 0; ps < a.npass; ++ps) {
        const int R = a.radix[ps];
        switch (R) {
            case 2: stockham_pass<2>(in, out, K, Ns, PG, Kp, tid, blockDim.x); break;
            case 4: stockham_pass<4>(in, out, K, Ns, PG, Kp, tid, blockDim.x); break;
            case 8: stockham_pass<8>(in, out, K, Ns, PG, Kp, tid, blockDim.x); break;
            default: stockham_pass<16>(in, out, K, Ns, PG, Kp, tid, blockDim.x); break;
        }
        __syncthreads();
        Ns *= R;
        float2* tmp = in;
        in = out;
        out = tmp;
    }

    // shifted ROI store, pulse-contiguous rows
    const size_t cbase = static_cast<size_t>(c_local) * a.R_slice * a.M;
    const float sc = OUT16 ? fp16_prescale(a.maxbits, K) : 1.0f;
    for (int idx = tid; idx < a.R_slice * PG; idx += blockDim.x) {
        const int r = idx / PG;
        const int p = idx - r * PG;
        int n = a.n_base + r + s_shift[p];
        n &= K - 1;
        const float2 v = cmul(in[p * Kp + padi(n)], s_pre[p]);
        const size_t o = cbase + static_cast<size_t>(r) * a.M + m0 + p;
        if (OUT16) {
            // x = x_hi + x_lo in fp16 (interleaved re, im along K)
            const float xr = v.x * sc, xi = v.y * sc;
            __half2 hi = __floats2half2_rn(xr, xi);
            const float2 hf = __half22float2(hi);
            __half2 lo = __floats2half2_rn(xr - hf.x, xi - hf.y);
            a.Xh[o] = *reinterpret_cast<uint32_t*>(&hi);
            a.Xl[o] = *reinterpret_cast<uint32_t*>(&lo);
        } else {
            a.X[o] = v;
        }
    }
}

// f64 interleaved host layout -> complex64 device cube
__global__ void f64_to_c64_kernel(const double2* __restrict__ in, float2* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double2 v = in[i];
        out[i] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
    }
}

// K4 keystone (reference proj/src/transforms.cpp:96-130): per frequency row
// resample slow time at x = fc/(f_k+fc) * (m+1) (1-based) with a taps-tap
// Hamming-windowed sinc renormalised to unit sum, clamped tap indices, and an
// exact copy when x is an integer.  Positions are formed in FP64; the sinc
// shares one sinpi over all taps (sin(pi(frac - n)) = (-1)^n sin(pi frac)).
struct KeystoneArgs {
    const float2* in;
    float2* out;
    int K, M, taps;
    double fc, delta_f;
};

__global__ void __launch_bounds__(256) keystone_kernel(KeystoneArgs a) {
    const size_t total = static_cast<size_t>(a.K) * a.M;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int k = static_cast<int>(i % a.K);
        const int m = static_cast<int>(i / a.K);
        const double fk = a.delta_f * static_cast<double>(k < a.K / 2 ? k : k - a.K);
        const double fbar = a.fc / (fk + a.fc);
        const double x = fbar * static_cast<double>(m + 1);
        const long long j0 = llround(x);
        const float2* col = a.in + k;
        if (x == static_cast<double>(j0)) {
            long long src = j0 - 1;
            src = src < 0 ? 0 : (src > a.M - 1 ? a.M - 1 : src);
            a.out[i] = col[static_cast<size_t>(src) * a.K];
            continue;
        }
        const int half = a.taps / 2;
        const double frac = x - static_cast<double>(j0);
        const float fr = static_cast<float>(frac);
        const float sfr = sinpif(fr);  // sin(pi * frac)
        float2 acc = make_float2(0.f, 0.f);
        float wsum = 0.f;
        for (long long j = j0 - half + 1; j <= j0 + half; ++j) {
            const int nshift = static_cast<int>(j0 - j);  // u = frac + nshift
            const float u = fr + static_cast<float>(nshift);
            const float sn = (nshift & 1) ? -sfr : sfr;
            const float sinc = sn / (3.14159265358979323846f * u);
            const float w = sinc * (0.54f + 0.46f * cospif(u / static_cast<float>(half)));
            wsum += w;
            long long src = j - 1;
            src = src < 0 ? 0 : (src > a.M - 1 ? a.M - 1 : src);
            const float2 y = col[static_cast<size_t>(src) * a.K];
            acc.x = fmaf(w, y.x, acc.x);
            acc.y = fmaf(w, y.y, acc.y);
        }
        a.out[i] = make_float2(acc.x / wsum, acc.y / wsum);
    }
}

}  // namespace ltcib
