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
    const float* deap;       // TAB = 1: per-frequency-row real scale (gather.cuh deapodisation)
    int pg;                  // pulses per CTA (0: coarse_pg_for; smaller for plans that would not fill the GPU)
    int npass;
    int radix[8];
};


// One CTA = PG pulses x one coarse cell, PG * K = coarse_samples(OUT16)
// (PG = 4 fp32 / 8 fp16 pulses at K = 2048: an output row segment is one full
// 32-byte sector either way).  The K-point transform is an in-place
// mixed-radix decimation-in-frequency FFT (radices 16, ..., 16, R_last):
// every butterfly reads and writes its own positions, so a pass needs one
// barrier and only R values per thread.
//   pass 1     global loads (all in flight) -> phase ramp -> DFT16 ->
//              twiddle -> shared
//   middle     shared -> DFT16 -> twiddle -> shared (same positions)
//   last       shared -> DFT_R -> global
// The pass-1 ramp carries the whole per-(cell, pulse) phase: the fractional
// delay and keystone terms, the preDFM factor and the integer part s of the
// shift as the exact linear phase (k s mod K) / K cycles (reduced in integers,
// so every FP32 sincos argument stays within 2.5 pi + |b| g^2).  The last pass
// therefore emits absolute bins: the thread of residue kl owns bins
// kl + G t, lanes p = 0..PG-1 of a warp write the same row (PG contiguous
// pulses), and a row's value depends only on its absolute bin (range-cell
// shards reproduce the 1-GPU map bit for bit).
constexpr int kCoarseThreads = 512;      // fp16-output (tcgen05 path) CTAs and fd_grft
constexpr int kCoarseSamples = 16384;
#ifndef LTCI_COARSE_NT32
#define LTCI_COARSE_NT32 256  // fp32-output CTA size
#endif
template <int OUT16>
__host__ __device__ constexpr int coarse_threads() { return OUT16 ? kCoarseThreads : LTCI_COARSE_NT32; }
#ifndef LTCI_COARSE_MINB32
#define LTCI_COARSE_MINB32 3  // fp32-output CTAs per SM (register cap 65536 / (256 x this))
#endif
#ifndef LTCI_COARSE_H32
#define LTCI_COARSE_H32 1  // fp32 output: pass-1 butterflies in flight per thread
#endif
template <int OUT16>
__host__ __device__ constexpr int coarse_min_blocks() { return OUT16 ? 1 : LTCI_COARSE_MINB32; }
__host__ __device__ constexpr int coarse_samples(int out16) { return out16 ? kCoarseSamples : 8192; }

__host__ __device__ constexpr int coarse_pg_for(int K, int M, int out16 = 1) {
    return (coarse_samples(out16) / K) < M ? (coarse_samples(out16) / K) : M;
}
// 8 float2 of padding per 128 (2-way worst case in the middle passes; keeps
// 8-element runs 16-byte aligned), plus 4 float2 per pulse buffer
__host__ __device__ constexpr int cpad(int i) { return i + ((i >> 7) << 3); }
__host__ __device__ constexpr int coarse_kp(int K) { return cpad(K) + 4; }

// Pulse-buffer layouts.  SW = false: the padded layout above.  SW = true
// (K = 2048, fp32 output; 16 radix-16 blocks of 128 per pulse): no padding;
// position i is XOR-swizzled in its low 4 bits by g(i >> 7), g(b) = rotr4(b),
// and pulses are K + 2 apart.  With that every access pattern of the three
// passes is conflict-free for 64-bit accesses: pass-1 stores (lanes j, one
// block), middle reads/writes (lanes j < 8 over block pairs b, b + 1:
// g(b) ^ g(b + 1) = 8), and last-pass reads (lanes = 4 pulses x 4 blocks:
// {r ^ g(b)} is a coset of {0, 1, 8, 9}, the pulse stride moves it by 2p).
template <int K, bool SW>
struct CLayout {
    static constexpr int kp = SW ? K + 2 : coarse_kp(K);
    static __device__ __forceinline__ int idx(int i) {
        if constexpr (SW) {
            const int b = (i >> 7) & 15;
            return i ^ (((b & 1) << 3) | (b >> 1));
        } else {
            return cpad(i);
        }
    }
};
template <int K, int OUT16>
constexpr bool coarse_swizzled() { return K == 2048 && !OUT16; }

// v[r] *= (e^{+j 2 pi num / den})^r, r = 1 .. R-1
template <int R>
__device__ __forceinline__ void twiddle_pow(float2 (&v)[R], int num, int den) {
    float s, c;
    __sincosf(6.28318530717958647692f * static_cast<float>(num) / static_cast<float>(den), &s, &c);
    const float2 w1 = make_float2(c, s);
    float2 w = w1;
#pragma unroll
    for (int r = 1; r < R; ++r) {
        v[r] = cmul(v[r], w);
        w = cmul(w, w1);
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

// compile-time radix plan for K = 16^a * rem: passes 16, ..., 16, last
__host__ __device__ constexpr int coarse_npass(int K) { return K <= 16 ? 1 : 1 + coarse_npass(K / 16); }
__host__ __device__ constexpr int coarse_last_radix(int K) { return K <= 16 ? K : coarse_last_radix(K / 16); }

// bin residue kl (mod K / R_last) -> its position after the DIF passes
// (mixed-radix digit reversal over the radix-16 passes)
template <int K, int NREV>
__device__ __forceinline__ int coarse_digit_rev(int kl) {
    int pos = 0, span = K;
#pragma unroll
    for (int s = 0; s < NREV; ++s) {
        span /= 16;
        pos += (kl & 15) * span;
        kl >>= 4;
    }
    return pos;
}

template <int K, int R, int OUT16, int NT, bool SW>
__device__ __forceinline__ void coarse_last_pass(const CoarseArgs& a, const float2* __restrict__ buf, int PG,
                                                 int lg_pg, float sc, int tid) {
    constexpr int Kp = CLayout<K, SW>::kp;
    constexpr int G = K / R;
    constexpr int NREV = R == 1 ? coarse_npass(K) : coarse_npass(K) - 1;  // R == 1: K = 16, one pass
    const int total = PG * G;
    const size_t cbase = static_cast<size_t>(blockIdx.y) * a.R_slice * a.M;
    const int m0 = blockIdx.x * PG;
    const bool full = a.n_base == 0 && a.R_slice == K;  // ROI = all range cells, one slice
    for (int idx = tid; idx < total; idx += NT) {
        const int p = idx & (PG - 1);  // lanes run over pulses first: one row per PG lanes
        const int kl = idx >> lg_pg;   // this thread's bins: kl + G t
        const int pos0 = coarse_digit_rev<K, NREV>(kl);
        const float2* src = buf + p * Kp;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[CLayout<K, SW>::idx(pos0 + r)];
        dft_reg<R>(v);
        if (!OUT16 && full) {
            // every bin is a stored row (n = bin): rows kl + G t, one pointer
            float2* dst = a.X + cbase + static_cast<size_t>(kl) * a.M + m0 + p;
            const size_t step = static_cast<size_t>(G) * a.M;
#pragma unroll
            for (int t = 0; t < R; ++t) dst[t * step] = v[t];
            continue;
        }
#pragma unroll
        for (int t = 0; t < R; ++t) {
            const int n = (kl + G * t - a.n_base) & (K - 1);  // row of bin kl + G t
            if (n < a.R_slice) {
                const size_t o = cbase + static_cast<size_t>(n) * a.M + m0 + p;
                if (OUT16) {
                    // x = x_hi + x_lo in fp16 (interleaved re, im along K)
                    const float2 x = make_float2(v[t].x * sc, v[t].y * sc);
                    __half2 hi = __floats2half2_rn(x.x, x.y);
                    const float2 hf = __half22float2(hi);
                    __half2 lo = __floats2half2_rn(x.x - hf.x, x.y - hf.y);
                    a.Xh[o] = *reinterpret_cast<uint32_t*>(&hi);
                    a.Xl[o] = *reinterpret_cast<uint32_t*>(&lo);
                } else {
                    a.X[o] = v[t];
                }
            }
        }
    }
}

// middle DIF passes: radix 16 within blocks of length L (K/16 >= L > R_last)
template <int K, int L, int NT = kCoarseThreads, bool SW = false>
__device__ __forceinline__ void coarse_middle_passes(float2* __restrict__ buf, int PG, int tid) {
    if constexpr (L > coarse_last_radix(K)) {
        constexpr int Kp = CLayout<K, SW>::kp;
        constexpr int S = L / 16;
        constexpr int per = K / 16;  // butterflies per pulse
        for (int idx = tid; idx < PG * per; idx += NT) {
            const int p = idx / per;
            const int rem = idx - p * per;
            const int blk = rem / S;
            const int j = rem - blk * S;
            float2* ptr = buf + p * Kp;
            const int base = blk * L + j;
            float2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = ptr[CLayout<K, SW>::idx(base + r * S)];
            dft_reg<16>(v);
            twiddle_pow<16>(v, j, L);
#pragma unroll
            for (int r = 0; r < 16; ++r) ptr[CLayout<K, SW>::idx(base + r * S)] = v[r];
        }
        __syncthreads();
        coarse_middle_passes<K, S, NT, SW>(buf, PG, tid);
    }
}

// grid: (M / PG, c_count); block coarse_threads<OUT16>(); dynamic smem = coarse_smem_bytes
// TAB = 1 builds the oversampled range profiles of gather.cuh with the same
// passes: "cell" blockIdx.y has cparams (delta in range cells, folding number
// q, -, -), no preDFM factor, and every frequency row is scaled by deap[k].
template <int K, int OUT16, int TAB = 0>
__global__ void __launch_bounds__(coarse_threads<OUT16>(), TAB ? 2 : coarse_min_blocks<OUT16>())
    coarse_rm_kernel(CoarseArgs a) {
    constexpr int NT = coarse_threads<OUT16>();
    constexpr bool SW = coarse_swizzled<K, OUT16>();
    extern __shared__ float2 smem[];
    constexpr int Kp = CLayout<K, SW>::kp;
    const int PG = a.pg ? a.pg : coarse_pg_for(K, a.M, OUT16);
    const int lg_pg = __ffs(PG) - 1;
    float2* buf = smem;
    int* s_shift = reinterpret_cast<int*>(smem + PG * Kp);
    float* s_ra = reinterpret_cast<float*>(s_shift + PG);
    float* s_rb = s_ra + PG;
    float* s_pre = s_rb + PG;

    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * PG;
    const unsigned long long c = a.c_begin + blockIdx.y;

    for (int q = tid; q < PG; q += NT) {
        const int m = m0 + q;
        const double t = static_cast<double>(m + 1) * a.inv_prf;
        const double* cp = a.cparams + 4 * c;
        double s_rm, s_predfm, b = 0.0;
        if constexpr (TAB) {
            s_rm = 0.0;
            s_predfm = 0.0;
            b = a.kt_b * cp[1] * a.Va * t;
        } else if (a.variant == 0) {
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
        const double delta = TAB ? cp[0] : s_rm * a.inv_dR;
        const double sh = floor(delta + 0.5);
        const double frac = delta - sh;
        long long shl = static_cast<long long>(sh) % K;
        if (shl < 0) shl += K;
        s_shift[q] = static_cast<int>(shl);
        s_ra[q] = static_cast<float>(6.283185307179586 * frac / K);
        s_rb[q] = static_cast<float>(b);
        const double cyc = s_predfm * a.two_over_lambda;  // 4pi/lambda * S = 2pi * (2S/lambda)
        s_pre[q] = static_cast<float>(6.283185307179586 * (cyc - rint(cyc)));
    }
    __syncthreads();

    // pass 1: radix 16 over span S = K/16, straight from global
    {
        constexpr int S = K / 16;
        const int total = PG * S;
        constexpr int H = OUT16 ? 2 : LTCI_COARSE_H32;  // butterflies in flight per thread (register budget)
#pragma unroll 1
        for (int i0 = tid; i0 < total; i0 += H * NT) {
            float2 v[H][16];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int idx = i0 + h * NT;
                if (idx < total) {
                    const int p = idx / S;
                    const int j = idx - p * S;
                    const float2* col = a.cube + static_cast<size_t>(m0 + p) * K + j;
#pragma unroll
                    for (int r = 0; r < 16; ++r) v[h][r] = __ldg(col + r * S);
                }
            }
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int idx = i0 + h * NT;
                if (idx < total) {
                    const int p = idx / S;
                    const int j = idx - p * S;
                    const float ra = s_ra[p], rb = s_rb[p], pre = s_pre[p];
                    const int sp = s_shift[p];
                    // integer shift in cycles, exact: ((j + r S) s mod K) / K = c0 + r c1 (mod 1)
                    constexpr float kInvK = 1.0f / static_cast<float>(K);
                    const float c0 = static_cast<float>((j * sp) & (K - 1)) * kInvK;
                    const float c1 = static_cast<float>((S * sp) & (K - 1)) * kInvK;
                    const float fj = static_cast<float>(j);
                    if (a.variant == 0) {
                        // GRFT: the phase is linear in r on each half (g jumps by -K at r = 8),
                        // so 3 sincos per 16 points: the two half bases and the common step,
                        // then an 8-long power chain per half (fp32 drift ~1e-6 rel).
                        constexpr float kTwoPi = 6.28318530717958647692f;
                        const float cy8 = fmaf(8.0f, c1, c0);
                        float sn, cs;
                        __sincosf(fmaf(kTwoPi, c0 - rintf(c0), fmaf(ra, fj, pre)), &sn, &cs);
                        float2 w0 = make_float2(cs, sn);
                        __sincosf(fmaf(kTwoPi, cy8 - rintf(cy8), fmaf(ra, fj + static_cast<float>(8 * S - K), pre)),
                                  &sn, &cs);
                        float2 w8 = make_float2(cs, sn);
                        __sincosf(fmaf(kTwoPi, c1 - rintf(c1), ra * static_cast<float>(S)), &sn, &cs);
                        const float2 st = make_float2(cs, sn);
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            v[h][r] = cmul(v[h][r], w0);
                            v[h][r + 8] = cmul(v[h][r + 8], w8);
                            if (r < 7) {
                                w0 = cmul(w0, st);
                                w8 = cmul(w8, st);
                            }
                        }
                        if constexpr (TAB) {
#pragma unroll
                            for (int r = 0; r < 16; ++r) {
                                const float dp = __ldg(a.deap + j + r * S);
                                v[h][r] = mul2(v[h][r], make_float2(dp, dp));
                            }
                        }
                    } else {
#pragma unroll
                        for (int r = 0; r < 16; ++r) {
                            const float gg = fj + static_cast<float>(r < 8 ? r * S : r * S - K);  // g(k), k = j + r S
                            const float cyc = fmaf(static_cast<float>(r), c1, c0);
                            const float ti = cyc - rintf(cyc);
                            float sn, cs;
                            __sincosf(fmaf(6.28318530717958647692f, ti, fmaf(rb * gg, gg, fmaf(ra, gg, pre))), &sn,
                                      &cs);
                            if constexpr (TAB) {
                                const float dp = __ldg(a.deap + j + r * S);
                                cs *= dp;
                                sn *= dp;
                            }
                            v[h][r] = cmul(v[h][r], make_float2(cs, sn));
                        }
                    }
                    dft_reg<16>(v[h]);
                    if constexpr (S > 1) twiddle_pow<16>(v[h], j, K);
                    float2* dst = buf + p * Kp;
#pragma unroll
                    for (int r = 0; r < 16; ++r) dst[CLayout<K, SW>::idx(j + r * S)] = v[h][r];
                }
            }
        }
        __syncthreads();
    }
    coarse_middle_passes<K, K / 16, NT, SW>(buf, PG, tid);

    const float sc = OUT16 ? fp16_prescale(a.maxbits, K) : 1.0f;
    constexpr int RL = K == 16 ? 1 : coarse_last_radix(K);
    coarse_last_pass<K, RL, OUT16, NT, SW>(a, buf, PG, lg_pg, sc, tid);
}

// fp32 output: fewer pulses per CTA (down to 4 = one 32-byte sector per row) until the grid has
// at least 3 CTAs per SM -- small plans (configs[0]: 11 coarse cells x 16 pulse groups = 176 CTAs)
// are latency-bound on one partial wave otherwise
inline int coarse_pg_launch(int K, int M, int out16, long long cells) {
    int pg = coarse_pg_for(K, M, out16);
    if (!out16)
        while (pg > 4 && (M / pg) * cells < 148 * 3) pg /= 2;
    return pg;
}

inline size_t coarse_smem_bytes(int K, int M, int out16 = 1, int pg = 0) {
    const int PG = pg ? pg : coarse_pg_for(K, M, out16);
    const int kp = (K == 2048 && !out16) ? CLayout<2048, true>::kp : coarse_kp(K);
    return static_cast<size_t>(PG) * kp * sizeof(float2) + static_cast<size_t>(PG) * (4 + 4 + 4 + 4);
}

// f64 interleaved host layout -> complex64 device cube
static __global__ void f64_to_c64_kernel(const double2* __restrict__ in, float2* __restrict__ out, size_t n) {
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

static __global__ void __launch_bounds__(256) keystone_kernel(KeystoneArgs a) {
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

// K4 tiled: the same resampling on 32-row x 64-pulse output tiles.  A CTA
// stages the input pulses its tile can touch (the union over its rows of
// [x_first - taps/2, x_last + taps/2], ~84 pulses at the BASELINE radars) as
// 256-byte coalesced row segments in shared memory, all loads in flight at
// once, then every lane (one frequency row) produces 8 outputs reading its
// taps from shared memory (lane-contiguous, conflict-free) and storing
// 256-byte coalesced rows.  Per output one FP64 multiply and round give j0
// and frac; the weights avoid every per-tap transcendental and division:
//   * sinc(frac + n) = (-1)^n sin(pi frac) / (pi (frac + n)); the factor
//     sin(pi frac)/pi / prod_i (frac + i) is common to all taps and cancels in
//     the unit-sum renormalisation, leaving (-1)^n prod_{i != n} (frac + i)
//     (prefix x suffix products);
//   * the Hamming window cos(pi (frac + n)/half) by angle addition from one
//     sincospi(frac / half) and the per-CTA table cos/sin(pi n / half).
// Tiles whose span exceeds the stage (very wide bands: fbar far from 1 across
// the tile) read their taps straight from global memory instead.
constexpr int kKtRows = 32, kKtTile = 64, kKtSpan = 96, kKtThreads = 256;

// one output at pulse m, j0 = lround(fbar (m + 1)) and frac given: the taps
// from shared memory (STAGED) or global memory, clamped to [0, M) when CLAMP.
// cw[i] = (-1)^n (0.54, 0.46 cos, -0.46 sin)(pi n / half) folds the tap sign
// into the Hamming window, evaluated by angle addition from one MUFU sin/cos
// of pi frac / half.
template <int HALF, bool STAGED, bool CLAMP>
__device__ __forceinline__ float2 keystone_point(const KeystoneArgs& a, const float2 (*s_in)[kKtRows],
                                                 const float2* __restrict__ col, const float3 (&cw)[2 * HALF],
                                                 int j0, float fr, int idx_lo, int lane) {
    constexpr int NTAP = 2 * HALF;
    const size_t K = static_cast<size_t>(a.K);
    // tap i reads 0-based pulse j0 - HALF + i (= j - 1, j = j0 - HALF + 1 + i)
    const float2* sp = STAGED && !CLAMP ? &s_in[j0 - HALF - idx_lo][lane] : nullptr;
    auto tap = [&](int i) -> float2 {
        if constexpr (STAGED && !CLAMP) {
            return sp[i * kKtRows];
        } else {
            const int j1 = j0 - HALF + i;
            const int src = CLAMP ? min(max(j1, 0), a.M - 1) : j1;
            return STAGED ? s_in[src - idx_lo][lane] : col[static_cast<size_t>(src) * K];
        }
    };
    if (fr == 0.0f) return tap(HALF - 1);  // exact copy of pulse j0 - 1
    float sa, ca;
    __sincosf(fr * (3.14159265358979323846f / static_cast<float>(HALF)), &sa, &ca);
    // tap i: n = j0 - j = HALF - 1 - i, u = fr + n
    float d[NTAP], pre[NTAP];
    float acc_p = 1.0f;
#pragma unroll
    for (int i = 0; i < NTAP; ++i) {
        d[i] = fr + static_cast<float>(HALF - 1 - i);
        pre[i] = acc_p;
        acc_p *= d[i];
    }
    float suf = 1.0f, wsum = 0.0f;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = NTAP - 1; i >= 0; --i) {
        const float win = fmaf(sa, cw[i].z, fmaf(ca, cw[i].y, cw[i].x));  // (-1)^n (0.54 + 0.46 cos(pi u / half))
        const float w = win * (pre[i] * suf);
        suf *= d[i];
        wsum += w;
        acc = fma2(make_float2(w, w), tap(i), acc);
    }
    const float inv = 1.0f / wsum;
    return make_float2(acc.x * inv, acc.y * inv);
}

// grid: (ceil(K / 32), ceil(M / 64)), kKtThreads threads.  Lane = frequency
// row k, warp w produces pulses m_a + w + 8 i.  Positions: x = fbar (m + 1) =
// (m + 1) + e, e = (fbar - 1)(m + 1); per thread e is split once in FP64 at
// its first pulse into an integer and a fraction, and advanced in FP32 by
// 8 (fbar - 1) per output (|8 i (fbar - 1)| < 0.3 over a tile at the BASELINE
// radars: ~1e-8 absolute error in frac, where x itself in FP32 would carry 6e-5).
template <int HALF>
__global__ void __launch_bounds__(kKtThreads) keystone_tiled_kernel(KeystoneArgs a) {
    constexpr int NTAP = 2 * HALF, NW = kKtThreads / 32;
    __shared__ float2 s_in[kKtSpan][kKtRows];
    __shared__ float3 s_cw[NTAP];
    __shared__ int s_lo, s_n, s_clamp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = blockIdx.x * kKtRows + lane;
    const bool live = k < a.K;
    const int m_a = blockIdx.y * kKtTile, m_b = min(a.M, m_a + kKtTile);
    const double fk = a.delta_f * static_cast<double>(k < a.K / 2 ? k : k - a.K);
    const double fbar = a.fc / (fk + a.fc);
    const double dlt = fbar - 1.0;  // exact (Sterbenz)
    if (threadIdx.x < NTAP) {
        const int n = HALF - 1 - static_cast<int>(threadIdx.x);
        float sn, cs;
        sincospif(static_cast<float>(n) / static_cast<float>(HALF), &sn, &cs);
        const float sg = (n & 1) ? -1.0f : 1.0f;
        s_cw[threadIdx.x] = make_float3(0.54f * sg, 0.46f * sg * cs, -0.46f * sg * sn);
    }
    if (warp == 0) {
        // the tile's input pulses: union over its rows of the tap windows (one
        // pulse of margin on each side for the FP32 position advance)
        int lo = 0x7fffffff, hi = -0x7fffffff;
        if (live) {
            lo = static_cast<int>(llround(fbar * static_cast<double>(m_a + 1))) - HALF - 1;
            hi = static_cast<int>(llround(fbar * static_cast<double>(m_b))) + HALF;
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0) {
            s_clamp = lo < 0 || hi > a.M - 1;
            lo = min(max(lo, 0), a.M - 1);
            hi = min(max(hi, 0), a.M - 1);
            s_lo = lo;
            s_n = hi - lo + 1;
        }
    }
    __syncthreads();
    const int idx_lo = s_lo, n = s_n;
    const bool clamp = s_clamp;
    const float2* __restrict__ col = a.in + (live ? k : 0);
    const size_t K = static_cast<size_t>(a.K);
    float3 cw[NTAP];
#pragma unroll
    for (int i = 0; i < NTAP; ++i) cw[i] = s_cw[i];
    const bool staged = n <= kKtSpan;
    if (staged) {
        for (int i = warp; i < n; i += NW)
            s_in[i][lane] = live ? col[static_cast<size_t>(idx_lo + i) * K] : make_float2(0.f, 0.f);
        __syncthreads();
    }
    if (!live) return;
    const int m_first = m_a + warp;
    const double e0 = dlt * static_cast<double>(m_first + 1);
    const double ea = floor(e0);
    const int jbase = m_first + 1 + static_cast<int>(ea);
    const float e0f = static_cast<float>(e0 - ea);
    const float step = static_cast<float>(dlt * NW);
    for (int it = 0, m = m_first; m < m_b; ++it, m += NW) {
        const float ef = fmaf(step, static_cast<float>(it), e0f);
        const float n1 = floorf(ef + 0.5f);
        const int j0 = jbase + NW * it + static_cast<int>(n1);
        const float fr = ef - n1;
        float2 r;
        if (staged && !clamp)
            r = keystone_point<HALF, true, false>(a, s_in, col, cw, j0, fr, idx_lo, lane);
        else if (staged)
            r = keystone_point<HALF, true, true>(a, s_in, col, cw, j0, fr, idx_lo, lane);
        else
            r = keystone_point<HALF, false, true>(a, s_in, col, cw, j0, fr, 0, lane);
        a.out[k + K * static_cast<size_t>(m)] = r;
    }
}

}  // namespace ltcib
