// fd_grft.cuh -- single-scale frequency-domain GRFT.
//
// Reference: ltci::fd_grft (proj/src/detectors.cpp:105-197).  Per motion cell
// c with S_c(t) = sum_p c_p t^p, the matched filter over the wrapped
// frequency rows r (g = r or r - K) and pulses m
//     acc_c[r] = sum_m y[r, m] exp(j (4 pi / lambda + 4 pi delta_f g / c) S_c(t_m))
// followed by the K-point dft_plus over r; the ROI bins are the map rows.
// The reference advances a per-pulse rotor along r; here every (r, m) term
// is evaluated independently from two per-(cell, pulse) phase scalars held as
// 32-bit fixed-point fractions of a cycle,
//     phase_u32 = A_m + B_m * g  (mod 2^32),  A_m = frac(2 S / lambda),
//                                              B_m = frac(2 delta_f S / c),
// formed in FP64 once per (cell, pulse): the integer multiply wraps exactly
// mod one cycle, so the angle handed to the SFU is always in [-pi, pi) and
// the phase error is <= 2^-32 (1 + |g|) cycles.
//
//   K5 fd_mf_kernel       CG cells per CTA share every cube load; threads over
//                         rows (one SFU sincos per thread, rows chained by exact
//                         per-pulse rotors), loop over pulses; acc written [cell][K]
//   K6 fd_fft_scan_kernel in-place mixed-radix DIF transform of PG = 16384/K
//                         cells per CTA (the coarse-stage passes), then the
//                         ROI scan: |v| > retain candidates, dense store,
//                         per-CTA argmax -> one 128-bit CAS publish
#pragma once

#include "coarse.cuh"
#include "fine_fft.cuh"

namespace ltcib {

struct FdArgs {
    const float2* cube;           // K x M complex64, column-major (k + K*m)
    float2* acc;                  // [cells in batch][K]
    unsigned long long c_begin;   // first motion cell of the batch
    unsigned long long c_count;   // cells in the batch
    int K, M, P;
    int count[4];                 // grid counts, order p at [p-1] (c_1 fastest in the cell index)
    double start[4], step[4];
    double inv_prf, two_over_lambda, two_df_over_c;
    // td_grft (td_grft.cuh): metres -> range bins, TrajectoryPolicy (0 zero outside, 1 wrap, 2 error)
    // and the flag the error policy raises
    double bin_scale;
    int policy;
    int* err;
    // scan
    int roi_first, R;
    float retain2;                // retain^2 (-1: retain everything)
    CandRec* cand;
    unsigned long long* cand_count;
    unsigned long long cand_cap;
    float2* dense;                // optional, [cells][R] by flat index
    PeakSlot* best;               // global argmax slot
};

constexpr int kFdCells = 4;  // max cells per MF CTA (batch granularity)

// MF CTA shape per K: rows per thread RPT = K / threads, cells x RPT <= 32
// accumulators per thread (64 registers) -- more rows per thread means fewer
// SFU sincos per term (one per thread, cell and pulse)
__host__ __device__ constexpr int fd_threads(int K) { return K / 4 < 32 ? 32 : (K / 4 > 256 ? 256 : K / 4); }
__host__ __device__ constexpr int fd_rpt(int K) { return K >= fd_threads(K) ? K / fd_threads(K) : 1; }
__host__ __device__ constexpr int fd_cells(int K) { return fd_rpt(K) <= 8 ? 4 : (fd_rpt(K) <= 16 ? 2 : 1); }

__device__ __forceinline__ unsigned fd_frac_u32(double cycles) {
    const double f = cycles - floor(cycles);  // [0, 1)
    return static_cast<unsigned>(static_cast<unsigned long long>(f * 4294967296.0) & 0xffffffffull);
}

constexpr int kFdTile = 256;  // pulses per staged tile of per-(cell, pulse) scalars

// grid: ceil(c_count / fd_cells(K)); block fd_threads(K); static smem (scalars of one pulse tile)
//
// Thread t owns rows r_q = t + T q (T threads).  Their wrapped indices differ
// by the thread-independent offsets  D_q = T q  (q < K/2T)  or  T q - K, so
//   e^{j phi(r_q)} = e^{j phi(r_0)} rho^q  (times omega once past K/2),
// rho = e^{j 2 pi T B_m}, omega = e^{-j 2 pi K B_m}: one SFU sincos per
// (thread, cell, pulse) instead of one per row.
template <int K>
__global__ void __launch_bounds__(fd_threads(K)) fd_mf_kernel(FdArgs a) {
    constexpr int kFdThreads = fd_threads(K);
    constexpr int RPT = fd_rpt(K);
    constexpr int CPB = fd_cells(K);
    constexpr int QH = K >= 2 * kFdThreads ? K / (2 * kFdThreads) : RPT;  // first row index past K/2
    __shared__ unsigned sA[CPB][kFdTile], sB[CPB][kFdTile];
    __shared__ float2 sRho[CPB][kFdTile], sRhoW[CPB][kFdTile];
    const int M = a.M;
    const unsigned long long cell0 = static_cast<unsigned long long>(blockIdx.x) * CPB;
    const int ncell = static_cast<int>(min(static_cast<unsigned long long>(CPB), a.c_count - cell0));

    float2 acc[CPB][RPT];
#pragma unroll
    for (int c = 0; c < CPB; ++c)
#pragma unroll
        for (int q = 0; q < RPT; ++q) acc[c][q] = make_float2(0.f, 0.f);
    const int r0 = threadIdx.x;
    const unsigned g0 = static_cast<unsigned>(r0 < K / 2 ? r0 : r0 - K);
    const bool live = K >= kFdThreads || threadIdx.x < K;

    for (int m0 = 0; m0 < M; m0 += kFdTile) {
        const int tm = min(kFdTile, M - m0);
        __syncthreads();  // previous tile consumed
        for (int i = threadIdx.x; i < CPB * kFdTile; i += kFdThreads) {
            const int g = i / kFdTile, mm = i - g * kFdTile;
            unsigned A = 0, B = 0;
            if (g < ncell && mm < tm) {
                // decode_motion (detectors.cpp:84-92): c_1 fastest
                unsigned long long rem = a.c_begin + cell0 + g;
                const double t = static_cast<double>(m0 + mm + 1) * a.inv_prf;
                double S = 0.0, tp = 1.0;
                for (int p = 0; p < a.P; ++p) {
                    const int ip = static_cast<int>(rem % static_cast<unsigned long long>(a.count[p]));
                    rem /= static_cast<unsigned long long>(a.count[p]);
                    tp *= t;
                    S += (a.start[p] + a.step[p] * static_cast<double>(ip)) * tp;
                }
                A = fd_frac_u32(S * a.two_over_lambda);
                B = fd_frac_u32(S * a.two_df_over_c);
            }
            sA[g][mm] = A;
            sB[g][mm] = B;
            // exact mod-one-cycle products, then an accurate FP32 sincospi
            float rs, rc, ws, wc;
            sincospif(static_cast<float>(static_cast<int>(B * static_cast<unsigned>(kFdThreads))) * 4.656612873077393e-10f, &rs, &rc);  // 2^-31
            sincospif(-static_cast<float>(static_cast<int>(B * static_cast<unsigned>(K))) * 4.656612873077393e-10f,
                      &ws, &wc);
            sRho[g][mm] = make_float2(rc, rs);
            sRhoW[g][mm] = make_float2(rc * wc - rs * ws, rc * ws + rs * wc);
        }
        __syncthreads();
        if (live) {
#pragma unroll 2
            for (int mm = 0; mm < tm; ++mm) {
                const int m = m0 + mm;
                float2 y[RPT];
#pragma unroll
                for (int q = 0; q < RPT; ++q) y[q] = __ldg(a.cube + static_cast<size_t>(m) * K + r0 + q * kFdThreads);
#pragma unroll
                for (int c = 0; c < CPB; ++c) {
                    const int ph = static_cast<int>(sA[c][mm] + sB[c][mm] * g0);  // signed cycles * 2^32
                    float s, co;
                    __sincosf(static_cast<float>(ph) * 1.46291807926715968e-09f, &s, &co);  // 2 pi / 2^32
                    float2 z = make_float2(co, s);
                    const float2 rho = sRho[c][mm];
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        if (q > 0) z = cmul(z, q == QH ? sRhoW[c][mm] : rho);
                        acc[c][q].x = fmaf(y[q].x, z.x, fmaf(-y[q].y, z.y, acc[c][q].x));
                        acc[c][q].y = fmaf(y[q].x, z.y, fmaf(y[q].y, z.x, acc[c][q].y));
                    }
                }
            }
        }
    }
    if (live) {
#pragma unroll
        for (int c = 0; c < CPB; ++c) {
            if (c < ncell) {
#pragma unroll
                for (int q = 0; q < RPT; ++q)
                    a.acc[(cell0 + c) * K + r0 + q * kFdThreads] = acc[c][q];
            }
        }
    }
}

// last DIF pass kept in shared memory (radix R, span 1, no twiddle)
template <int K, int R>
__device__ __forceinline__ void fd_last_pass_inplace(float2* __restrict__ buf, int PG, int tid) {
    constexpr int Kp = coarse_kp(K);
    constexpr int G = K / R;
    for (int idx = tid; idx < PG * G; idx += kCoarseThreads) {
        const int p = idx / G;
        const int b = idx - p * G;
        float2* ptr = buf + p * Kp;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = ptr[cpad(b * R + r)];
        dft_reg<R>(v);
#pragma unroll
        for (int r = 0; r < R; ++r) ptr[cpad(b * R + r)] = v[r];
    }
    __syncthreads();
}

// grid: ceil(c_count / PG), PG = coarse_pg_for(K, huge); block kCoarseThreads;
// dynamic smem PG * coarse_kp(K) float2
template <int K>
__global__ void __launch_bounds__(kCoarseThreads, 1) fd_fft_scan_kernel(FdArgs a) {
    extern __shared__ float2 smem[];
    constexpr int Kp = coarse_kp(K);
    constexpr int PG = kCoarseSamples / K;
    constexpr int NP = coarse_npass(K);
    constexpr int RL = coarse_last_radix(K);
    float2* buf = smem;
    const int tid = threadIdx.x;
    const unsigned long long cell0 = static_cast<unsigned long long>(blockIdx.x) * PG;
    const int ncell = static_cast<int>(min(static_cast<unsigned long long>(PG), a.c_count - cell0));

    // pass 1 (radix 16, span K/16) straight from the MF output
    {
        constexpr int S = K / 16;
        for (int idx = tid; idx < PG * S; idx += kCoarseThreads) {
            const int p = idx / S;
            const int j = idx - p * S;
            float2 v[16];
            if (p < ncell) {
                const float2* col = a.acc + (cell0 + p) * K + j;
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = col[r * S];
            } else {
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = make_float2(0.f, 0.f);
            }
            dft_reg<16>(v);
            if constexpr (S > 1) twiddle_pow<16>(v, j, K);
            float2* dst = buf + p * Kp;
#pragma unroll
            for (int r = 0; r < 16; ++r) dst[cpad(j + r * S)] = v[r];
        }
        __syncthreads();
    }
    if constexpr (NP > 1) {
        coarse_middle_passes<K, K / 16>(buf, PG, tid);
        fd_last_pass_inplace<K, RL>(buf, PG, tid);
    }

    // ROI scan: bin k sits at its digit-reversed position
    constexpr int G = NP > 1 ? K / RL : 1;
    float bm = -1.0f;
    unsigned long long bidx = ~0ull;
    float2 bv = make_float2(0.f, 0.f);
    for (int idx = tid; idx < ncell * a.R; idx += kCoarseThreads) {
        const int p = idx / a.R;
        const int r = idx - p * a.R;
        const int k = a.roi_first + r;
        const int pos = NP > 1 ? coarse_digit_rev<K, NP - 1>(k & (G - 1)) + k / G : k;
        const float2 v = buf[p * Kp + cpad(pos)];
        const float m2 = mag2f(v.x, v.y);
        const unsigned long long flat = (a.c_begin + cell0 + p) * static_cast<unsigned long long>(a.R) + r;
        if (a.dense) a.dense[flat] = v;
        if (m2 > a.retain2) {
            const unsigned long long at = atomicAdd(a.cand_count, 1ull);
            if (at < a.cand_cap) {
                CandRec rec;
                rec.idx = flat;
                rec.re = v.x;
                rec.im = v.y;
                a.cand[at] = rec;
            }
        }
        if (m2 > bm || (m2 == bm && flat < bidx)) {
            bm = m2;
            bidx = flat;
            bv = v;
        }
    }
    // CTA argmax (ties to the lowest flat index), one publish per CTA
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, bm, off);
        const unsigned long long oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        const float ore = __shfl_xor_sync(0xffffffffu, bv.x, off);
        const float oim = __shfl_xor_sync(0xffffffffu, bv.y, off);
        if (om > bm || (om == bm && oi < bidx)) {
            bm = om;
            bidx = oi;
            bv = make_float2(ore, oim);
        }
    }
    __shared__ float s_m[kCoarseThreads / 32];
    __shared__ unsigned long long s_i[kCoarseThreads / 32];
    __shared__ float2 s_v[kCoarseThreads / 32];
    if ((tid & 31) == 0) {
        s_m[tid >> 5] = bm;
        s_i[tid >> 5] = bidx;
        s_v[tid >> 5] = bv;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kCoarseThreads / 32; ++w)
            if (s_m[w] > bm || (s_m[w] == bm && s_i[w] < bidx)) {
                bm = s_m[w];
                bidx = s_i[w];
                bv = s_v[w];
            }
        if (bidx != ~0ull) peak_publish(a.best, bv.x, bv.y, bidx);
    }
}

// K < 16 (the reference accepts any power of two): one cell per thread, the
// K-point dft_plus in registers, then the same ROI scan and argmax publish.
template <int K>
__global__ void __launch_bounds__(256) fd_small_scan_kernel(FdArgs a) {
    static_assert(K >= 2 && K < 16, "small-K transform");
    const unsigned long long cell = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    float bm = -1.0f;
    unsigned long long bidx = ~0ull;
    float2 bv = make_float2(0.f, 0.f);
    if (cell < a.c_count) {
        float2 v[K];
#pragma unroll
        for (int r = 0; r < K; ++r) v[r] = a.acc[cell * K + r];
        dft_reg<K>(v);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = k - a.roi_first;
            if (r < 0 || r >= a.R) continue;
            const float m2 = mag2f(v[k].x, v[k].y);
            const unsigned long long flat = (a.c_begin + cell) * static_cast<unsigned long long>(a.R) + r;
            if (a.dense) a.dense[flat] = v[k];
            if (m2 > a.retain2) {
                const unsigned long long at = atomicAdd(a.cand_count, 1ull);
                if (at < a.cand_cap) {
                    CandRec rec;
                    rec.idx = flat;
                    rec.re = v[k].x;
                    rec.im = v[k].y;
                    a.cand[at] = rec;
                }
            }
            if (m2 > bm || (m2 == bm && flat < bidx)) {
                bm = m2;
                bidx = flat;
                bv = v[k];
            }
        }
    }
    // warp argmax, one publish per warp
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, bm, off);
        const unsigned long long oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        const float ore = __shfl_xor_sync(0xffffffffu, bv.x, off);
        const float oim = __shfl_xor_sync(0xffffffffu, bv.y, off);
        if (om > bm || (om == bm && oi < bidx)) {
            bm = om;
            bidx = oi;
            bv = make_float2(ore, oim);
        }
    }
    if ((threadIdx.x & 31) == 0 && bidx != ~0ull) peak_publish(a.best, bv.x, bv.y, bidx);
}

}  // namespace ltcib
