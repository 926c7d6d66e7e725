// td_grft.cuh -- single-scale time-domain GRFT: the literal trajectory gather.
//
// Reference: ltci::td_grft (proj/src/detectors.cpp:199-264).  Per motion cell c
// with S_c(t) = sum_p c_p t^p and ROI row r (range bin n0 = roi.first + r)
//     acc_c[r] = sum_m s[n(m), m] exp(j 4 pi S_c(t_m) / lambda),
//     n(m) = lround(n0 + (2 fs / c) S_c(t_m))
// over the RANGE-pulse cube s (nearest-bin gather: no interpolation, the
// paper's TD-GRFT baseline).  Samples whose bin rounds outside [0, K) follow
// the reference's TrajectoryPolicy: contribute zero, wrap modulo K, or raise.
//
// K7 td_gather_scan_kernel: one CTA = one motion cell x 256 ROI rows.  The
// per-(cell, pulse) scalars -- the FP64 bin offset and the Doppler phase
// (FP64 sincos of the cycle fraction) -- are staged per 256-pulse tile in
// shared memory; a thread owns one row and walks the pulses: the bin is
// llround(n0 + offset) in FP64 exactly as the reference forms it (ties and
// all), the loads of a warp are 32 consecutive bins of one pulse column
// (coalesced; the 16.8 MB cube lives in L2), the sum runs in packed FP32.
// Measured on the C0 radar's full single-scale grid (82 971 cells x 512 rows x
// 256 pulses): 12.8 ms = 852 G trajectory samples/s, 6.8 TB/s of 8-byte
// gathers; the reference's td_grft on 16 host threads: 3.3 G/s
// (profiles/r02_side_td.json).  Two variants measured and dropped: an
// integer-only bin computation in place of the FP64 llround (13.5 ms), and 8
// neighbouring velocity cells per CTA sharing their loads through L1 (20.4 ms).
// The ROI scan (threshold candidates, dense store, argmax with the lowest
// flat index on ties, one 128-bit CAS publish per CTA) is fused.
#pragma once

#include "fd_grft.cuh"

namespace ltcib {

constexpr int kTdThreads = 256;
constexpr int kTdTile = 256;

// grid: (cells in batch, ceil(R / kTdThreads)); block kTdThreads
__global__ void __launch_bounds__(kTdThreads) td_gather_scan_kernel(FdArgs a) {
    __shared__ double s_off[kTdTile];
    __shared__ float2 s_ph[kTdTile];
    const int tid = threadIdx.x;
    const unsigned long long cell = a.c_begin + blockIdx.x;
    const int r = blockIdx.y * kTdThreads + tid;
    const bool live = r < a.R;
    const double n0 = static_cast<double>(a.roi_first + r);
    const long long K = a.K;
    float2 acc = make_float2(0.f, 0.f);
    bool left = false;

    // decode_motion (detectors.cpp:84-92): c_1 fastest
    double cv[4] = {0.0, 0.0, 0.0, 0.0};
    {
        unsigned long long rem = cell;
        for (int p = 0; p < a.P; ++p) {
            const int ip = static_cast<int>(rem % static_cast<unsigned long long>(a.count[p]));
            rem /= static_cast<unsigned long long>(a.count[p]);
            cv[p] = a.start[p] + a.step[p] * static_cast<double>(ip);
        }
    }
    for (int m0 = 0; m0 < a.M; m0 += kTdTile) {
        const int tm = min(kTdTile, a.M - m0);
        __syncthreads();  // previous tile consumed
        for (int mm = tid; mm < tm; mm += kTdThreads) {
            const double t = static_cast<double>(m0 + mm + 1) * a.inv_prf;
            double S = 0.0, tp = 1.0;
            for (int p = 0; p < a.P; ++p) {
                tp *= t;
                S += cv[p] * tp;
            }
            s_off[mm] = a.bin_scale * S;
            const double cyc = S * a.two_over_lambda;  // 4 pi S / lambda = 2 pi (2 S / lambda)
            double sn, cs;
            sincospi(2.0 * (cyc - rint(cyc)), &sn, &cs);
            s_ph[mm] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
        }
        __syncthreads();
        if (live) {
            const float2* col = a.cube + static_cast<size_t>(m0) * K;
#pragma unroll 4
            for (int mm = 0; mm < tm; ++mm) {
                long long n = llround(n0 + s_off[mm]);
                if (n < 0 || n >= K) {
                    if (a.policy == 1) {
                        n = ((n % K) + K) % K;
                    } else {
                        left = left || a.policy == 2;
                        continue;
                    }
                }
                const float2 v = __ldg(col + static_cast<size_t>(mm) * K + n);
                const float2 w = s_ph[mm];
                acc = fma2(make_float2(-v.y, v.x), make_float2(w.y, w.y), fma2(v, make_float2(w.x, w.x), acc));
            }
        }
    }
    if (left) *a.err = 1;

    float bm = -1.0f;
    unsigned long long bidx = ~0ull;
    float2 bv = make_float2(0.f, 0.f);
    if (live) {
        const float m2 = mag2f(acc.x, acc.y);
        const unsigned long long flat = cell * static_cast<unsigned long long>(a.R) + r;
        if (a.dense) a.dense[flat] = acc;
        if (m2 > a.retain2) {
            const unsigned long long at = atomicAdd(a.cand_count, 1ull);
            if (at < a.cand_cap) {
                CandRec rec;
                rec.idx = flat;
                rec.re = acc.x;
                rec.im = acc.y;
                a.cand[at] = rec;
            }
        }
        bm = m2;
        bidx = flat;
        bv = acc;
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
    __shared__ float s_m[kTdThreads / 32];
    __shared__ unsigned long long s_i[kTdThreads / 32];
    __shared__ float2 s_v[kTdThreads / 32];
    if ((tid & 31) == 0) {
        s_m[tid >> 5] = bm;
        s_i[tid >> 5] = bidx;
        s_v[tid >> 5] = bv;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kTdThreads / 32; ++w)
            if (s_m[w] > bm || (s_m[w] == bm && s_i[w] < bidx)) {
                bm = s_m[w];
                bidx = s_i[w];
                bv = s_v[w];
            }
        if (bidx != ~0ull) peak_publish(a.best, bv.x, bv.y, bidx);
    }
}

}  // namespace ltcib
