// coarse2k.cuh -- K1 specialised for K = 2048 with complex64 output (C1, C3).
//
// Same transform as coarse_rm_kernel (mgift = gift + compensated_ifft +
// build_mf(RM|KtRm, PreDfm), reference proj/src/transforms.cpp:32-94,134-173;
// see coarse.cuh for the fractional-delay formulation): per (coarse cell,
// pulse) the ramped echo column goes through a 2048-point DIF transform
// 16 x 16 x 8, the same passes writing the same positions.  What changes is
// how the work maps onto the SM (the generic kernel issued ~50 instructions
// per point at 46 % issue efficiency, latency-bound between its barriers):
//
//  * every thread owns two ADJACENT butterflies (j, j+1) in the radix-16
//    passes, so each echo load is one 16-byte LDG and every shared-memory
//    access is a 16-byte LDS/STS (half the LSU instructions, no swizzle
//    arithmetic); the padded layout (8 float2 per 128, pulse stride 2178 =
//    2 mod 16 float2) keeps all three passes' 16-byte phases conflict-free;
//  * the GRFT ramp is factored: for k = j + 128 r the phase is a_j + b_r, so
//    a per-pulse table B_r = e^{2 pi i b_r} (16 entries, FP64-reduced) is
//    applied before the radix-16 DFT and A_j = e^{2 pi i a_j} -- constant over
//    r, so it commutes with the DFT -- starts the inter-pass twiddle chain
//    for free (2 + ~0 instead of ~5.5 instructions per point);
//  * the second pass reads its twiddles w_128^{j r} from a 1 KB table.
//
// CTA: 256 threads = 4 pulses x 64 butterfly pairs; 3 CTAs per SM.
#pragma once

#include "coarse.cuh"

namespace ltcib {

#ifndef LTCI_C2K_MINB
#define LTCI_C2K_MINB 3  // CTAs per SM (register cap 65536 / (256 x this)); A/B: -DLTCI_C2K_MINB=2
#endif
constexpr int k2kThreads = 256;
constexpr int k2kPG = 4;      // pulses per CTA (one 32-byte output sector per row)
constexpr int k2kKp = 2178;   // pulse stride in float2: cpad(2048) + 2, = 2 (mod 16)

__host__ __device__ constexpr size_t coarse2k_smem_bytes() {
    return static_cast<size_t>(k2kPG) * k2kKp * 8 + k2kPG * 16 * 8 + 16 * 8 * 8 + k2kPG * 16;
}

__device__ __forceinline__ float4 pack2(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }

// grid: (M / 4, c_count); block k2kThreads; dynamic smem = coarse2k_smem_bytes()
__global__ void __launch_bounds__(k2kThreads, LTCI_C2K_MINB) coarse2k_kernel(CoarseArgs a) {
    constexpr int K = 2048, S = 128;
    extern __shared__ float4 smem4[];
    float2* buf = reinterpret_cast<float2*>(smem4);
    float2* sB = buf + k2kPG * k2kKp;          // [4][16] GRFT ramp table B_r per pulse
    float2* sT = sB + k2kPG * 16;              // [16][8] w_128^{j2 r}
    int* s_shift = reinterpret_cast<int*>(sT + 16 * 8);
    float* s_fr = reinterpret_cast<float*>(s_shift + k2kPG);  // GRFT: frac / K ; KT: 2 pi frac / K
    float* s_rb = s_fr + k2kPG;
    float* s_pre = s_rb + k2kPG;                // GRFT: preDFM cycles ; KT: radians

    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * k2kPG;
    const unsigned long long c = a.c_begin + blockIdx.y;
    const bool grft = a.variant == 0;

    // ---- prologue: per-pulse FP64 scalars (same expressions as coarse_rm_kernel)
    if (tid < 64) {
        const int q = tid >> 4, r = tid & 15;
        const int m = m0 + q;
        const double t = static_cast<double>(m + 1) * a.inv_prf;
        const double* cp = a.cparams + 4 * c;
        double s_rm, s_predfm, b = 0.0;
        if (grft) {
            double tp = 1.0, acc = 0.0;  // poly_from(c, t, 1), transforms.cpp:12-22
            for (int pp = 0; pp < a.P; ++pp) {
                tp *= t;
                acc += cp[pp] * tp;
            }
            s_rm = acc;
            s_predfm = acc;
        } else {
            const double qva = cp[0] * a.Va;  // KtRm (transforms.cpp:53-70)
            s_rm = qva * t - cp[1] * t * t;
            s_predfm = cp[1] * t * t;
            b = a.kt_b * qva * t;
        }
        const double delta = s_rm * a.inv_dR;
        const double sh = floor(delta + 0.5);
        const double frac = delta - sh;
        long long shl = static_cast<long long>(sh) % K;
        if (shl < 0) shl += K;
        const double cyc = s_predfm * a.two_over_lambda;
        if (grft) {
            // b_r = r (128 s mod K) / K + frac 128 r / K - [r >= 8] frac   (cycles)
            double br = static_cast<double>(r) * static_cast<double>((S * shl) & (K - 1)) / K +
                        frac * static_cast<double>(S * r) / K - (r >= 8 ? frac : 0.0);
            br -= rint(br);
            double sn, cs;
            sincospi(2.0 * br, &sn, &cs);
            sB[q * 16 + r] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
        }
        if (r == 0) {
            s_shift[q] = static_cast<int>(shl);
            s_fr[q] = grft ? static_cast<float>(frac / K) : static_cast<float>(6.283185307179586 * frac / K);
            s_rb[q] = static_cast<float>(b);
            s_pre[q] = grft ? static_cast<float>(cyc - rint(cyc))
                            : static_cast<float>(6.283185307179586 * (cyc - rint(cyc)));
        }
    } else if (tid < 64 + 128) {
        const int e = tid - 64, r = e >> 3, jj = e & 7;
        float sn, cs;
        sincospif(static_cast<float>(jj * r) / 64.0f, &sn, &cs);  // w_128^{jj r}
        sT[r * 8 + jj] = make_float2(cs, sn);
    }
    __syncthreads();

    const int p = tid >> 6, t = tid & 63;
    // ---- pass 1: radix 16 over span 128, from global, butterflies j, j + 1
    {
        const int j = 2 * t;
        const float4* src = reinterpret_cast<const float4*>(a.cube + static_cast<size_t>(m0 + p) * K + j);
        float2 v0[16], v1[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float4 q = __ldg(src + r * (S / 2));
            v0[r] = make_float2(q.x, q.y);
            v1[r] = make_float2(q.z, q.w);
        }
        const int sp = s_shift[p];
        constexpr float kInvK = 1.0f / static_cast<float>(K);
        float2 T0, T1;  // twiddle chain seeds
        if (grft) {
            const float2* B = sB + p * 16;
#pragma unroll
            for (int r = 1; r < 16; ++r) {
                const float2 br = B[r];
                v0[r] = cmul(v0[r], br);
                v1[r] = cmul(v1[r], br);
            }
            // A_j = e^{2 pi i a_j}, a_j = (j s mod K)/K + frac j / K + preDFM
            const float fr = s_fr[p], pre = s_pre[p];
            float a0 = fmaf(fr, static_cast<float>(j), static_cast<float>((j * sp) & (K - 1)) * kInvK + pre);
            float a1 = fmaf(fr, static_cast<float>(j + 1), static_cast<float>(((j + 1) * sp) & (K - 1)) * kInvK + pre);
            a0 -= rintf(a0);
            a1 -= rintf(a1);
            float sn, cs;
            sincospif(2.0f * a0, &sn, &cs);
            T0 = make_float2(cs, sn);
            sincospif(2.0f * a1, &sn, &cs);
            T1 = make_float2(cs, sn);
        } else {
            // KT: phase 2 pi (k s mod K)/K + ra g + rb g^2 + pre per point (as coarse_rm_kernel)
            const float ra = s_fr[p], rb = s_rb[p], pre = s_pre[p];
            const float c1 = static_cast<float>((S * sp) & (K - 1)) * kInvK;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int jh = j + h;
                const float c0 = static_cast<float>((jh * sp) & (K - 1)) * kInvK;
                const float fj = static_cast<float>(jh);
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const float gg = fj + static_cast<float>(r < 8 ? r * S : r * S - K);
                    const float cyc = fmaf(static_cast<float>(r), c1, c0);
                    const float ti = cyc - rintf(cyc);
                    float sn, cs;
                    __sincosf(fmaf(6.28318530717958647692f, ti, fmaf(rb * gg, gg, fmaf(ra, gg, pre))), &sn, &cs);
                    if (h == 0)
                        v0[r] = cmul(v0[r], make_float2(cs, sn));
                    else
                        v1[r] = cmul(v1[r], make_float2(cs, sn));
                }
            }
            T0 = T1 = make_float2(1.f, 0.f);
        }
        dft_reg<16>(v0);
        dft_reg<16>(v1);
        // v[r] *= T_j w_K^{j r}
        float sn, cs;
        sincospif(static_cast<float>(j) / 1024.0f, &sn, &cs);
        const float2 w0 = make_float2(cs, sn);
        sincospif(static_cast<float>(j + 1) / 1024.0f, &sn, &cs);
        const float2 w1 = make_float2(cs, sn);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            v0[r] = cmul(v0[r], T0);
            v1[r] = cmul(v1[r], T1);
            if (r < 15) {
                T0 = cmul(T0, w0);
                T1 = cmul(T1, w1);
            }
        }
        float4* dst = reinterpret_cast<float4*>(buf + p * k2kKp) + t;  // position j + 128 r -> j + 136 r
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r * 68] = pack2(v0[r], v1[r]);
    }
    __syncthreads();
    // ---- pass 2: radix 16 within blocks of 128 (span 8), butterflies (blk, j2), (blk, j2 + 1)
    {
        const int blk = t >> 2, j2 = 2 * (t & 3);
        float4* ptr = reinterpret_cast<float4*>(buf + p * k2kKp + blk * 136 + j2);
        float2 v0[16], v1[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float4 q = ptr[r * 4];
            v0[r] = make_float2(q.x, q.y);
            v1[r] = make_float2(q.z, q.w);
        }
        dft_reg<16>(v0);
        dft_reg<16>(v1);
        const float4* tw = reinterpret_cast<const float4*>(sT + j2);
#pragma unroll
        for (int r = 1; r < 16; ++r) {
            const float4 w = tw[r * 4];
            v0[r] = cmul(v0[r], make_float2(w.x, w.y));
            v1[r] = cmul(v1[r], make_float2(w.z, w.w));
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) ptr[r * 4] = pack2(v0[r], v1[r]);
    }
    __syncthreads();
    // ---- pass 3: radix 8 over contiguous octets, fused with the store
    {
        const size_t cbase = static_cast<size_t>(blockIdx.y) * a.R_slice * a.M;
        const bool full = a.n_base == 0 && a.R_slice == K;
#pragma unroll 1
        for (int idx = tid; idx < k2kPG * 256; idx += k2kThreads) {
            const int pp = idx & 3;   // lanes over pulses first: one 32-byte row sector per 4 lanes
            const int kl = idx >> 2;  // this thread's bins: kl + 256 t
            const float4* src = reinterpret_cast<const float4*>(buf + pp * k2kKp + (kl & 15) * 136 + ((kl >> 4) & 15) * 8);
            float2 v[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float4 q = src[i];
                v[2 * i] = make_float2(q.x, q.y);
                v[2 * i + 1] = make_float2(q.z, q.w);
            }
            dft_reg<8>(v);
            if (full) {
                float2* dst = a.X + cbase + static_cast<size_t>(kl) * a.M + m0 + pp;
                const size_t step = static_cast<size_t>(256) * a.M;
#pragma unroll
                for (int tt = 0; tt < 8; ++tt) dst[tt * step] = v[tt];
            } else {
#pragma unroll
                for (int tt = 0; tt < 8; ++tt) {
                    const int n = (kl + 256 * tt - a.n_base) & (K - 1);
                    if (n < a.R_slice) a.X[cbase + static_cast<size_t>(n) * a.M + m0 + pp] = v[tt];
                }
            }
        }
    }
}

}  // namespace ltcib
