// gather.cuh -- K1g: the coarse range-migration gather as an interpolation of
// 2x-oversampled range profiles.
//
// mgift (reference proj/src/transforms.cpp:134-173; build_mf RM/KtRm/PreDfm
// :32-94) is, per coarse cell c and pulse m, the trigonometric polynomial of
// the pulse's range spectrum evaluated on the range grid displaced by the
// coarse trajectory:
//   X_c[n, m] = preDFM_c(m) * P_m(n + delta_c(m)),
//   P_m(x)    = sum_g y[g, m] e^{j b(m) g^2} e^{j 2 pi g x / K},  g in [-K/2, K/2)
// with delta_c(m) = S_c(t_m) / dR.  P_m does not depend on the coarse cell
// (b is zero for DS-GRFT and depends only on the folding number q for
// DS-KT-MFP), so instead of one K-point transform per (cell, pulse) -- K1,
// coarse.cuh -- the polynomial is tabulated ONCE per pulse on the grid of
// half range cells and every coarse cell gathers from that table:
//   U[l, m] = sum_g (y[g, m] / D(g)) e^{j b g^2} e^{j 2 pi g l / (2K)}
//   X_c[n, m] = preDFM * sum_{i < 8} phi(eps + 3 - i) U[2n + L - 3 + i, m],
//   2 delta = L + eps,  L = floor(2 delta)
// phi(z) = exp(beta (sqrt(1 - (z/4)^2) - 1)) is the "exponential of
// semicircle" window of width 8 on the fine grid (beta = 18.4) and
// D(g) = int phi(z) cos(pi g z / K) dz its transform: the type-2 non-uniform
// FFT with oversampling 2, whose aliasing error for this window is 1.3e-7 of
// the profile maximum (measured against the exact transform in FP64) -- FP32
// rounding level, under the 2e-5 the kernel-level parity tests hold K1 to.
// The table is two K-point transforms per pulse (even l: delta = 0, odd l:
// delta = 1/2) done by K1's own passes (coarse_rm_kernel<K, 0, TAB = 1>).
//
// Per output the gather costs 8 packed FMAs on two 4-tap streams (the even and
// odd fine samples live in separate planes, so the 8 taps are rows r .. r+3 of
// each plane), one complex multiply and one store, against ~50 instructions
// per point of the transform: the stage becomes a streaming write of X.
#pragma once

#include "common.cuh"
#include "gather_launch.hpp"

namespace ltcib {

constexpr int kGatherTaps = 8;
constexpr double kGatherBeta = 2.30 * kGatherTaps;
#ifndef LTCI_GATHER_CELLS
#define LTCI_GATHER_CELLS 16      // coarse cells (one warp each) per CTA
#endif
constexpr int kGatherCells = LTCI_GATHER_CELLS;
#ifndef LTCI_GATHER_ROWS
#define LTCI_GATHER_ROWS 128      // range cells per CTA tile
#endif
constexpr int kGatherRows = LTCI_GATHER_ROWS;
#ifndef LTCI_GATHER_MINB
#define LTCI_GATHER_MINB 2        // CTAs per SM the tile leaves room for
#endif
#ifndef LTCI_GATHER_STORE
#define LTCI_GATHER_STORE 1       // 1: evict-first (streaming) stores of X
#endif
constexpr int kGatherHalo = 24;   // staged rows beyond the tile: 4 taps + the CTA's spread of shifts
constexpr int kGatherThreads = 32 * kGatherCells;


// D(g), g = 0 .. K/2 (even in g); deap[k] = 1 / D(g(k)) for every frequency
// row.  Simpson over z = 4 sin(theta): the integrand is analytic in theta
// (128 intervals reach 3e-13).
__global__ void __launch_bounds__(128) gather_deap_kernel(float* __restrict__ deap, int K) {
    constexpr int N = 128;
    constexpr double kPiD = 3.14159265358979323846;
    __shared__ double s_f[N + 1], s_z[N + 1];
    const double h = kPiD / N;
    for (int i = threadIdx.x; i <= N; i += blockDim.x) {
        double sn, cs;
        sincos(-0.5 * kPiD + h * i, &sn, &cs);
        const double wgt = (i == 0 || i == N) ? 1.0 : (i & 1) ? 4.0 : 2.0;
        s_z[i] = 0.5 * kGatherTaps * sn;
        s_f[i] = wgt * exp(kGatherBeta * (cs - 1.0)) * (0.5 * kGatherTaps) * cs;
    }
    __syncthreads();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g > K / 2) return;
    const double kz = kPiD * static_cast<double>(g) / K;
    double acc = 0.0;
    for (int i = 0; i <= N; ++i) acc += s_f[i] * cos(kz * s_z[i]);
    const float v = static_cast<float>(1.0 / (acc * h / 3.0));
    deap[g] = v;
    if (g > 0 && g < K / 2) deap[K - g] = v;
}

// per (cell, pulse): L, the 8 taps and the preDFM factor, FP64
__global__ void __launch_bounds__(256) gather_weights_kernel(GatherArgs a) {
    const size_t total = static_cast<size_t>(a.c_count) * a.M;
    const size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (idx >= total) return;
    const int cl = static_cast<int>(idx / a.M);
    const int m = static_cast<int>(idx - static_cast<size_t>(cl) * a.M);
    const double* cp = a.cparams + 4 * (a.c_begin + cl);
    const double t = static_cast<double>(m + 1) * a.inv_prf;
    double s_rm, s_predfm;
    if (a.variant == 0) {
        // poly_from(c, t, 1) (transforms.cpp:12-22)
        double tp = 1.0, acc = 0.0;
        for (int p = 0; p < a.P; ++p) {
            tp *= t;
            acc += cp[p] * tp;
        }
        s_rm = acc;
        s_predfm = acc;
    } else {
        // KtRm (transforms.cpp:53-70): the part linear in f_r; the f_r^2 term is in the table
        s_rm = cp[0] * a.Va * t - cp[1] * t * t;
        s_predfm = cp[1] * t * t;
    }
    const double two_delta = 2.0 * s_rm * a.inv_dR;
    const double Lf = floor(two_delta);
    const double eps = two_delta - Lf;
    long long Lm = static_cast<long long>(fmod(Lf, 2.0 * a.K));
    if (Lm < 0) Lm += 2 * a.K;
    float w[kGatherTaps];
#pragma unroll
    for (int i = 0; i < kGatherTaps; ++i) {
        const double z = (eps + (kGatherTaps / 2 - 1) - i) * (2.0 / kGatherTaps);
        const double x = fmax(1.0 - z * z, 0.0);
        w[i] = static_cast<float>(exp(kGatherBeta * (sqrt(x) - 1.0)));
    }
    const double cyc = s_predfm * a.two_over_lambda;
    double sn, cs;
    sincospi(2.0 * (cyc - rint(cyc)), &sn, &cs);
    const size_t o = static_cast<size_t>(a.c_begin - a.w_first) * a.M + idx;
    a.W[o] = make_float4(w[0], w[2], w[4], w[6]);
    a.W[a.w_plane + o] = make_float4(w[1], w[3], w[5], w[7]);
    a.W[2 * a.w_plane + o] = make_float4(static_cast<float>(cs), static_cast<float>(sn),
                                         __int_as_float(static_cast<int>(Lm)), 0.0f);
}

// 1-D bulk copy (TMA unit) of one 256-byte table row segment into the tile,
// completion counted in bytes on the CTA's mbarrier
__device__ __forceinline__ void gather_bulk_row(void* smem, const void* gmem, unsigned bytes, unsigned bar) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
                 "l"(gmem), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void gather_bar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// one tile's outputs of a thread.  STAGED: pa / pb point at the thread's first
// row of each stream in the shared tile (32 float2 per row).  Otherwise they
// point at the plane's column in global memory and rows RA + i, RB + i wrap
// modulo K.
template <bool STAGED>
__device__ __forceinline__ void gather_run(const float2* __restrict__ pa, const float2* __restrict__ pb, int RA,
                                           int RB, int K, size_t M, const float4 wa, const float4 wb,
                                           const float2 pre, float2* __restrict__ out, int nmax) {
    const float2 a0w = make_float2(wa.x, wa.x), a1w = make_float2(wa.y, wa.y), a2w = make_float2(wa.z, wa.z),
                 a3w = make_float2(wa.w, wa.w);
    const float2 b0w = make_float2(wb.x, wb.x), b1w = make_float2(wb.y, wb.y), b2w = make_float2(wb.z, wb.z),
                 b3w = make_float2(wb.w, wb.w);
    auto la = [&](int i) -> float2 {
        if constexpr (STAGED) return pa[i * 32];
        return __ldg(pa + static_cast<size_t>((RA + i) & (K - 1)) * M);
    };
    auto lb = [&](int i) -> float2 {
        if constexpr (STAGED) return pb[i * 32];
        return __ldg(pb + static_cast<size_t>((RB + i) & (K - 1)) * M);
    };
    float2 a0 = la(0), a1 = la(1), a2 = la(2), a3;
    float2 b0 = lb(0), b1 = lb(1), b2 = lb(2), b3;
    int left = nmax;
    auto emit = [&](int u, float2 x0, float2 x1, float2 x2, float2 x3, float2 y0, float2 y1, float2 y2, float2 y3) {
        const float2 sa = fma2(a3w, x3, fma2(a2w, x2, fma2(a1w, x1, mul2(a0w, x0))));
        const float2 sb = fma2(b3w, y3, fma2(b2w, y2, fma2(b1w, y1, mul2(b0w, y0))));
        const float2 v = cmul(add2(sa, sb), pre);
        if (u < left) {
            if constexpr (LTCI_GATHER_STORE)
                __stcs(out + static_cast<size_t>(u) * M, v);
            else
                out[static_cast<size_t>(u) * M] = v;
        }
    };
#pragma unroll 1
    for (; left > 0; left -= 4) {
        a3 = la(3);
        b3 = lb(3);
        emit(0, a0, a1, a2, a3, b0, b1, b2, b3);
        a0 = la(4);
        b0 = lb(4);
        emit(1, a1, a2, a3, a0, b1, b2, b3, b0);
        a1 = la(5);
        b1 = lb(5);
        emit(2, a2, a3, a0, a1, b2, b3, b0, b1);
        a2 = la(6);
        b2 = lb(6);
        emit(3, a3, a0, a1, a2, b3, b0, b1, b2);
        if constexpr (STAGED) {
            pa += 4 * 32;
            pb += 4 * 32;
        } else {
            RA += 4;
            RB += 4;
        }
        out += 4 * M;
    }
}

// grid: (M / 32, tables x groups, ceil(R_slice / kGatherRows)); block = 16
// warps, warp = one coarse cell, lane = pulse m0 + lane.  The range tile is
// the slowest grid index: all cell groups of a tile run back to back on the
// same ~2 MB of table rows, so the table is read from HBM once (with the
// groups slowest every group swept the whole table again after 130 MB of X
// had passed through L2: 1.08 GB of DRAM reads at C1 for a 33.5 MB table).
// The CTA stages the plane rows its 16 cells x 32 pulses can touch (one
// 256-byte bulk copy per row on the TMA unit, rows taken modulo K: the gather
// is circular like the transform; all threads wait on the CTA's mbarrier),
// then every thread slides its two 4-tap windows down the tile.  Warps store
// 256 contiguous bytes per range cell; blockIdx.x walks the pulses so
// co-resident CTAs complete whole rows in L2.  When the shifts of a CTA's
// cells spread over more than the halo (not the case for the reference's grid
// rules, where neighbouring coarse cells differ by one range cell at the end
// of the CPI) the taps are read from global memory instead.
__global__ void __launch_bounds__(kGatherThreads, LTCI_GATHER_MINB) gather_interp_kernel(GatherArgs a, int rows_cap) {
    extern __shared__ __align__(16) float2 g_tile[];  // [2][rows_cap][32]
    __shared__ int s_ref, s_min, s_max;
    __shared__ __align__(8) unsigned long long s_bar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = a.K, M = a.M;
    const int m0 = blockIdx.x * 32, r0 = blockIdx.z * kGatherRows;
    const unsigned long long cpt = a.cells_per_table;
    const unsigned gpt = static_cast<unsigned>((cpt + kGatherCells - 1) / kGatherCells);
    const unsigned long long tq = a.c_begin / cpt + blockIdx.y / gpt;
    const unsigned long long c_first = tq * cpt + static_cast<unsigned long long>(blockIdx.y % gpt) * kGatherCells;
    const unsigned long long c_end = min(a.c_begin + static_cast<unsigned long long>(a.c_count), (tq + 1) * cpt);
    const unsigned long long c_lo = max(a.c_begin, c_first);
    if (c_lo >= c_end || c_lo >= c_first + kGatherCells) return;  // whole CTA outside the batch
    const unsigned long long c = c_first + warp;
    const bool active = c >= c_lo && c < c_end;
    const int warp_ref = static_cast<int>(c_lo - c_first);

    const size_t widx = active ? static_cast<size_t>(c - a.w_first) * M + m0 + lane : 0;
    float4 wa = make_float4(0, 0, 0, 0), wb = wa, wc = wa;
    if (active) {
        wa = __ldg(a.W + widx);
        wb = __ldg(a.W + a.w_plane + widx);
        wc = __ldg(a.W + 2 * a.w_plane + widx);
    }
    const int L = __float_as_int(wc.z);
    const unsigned bar = static_cast<unsigned>(__cvta_generic_to_shared(&s_bar));
    if (tid == 0) {
        s_min = 0x7fffffff;
        s_max = -0x7fffffff;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == warp_ref && lane == 0) s_ref = L;
    __syncthreads();
    // circular distance of this thread's shift to the reference, in [-K, K)
    const int d = ((L - s_ref + 3 * K) & (2 * K - 1)) - K;
    {
        int dmin = active ? d : 0x7fffffff, dmax = active ? d : -0x7fffffff;
        dmin = __reduce_min_sync(0xffffffffu, dmin);
        dmax = __reduce_max_sync(0xffffffffu, dmax);
        if (lane == 0 && active) {
            atomicMin(&s_min, dmin);
            atomicMax(&s_max, dmax);
        }
    }
    __syncthreads();
    // fine index of tap 0 at the tile's first range cell: B = 2 bin + L - 3
    const int base = 2 * (a.n_base + r0) + s_ref - (kGatherTaps / 2 - 1);
    const int row_lo = (base + s_min) >> 1;
    const int rows_need = ((base + s_max + 1) >> 1) + kGatherRows + 2 - row_lo + 1;
    const bool staged = rows_need <= rows_cap;
    const float2* Ut = a.U + static_cast<size_t>(tq) * 2 * K * M;
    if (staged) {
        // one elected thread per table row: 2 planes x rows_need segments of 256 bytes
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"(static_cast<unsigned>(2 * rows_need * 256))
                         : "memory");
        for (int rr = tid; rr < 2 * rows_need; rr += kGatherThreads) {
            const int plane = rr >= rows_need ? 1 : 0;
            const int row = rr - plane * rows_need;
            const float2* src = Ut + (static_cast<size_t>(plane) * K + ((row_lo + row) & (K - 1))) * M + m0;
            gather_bulk_row(g_tile + (static_cast<size_t>(plane) * rows_cap + row) * 32, src, 256, bar);
        }
    }
    if (!active) return;
    if (staged) gather_bar_wait(bar, 0);
    const int nmax = min(kGatherRows, a.R_slice - r0);
    const int B = base + d;
    const int pA = B & 1, RA = B >> 1, RB = (B + 1) >> 1;
    const float2 pre = make_float2(wc.x, wc.y);
    float2* out = a.X + (static_cast<size_t>(c - a.c_begin) * a.R_slice + r0) * M + m0 + lane;
    if (staged) {
        const float2* sa = g_tile + (static_cast<size_t>(pA) * rows_cap + (RA - row_lo)) * 32 + lane;
        const float2* sb = g_tile + (static_cast<size_t>(1 - pA) * rows_cap + (RB - row_lo)) * 32 + lane;
        gather_run<true>(sa, sb, 0, 0, K, static_cast<size_t>(M), wa, wb, pre, out, nmax);
    } else {
        const float2* ga = Ut + static_cast<size_t>(pA) * K * M + m0 + lane;
        const float2* gb = Ut + static_cast<size_t>(1 - pA) * K * M + m0 + lane;
        gather_run<false>(ga, gb, RA, RB, K, static_cast<size_t>(M), wa, wb, pre, out, nmax);
    }
}

inline size_t gather_smem_bytes(int rows_cap) { return static_cast<size_t>(2) * rows_cap * 32 * sizeof(float2); }

}  // namespace ltcib
