// fine_tc.cuh -- K2a: the fine Doppler-frequency-migration stage as a dense
// complex contraction on the 5th-generation tensor cores (tcgen05 + TMEM +
// TMA), fused with the K3 statistic reduction.
//
// For a batch of coarse-compensated rows X[rho, m] (rho = (coarse cell,
// range cell)) the fine stage of the reference (gft over the Doppler window,
// proj/src/transforms.cpp:180-214, scanned by UnitScan, detectors.cpp:23-31)
// is
//     Y[rho, q] = sum_m X[rho, m] * B[m, q],   q = f*D + jj,
//     B[m, q]   = H_f(m) * w_M^{d m},  d = dop_first + jj - M/2,
// (pre-recentring convention, like the FFT path: the unit-modulus factor
// e^{j 2 pi d/M} is applied on the host to returned values).  B does not
// depend on the coarse cell, so the whole stage is one GEMM.
//
// Real-ified with complex interleaving along K (k' = 2m + {re, im}):
//   A operand (MMA M = 128): X rows, K-major fp16, loaded by TMA (SW128);
//   B operand (MMA N = 256): generated steering tile, row n' = 2q + part,
//        part 0 -> (Br, -Bi), part 1 -> (Bi, Br) at (k' = 2m, 2m + 1);
//   D (TMEM, fp32, 128 lanes x 256 columns): lane = X row, Re Y / Im Y of
//        output q in adjacent columns 2q, 2q + 1.
// Split precision: x = x_hi + x_lo in fp16 (global power-of-two prescale s
// keeps X in fp16's normal range); TERMS = 3 accumulates X_hi G_hi + X_hi G_lo
// + X_lo G_hi (error ~1e-7 rel., FP32 class); TERMS = 1 is X_hi G_hi (~3e-4 of
// the row maximum, inside the 1e-3 contract; opt-in).
//
// Persistent CTAs (one per SM) walk (128-row, 128-output) tiles; warp roles
// (448 threads):
//   warp 0      TMEM allocation (512 columns = two accumulators); one lane
//               issues the TMA loads of X tiles
//   warp 1      one lane issues tcgen05.mma / tcgen05.commit
//   warps 2-9   generate the steering tile in swizzled smem from the FP64
//               H table (global, L1-resident per tile) and w_M^k
//   warps 10-13 epilogue, one X row per thread: tcgen05.ld, |Y|^2, threshold
//               compaction, in-thread row argmax (lowest q on ties), one
//               128-bit CAS per row and tile into the per-cell peak slot;
//               overlaps the next tile's MMAs (double-buffered TMEM).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include "coarse.cuh"
#include "fine_fft.cuh"

namespace ltcib {

constexpr int TC_BM = 128;    // X rows per tile (MMA M)
constexpr int TC_BN = 256;    // real output columns per tile (MMA N) = 128 complex outputs
constexpr int TC_BK = 64;     // real K per k-block: 128-byte rows, SW128
constexpr int TC_QT = TC_BN / 2;
constexpr int TC_GEN_WARPS = 8;
constexpr int TC_EPI_WARPS = 4;
constexpr int TC_THREADS = 32 * (2 + TC_GEN_WARPS + TC_EPI_WARPS);
constexpr int TC_X_BYTES = TC_BM * TC_BK * 2;
constexpr int TC_G_BYTES = TC_BN * TC_BK * 2;

struct TcArgs {
    FineArgs f;                 // shared indexing / output fields
    int M, K;
    int nfa;                    // fine axes (0..3)
    int fcount[3], ford[3];
    double fstart[3], fstep[3];
    double coef_cycles;         // 2 kappa / lambda
    double inv_prf;
    const float2* htab;         // [F][M] H_f(m), built by build_htab_kernel
    const unsigned* maxbits;    // max |y|^2 of the coarse-stage input (float bits)
};

// ------------------------------------------------------------- PTX glue ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
// try_wait carries a suspend-time hint, so a waiting warp sleeps in hardware
// until the phase completes instead of spinning on issue slots the generator
// warps need.
__device__ __noinline__ void mbar_wait_slow(uint32_t bar, uint32_t parity) {
    const long long t0 = clock64();
#pragma unroll 1
    for (;;) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(1000000u)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 20000000000ll) __trap();  // ~10 s: protocol bug, fail the launch
    }
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (!done) mbar_wait_slow(bar, parity);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte swizzle, 8-row core groups 1024 B apart (SBO), sm100 version bit.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;             // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;     // SBO
    d |= static_cast<uint64_t>(1) << 46;             // descriptor version (Blackwell)
    d |= static_cast<uint64_t>(2) << 61;             // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: F32 accumulate, F16 A/B, both K-major.
__host__ __device__ constexpr uint32_t tc_idesc(int m, int n) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// exp(+j 2 pi idx / M) for an exact integer index (reduced to [-M/2, M/2), so
// the MUFU argument stays in [-pi, pi): abs error < 4e-7).
__device__ __forceinline__ float2 wpow(int idx, int M) {
    int k = idx & (M - 1);
    if (k >= M / 2) k -= M;
    float s, c;
    __sincosf(6.28318530717958647692f * static_cast<float>(k) / static_cast<float>(M), &s, &c);
    return make_float2(c, s);
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float2 unpack_half2(uint32_t u) {
    __half2 h = *reinterpret_cast<__half2*>(&u);
    return __half22float2(h);
}

template <int TERMS>
__host__ __device__ constexpr int tc_stages() {
    return TERMS == 3 ? 2 : 4;
}

template <int TERMS>
__host__ __device__ constexpr int tc_stage_bytes() {
    return (TERMS == 3 ? 2 : 1) * (TC_X_BYTES + TC_G_BYTES);
}

// ------------------------------------------------------------- kernel -----
// Persistent: each CTA walks tiles t = blockIdx.x, + gridDim.x, ...; tile t =
// (row tile t / nq, q tile t % nq), q fastest so co-resident CTAs share the
// X row tile in L2.  TMEM holds two 128 x 256 fp32 accumulators so the
// epilogue of tile i overlaps the MMAs of tile i + 1.
template <int TERMS>
__global__ void __launch_bounds__(TC_THREADS, 1)
    fine_tc_kernel(const __grid_constant__ TcArgs a, const __grid_constant__ CUtensorMap tm_hi,
                   const __grid_constant__ CUtensorMap tm_lo) {
    constexpr int STAGES = tc_stages<TERMS>();
    constexpr int PLANES = TERMS == 3 ? 2 : 1;
    constexpr int SB = tc_stage_bytes<TERMS>();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment by offsetting the shared array itself, so every
    // derived pointer stays in the shared state space (LDS/STS, not LD/ST).
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const FineArgs& fa = a.f;
    const int M = a.M;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Q = static_cast<int>(fa.F) * fa.D;
    const int nq = (Q + TC_QT - 1) / TC_QT;
    const int nrt = (fa.rows + TC_BM - 1) / TC_BM;
    const int ntiles = nq * nrt;
    const int nkb = (2 * M) / TC_BK;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1 + TC_GEN_WARPS);  // TMA producer + generator warps
            mbar_init(empty0 + 8 * s, 1);                 // tcgen05.commit
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);                 // tcgen05.commit after a tile's last k-block
            mbar_init(tempty0 + 8 * b, TC_EPI_WARPS);     // epilogue warps drained the accumulator
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(2 * TC_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        // ---------------- TMA producer: X tiles (MMA A operand) ----------------
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int row0 = (t / nq) * TC_BM;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(empty0 + 8 * s, ph ^ 1);
                    uint8_t* st = smem + s * SB;
                    mbar_expect_tx(full0 + 8 * s, PLANES * TC_X_BYTES);
                    tma_load_2d(smem_u32(st), &tm_hi, kb * TC_BK, row0, full0 + 8 * s);
                    if (TERMS == 3) tma_load_2d(smem_u32(st + TC_X_BYTES), &tm_lo, kb * TC_BK, row0, full0 + 8 * s);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = tc_idesc(TC_BM, TC_BN);
            int it = 0, i = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                const int ab = i & 1;
                mbar_wait(tempty0 + 8 * ab, ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + ab * TC_BN;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(full0 + 8 * s, ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * SB);
                    const uint32_t x_hi = st, x_lo = st + TC_X_BYTES;
                    const uint32_t g_hi = st + PLANES * TC_X_BYTES, g_lo = g_hi + TC_G_BYTES;
#pragma unroll
                    for (int ks = 0; ks < TC_BK / 16; ++ks) {
                        const uint32_t off = ks * 32;  // 16 fp16 along K
                        tc_mma(dcol, sw128_desc(x_hi + off), sw128_desc(g_hi + off), idesc, (kb | ks) != 0);
                        if (TERMS == 3) {
                            tc_mma(dcol, sw128_desc(x_hi + off), sw128_desc(g_lo + off), idesc, 1);
                            tc_mma(dcol, sw128_desc(x_lo + off), sw128_desc(g_hi + off), idesc, 1);
                        }
                    }
                    tc_commit(empty0 + 8 * s);
                }
                tc_commit(tfull0 + 8 * ab);
            }
        }
    } else if (warp < 2 + TC_GEN_WARPS) {
        // ---------------- steering generators (MMA B operand) ----------------
        // Each complex steering value is computed once and written to both of
        // its real rows (2q: (Br, -Bi) -> Re Y, 2q+1: (Bi, Br) -> Im Y).
        // Lane bits 0-1 pick the q (row swizzle residue), bits 2-4 the 16-byte
        // chunk, so every 8-lane phase of a 128-bit store hits 8 distinct bank
        // groups; 4 passes of 32 q per warp cover the 128 q of a tile.
        const int wg = warp - 2;                       // 0..7
        const int c = lane >> 2;                       // chunk 0..7 (4 pulses each)
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int q0 = (t % nq) * TC_QT;
            int dq[4];
            const float2* Hq[4];
            bool vq[4];
            float2 wd[4];  // w_M^d: per-pulse step of the Doppler phase
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int qc = q0 + (lane & 3) + 4 * wg + 32 * u;
                vq[u] = qc < Q;
                const int f = vq[u] ? qc / fa.D : 0;
                const int jj = vq[u] ? qc - f * fa.D : 0;
                dq[u] = jj + fa.dop_first - M / 2;
                Hq[u] = a.htab + static_cast<size_t>(f) * M;
                wd[u] = wpow(dq[u], M);
            }
            for (int kb = 0; kb < nkb; ++kb, ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                mbar_wait(empty0 + 8 * s, ph ^ 1);
                uint8_t* g_hi = smem + s * SB + PLANES * TC_X_BYTES;
                uint8_t* g_lo = g_hi + TC_G_BYTES;
                const int mf = kb * (TC_BK / 2) + 4 * c;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int L0 = 2 * ((lane & 3) + 4 * wg + 32 * u), L1 = L0 + 1;
                    const uint32_t o0 = (L0 >> 3) * 1024 + (L0 & 7) * 128 + ((c ^ (L0 & 7)) << 4);
                    const uint32_t o1 = (L1 >> 3) * 1024 + (L1 & 7) * 128 + ((c ^ (L1 & 7)) << 4);
                    uint32_t h0[4], h1[4], l0[4], l1[4];
                    // exact-index w_M^{d m} for the chunk's first pulse, then w_M^d steps
                    float2 wv = wpow(dq[u] * mf, M);
                    const float4 hA = __ldg(reinterpret_cast<const float4*>(Hq[u] + mf));
                    const float4 hB = __ldg(reinterpret_cast<const float4*>(Hq[u] + mf + 2));
                    const float2 hv[4] = {make_float2(hA.x, hA.y), make_float2(hA.z, hA.w),
                                          make_float2(hB.x, hB.y), make_float2(hB.z, hB.w)};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float2 b = cmul(hv[e], wv);
                        if (e < 3) wv = cmul(wv, wd[u]);
                        if (!vq[u]) b = make_float2(0.f, 0.f);
                        const uint32_t hb = pack_half2(b.x, b.y);     // (Br, Bi) hi
                        h0[e] = hb ^ 0x80000000u;                     // (Br, -Bi)
                        h1[e] = __byte_perm(hb, 0, 0x1032);           // (Bi, Br)
                        if (TERMS == 3) {
                            const float2 hf = unpack_half2(hb);
                            const uint32_t lb = pack_half2(b.x - hf.x, b.y - hf.y);
                            l0[e] = lb ^ 0x80000000u;
                            l1[e] = __byte_perm(lb, 0, 0x1032);
                        }
                    }
                    *reinterpret_cast<uint4*>(g_hi + o0) = make_uint4(h0[0], h0[1], h0[2], h0[3]);
                    *reinterpret_cast<uint4*>(g_hi + o1) = make_uint4(h1[0], h1[1], h1[2], h1[3]);
                    if (TERMS == 3) {
                        *reinterpret_cast<uint4*>(g_lo + o0) = make_uint4(l0[0], l0[1], l0[2], l0[3]);
                        *reinterpret_cast<uint4*>(g_lo + o1) = make_uint4(l1[0], l1[1], l1[2], l1[3]);
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(full0 + 8 * s);
            }
        }
    } else {
        // ---------------- epilogue: one X row per thread ----------------
        const int quad = warp & 3;                 // TMEM lane quadrant (warps 10..13 -> 2,3,0,1)
        const float inv_s = 1.0f / fp16_prescale(a.maxbits, a.K);
        int i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int ab = i & 1;
            const int q0 = (t % nq) * TC_QT;
            const int rho = (t / nq) * TC_BM + 32 * quad + lane;
            const bool rvalid = rho < fa.rows;
            const int c_local = rvalid ? rho / fa.R_slice : 0;
            const int r_local = rho - c_local * fa.R_slice;
            const unsigned long long c_glob = fa.c_begin + c_local;
            const int r_glob = fa.row_begin + r_local;
            mbar_wait(tfull0 + 8 * ab, (i >> 1) & 1);
            tc_fence_after();
            RowBest best{-1.0f, 0xffffffffu, 0.f, 0.f};
            int qf = q0 / fa.D, qj = q0 - qf * fa.D;    // (f, jj) of the current q, advanced incrementally
            for (int cb = 0; cb < TC_BN / 32; ++cb) {
                uint32_t r[32];
                tmem_ld32(tmem + (static_cast<uint32_t>(32 * quad) << 16) + ab * TC_BN + cb * 32, r);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int q = q0 + cb * 16 + j;
                    const float re = __uint_as_float(r[2 * j]) * inv_s;
                    const float im = __uint_as_float(r[2 * j + 1]) * inv_s;
                    if (rvalid && q < Q) {
                        const float m2 = mag2f(re, im);
                        const unsigned lidx = static_cast<unsigned>(q);
                        if (m2 > best.m) {  // q ascends: strict > keeps the lowest q on ties
                            best.m = m2;
                            best.lidx = lidx;
                            best.re = re;
                            best.im = im;
                        }
                        if (fa.dense != nullptr || m2 > fa.retain2)
                            emit_cell(fa, make_float2(re, im), m2, static_cast<unsigned>(qf), qj, c_glob, r_glob,
                                      fa.dense != nullptr);
                    }
                    if (++qj == fa.D) {
                        qj = 0;
                        ++qf;
                    }
                }
            }
            // accumulator buffer drained: hand it back to the MMA issuer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty0 + 8 * ab);
            if (rvalid && best.lidx != 0xffffffffu) {
                const unsigned fb = best.lidx / static_cast<unsigned>(fa.D);
                const unsigned jb = best.lidx - fb * static_cast<unsigned>(fa.D);
                const unsigned long long flat =
                    ((c_glob * fa.F + fb) * fa.R_total + static_cast<unsigned long long>(r_glob)) * fa.D + jb;
                peak_publish(fa.slots + r_local, best.re, best.im, flat);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_BN));
    }
}

// ===================== CTA-pair variant (cta_group::2) =====================
// A cluster of two CTAs on one TPC computes a 256-row x 256-column tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA loads its own 128 X rows and
// generates HALF of the steering columns (64 complex outputs), so the
// generator work and the smem operand reads per SM halve; D lands in each
// CTA's TMEM as its 128 rows x 256 columns.  Protocol (CUTLASS 2-SM style):
//   full[s]   leader's barrier: leader producer expect_tx (both CTAs' bytes),
//             both CTAs' TMA complete_tx, 8 generator warps per CTA arrive
//   empty[s]  per CTA: leader's tcgen05.commit multicast to both CTAs
//   tfull[b]  per CTA: commit multicast after a tile's last k-block
//   tempty[b] leader's barrier: 4 epilogue warps per CTA arrive
constexpr int TC2_BM = 128;                    // X rows per CTA
constexpr int TC2_GN = 128;                    // generated real columns per CTA (64 q)
constexpr int TC2_X_BYTES = TC2_BM * TC_BK * 2;
constexpr int TC2_G_BYTES = TC2_GN * TC_BK * 2;

template <int TERMS>
__host__ __device__ constexpr int tc2_stages() {
    return TERMS == 3 ? 3 : 6;
}

template <int TERMS>
__host__ __device__ constexpr int tc2_stage_bytes() {
    return (TERMS == 3 ? 2 : 1) * (TC2_X_BYTES + TC2_G_BYTES);
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Arrive on a (possibly peer) CTA's barrier.  Writers of async-proxy
// operands precede this with fence.proxy.async, as CUTLASS does.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __noinline__ void mbar_wait_cluster_slow(uint32_t bar, uint32_t parity) {
    const long long t0 = clock64();
#pragma unroll 1
    for (;;) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(1000000u)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 20000000000ll) __trap();
    }
}

// wait with cluster-scope acquire (arrivals come from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (!done) mbar_wait_cluster_slow(bar, parity);
}

__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
        : "memory");
}

__device__ __forceinline__ void tc2_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tc2_commit_both(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            bar),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

template <int TERMS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    fine_tc2_kernel(const __grid_constant__ TcArgs a, const __grid_constant__ CUtensorMap tm_hi,
                    const __grid_constant__ CUtensorMap tm_lo) {
    constexpr int STAGES = tc2_stages<TERMS>();
    constexpr int PLANES = TERMS == 3 ? 2 : 1;
    constexpr int SB = tc2_stage_bytes<TERMS>();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const FineArgs& fa = a.f;
    const int M = a.M;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int Q = static_cast<int>(fa.F) * fa.D;
    const int nq = (Q + TC_QT - 1) / TC_QT;
    const int nrt = (fa.rows + 2 * TC2_BM - 1) / (2 * TC2_BM);
    const int ntiles = nq * nrt;
    const int nkb = (2 * M) / TC_BK;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);
    const uint32_t full0_l = mapa_shared(full0, 0), tempty0_l = mapa_shared(tempty0, 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1 + 2 * TC_GEN_WARPS);  // leader producer + generators of both CTAs
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, 2 * TC_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(2 * TC_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int t = pair; t < ntiles; t += npairs) {
                const int row0 = (t / nq) * (2 * TC2_BM) + rank * TC2_BM;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(empty0 + 8 * s, ph ^ 1);
                    uint8_t* st = smem + s * SB;
                    if (rank == 0) mbar_expect_tx(full0 + 8 * s, 2 * PLANES * TC2_X_BYTES);
                    tma_load_2d_pair(smem_u32(st), &tm_hi, kb * TC_BK, row0, full0_l + 8 * s);
                    if (TERMS == 3)
                        tma_load_2d_pair(smem_u32(st + TC2_X_BYTES), &tm_lo, kb * TC_BK, row0, full0_l + 8 * s);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = tc_idesc(2 * TC2_BM, TC_BN);
            int it = 0, i = 0;
            for (int t = pair; t < ntiles; t += npairs, ++i) {
                const int ab = i & 1;
                mbar_wait_cluster(tempty0 + 8 * ab, ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + ab * TC_BN;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait_cluster(full0 + 8 * s, ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * SB);
                    const uint32_t x_hi = st, x_lo = st + TC2_X_BYTES;
                    const uint32_t g_hi = st + PLANES * TC2_X_BYTES, g_lo = g_hi + TC2_G_BYTES;
#pragma unroll
                    for (int ks = 0; ks < TC_BK / 16; ++ks) {
                        const uint32_t off = ks * 32;
                        tc2_mma(dcol, sw128_desc(x_hi + off), sw128_desc(g_hi + off), idesc, (kb | ks) != 0);
                        if (TERMS == 3) {
                            tc2_mma(dcol, sw128_desc(x_hi + off), sw128_desc(g_lo + off), idesc, 1);
                            tc2_mma(dcol, sw128_desc(x_lo + off), sw128_desc(g_hi + off), idesc, 1);
                        }
                    }
                    tc2_commit_both(empty0 + 8 * s);
                }
                tc2_commit_both(tfull0 + 8 * ab);
            }
        }
    } else if (warp < 2 + TC_GEN_WARPS) {
        // generators: this CTA's 64 q of the tile (q0 + 64 rank ...), 2 per thread
        const int wg = warp - 2;
        const int c = lane >> 2;
        int it = 0;
        for (int t = pair; t < ntiles; t += npairs) {
            const int q0 = (t % nq) * TC_QT + 64 * static_cast<int>(rank);
            int dq[2];
            const float2* Hq[2];
            bool vq[2];
            float2 wd[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int qc = q0 + (lane & 3) + 4 * wg + 32 * u;
                vq[u] = qc < Q;
                const int f = vq[u] ? qc / fa.D : 0;
                const int jj = vq[u] ? qc - f * fa.D : 0;
                dq[u] = jj + fa.dop_first - M / 2;
                Hq[u] = a.htab + static_cast<size_t>(f) * M;
                wd[u] = wpow(dq[u], M);
            }
            for (int kb = 0; kb < nkb; ++kb, ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                const int mf = kb * (TC_BK / 2) + 4 * c;
                // operand inputs do not depend on the stage: load them before waiting
                float4 hA[2], hB[2];
                float2 w0[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    hA[u] = __ldg(reinterpret_cast<const float4*>(Hq[u] + mf));
                    hB[u] = __ldg(reinterpret_cast<const float4*>(Hq[u] + mf + 2));
                    w0[u] = wpow(dq[u] * mf, M);
                }
                mbar_wait(empty0 + 8 * s, ph ^ 1);
                uint8_t* g_hi = smem + s * SB + PLANES * TC2_X_BYTES;
                uint8_t* g_lo = g_hi + TC2_G_BYTES;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int L0 = 2 * ((lane & 3) + 4 * wg + 32 * u), L1 = L0 + 1;
                    const uint32_t o0 = (L0 >> 3) * 1024 + (L0 & 7) * 128 + ((c ^ (L0 & 7)) << 4);
                    const uint32_t o1 = (L1 >> 3) * 1024 + (L1 & 7) * 128 + ((c ^ (L1 & 7)) << 4);
                    uint32_t h0[4], h1[4], l0[4], l1[4];
                    float2 wv = w0[u];
                    const float2 hv[4] = {make_float2(hA[u].x, hA[u].y), make_float2(hA[u].z, hA[u].w),
                                          make_float2(hB[u].x, hB[u].y), make_float2(hB[u].z, hB[u].w)};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float2 b = cmul(hv[e], wv);
                        if (e < 3) wv = cmul(wv, wd[u]);
                        if (!vq[u]) b = make_float2(0.f, 0.f);
                        const uint32_t hb = pack_half2(b.x, b.y);
                        h0[e] = hb ^ 0x80000000u;
                        h1[e] = __byte_perm(hb, 0, 0x1032);
                        if (TERMS == 3) {
                            const float2 hf = unpack_half2(hb);
                            const uint32_t lb = pack_half2(b.x - hf.x, b.y - hf.y);
                            l0[e] = lb ^ 0x80000000u;
                            l1[e] = __byte_perm(lb, 0, 0x1032);
                        }
                    }
                    *reinterpret_cast<uint4*>(g_hi + o0) = make_uint4(h0[0], h0[1], h0[2], h0[3]);
                    *reinterpret_cast<uint4*>(g_hi + o1) = make_uint4(h1[0], h1[1], h1[2], h1[3]);
                    if (TERMS == 3) {
                        *reinterpret_cast<uint4*>(g_lo + o0) = make_uint4(l0[0], l0[1], l0[2], l0[3]);
                        *reinterpret_cast<uint4*>(g_lo + o1) = make_uint4(l1[0], l1[1], l1[2], l1[3]);
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(full0_l + 8 * s);
            }
        }
    } else {
        // epilogue: this CTA's 128 rows, all 256 columns (128 q) of the tile
        const int quad = warp & 3;
        const float inv_s = 1.0f / fp16_prescale(a.maxbits, a.K);
        int i = 0;
        for (int t = pair; t < ntiles; t += npairs, ++i) {
            const int ab = i & 1;
            const int q0 = (t % nq) * TC_QT;
            const int rho = (t / nq) * (2 * TC2_BM) + rank * TC2_BM + 32 * quad + lane;
            const bool rvalid = rho < fa.rows;
            const int c_local = rvalid ? rho / fa.R_slice : 0;
            const int r_local = rho - c_local * fa.R_slice;
            const unsigned long long c_glob = fa.c_begin + c_local;
            const int r_glob = fa.row_begin + r_local;
            mbar_wait(tfull0 + 8 * ab, (i >> 1) & 1);
            tc_fence_after();
            RowBest best{-1.0f, 0xffffffffu, 0.f, 0.f};
            int qf = q0 / fa.D, qj = q0 - qf * fa.D;
            for (int cb = 0; cb < TC_BN / 32; ++cb) {
                uint32_t r[32];
                tmem_ld32(tmem + (static_cast<uint32_t>(32 * quad) << 16) + ab * TC_BN + cb * 32, r);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int q = q0 + cb * 16 + j;
                    const float re = __uint_as_float(r[2 * j]) * inv_s;
                    const float im = __uint_as_float(r[2 * j + 1]) * inv_s;
                    if (rvalid && q < Q) {
                        const float m2 = mag2f(re, im);
                        if (m2 > best.m) {
                            best.m = m2;
                            best.lidx = static_cast<unsigned>(q);
                            best.re = re;
                            best.im = im;
                        }
                        if (fa.dense != nullptr || m2 > fa.retain2)
                            emit_cell(fa, make_float2(re, im), m2, static_cast<unsigned>(qf), qj, c_glob, r_glob,
                                      fa.dense != nullptr);
                    }
                    if (++qj == fa.D) {
                        qj = 0;
                        ++qf;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty0_l + 8 * ab);
            if (rvalid && best.lidx != 0xffffffffu) {
                const unsigned fb = best.lidx / static_cast<unsigned>(fa.D);
                const unsigned jb = best.lidx - fb * static_cast<unsigned>(fa.D);
                const unsigned long long flat =
                    ((c_glob * fa.F + fb) * fa.R_total + static_cast<unsigned long long>(r_glob)) * fa.D + jb;
                peak_publish(fa.slots + r_local, best.re, best.im, flat);
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_BN));
    }
}

inline size_t tc2_smem_bytes(int terms) {
    const size_t stages = terms == 3 ? static_cast<size_t>(tc2_stages<3>()) * tc2_stage_bytes<3>()
                                     : static_cast<size_t>(tc2_stages<1>()) * tc2_stage_bytes<1>();
    return 1024 + stages + 8 * (2 * 6 + 4) + 16;
}

// H_f(m) = exp(+j 4pi/lambda * kappa * sum_axes val * t^ord) for every fine
// cell f (mixed radix over the fine axes, last fastest), phase in FP64 cycles.
__global__ void build_htab_kernel(TcArgs a, float2* htab) {
    const size_t total = static_cast<size_t>(a.f.F) * a.M;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(i % a.M);
        long long rem = static_cast<long long>(i / a.M);
        const double t = static_cast<double>(m + 1) * a.inv_prf;
        double cyc = 0.0;
        for (int ax = a.nfa - 1; ax >= 0; --ax) {
            const int idx = static_cast<int>(rem % a.fcount[ax]);
            rem /= a.fcount[ax];
            double tp = 1.0;
            for (int p = 0; p < a.ford[ax]; ++p) tp *= t;
            cyc += a.coef_cycles * (a.fstart[ax] + a.fstep[ax] * idx) * tp;
        }
        const double fr = cyc - rint(cyc);
        float s, c;
        sincospif(static_cast<float>(2.0 * fr), &s, &c);
        htab[i] = make_float2(c, s);
    }
}

// Max |y|^2 over the coarse-stage input (for the fp16 prescale).
__global__ void cube_maxabs_kernel(const float2* __restrict__ y, size_t n, unsigned* maxbits) {
    float m = 0.f;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        m = fmaxf(m, mag2f(y[i].x, y[i].y));
    unsigned u = __float_as_uint(m);
    u = __reduce_max_sync(0xffffffffu, u);
    if ((threadIdx.x & 31) == 0) atomicMax(maxbits, u);
}

// ------------------------------------------------------------- host -------
inline int tc_terms_for(int fine_path) { return fine_path == 3 /* LTCI_FINE_TC_FAST */ ? 1 : 3; }

inline bool tc_fine_selected(int fine_path, int M, int D, bool keep_dense) {
    (void)D;
    (void)keep_dense;
    if (fine_path == 2 || fine_path == 3) {
        if (M < 32) throw std::invalid_argument("ltci_cuda: tcgen05 fine path needs M >= 32");
        return true;
    }
    if (fine_path == 1) return false;  // explicit CUDA-core FFT path
    // AUTO (by measurement): M = 256..1024 runs the CUDA-core
    // FFT path with TMEM-resident rows (C1: 222 vs 246 ms tensor 3-term; C4:
    // 8.7 vs 12.3 ms per CPI; C0: 0.56 vs 0.69 ms; C3 KT, D = M: the dense
    // form is ~8x the work); M = 2048 likewise for a narrow window; below 256 the
    // 3-term (FP32-class) tensor path for a narrow Doppler window, else FFT.
    if (M >= 256 && M <= 1024) return false;
    if (M == 2048) {
        // CUDA-core FFT (radix-2 split onto two 1024-point halves) when the
        // Doppler window fits its pruned second pass (symmetric window of D
        // bins: at most 6 32-bin blocks per side of each half axis)
        const int keep = (D - 1) / 2;
        const int nbp = (keep / 2) / 32 + 1, nbn = 32 - ((M - keep - 1) / 2) / 32;
        return std::max(nbp, nbn) > 6;
    }
    if (keep_dense) return M > 1024;
    return M > 1024 || (M >= 64 && (D <= 160 || 2 * D <= M));
}

inline size_t tc_smem_bytes(int terms, int M) {
    const size_t stages = terms == 3 ? static_cast<size_t>(tc_stages<3>()) * tc_stage_bytes<3>()
                                     : static_cast<size_t>(tc_stages<1>()) * tc_stage_bytes<1>();
    (void)M;
    return 1024 + stages + 8 * (2 * 4 + 4) + 16;
}

}  // namespace ltcib
