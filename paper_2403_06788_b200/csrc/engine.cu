// engine.cu -- host plan, device engine and C-ABI of the B200 dual-scale
// cascade (include/ltci_cuda.h).  One translation unit: the kernels live in
// coarse.cuh (K1 coarse RM "gather", K4 keystone) and fine_fft.cuh (K2b fine
// DFM stage + fused K3 reduction); fine_tc.cuh adds the tcgen05 K2a path.
//
// Host-side plan mirrors run_dual_scale / ds_grft / ds_kt_mfp control flow
// (reference proj/src/detectors.cpp:337-481): coarse cells are enumerated
// mixed-radix over the map's coarse axes (last fastest), fine cells over the
// fine axes, the flat cell index is ((c*F + f)*R + r)*D + jj, counters follow
// predict_counters (proj/src/bench.cpp:180-189).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cuda.h>

#include "../../include/ltci_cuda.h"
#include "coarse.cuh"
#include "cube_io.hpp"
#include "fine_fft.cuh"
#include "fine_tc.cuh"
#include "fd_grft.cuh"
#include "td_grft.cuh"
#include "range_fft.cuh"
#include "fine_launch.hpp"
#include "gather_launch.hpp"
#include "launch_util.hpp"

using namespace ltcib;

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kC = 3.0e8;  // kSpeedOfLight, proj/include/ltci/common.hpp:12

thread_local std::string g_err;

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            fail(e_ == cudaErrorMemoryAllocation ? LTCI_BAD_ALLOC : LTCI_RUNTIME_ERROR,     \
                 std::string(#call) + ": " + cudaGetErrorString(e_));                       \
    } while (0)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LTCI_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const ltcib::CubeError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_err = std::string("allocation failed: ") + e.what();
        return LTCI_BAD_ALLOC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LTCI_RUNTIME_ERROR;
    }
}

bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }

double lambda_of(const ltci_radar& r) { return kC / r.fc; }
double va_of(const ltci_radar& r) { return lambda_of(r) * r.PRF / 2.0; }
double dR_of(const ltci_radar& r) { return kC / (2.0 * r.fs); }

// RadarParams::validate (proj/src/radar_params.cpp:30-45)
void validate_radar(const ltci_radar& p) {
    if (!(p.fc > 0) || !(p.fs > 0) || !(p.Br > 0) || !(p.PRF > 0) || p.M <= 0 || p.K <= 0)
        fail(LTCI_INVALID_ARGUMENT, "RadarParams: fc, fs, Br, PRF, M, K must be positive");
    if (!is_pow2(p.M) || !is_pow2(p.K))
        fail(LTCI_INVALID_ARGUMENT, "RadarParams: M and K must be powers of two");
}

// check_same_params (proj/src/detectors.cpp:52-55)
void check_same_params(const ltci_radar& a, const ltci_radar& b) {
    if (a.K != b.K || a.M != b.M || a.fc != b.fc || a.fs != b.fs || a.PRF != b.PRF)
        fail(LTCI_INVALID_ARGUMENT, "detector: cube and search space use different radar parameters");
}

// ---------------------------------------------------------------- plan ----

struct Plan {
    ltci_radar rp{};
    int variant = 0;
    int P = 0;
    std::vector<ltci_grid> coarse_axes;  // map order, last fastest
    int q_min = 0, q_count = 1;          // KT folding axis (slowest)
    unsigned long long coarse_cells = 1;
    std::vector<ltci_grid> fine_axes;
    std::vector<int> fine_orders;        // motion order of each fine axis
    unsigned long long fine_cells = 1;
    int n_outer = 1, n_inner = 1;
    int n_split = 1, chunk = 1;           // inner fine axis split across CTAs (small grids)
    int R_total = 0, roi_first = 0;
    int row_begin = 0, row_end = 0, R_slice = 0;
    int D = 0, dop_first = 0;
    double kappa = 1.0;
    double retain = 0.0;
    bool keep_dense = false;
    int taps = 8;
    int fine_path = LTCI_FINE_AUTO;
    std::vector<double> cparams;          // [coarse][4]
    std::vector<float2> h0, hstep;        // fine chirp tables
    std::vector<ltci_axis> axes;
    unsigned long long counters[4] = {0, 0, 0, 0};
};

// exp(+j 4pi/lambda * x) with the phase reduced in FP64 cycles
float2 phase_lambda(double x, double lambda) {
    const double cyc = 2.0 * x / lambda;
    const double fr = cyc - std::nearbyint(cyc);
    return make_float2(static_cast<float>(std::cos(2.0 * kPi * fr)), static_cast<float>(std::sin(2.0 * kPi * fr)));
}

void build_fine_tables(Plan& pl) {
    const int M = pl.rp.M;
    const double lam = lambda_of(pl.rp);
    const int nf = static_cast<int>(pl.fine_axes.size());
    pl.n_inner = nf > 0 ? pl.fine_axes[nf - 1].count : 1;
    pl.n_outer = 1;
    for (int i = 0; i + 1 < nf; ++i) pl.n_outer *= pl.fine_axes[i].count;
    pl.n_split = 1;
    pl.chunk = pl.n_inner;
    // Small problems (C0: 11 coarse cells x 512 rows = 1 408 warps of the
    // M = 256 TMEM kernel, under one wave of 148 SMs x 16 warps) split the
    // inner fine axis across CTAs: chunk sp starts from its own FP64 seed.
    if (nf > 0 && M >= 256 && M <= 1024 && !tc_fine_selected(pl.fine_path, M, pl.D, pl.keep_dense) &&
        !std::getenv("LTCI_FINE_NOSPLIT")) {
        // global sizes only (R_total, not the slice): every shard picks the same split, so
        // range-cell shards still reproduce the 1-GPU map bit for bit
        const double warps = static_cast<double>(pl.coarse_cells) * pl.R_total * M / 1024.0;
        const double want = 148.0 * 16.0 * 3.0;
        int ns = 1;
        if (warps < want) {
            // under ~3 waves: pick the split with the smallest wave-quantised makespan,
            // waves x (chunk + 2) fine cells (2 ~ the per-CTA row load and seeding);
            // 8-warp CTAs of 8 x 32/G rows, 2 per SM (fine_fft_tm_kernel launch bounds)
            const long long rows_per_cta = 8LL * (32 / (M / 32));
            const long long ctas = (static_cast<long long>(pl.coarse_cells) * pl.R_total + rows_per_cta - 1) /
                                   rows_per_cta;
            const long long slots = 148LL * 2;
            long long best = -1;
            for (int cand = 1; cand <= std::max(1, pl.n_inner / 16); ++cand) {
                const int ch = (pl.n_inner + cand - 1) / cand;
                const int nsp = (pl.n_inner + ch - 1) / ch;
                const long long cost = (ctas * nsp + slots - 1) / slots * (ch + 2);
                if (best < 0 || cost < best) {
                    best = cost;
                    ns = cand;
                }
            }
        }
        if (const char* env = std::getenv("LTCI_FINE_NSPLIT")) ns = std::max(1, std::atoi(env));  // A/B only
        if (ns > 1) {
            pl.chunk = (pl.n_inner + ns - 1) / ns;
            pl.n_split = (pl.n_inner + pl.chunk - 1) / pl.chunk;
        }
    }
    pl.h0.assign(static_cast<size_t>(pl.n_outer) * pl.n_split * M, make_float2(1.f, 0.f));
    pl.hstep.assign(M, make_float2(1.f, 0.f));
    if (nf == 0) return;
    for (int outer = 0; outer < pl.n_outer * pl.n_split; ++outer) {
        const int sp = outer % pl.n_split;
        // decode outer over fine axes 0..nf-2 (last fastest)
        std::vector<int> fi(nf, 0);
        int rem = outer / pl.n_split;
        for (int i = nf - 2; i >= 0; --i) {
            fi[i] = rem % pl.fine_axes[i].count;
            rem /= pl.fine_axes[i].count;
        }
        for (int m = 0; m < M; ++m) {
            const double t = static_cast<double>(m + 1) / pl.rp.PRF;
            double s = 0.0;
            for (int i = 0; i < nf; ++i) {
                const double val = i + 1 < nf ? pl.fine_axes[i].start + pl.fine_axes[i].step * fi[i]
                                              : pl.fine_axes[i].start + pl.fine_axes[i].step * (sp * pl.chunk);
                s += pl.kappa * val * std::pow(t, pl.fine_orders[i]);
            }
            pl.h0[static_cast<size_t>(outer) * M + m] = phase_lambda(s, lam);
        }
    }
    for (int m = 0; m < M; ++m) {
        const double t = static_cast<double>(m + 1) / pl.rp.PRF;
        pl.hstep[m] = phase_lambda(pl.kappa * pl.fine_axes[nf - 1].step * std::pow(t, pl.fine_orders[nf - 1]), lam);
    }
}

void set_slice(Plan& pl, int row_begin, int row_end) {
    if (row_end < 0) row_end = pl.R_total;
    if (row_begin < 0 || row_end > pl.R_total || row_begin >= row_end)
        fail(LTCI_INVALID_ARGUMENT, "engine: empty or out-of-range row slice");
    pl.row_begin = row_begin;
    pl.row_end = row_end;
    pl.R_slice = row_end - row_begin;
}

void check_roi(const ltci_dual_space& s) {
    const int count = s.roi_last - s.roi_first + 1;
    // gft's check (proj/src/transforms.cpp:183-184)
    if (count <= 0 || s.roi_first < 0 || s.roi_last >= s.radar.K)
        fail(LTCI_INVALID_ARGUMENT, "gft: empty or out-of-range roi");
}

void check_grids(const ltci_dual_space& s) {
    if (s.order < 1 || s.order > LTCI_MAX_ORDER)
        fail(LTCI_INVALID_ARGUMENT, "dual-scale space: order must be in 1..4");
    for (int p = 0; p < s.order; ++p)
        if (s.coarse[p].count < 1 || s.fine[p].count < 1)
            fail(LTCI_INVALID_ARGUMENT, "dual-scale space: empty grid");
}

void check_supported(const ltci_radar& r, int fine_path = LTCI_FINE_AUTO) {
    // CUDA-core FFT path: M in [4, 2048] (M = 2048 for Doppler-windowed
    // searches, checked at launch); tcgen05 path: M in [32, 2048]
    const bool tc = fine_path == LTCI_FINE_TC_DENSE || fine_path == LTCI_FINE_TC_FAST;
    if (r.M < 4 || r.M > 2048 || (tc && r.M < 32))
        fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: pulse count M must be a power of two in [4, 2048] "
                                    "(CUDA-core path) or [32, 2048] (tcgen05 path)");
    if (r.K < 16 || r.K > 8192)
        fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: frequency bins K must be a power of two in [16, 8192]");
}

Plan make_plan(const ltci_radar& cube_params, const ltci_dual_space& s, const ltci_ambiguity* amb,
               int variant, const ltci_options* opt, int row_begin, int row_end) {
    Plan pl;
    validate_radar(cube_params);
    check_same_params(cube_params, s.radar);
    pl.rp = cube_params;
    pl.variant = variant;
    pl.P = s.order;
    if (variant == LTCI_VARIANT_KTMFP && s.order != 2)
        fail(LTCI_INVALID_ARGUMENT, "ds_kt_mfp: needs a P = 2 search space");
    if (variant == LTCI_VARIANT_KTMFP && !amb) fail(LTCI_INVALID_ARGUMENT, "ds_kt_mfp: ambiguity space required");
    check_grids(s);
    check_roi(s);
    check_supported(cube_params, opt ? opt->fine_path : LTCI_FINE_AUTO);
    const int M = pl.rp.M;
    pl.kappa = s.kappa;
    pl.R_total = s.roi_last - s.roi_first + 1;
    pl.roi_first = s.roi_first;
    set_slice(pl, row_begin, row_end);
    if (opt) {
        pl.retain = opt->retain_threshold;
        pl.keep_dense = opt->keep_dense != 0;
        pl.taps = opt->keystone_taps;
        pl.fine_path = opt->fine_path;
    }

    if (variant == LTCI_VARIANT_GRFT) {
        // ds_grft: Doppler window (proj/src/detectors.cpp:420-432)
        const double dop_bin = va_of(pl.rp) / M;
        int keep = static_cast<int>(std::ceil(s.kappa * s.rm_step[0] / 2.0 / dop_bin - 1e-9));
        keep = std::min(keep, M / 2 - 1);
        if (keep < 0) fail(LTCI_INVALID_ARGUMENT, "ds_grft: empty Doppler window");
        pl.dop_first = M / 2 - keep;
        pl.D = 2 * keep + 1;
        for (int p = 0; p < s.order; ++p) pl.coarse_axes.push_back(s.coarse[p]);
        for (int p = 2; p <= s.order; ++p) {
            pl.fine_axes.push_back(s.fine[p - 1]);
            pl.fine_orders.push_back(p);
        }
        for (int p = 1; p <= s.order; ++p) pl.axes.push_back({LTCI_AXIS_COARSE, p, s.coarse[p - 1].count});
        for (int p = 2; p <= s.order; ++p) pl.axes.push_back({LTCI_AXIS_FINE, p, s.fine[p - 1].count});
        pl.axes.push_back({LTCI_AXIS_RANGE, 0, pl.R_total});
        pl.axes.push_back({LTCI_AXIS_DOPPLER, 0, pl.D});
    } else {
        if (pl.taps < 2) fail(LTCI_INVALID_ARGUMENT, "keystone: need at least 2 taps");
        pl.dop_first = 0;
        pl.D = M;
        pl.q_min = amb->q_min;
        pl.q_count = amb->q_max - amb->q_min + 1;
        if (pl.q_count < 1) fail(LTCI_INVALID_ARGUMENT, "ds_kt_mfp: empty ambiguity space");
        pl.coarse_axes.push_back(s.coarse[1]);
        pl.fine_axes.push_back(s.fine[1]);
        pl.fine_orders.push_back(2);
        pl.axes.push_back({LTCI_AXIS_FOLDING, 0, pl.q_count});
        pl.axes.push_back({LTCI_AXIS_COARSE, 2, s.coarse[1].count});
        pl.axes.push_back({LTCI_AXIS_FINE, 2, s.fine[1].count});
        pl.axes.push_back({LTCI_AXIS_RANGE, 0, pl.R_total});
        pl.axes.push_back({LTCI_AXIS_DOPPLER, 0, M});
    }
    pl.coarse_cells = 1;
    for (const ltci_grid& g : pl.coarse_axes) pl.coarse_cells *= static_cast<unsigned long long>(g.count);
    if (variant == LTCI_VARIANT_KTMFP) pl.coarse_cells *= static_cast<unsigned long long>(pl.q_count);
    pl.fine_cells = 1;
    for (const ltci_grid& g : pl.fine_axes) pl.fine_cells *= static_cast<unsigned long long>(g.count);
    if (pl.fine_cells * static_cast<unsigned long long>(pl.D) >= 0xffffffffull)
        fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: fine cells x Doppler bins must fit in 32 bits");

    // per-coarse-cell parameters (decode exactly as run_dual_scale, detectors.cpp:360-374)
    pl.cparams.assign(pl.coarse_cells * 4, 0.0);
    const size_t na = pl.coarse_axes.size();
    for (unsigned long long cidx = 0; cidx < pl.coarse_cells; ++cidx) {
        unsigned long long rem = cidx;
        std::vector<int> ci(na);
        for (size_t i = na; i-- > 0;) {
            ci[i] = static_cast<int>(rem % static_cast<unsigned long long>(pl.coarse_axes[i].count));
            rem /= static_cast<unsigned long long>(pl.coarse_axes[i].count);
        }
        double* cp = &pl.cparams[cidx * 4];
        if (variant == LTCI_VARIANT_KTMFP) {
            cp[0] = static_cast<double>(pl.q_min + static_cast<int>(rem));
            cp[1] = pl.coarse_axes[0].start + pl.coarse_axes[0].step * ci[0];
        } else {
            for (size_t i = 0; i < na; ++i) cp[i] = pl.coarse_axes[i].start + pl.coarse_axes[i].step * ci[i];
        }
    }
    build_fine_tables(pl);

    // predict_counters (proj/src/bench.cpp:180-189)
    const unsigned long long Mu = static_cast<unsigned long long>(M);
    const unsigned long long Nt = static_cast<unsigned long long>(pl.R_total);
    if (variant == LTCI_VARIANT_GRFT) {
        pl.counters[2] = pl.coarse_cells * Mu;
        pl.counters[1] = pl.coarse_cells * pl.fine_cells * Nt;
        pl.counters[3] = pl.coarse_cells * pl.fine_cells * Nt;
    } else {
        pl.counters[0] = 1;
        pl.counters[2] = pl.coarse_cells * Mu;
        pl.counters[1] = pl.coarse_cells * pl.fine_cells * Nt;
        pl.counters[3] = pl.coarse_cells * pl.fine_cells * Nt;
    }
    return pl;
}

// ----------------------------------------------------------- dispatch -----

void radix_plan(int K, int* radix, int* npass) {
    int n = 0, rem = K;
    while (rem >= 16) {
        radix[n++] = 16;
        rem /= 16;
    }
    if (rem > 1) radix[n++] = rem;
    *npass = n;
}

int coarse_pg(int K, int M) { return coarse_pg_for(K, M); }

// K4 launch: the tiled kernel for 2..16 taps (HALF = taps / 2 <= 8), the
// per-element kernel beyond
void launch_keystone(const KeystoneArgs& ka, cudaStream_t st) {
    const int half = ka.taps / 2;
    const dim3 grid((ka.K + kKtRows - 1) / kKtRows, (ka.M + kKtTile - 1) / kKtTile);
    switch (half) {
        case 1: keystone_tiled_kernel<1><<<grid, kKtThreads, 0, st>>>(ka); break;
        case 2: keystone_tiled_kernel<2><<<grid, kKtThreads, 0, st>>>(ka); break;
        case 3: keystone_tiled_kernel<3><<<grid, kKtThreads, 0, st>>>(ka); break;
        case 4: keystone_tiled_kernel<4><<<grid, kKtThreads, 0, st>>>(ka); break;
        case 5: keystone_tiled_kernel<5><<<grid, kKtThreads, 0, st>>>(ka); break;
        case 6: keystone_tiled_kernel<6><<<grid, kKtThreads, 0, st>>>(ka); break;
        case 7: keystone_tiled_kernel<7><<<grid, kKtThreads, 0, st>>>(ka); break;
        case 8: keystone_tiled_kernel<8><<<grid, kKtThreads, 0, st>>>(ka); break;
        default: {
            const size_t total = static_cast<size_t>(ka.K) * ka.M;
            keystone_kernel<<<static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16)), 256, 0, st>>>(ka);
        }
    }
    CK(cudaGetLastError());
}

__global__ void module_anchor_kernel() {}

// The runtime loads kernels lazily, on their first launch, so module-loading
// time would land in whichever detector call first needs an instantiation
// (a latency spike inside a timed or real-time call).  The first engine on a
// device therefore loads every function of this module up front through the
// driver's module enumeration; best effort: any failure leaves lazy loading.
void preload_module() {
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(mu);
    if (!done.insert(dev).second) return;
    using GetModule = CUresult (*)(CUmodule*, CUfunction);
    using Count = CUresult (*)(unsigned int*, CUmodule);
    using Enumerate = CUresult (*)(CUfunction*, unsigned int, CUmodule);
    using Load = CUresult (*)(CUfunction);
    void *p_mod = nullptr, *p_cnt = nullptr, *p_enum = nullptr, *p_load = nullptr;
    if (cudaGetDriverEntryPoint("cuFuncGetModule", &p_mod, cudaEnableDefault) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuModuleGetFunctionCount", &p_cnt, cudaEnableDefault) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuModuleEnumerateFunctions", &p_enum, cudaEnableDefault) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuFuncLoad", &p_load, cudaEnableDefault) != cudaSuccess || !p_mod || !p_cnt ||
        !p_enum || !p_load) {
        cudaGetLastError();
        return;
    }
    // this translation unit's module and the fine-kernel one (fine_launch.cu)
    for (const void* sym : {reinterpret_cast<const void*>(module_anchor_kernel), ltcib::fine_module_anchor(),
                            ltcib::gather_module_anchor()}) {
        cudaFunction_t anchor = nullptr;
        if (cudaGetFuncBySymbol(&anchor, sym) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        CUmodule mod = nullptr;
        unsigned int n = 0;
        if (reinterpret_cast<GetModule>(p_mod)(&mod, reinterpret_cast<CUfunction>(anchor)) != CUDA_SUCCESS ||
            reinterpret_cast<Count>(p_cnt)(&n, mod) != CUDA_SUCCESS || n == 0)
            continue;
        std::vector<CUfunction> fns(n);
        if (reinterpret_cast<Enumerate>(p_enum)(fns.data(), n, mod) != CUDA_SUCCESS) continue;
        for (CUfunction f : fns) reinterpret_cast<Load>(p_load)(f);
    }
}

template <int K, int OUT16>
void launch_coarse_k(const CoarseArgs& a0, cudaStream_t st) {
    auto kern = coarse_rm_kernel<K, OUT16>;
    CoarseArgs a = a0;
    static const bool fixed_pg = std::getenv("LTCI_COARSE_FIXED_PG") != nullptr;  // A/B
    a.pg = fixed_pg ? coarse_pg_for(K, a.M, OUT16) : coarse_pg_launch(K, a.M, OUT16, a.c_count);
    const size_t smem = coarse_smem_bytes(K, a.M, OUT16, a.pg);
    ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(std::max<size_t>(smem, 160 * 1024)));
    dim3 grid(a.M / a.pg, a.c_count);
    kern<<<grid, coarse_threads<OUT16>(), smem, st>>>(a);
    CK(cudaGetLastError());
}

template <int OUT16>
void launch_coarse_out(const CoarseArgs& a, cudaStream_t st) {
    switch (a.K) {
        case 16: launch_coarse_k<16, OUT16>(a, st); break;
        case 32: launch_coarse_k<32, OUT16>(a, st); break;
        case 64: launch_coarse_k<64, OUT16>(a, st); break;
        case 128: launch_coarse_k<128, OUT16>(a, st); break;
        case 256: launch_coarse_k<256, OUT16>(a, st); break;
        case 512: launch_coarse_k<512, OUT16>(a, st); break;
        case 1024: launch_coarse_k<1024, OUT16>(a, st); break;
        case 2048: launch_coarse_k<2048, OUT16>(a, st); break;
        case 4096: launch_coarse_k<4096, OUT16>(a, st); break;
        case 8192: launch_coarse_k<8192, OUT16>(a, st); break;
        default: fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: unsupported K");
    }
}

void launch_coarse(const CoarseArgs& a, int /*pg*/, cudaStream_t st, bool out16 = false) {
    if (out16)
        launch_coarse_out<1>(a, st);
    else
        launch_coarse_out<0>(a, st);
}

// K0 range FFT launch (range-pulse -> freq-pulse, ltci::range_fft)
template <int K, int IN64>
void launch_range_fft_k(const void* in, float2* out, int M, cudaStream_t st) {
    auto kern = range_fft_kernel<K, IN64>;
    const size_t smem = range_fft_smem_bytes(K, M);
    ensure_smem_attr(reinterpret_cast<const void*>(kern), 96 * 1024);
    const int pg = range_fft_pg(K, M);
    range_fft_kernel<K, IN64><<<(M + pg - 1) / pg, kRangeFftThreads, smem, st>>>(in, out, M);
    CK(cudaGetLastError());
}

template <int IN64>
void launch_range_fft_in(const void* in, float2* out, int K, int M, cudaStream_t st) {
    switch (K) {
        case 16: launch_range_fft_k<16, IN64>(in, out, M, st); break;
        case 32: launch_range_fft_k<32, IN64>(in, out, M, st); break;
        case 64: launch_range_fft_k<64, IN64>(in, out, M, st); break;
        case 128: launch_range_fft_k<128, IN64>(in, out, M, st); break;
        case 256: launch_range_fft_k<256, IN64>(in, out, M, st); break;
        case 512: launch_range_fft_k<512, IN64>(in, out, M, st); break;
        case 1024: launch_range_fft_k<1024, IN64>(in, out, M, st); break;
        case 2048: launch_range_fft_k<2048, IN64>(in, out, M, st); break;
        case 4096: launch_range_fft_k<4096, IN64>(in, out, M, st); break;
        case 8192: launch_range_fft_k<8192, IN64>(in, out, M, st); break;
        default: fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: range_fft needs K a power of two in [16, 8192]");
    }
}

void launch_range_fft(const void* in, bool in64, float2* out, int K, int M, cudaStream_t st) {
    if (in64)
        launch_range_fft_in<1>(in, out, K, M, st);
    else
        launch_range_fft_in<0>(in, out, K, M, st);
}

// ---- tcgen05 fine path: TMA tensor maps over the fp16 X planes ----------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) fail(LTCI_RUNTIME_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// [rows][2M] fp16, box 64 (K) x 128 (rows), 128-byte swizzle (matches sw128_desc)
CUtensorMap make_x16_map(void* base, int M, unsigned long long rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * M), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * M) * 2};
    const cuuint32_t box[2] = {TC_BK, TC_BM};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(LTCI_RUNTIME_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

template <int TERMS>
void launch_tc2_terms(const TcArgs& a, const CUtensorMap& hi, const CUtensorMap& lo, cudaStream_t st) {
    auto kern = fine_tc2_kernel<TERMS>;
    const size_t smem = tc2_smem_bytes(TERMS);
    ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    const long long Q = static_cast<long long>(a.f.F) * a.f.D;
    const long long tiles = ((Q + TC_QT - 1) / TC_QT) * ((a.f.rows + 2 * TC2_BM - 1) / (2 * TC2_BM));
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int pairs = static_cast<int>(std::min<long long>(tiles, sms / 2));  // persistent CTA pairs
    kern<<<2 * pairs, TC_THREADS, smem, st>>>(a, hi, lo);
    CK(cudaGetLastError());
}

bool tc_pair_enabled() {
    const char* e = std::getenv("LTCI_TC_PAIR");
    return !(e && e[0] == '0');
}

template <int TERMS>
void launch_tc_terms(const TcArgs& a, const CUtensorMap& hi, const CUtensorMap& lo, cudaStream_t st) {
    if (tc_pair_enabled()) {
        launch_tc2_terms<TERMS>(a, hi, lo, st);
        return;
    }
    auto kern = fine_tc_kernel<TERMS>;
    const size_t smem = tc_smem_bytes(TERMS, a.M);
    if (smem > 227 * 1024) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: tcgen05 tiles exceed shared memory");
    ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    const long long Q = static_cast<long long>(a.f.F) * a.f.D;
    const long long tiles = ((Q + TC_QT - 1) / TC_QT) * ((a.f.rows + TC_BM - 1) / TC_BM);
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = static_cast<int>(std::min<long long>(tiles, sms));  // persistent: one CTA per SM
    kern<<<grid, TC_THREADS, smem, st>>>(a, hi, lo);
    CK(cudaGetLastError());
}

// --------------------------------------------------------------- engine ---

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void ensure(size_t count) {
        if (count <= n) return;
        release();
        CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
};

// grow-only pinned host buffer (mapped when asked: small results are written
// there by the device)
template <typename T>
struct HostBuf {
    T* p = nullptr;
    size_t n = 0;
    // portable: pinned (and, with cudaHostAllocMapped, mapped) for every device's
    // context, so one process may drive engines on several GPUs
    void ensure(size_t count, unsigned flags = cudaHostAllocDefault) {
        if (count <= n) return;
        release();
        CK(cudaHostAlloc(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T),
                         flags | cudaHostAllocPortable));
        n = count;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
    ~HostBuf() { release(); }
};

// Pinned staging for H2D of a caller's pageable host cube: one host memcpy
// into the block, then an async DMA (no driver-side pageable path).  The event
// guards reuse: a block is refilled only after its previous DMA completed.
struct Stager {
    HostBuf<double2> buf;
    cudaEvent_t ev = nullptr;
    ~Stager() {
        if (ev) cudaEventDestroy(ev);
    }
};

}  // namespace

void ltcib_set_last_error(const char* msg) { g_err = msg ? msg : ""; }

// K1g workspace (gather.cuh): the oversampled range profiles of the current
// cube, the deapodisation row scales (depend on K only) and the per-batch
// (cell, pulse) weights.
struct GatherStage {
    DevBuf<float2> U;
    DevBuf<float> deap;
    DevBuf<float4> W;
    DevBuf<double> tparams;
    int deap_K = 0;
    int tables = 0;
    unsigned long long cells_per_table = 1;
    // the weights depend on the plan only: kept for every coarse cell of the
    // plan when they fit 1 GiB (w_ready after the first run), else per batch
    bool w_whole = false, w_ready = false;
    size_t w_plane = 0;
    // q: the folding number of each table (KT), one zero for GRFT
    void init(int K, int M, const std::vector<double>& q, unsigned long long cpt, unsigned long long batch,
              unsigned long long plan_cells) {
        tables = static_cast<int>(q.size());
        cells_per_table = cpt;
        U.ensure(static_cast<size_t>(tables) * 2 * K * M);
        size_t cache_cap = 1ull << 30;  // LTCI_GATHER_WCACHE_MB overrides (0: weights per batch)
        if (const char* env = std::getenv("LTCI_GATHER_WCACHE_MB")) cache_cap = std::strtoull(env, nullptr, 10) << 20;
        w_whole = gather_weight_bytes(plan_cells, M) <= cache_cap;
        w_ready = false;
        w_plane = static_cast<size_t>(w_whole ? plan_cells : batch) * M;
        W.ensure(3 * w_plane);
        if (static_cast<size_t>(K) > deap.n) {
            deap.ensure(K);
            deap_K = 0;
        }
        std::vector<double> tp(static_cast<size_t>(tables) * 8, 0.0);
        for (int t = 0; t < tables; ++t) {
            tp[8 * t + 1] = q[t];       // even fine samples: delta = 0
            tp[8 * t + 4] = 0.5;        // odd fine samples: delta = 1/2
            tp[8 * t + 5] = q[t];
        }
        tparams.ensure(tp.size());
        CK(cudaMemcpy(tparams.p, tp.data(), tp.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    // tables of `base.cube` (base: the coarse stage's radar scalars); returns the kernels launched
    int build(const CoarseArgs& base, cudaStream_t st) {
        int n = 1;
        if (deap_K != base.K) {
            launch_gather_deap(deap.p, base.K, st);
            deap_K = base.K;
            ++n;
        }
        CoarseArgs ta = base;
        ta.cparams = tparams.p;
        ta.X = U.p;
        ta.c_begin = 0;
        ta.c_count = 2 * tables;
        ta.n_base = 0;
        ta.R_slice = base.K;
        ta.deap = deap.p;
        launch_gather_tables(ta, st);
        return n;
    }
    GatherArgs args(const CoarseArgs& base) const {
        GatherArgs g{};
        g.U = U.p;
        g.W = W.p;
        g.w_plane = w_plane;
        g.w_first = 0;
        g.cparams = base.cparams;
        g.X = base.X;
        g.cells_per_table = cells_per_table;
        g.K = base.K;
        g.M = base.M;
        g.P = base.P;
        g.variant = base.variant;
        g.n_base = base.n_base;
        g.R_slice = base.R_slice;
        g.inv_prf = base.inv_prf;
        g.inv_dR = base.inv_dR;
        g.two_over_lambda = base.two_over_lambda;
        g.Va = base.Va;
        return g;
    }
};

// LTCI_COARSE = transform | gather forces the coarse kernel (A/B and tests);
// otherwise K1g runs whenever the FP32 fine path follows, the shape fits and a
// table (two transforms per pulse) serves at least 16 coarse cells (measured:
// C3's 4 cells per folding number are faster through K1, 0.31 vs 0.44 ms).
bool gather_selected(int K, int M, bool use_tc, unsigned long long cells_per_table) {
    if (use_tc || !gather_supported(K, M)) return false;
    if (const char* env = std::getenv("LTCI_COARSE")) {
        if (!std::strcmp(env, "transform")) return false;
        if (!std::strcmp(env, "gather")) return true;
    }
    return cells_per_table >= 16;
}

struct ltci_engine {
    Plan pl;
    int device = 0;
    DevBuf<float2> cube_c64, cube_kt, X, h0, hstep, dense;
    DevBuf<double2> cube_f64;
    DevBuf<double> cparams;
    DevBuf<PeakSlot> slots;
    DevBuf<CandRec> cand;
    DevBuf<unsigned long long> cand_count;
    unsigned long long cand_cap = 0;
    unsigned long long batch = 0;  // coarse cells per X batch
    const float2* last_cube = nullptr;
    bool ran = false;
    bool timing = false;
    int64_t launches = 0;
    double fine_ms = 0, coarse_ms = 0, keystone_ms = 0;
    std::vector<cudaEvent_t> ev;
    // tcgen05 fine path
    bool use_tc = false;
    int tc_terms = 3;
    DevBuf<uint32_t> x16h, x16l;
    DevBuf<unsigned> maxbits;
    DevBuf<float2> htab;
    bool htab_ready = false;
    CUtensorMap tm_hi{}, tm_lo{};
    // interpolating coarse gather (K1g)
    bool use_gather = false;
    GatherStage gs;
    // coarse-cell slice searched by this engine (coarse-cell sharding across GPUs)
    unsigned long long c_lo = 0, c_hi = ~0ull;
    // candidate assembly on the device (radix sort by flat index + recentring)
    DevBuf<unsigned long long> ck0, ck1;
    DevBuf<float2> cv0, cv1;
    DevBuf<double2> cvals;
    DevBuf<unsigned char> csort_tmp;
    // cube-file wire path: two pinned staging blocks, reused across runs
    double* stage[2] = {nullptr, nullptr};
    size_t stage_doubles = 0;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    // small-result fast path (mapped) and pinned staging for dense maps
    HostBuf<unsigned char> small;
    HostBuf<float2> dense_h;
    Stager stager;
};

namespace {

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev != prev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// Bounded per-device pool of reusable objects (one-shot engines, fd_grft
// workspaces).  A call leases one (or makes one), returns it afterwards; at
// most LTCI_POOL_IDLE (default 2) idle objects per device are kept, the rest
// are destroyed on return, so N calling threads never pin N x the buffers.
template <typename T>
struct ObjectPool {
    std::mutex mu;
    std::vector<std::vector<std::unique_ptr<T>>> idle;  // [device]
    size_t cap = [] {
        const char* env = std::getenv("LTCI_POOL_IDLE");
        return env ? static_cast<size_t>(std::strtoull(env, nullptr, 10)) : size_t{2};
    }();
    std::unique_ptr<T> take(int device) {
        std::lock_guard<std::mutex> g(mu);
        if (static_cast<int>(idle.size()) <= device) idle.resize(device + 1);
        auto& v = idle[device];
        if (v.empty()) return std::make_unique<T>();
        std::unique_ptr<T> o = std::move(v.back());
        v.pop_back();
        return o;
    }
    void give(int device, std::unique_ptr<T> o) {
        {
            std::lock_guard<std::mutex> g(mu);
            auto& v = idle[device];
            if (v.size() < cap) {
                v.push_back(std::move(o));
                return;
            }
        }
        DeviceGuard dg(device);
        o.reset();  // frees the device buffers outside the lock
    }
    size_t idle_count(int device) {
        std::lock_guard<std::mutex> g(mu);
        return device < static_cast<int>(idle.size()) ? idle[device].size() : 0;
    }
};

template <typename T>
struct PoolLease {
    ObjectPool<T>& pool;
    int device;
    std::unique_ptr<T> obj;
    PoolLease(ObjectPool<T>& p, int dev) : pool(p), device(dev), obj(p.take(dev)) {}
    ~PoolLease() { pool.give(device, std::move(obj)); }
    T& operator*() { return *obj; }
};

ObjectPool<ltci_engine>& engine_pool() {
    static auto* p = new ObjectPool<ltci_engine>();  // leaked: no teardown after the CUDA runtime
    return *p;
}

void engine_init(ltci_engine* e) {
    const Plan& pl = e->pl;
    const int M = pl.rp.M;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        fail(LTCI_NO_DEVICE, "ltci_cuda: no CUDA device available");
    if (e->device < 0 || e->device >= ndev) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: bad device ordinal");
    DeviceGuard dg(e->device);
    preload_module();
    e->cparams.ensure(pl.cparams.size());
    CK(cudaMemcpy(e->cparams.p, pl.cparams.data(), pl.cparams.size() * sizeof(double), cudaMemcpyHostToDevice));
    e->h0.ensure(pl.h0.size());
    CK(cudaMemcpy(e->h0.p, pl.h0.data(), pl.h0.size() * sizeof(float2), cudaMemcpyHostToDevice));
    e->hstep.ensure(pl.hstep.size());
    CK(cudaMemcpy(e->hstep.p, pl.hstep.data(), pl.hstep.size() * sizeof(float2), cudaMemcpyHostToDevice));
    e->slots.ensure(pl.R_slice);
    e->cand_count.ensure(1);
    // X batch: bounded device footprint (default 6 GiB -- all of C1 in one batch -- LTCI_X_BUDGET_MB overrides)
    size_t budget = 6ull << 30;
    if (const char* env = std::getenv("LTCI_X_BUDGET_MB")) budget = std::strtoull(env, nullptr, 10) << 20;
    const size_t per_coarse = static_cast<size_t>(pl.R_slice) * M * sizeof(float2);
    e->batch = std::max<unsigned long long>(1, std::min<unsigned long long>(pl.coarse_cells, budget / per_coarse));
    // the fine kernel indexes rows with int; the coarse kernels put the batch's cells on grid.y
    e->batch = std::min<unsigned long long>(e->batch, (1ull << 30) / std::max(1, pl.R_slice));
    e->batch = std::min<unsigned long long>(e->batch, 65535);
    e->use_tc = tc_fine_selected(pl.fine_path, M, pl.D, pl.keep_dense);
    e->tc_terms = tc_terms_for(pl.fine_path);
    if (!e->use_tc && M == 2048) {
        const int dlo = pl.dop_first - M / 2;
        if (tm2k_nb(dlo + pl.D - 1, M + dlo) == 0)
            fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: CUDA-core fine path at M = 2048 needs a Doppler window of "
                                        "at most 12 x 64 bins (use the tcgen05 path)");
    }
    if (e->use_tc) {
        const size_t words = e->batch * static_cast<size_t>(pl.R_slice) * M;  // one half2 per complex sample
        e->x16h.ensure(words);
        e->x16l.ensure(words);
        e->maxbits.ensure(1);
        const unsigned long long rows_cap = e->batch * static_cast<unsigned long long>(pl.R_slice);
        e->tm_hi = make_x16_map(e->x16h.p, M, rows_cap);
        e->tm_lo = make_x16_map(e->x16l.p, M, rows_cap);
    } else {
        e->X.ensure(e->batch * per_coarse / sizeof(float2));
    }
    {
        const bool kt = pl.variant == LTCI_VARIANT_KTMFP;
        const unsigned long long cpt = kt ? pl.coarse_cells / static_cast<unsigned long long>(pl.q_count) : pl.coarse_cells;
        e->use_gather = gather_selected(pl.rp.K, M, e->use_tc, cpt);
        if (e->use_gather) {
            std::vector<double> q(kt ? pl.q_count : 1, 0.0);
            if (kt)
                for (int i = 0; i < pl.q_count; ++i) q[i] = static_cast<double>(pl.q_min + i);
            e->gs.init(pl.rp.K, M, q, cpt, e->batch, pl.coarse_cells);
        }
    }
    const unsigned long long H = pl.coarse_cells * pl.fine_cells * pl.R_slice * pl.D;
    unsigned long long cap0 = 1ull << 22;  // initial candidate buffer (grown by the overflow re-run)
    if (const char* env = std::getenv("LTCI_CAND_CAP")) cap0 = std::strtoull(env, nullptr, 10);
    e->cand_cap = std::max<unsigned long long>(1, std::min<unsigned long long>(H, cap0));
    e->cand.ensure(e->cand_cap);
    if (pl.keep_dense) {
        const unsigned long long cells = pl.coarse_cells * pl.fine_cells * pl.R_total * pl.D;
        e->dense.ensure(cells);
    }
    if (pl.variant == LTCI_VARIANT_KTMFP) e->cube_kt.ensure(static_cast<size_t>(pl.rp.K) * M);
}

__global__ void init_slots_kernel(PeakSlot* __restrict__ slots, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        slots[i] = PeakSlot{0.f, 0.f, ~0ull};
}

void run_device_impl(ltci_engine* e, const float2* d_cube, cudaStream_t st) {
    const Plan& pl = e->pl;
    DeviceGuard dg(e->device);
    const int K = pl.rp.K, M = pl.rp.M;
    e->launches = 0;
    const bool tm = e->timing;
    if (tm && e->ev.empty()) {
        e->ev.resize(64);
        for (auto& x : e->ev) CK(cudaEventCreate(&x));
    }
    int evi = 0;
    std::vector<std::pair<int, int>> fine_ev, coarse_ev;
    std::pair<int, int> kt_ev{-1, -1};

    CK(cudaMemsetAsync(e->cand_count.p, 0, sizeof(unsigned long long), st));
    // slots: re = im = 0, idx = ~0 (on the stream: run_device never blocks the host)
    init_slots_kernel<<<std::max(1, std::min(148, (pl.R_slice + 255) / 256)), 256, 0, st>>>(e->slots.p, pl.R_slice);
    CK(cudaGetLastError());
    if (pl.keep_dense)
        CK(cudaMemsetAsync(e->dense.p, 0,
                           static_cast<size_t>(pl.coarse_cells * pl.fine_cells * pl.R_total * pl.D) * sizeof(float2), st));

    const float2* input = d_cube;
    if (pl.variant == LTCI_VARIANT_KTMFP) {
        KeystoneArgs ka;
        ka.in = d_cube;
        ka.out = e->cube_kt.p;
        ka.K = K;
        ka.M = M;
        ka.taps = pl.taps;
        ka.fc = pl.rp.fc;
        ka.delta_f = pl.rp.delta_f;
        if (tm && evi + 2 <= static_cast<int>(e->ev.size())) {
            kt_ev = {evi, evi + 1};
            CK(cudaEventRecord(e->ev[evi], st));
        }
        launch_keystone(ka, st);
        ++e->launches;
        if (kt_ev.first >= 0) {
            CK(cudaEventRecord(e->ev[evi + 1], st));
            evi += 2;
        }
        input = e->cube_kt.p;
    }

    CoarseArgs ca{};
    ca.cube = input;
    ca.cparams = e->cparams.p;
    ca.X = e->X.p;
    ca.K = K;
    ca.M = M;
    ca.P = pl.P;
    ca.variant = pl.variant;
    ca.n_base = pl.roi_first + pl.row_begin;
    ca.R_slice = pl.R_slice;
    ca.inv_prf = 1.0 / pl.rp.PRF;
    ca.inv_dR = 1.0 / dR_of(pl.rp);
    ca.two_over_lambda = 2.0 / lambda_of(pl.rp);
    ca.Va = va_of(pl.rp);
    ca.kt_b = -(4.0 * kPi / kC) * pl.rp.delta_f * pl.rp.delta_f / pl.rp.fc;
    radix_plan(K, ca.radix, &ca.npass);
    const int pg = coarse_pg(K, M);

    FineArgs fa{};
    fa.X = e->X.p;
    fa.H0 = e->h0.p;
    fa.Hstep = e->hstep.p;
    fa.slots = e->slots.p;
    fa.cand = e->cand.p;
    fa.cand_count = e->cand_count.p;
    fa.dense = pl.keep_dense ? e->dense.p : nullptr;
    fa.cand_cap = e->cand_cap;
    fa.F = pl.fine_cells;
    fa.R_total = static_cast<unsigned long long>(pl.R_total);
    fa.R_slice = pl.R_slice;
    fa.row_begin = pl.row_begin;
    fa.D = pl.D;
    fa.dop_first = pl.dop_first;
    {
        const int dlo = pl.dop_first - M / 2, dhi = dlo + pl.D - 1;
        fa.kA = dhi;
        fa.kB = M + dlo;
    }
    fa.n_outer = pl.n_outer;
    fa.n_inner = pl.n_inner;
    fa.n_split = pl.n_split;
    fa.chunk = pl.chunk;
    {
        const double r2 = pl.retain * pl.retain;
        fa.retain2 = pl.retain < 0 ? -1.0f : static_cast<float>(r2);
    }

    const bool use_tc = e->use_tc;
    TcArgs ta{};
    if (use_tc) {
        ca.Xh = e->x16h.p;
        ca.Xl = e->x16l.p;
        ca.maxbits = e->maxbits.p;
        CK(cudaMemsetAsync(e->maxbits.p, 0, sizeof(unsigned), st));
        const size_t n = static_cast<size_t>(K) * M;
        cube_maxabs_kernel<<<static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 4)), 256, 0, st>>>(input, n,
                                                                                                        e->maxbits.p);
        CK(cudaGetLastError());
        ++e->launches;
        ta.f = fa;
        ta.M = M;
        ta.K = K;
        ta.nfa = static_cast<int>(pl.fine_axes.size());
        for (int i = 0; i < ta.nfa && i < 3; ++i) {
            ta.fcount[i] = pl.fine_axes[i].count;
            ta.fstart[i] = pl.fine_axes[i].start;
            ta.fstep[i] = pl.fine_axes[i].step;
            ta.ford[i] = pl.fine_orders[i];
        }
        ta.coef_cycles = 2.0 * pl.kappa / lambda_of(pl.rp);
        ta.inv_prf = 1.0 / pl.rp.PRF;
        ta.maxbits = e->maxbits.p;
        if (!e->htab_ready) {
            // H_f(m) for every fine cell, FP64 phases, built once per engine
            e->htab.ensure(static_cast<size_t>(pl.fine_cells) * M);
            const size_t total = static_cast<size_t>(pl.fine_cells) * M;
            build_htab_kernel<<<static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16)), 256, 0, st>>>(
                ta, e->htab.p);
            CK(cudaGetLastError());
            ++e->launches;
            e->htab_ready = true;
        }
        ta.htab = e->htab.p;
    }
    const unsigned long long c_end = std::min(e->c_hi, pl.coarse_cells);
    GatherArgs ga{};
    if (e->use_gather && e->c_lo < c_end) {
        // the oversampled profiles of this cube, once per run (counted in coarse_ms)
        int evt = -1;
        if (tm && evi + 2 <= static_cast<int>(e->ev.size())) {
            evt = evi;
            evi += 2;
            CK(cudaEventRecord(e->ev[evt], st));
        }
        e->launches += e->gs.build(ca, st);
        if (evt >= 0) {
            CK(cudaEventRecord(e->ev[evt + 1], st));
            coarse_ev.push_back({evt, evt + 1});
        }
        ga = e->gs.args(ca);
        if (e->gs.w_whole && !e->gs.w_ready) {
            ga.c_begin = 0;
            ga.c_count = static_cast<int>(pl.coarse_cells);
            launch_gather_weights(ga, st);
            ++e->launches;
            e->gs.w_ready = true;
        }
    }
    for (unsigned long long c0 = e->c_lo; c0 < c_end; c0 += e->batch) {
        const unsigned long long cc = std::min<unsigned long long>(e->batch, c_end - c0);
        ca.c_begin = c0;
        ca.c_count = static_cast<int>(cc);
        int evc = -1;
        if (tm && evi + 4 <= static_cast<int>(e->ev.size())) {
            evc = evi;
            evi += 4;
            CK(cudaEventRecord(e->ev[evc], st));
        }
        if (e->use_gather) {
            ga.c_begin = c0;
            ga.c_count = static_cast<int>(cc);
            if (!e->gs.w_whole) {
                ga.w_first = c0;
                launch_gather_weights(ga, st);
                ++e->launches;
            }
            launch_gather_cells(ga, st);
            ++e->launches;
        } else {
            launch_coarse(ca, pg, st, use_tc);
            ++e->launches;
        }
        if (evc >= 0) CK(cudaEventRecord(e->ev[evc + 1], st));
        fa.c_begin = c0;
        fa.rows = static_cast<int>(cc) * pl.R_slice;
        if (evc >= 0) CK(cudaEventRecord(e->ev[evc + 2], st));
        if (use_tc) {
            ta.f.c_begin = c0;
            ta.f.rows = fa.rows;
            if (e->tc_terms == 1)
                launch_tc_terms<1>(ta, e->tm_hi, e->tm_lo, st);
            else
                launch_tc_terms<3>(ta, e->tm_hi, e->tm_lo, st);
            ++e->launches;
        } else {
            if (pl.keep_dense)
                launch_fine_m(fa, M, true, st);
            else
                launch_fine_m(fa, M, false, st);
            ++e->launches;
        }
        if (evc >= 0) {
            CK(cudaEventRecord(e->ev[evc + 3], st));
            coarse_ev.push_back({evc, evc + 1});
            fine_ev.push_back({evc + 2, evc + 3});
        }
    }
    if (d_cube != e->cube_c64.p) {
        // The candidate-overflow re-run in assemble() must see this run's echo,
        // not whatever a caller-owned buffer holds by the time result() is
        // called (double-buffered CPI streams reuse it): keep a private copy,
        // queued behind the run so it costs no latency (~5 us at C1).
        const size_t n = static_cast<size_t>(K) * M;
        e->cube_c64.ensure(n);
        CK(cudaMemcpyAsync(e->cube_c64.p, d_cube, n * sizeof(float2), cudaMemcpyDeviceToDevice, st));
    }
    e->last_cube = e->cube_c64.p;
    e->ran = true;
    if (tm) {
        CK(cudaStreamSynchronize(st));
        float ms = 0;
        e->fine_ms = e->coarse_ms = e->keystone_ms = 0;
        for (auto& pr : fine_ev) {
            CK(cudaEventElapsedTime(&ms, e->ev[pr.first], e->ev[pr.second]));
            e->fine_ms += ms;
        }
        for (auto& pr : coarse_ev) {
            CK(cudaEventElapsedTime(&ms, e->ev[pr.first], e->ev[pr.second]));
            e->coarse_ms += ms;
        }
        if (kt_ev.first >= 0) {
            CK(cudaEventElapsedTime(&ms, e->ev[kt_ev.first], e->ev[kt_ev.second]));
            e->keystone_ms = ms;
        }
    }
}

// H2D of a host float64 cube: pinned (or registered) memory goes straight to
// the DMA engine; small pageable cubes (<= 8 MiB, the one-shot drop-in calls
// of Monte-Carlo loops) are staged through a pinned block; large pageable
// cubes go direct (the driver pipelines them).
void h2d_cube(double2* dst, const double* src, size_t n, Stager& sg, cudaStream_t st) {
    const size_t bytes = n * sizeof(double2);
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();  // unregistered pointers may leave an error behind on old runtimes
    if (pinned || bytes > (8u << 20)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    if (!sg.ev) CK(cudaEventCreateWithFlags(&sg.ev, cudaEventDisableTiming));
    CK(cudaEventSynchronize(sg.ev));  // the block's previous DMA is done
    sg.buf.ensure(n);
    std::memcpy(sg.buf.p, src, bytes);
    CK(cudaMemcpyAsync(dst, sg.buf.p, bytes, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(sg.ev, st));
}

void upload_host_cube(ltci_engine* e, const double* cube, cudaStream_t st) {
    const size_t n = static_cast<size_t>(e->pl.rp.K) * e->pl.rp.M;
    e->cube_f64.ensure(n);
    e->cube_c64.ensure(n);
    h2d_cube(e->cube_f64.p, cube, n, e->stager, st);
    const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 8));
    f64_to_c64_kernel<<<blocks, 256, 0, st>>>(e->cube_f64.p, e->cube_c64.p, n);
    CK(cudaGetLastError());
}

__global__ void cand_split_kernel(const CandRec* __restrict__ in, unsigned long long* __restrict__ keys,
                                  float2* __restrict__ vals, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const CandRec r = in[i];
        keys[i] = r.idx;
        vals[i] = make_float2(r.re, r.im);
    }
}

// the recentring twiddle of recenter() below, in FP64 on the device
__global__ void cand_recenter_kernel(const unsigned long long* __restrict__ keys, const float2* __restrict__ vals,
                                     double2* __restrict__ out, unsigned long long n, int D, int dop_first, int M) {
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int jj = static_cast<int>(keys[i] % static_cast<unsigned long long>(D));
        const int d = dop_first + jj - M / 2;
        double s, c;
        sincospi(2.0 * d / M, &s, &c);
        const double re = vals[i].x, im = vals[i].y;
        out[i] = make_double2(re * c - im * s, re * s + im * c);
    }
}

// exp(+j 2pi d / M) for the flat index's Doppler bin (RangeDopplerMap recentring,
// proj/src/transforms.cpp:197-212)
void recenter(const Plan& pl, unsigned long long idx, float re, float im, double* out) {
    const int jj = static_cast<int>(idx % static_cast<unsigned long long>(pl.D));
    const int d = pl.dop_first + jj - pl.rp.M / 2;
    const double ang = 2.0 * kPi * d / pl.rp.M;
    const double c = std::cos(ang), s = std::sin(ang);
    out[0] = re * c - im * s;
    out[1] = re * s + im * c;
}

void* xmalloc(size_t bytes) {
    if (bytes == 0) return nullptr;
    void* p = std::malloc(bytes);
    if (!p) throw std::bad_alloc();
    return p;
}

struct CandSortBufs {
    DevBuf<unsigned long long>& k0;
    DevBuf<unsigned long long>& k1;
    DevBuf<float2>& v0;
    DevBuf<float2>& v1;
    DevBuf<double2>& out;
    DevBuf<unsigned char>& tmp;
};

// Candidates: radix sort by flat index and recentre on the device (D = 1,
// dop_first = M/2 is the identity), then one D2H per array straight into the
// map (scales to 1e8+ retained cells).
void sort_candidates(const CandRec* d_cand, unsigned long long count, unsigned long long cells, int D,
                     int dop_first, int M, CandSortBufs& b, uint64_t* h_idx, double* h_val, cudaStream_t st) {
    b.k0.ensure(count);
    b.k1.ensure(count);
    b.v0.ensure(count);
    b.v1.ensure(count);
    b.out.ensure(count);
    const int blocks = static_cast<int>(std::min<unsigned long long>((count + 255) / 256, 148 * 8));
    cand_split_kernel<<<blocks, 256, 0, st>>>(d_cand, b.k0.p, b.v0.p, count);
    CK(cudaGetLastError());
    int end_bit = 1;
    while (end_bit < 64 && (cells >> end_bit) != 0) ++end_bit;
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, b.k0.p, b.k1.p, b.v0.p, b.v1.p, count, 0, end_bit, st));
    b.tmp.ensure(tmp);
    CK(cub::DeviceRadixSort::SortPairs(b.tmp.p, tmp, b.k0.p, b.k1.p, b.v0.p, b.v1.p, count, 0, end_bit, st));
    cand_recenter_kernel<<<blocks, 256, 0, st>>>(b.k1.p, b.v1.p, b.out.p, count, D, dop_first, M);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_idx, b.k1.p, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_val, b.out.p, count * sizeof(double2), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

// ---- small-result fast path --------------------------------------------------
// One kernel turns a run's reduced output into host-visible results: the
// retained-candidate count, the peak slots, and -- when at most kSmallCand
// cells were retained (the normal case at a sensible threshold) -- the
// candidates sorted by flat index (bitonic sort in shared memory) and
// recentred in FP64 with the same expression as cand_recenter_kernel, so the
// values are bit-identical whichever path produced them.  It writes straight
// into mapped pinned host memory, so a detector call needs one
// synchronisation instead of a D2H round trip per array plus the multi-kernel
// radix sort (which stays the path for larger candidate sets).
constexpr unsigned long long kSmallCand = 2048;  // 32 KB of static shared memory


// mapped result block: [u64 count, pad x7][n_slots PeakSlot][kSmallCand u64 idx][kSmallCand double2 val]
struct SmallLayout {
    size_t slots, idx, val, bytes;
    explicit SmallLayout(int n_slots) {
        slots = 64;
        idx = slots + static_cast<size_t>(n_slots) * sizeof(PeakSlot);
        val = idx + kSmallCand * sizeof(unsigned long long);
        bytes = val + kSmallCand * sizeof(double2);
    }
};

__global__ void __launch_bounds__(1024) small_result_kernel(const unsigned long long* __restrict__ count_p,
                                                            const CandRec* __restrict__ cand,
                                                            unsigned long long limit, const PeakSlot* __restrict__ slots,
                                                            int n_slots, int D, int dop_first, int M,
                                                            unsigned char* __restrict__ out, SmallLayout L) {
    __shared__ unsigned long long key[kSmallCand];
    __shared__ float2 val[kSmallCand];
    const int tid = threadIdx.x, nt = blockDim.x;
    const unsigned long long count = *count_p;
    auto* h_slots = reinterpret_cast<PeakSlot*>(out + L.slots);
    for (int r = tid; r < n_slots; r += nt) h_slots[r] = slots[r];
    if (tid == 0) reinterpret_cast<unsigned long long*>(out)[0] = count;
    if (count > limit || count == 0) return;  // host falls back (or nothing to sort)
    const int n = static_cast<int>(count);
    int N = 2;
    while (N < n) N <<= 1;
    for (int i = tid; i < N; i += nt) {
        if (i < n) {
            const CandRec c = cand[i];
            key[i] = c.idx;
            val[i] = make_float2(c.re, c.im);
        } else {
            key[i] = ~0ull;  // flat indices are < 2^64 - 1 and unique
        }
    }
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < N; i += nt) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const unsigned long long a = key[i], b = key[ixj];
                    if ((a > b) == up) {
                        key[i] = b;
                        key[ixj] = a;
                        const float2 t = val[i];
                        val[i] = val[ixj];
                        val[ixj] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
    auto* h_idx = reinterpret_cast<unsigned long long*>(out + L.idx);
    auto* h_val = reinterpret_cast<double2*>(out + L.val);
    for (int i = tid; i < n; i += nt) {
        const unsigned long long kk = key[i];
        const int jj = static_cast<int>(kk % static_cast<unsigned long long>(D));
        const int d = dop_first + jj - M / 2;
        double sn, cs;
        sincospi(2.0 * d / M, &sn, &cs);
        const double re = val[i].x, im = val[i].y;
        h_idx[i] = kk;
        h_val[i] = make_double2(re * cs - im * sn, re * sn + im * cs);
    }
}

// Enqueue the fast path into a (grow-only) mapped block; returns its host pointer.
unsigned char* enqueue_small_result(HostBuf<unsigned char>& buf, const unsigned long long* d_count,
                                    const CandRec* d_cand, unsigned long long cand_cap, const PeakSlot* d_slots,
                                    int n_slots, int D, int dop_first, int M, cudaStream_t st) {
    const SmallLayout L(n_slots);
    buf.ensure(L.bytes, cudaHostAllocMapped);
    unsigned char* dptr = nullptr;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), buf.p, 0));
    small_result_kernel<<<1, 1024, 0, st>>>(d_count, d_cand, std::min(kSmallCand, cand_cap), d_slots, n_slots, D,
                                           dop_first, M, dptr, L);
    CK(cudaGetLastError());
    return buf.p;
}

ltci_detection_map* assemble(ltci_engine* e, cudaStream_t st) {
    const Plan& pl = e->pl;
    DeviceGuard dg(e->device);
    // the count, the per-row peak slots, small candidate sets (sorted and
    // recentred) and the optional dense map come back behind one
    // synchronisation (re-fetched below in the rare re-run case)
    const SmallLayout L(pl.R_slice);
    const size_t nd = pl.keep_dense ? static_cast<size_t>(pl.coarse_cells * pl.fine_cells * pl.R_total * pl.D) : 0;
    unsigned char* hb = nullptr;
    unsigned long long count = 0;
    auto fetch = [&] {
        hb = enqueue_small_result(e->small, e->cand_count.p, e->cand.p, e->cand_cap, e->slots.p, pl.R_slice, pl.D,
                                  pl.dop_first, pl.rp.M, st);
        if (nd) {
            e->dense_h.ensure(nd);  // not the (grow-only) device buffer's size
            CK(cudaMemcpyAsync(e->dense_h.p, e->dense.p, nd * sizeof(float2), cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
        count = *reinterpret_cast<volatile unsigned long long*>(hb);
    };
    fetch();
    if (count > e->cand_cap) {
        // The reference would try to hold every retained cell in host memory
        // (24 B each); refuse what cannot fit rather than hang.
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        const double host_bytes = static_cast<double>(count) * 24.0;
        const double dev_bytes = static_cast<double>(count) * sizeof(CandRec);
        if (dev_bytes > 0.8 * static_cast<double>(free_b) || host_bytes > 64.0 * (1ull << 30))
            fail(LTCI_BAD_ALLOC, "ltci_cuda: " + std::to_string(count) +
                                     " retained cells exceed the result memory (raise retain_threshold)");
        e->cand.release();
        e->cand_cap = count;
        e->cand.ensure(count);
        run_device_impl(e, e->last_cube, st);
        fetch();
    }
    const PeakSlot* slots = reinterpret_cast<const PeakSlot*>(hb + L.slots);

    auto* out = static_cast<ltci_detection_map*>(std::calloc(1, sizeof(ltci_detection_map)));
    if (!out) throw std::bad_alloc();
    try {
        out->kind = pl.variant == LTCI_VARIANT_GRFT ? LTCI_DS_GRFT : LTCI_DS_KT_MFP;
        if (pl.axes.size() > LTCI_MAX_AXES) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: too many map axes");
        out->n_axes = static_cast<int32_t>(pl.axes.size());
        for (size_t i = 0; i < pl.axes.size(); ++i) out->axes[i] = pl.axes[i];
        for (int i = 0; i < 4; ++i) out->counters[i] = pl.counters[i];
        out->retain_threshold = pl.retain;
        out->doppler_first = pl.dop_first;

        // peak slots -> per-row peaks + global argmax
        out->n_rows = pl.R_slice;
        out->peak_index = static_cast<uint64_t*>(xmalloc(pl.R_slice * sizeof(uint64_t)));
        out->peak_value = static_cast<double*>(xmalloc(2 * pl.R_slice * sizeof(double)));
        int best = -1;
        for (int r = 0; r < pl.R_slice; ++r) {
            out->peak_index[r] = slots[r].idx;
            recenter(pl, slots[r].idx, slots[r].re, slots[r].im, out->peak_value + 2 * r);
            if (best < 0) {
                best = r;
                continue;
            }
            const float mb = mag2f(slots[best].re, slots[best].im);
            const float mr = mag2f(slots[r].re, slots[r].im);
            if (mr > mb || (mr == mb && slots[r].idx < slots[best].idx)) best = r;
        }
        out->argmax = slots[best].idx;
        out->argmax_value[0] = out->peak_value[2 * best];
        out->argmax_value[1] = out->peak_value[2 * best + 1];

        // candidates: radix sort by flat index and recentre on the device, then
        // one D2H per array straight into the map (scales to 1e8+ retained cells)
        out->n_candidates = count;
        out->cand_index = static_cast<uint64_t*>(xmalloc(count * sizeof(uint64_t)));
        out->cand_value = static_cast<double*>(xmalloc(2 * count * sizeof(double)));
        if (count && count <= std::min(kSmallCand, e->cand_cap)) {
            std::memcpy(out->cand_index, hb + L.idx, count * sizeof(uint64_t));
            std::memcpy(out->cand_value, hb + L.val, count * sizeof(double2));
        } else if (count) {
            const unsigned long long cells = static_cast<unsigned long long>(pl.coarse_cells) * pl.fine_cells *
                                             static_cast<unsigned long long>(pl.R_total) * pl.D;
            CandSortBufs b{e->ck0, e->ck1, e->cv0, e->cv1, e->cvals, e->csort_tmp};
            sort_candidates(e->cand.p, count, cells, pl.D, pl.dop_first, pl.rp.M, b, out->cand_index,
                            out->cand_value, st);
        }
        if (pl.keep_dense) {
            out->dense_stored = 1;
            out->dense_count = nd;
            out->dense = static_cast<double*>(xmalloc(2 * nd * sizeof(double)));
            const float2* dh = e->dense_h.p;
            for (size_t i = 0; i < nd; ++i) recenter(pl, i, dh[i].x, dh[i].y, out->dense + 2 * i);
        }
    } catch (...) {
        ltci_cuda_free_map(out);
        throw;
    }
    return out;
}

int detect(const double* cube, const ltci_radar* cp, const ltci_ambiguity* amb, const ltci_dual_space* s,
           const ltci_options* opt, int variant, ltci_detection_map** out) {
    return guarded([&] {
        if (!cube || !cp || !s || !out) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        const int device = opt ? opt->device : 0;
        if (device < 0) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: bad device ordinal");
        // One-shot calls lease an engine from a process-wide, per-device pool:
        // its device buffers only grow, so a stream of small calls
        // (Monte-Carlo trials, the reference's timing loops) pays no
        // cudaMalloc/cudaFree per call, while the number of idle engines kept
        // is bounded (LTCI_POOL_IDLE, default 2 per device) however many host
        // threads fan calls out (proj/src/bench.cpp:94-110).
        PoolLease<ltci_engine> lease(engine_pool(), device);
        ltci_engine& eng = *lease;
        static const bool trace = std::getenv("LTCI_TRACE") != nullptr;  // per-phase wall times on stderr
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        eng.pl = make_plan(*cp, *s, amb, variant, opt, 0, -1);
        eng.device = device;
        eng.htab_ready = false;  // the chirp table belongs to the previous plan
        eng.c_lo = 0;
        eng.c_hi = ~0ull;
        eng.timing = false;
        const auto t1 = clk::now();
        engine_init(&eng);
        const auto t2 = clk::now();
        DeviceGuard dg(eng.device);
        cudaStream_t st = nullptr;
        upload_host_cube(&eng, cube, st);
        run_device_impl(&eng, eng.cube_c64.p, st);
        if (trace) CK(cudaStreamSynchronize(st));
        const auto t3 = clk::now();
        *out = assemble(&eng, st);
        if (trace) {
            const auto t4 = clk::now();
            auto ms = [](clk::time_point a, clk::time_point b) {
                return std::chrono::duration<double, std::milli>(b - a).count();
            };
            std::fprintf(stderr, "[ltci] %s M=%d K=%d D=%d tc=%d plan %.2f init %.2f run %.2f assemble %.2f ms\n",
                         variant == LTCI_VARIANT_KTMFP ? "ds_kt_mfp" : "ds_grft", eng.pl.rp.M, eng.pl.rp.K,
                         eng.pl.D, eng.use_tc ? 1 : 0, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
        }
    });
}

}  // namespace

namespace {

// 8 independent FMA chains per thread keep the FMA pipe issue-bound.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __fmaf_rn(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[threadIdx.x] = s;  // keep the chains alive
}

}  // namespace

namespace {

// ---- fd_grft (reference proj/src/detectors.cpp:105-197)
template <int K>
void fd_launch_batch(const FdArgs& a, cudaStream_t st) {
    auto mf = fd_mf_kernel<K>;
    mf<<<static_cast<unsigned>((a.c_count + fd_cells(K) - 1) / fd_cells(K)), fd_threads(K), 0, st>>>(a);
    CK(cudaGetLastError());
    if constexpr (K < 16) {
        fd_small_scan_kernel<K><<<static_cast<unsigned>((a.c_count + 255) / 256), 256, 0, st>>>(a);
    } else {
        auto sc = fd_fft_scan_kernel<K>;
        constexpr int PG = kCoarseSamples / K;
        const size_t smem_sc = static_cast<size_t>(PG) * coarse_kp(K) * sizeof(float2);
        ensure_smem_attr(reinterpret_cast<const void*>(sc), 200 * 1024);
        sc<<<static_cast<unsigned>((a.c_count + PG - 1) / PG), kCoarseThreads, smem_sc, st>>>(a);
    }
    CK(cudaGetLastError());
}

void fd_launch(const FdArgs& a, cudaStream_t st) {
    switch (a.K) {
        case 2: fd_launch_batch<2>(a, st); break;
        case 4: fd_launch_batch<4>(a, st); break;
        case 8: fd_launch_batch<8>(a, st); break;
        case 16: fd_launch_batch<16>(a, st); break;
        case 32: fd_launch_batch<32>(a, st); break;
        case 64: fd_launch_batch<64>(a, st); break;
        case 128: fd_launch_batch<128>(a, st); break;
        case 256: fd_launch_batch<256>(a, st); break;
        case 512: fd_launch_batch<512>(a, st); break;
        case 1024: fd_launch_batch<1024>(a, st); break;
        case 2048: fd_launch_batch<2048>(a, st); break;
        case 4096: fd_launch_batch<4096>(a, st); break;
        case 8192: fd_launch_batch<8192>(a, st); break;
        default: fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: unsupported K");
    }
}

struct FdWorkspace {
    DevBuf<double2> f64;
    DevBuf<float2> c64, acc, dense;
    DevBuf<CandRec> cand;
    DevBuf<unsigned long long> ccount, k0, k1;
    DevBuf<PeakSlot> best;
    DevBuf<float2> v0, v1;
    DevBuf<double2> vo;
    DevBuf<unsigned char> tmp;
    DevBuf<int> err;
    HostBuf<unsigned char> small;
    HostBuf<float2> dense_h;
    HostBuf<int> err_h;
    Stager stager;
};

ObjectPool<FdWorkspace>& fd_pool() {
    static auto* p = new ObjectPool<FdWorkspace>();  // leaked: no teardown after the CUDA runtime
    return *p;
}

// The single-scale searches fd_grft (frequency-pulse cube; K5 + K6) and td_grft
// (range-pulse cube; K7, proj/src/detectors.cpp:199-264) share everything but
// the kernels: the motion grid and its cell index, the ROI scan, the result.
ltci_detection_map* single_scale_run(int kind, const double* cube, const float2* d_cube, const ltci_radar& rp,
                                     const ltci_single_space& s, const ltci_options* opt) {
    const bool td = kind == LTCI_TD_GRFT;
    const std::string who = td ? "td_grft" : "fd_grft";
    validate_radar(rp);
    check_same_params(rp, s.radar);
    if (rp.K < 2 || rp.K > 8192) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: frequency bins K must be in [2, 8192]");
    if (rp.M > 1 << 20) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: " + who + " supports M <= 2^20");
    const int P = s.order;
    if (P < 1 || P > LTCI_MAX_ORDER) fail(LTCI_INVALID_ARGUMENT, who + ": order must be in [1, 4]");
    unsigned long long cells = 1;
    for (int p = 0; p < P; ++p) {
        if (s.c[p].count < 1) fail(LTCI_INVALID_ARGUMENT, "grid is empty");
        cells *= static_cast<unsigned long long>(s.c[p].count);
    }
    if (s.roi_first < 0 || s.roi_last >= rp.K || s.roi_first > s.roi_last)
        fail(LTCI_INVALID_ARGUMENT, who + ": ROI outside the range axis");
    const int R = s.roi_last - s.roi_first + 1;
    const int policy = opt ? opt->trajectory : 0;
    if (td && (policy < 0 || policy > 2)) fail(LTCI_INVALID_ARGUMENT, "td_grft: unknown trajectory policy");
    const int device = opt ? opt->device : 0;
    const double retain = opt ? opt->retain_threshold : 0.0;
    const bool keep_dense = opt && opt->keep_dense;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        fail(LTCI_NO_DEVICE, "ltci_cuda: no CUDA device available");
    if (device < 0 || device >= ndev) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: bad device ordinal");
    DeviceGuard dg(device);
    preload_module();
    cudaStream_t st = nullptr;
    const int K = rp.K, M = rp.M;
    const size_t n = static_cast<size_t>(K) * M;
    // per-device workspace leased from a bounded process-wide pool: grow-only
    // buffers reused across calls (many small calls -- e.g. noise-only
    // Monte-Carlo trials -- pay no cudaMalloc), at most LTCI_POOL_IDLE idle
    PoolLease<FdWorkspace> lease(fd_pool(), device);
    FdWorkspace& w = *lease;
    auto& f64 = w.f64;
    auto& c64 = w.c64;
    auto& acc = w.acc;
    auto& dense = w.dense;
    auto& cand = w.cand;
    auto& ccount = w.ccount;
    auto& best = w.best;
    if (!d_cube) {
        f64.ensure(n);
        c64.ensure(n);
        h2d_cube(f64.p, cube, n, w.stager, st);
        f64_to_c64_kernel<<<static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(f64.p, c64.p,
                                                                                                          n);
        CK(cudaGetLastError());
    }

    size_t free_b = 0, total_b = 0;
    const size_t nd = keep_dense ? static_cast<size_t>(cells) * R : 0;
    if (keep_dense) {
        const double bytes = static_cast<double>(nd) * sizeof(float2);
        if (bytes > static_cast<double>(256u << 20)) {  // the (slow) memory query only for big maps
            CK(cudaMemGetInfo(&free_b, &total_b));
            if (bytes > 0.5 * static_cast<double>(free_b) || bytes * 2 > 64.0 * (1ull << 30))
                fail(LTCI_BAD_ALLOC, "ltci_cuda: dense " + who + " map exceeds the result memory");
        }
        dense.ensure(static_cast<size_t>(cells) * R);
    }
    // MF output per batch: bounded at 2 GiB, whole CTAs of both kernels
    const unsigned long long gran = std::max<unsigned long long>(kFdCells, kCoarseSamples / K);
    unsigned long long batch = std::max<unsigned long long>(gran, ((2ull << 30) / (8ull * K)) / gran * gran);
    batch = std::min(batch, (cells + gran - 1) / gran * gran);
    if (td)
        batch = std::min<unsigned long long>(cells, 1u << 30);  // one CTA column per cell: the grid's x extent
    else
        acc.ensure(static_cast<size_t>(batch) * K);
    ccount.ensure(1);
    best.ensure(1);
    w.err.ensure(1);
    w.err_h.ensure(1);

    FdArgs a{};
    a.cube = d_cube ? d_cube : c64.p;
    a.acc = acc.p;
    a.K = K;
    a.M = M;
    a.P = P;
    for (int p = 0; p < P; ++p) {
        a.count[p] = s.c[p].count;
        a.start[p] = s.c[p].start;
        a.step[p] = s.c[p].step;
    }
    a.inv_prf = 1.0 / rp.PRF;
    a.two_over_lambda = 2.0 / lambda_of(rp);
    a.two_df_over_c = 2.0 * rp.delta_f / kC;
    a.bin_scale = 2.0 * rp.fs / kC;  // metres -> range bins (detectors.cpp:220)
    a.policy = policy;
    a.err = w.err.p;
    a.roi_first = s.roi_first;
    a.R = R;
    a.retain2 = retain < 0 ? -1.0f : static_cast<float>(retain * retain);
    a.dense = keep_dense ? dense.p : nullptr;
    a.best = best.p;
    a.cand_count = ccount.p;

    unsigned long long cap = std::max<unsigned long long>(cand.n, 1ull << 16), count = 0;
    const SmallLayout L(1);
    unsigned char* hb = nullptr;
    for (int attempt = 0; attempt < 2; ++attempt) {
        cand.ensure(cap);
        a.cand = cand.p;
        a.cand_cap = cap;
        CK(cudaMemsetAsync(ccount.p, 0, sizeof(unsigned long long), st));
        init_slots_kernel<<<1, 32, 0, st>>>(best.p, 1);
        CK(cudaGetLastError());
        if (td) CK(cudaMemsetAsync(w.err.p, 0, sizeof(int), st));
        for (unsigned long long c0 = 0; c0 < cells; c0 += batch) {
            a.c_begin = c0;
            a.c_count = std::min(batch, cells - c0);
            if (td) {
                td_gather_scan_kernel<<<dim3(static_cast<unsigned>(a.c_count), (R + kTdThreads - 1) / kTdThreads),
                                        kTdThreads, 0, st>>>(a);
                CK(cudaGetLastError());
            } else {
                fd_launch(a, st);
            }
        }
        if (td) CK(cudaMemcpyAsync(w.err_h.p, w.err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        // count, best cell and small candidate sets behind one synchronisation
        hb = enqueue_small_result(w.small, ccount.p, cand.p, cap, best.p, 1, 1, M / 2, M, st);
        if (nd) {
            w.dense_h.ensure(nd);
            CK(cudaMemcpyAsync(w.dense_h.p, dense.p, nd * sizeof(float2), cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
        if (td && *w.err_h.p) fail(LTCI_OUT_OF_RANGE, "td_grft: trajectory leaves the cube");
        count = *reinterpret_cast<volatile unsigned long long*>(hb);
        if (count <= cap) break;
        CK(cudaMemGetInfo(&free_b, &total_b));
        if (static_cast<double>(count) * 64.0 > 0.8 * static_cast<double>(free_b) ||
            static_cast<double>(count) * 24.0 > 64.0 * (1ull << 30))
            fail(LTCI_BAD_ALLOC, "ltci_cuda: " + std::to_string(count) +
                                     " retained cells exceed the result memory (raise retain_threshold)");
        cap = count;
    }

    auto* out = static_cast<ltci_detection_map*>(std::calloc(1, sizeof(ltci_detection_map)));
    if (!out) throw std::bad_alloc();
    try {
        out->kind = kind;
        // single_scale_axes (detectors.cpp:94-101): c_P .. c_2, c_1, range
        int na = 0;
        for (int p = P; p >= 2; --p) out->axes[na++] = ltci_axis{LTCI_AXIS_HIGHER, p, s.c[p - 1].count};
        out->axes[na++] = ltci_axis{LTCI_AXIS_VELOCITY, 1, s.c[0].count};
        out->axes[na++] = ltci_axis{LTCI_AXIS_RANGE, 0, R};
        out->n_axes = na;
        if (td) {
            out->counters[1] = cells * static_cast<unsigned long long>(R);  // mf += 1 per (cell, row)
        } else {
            out->counters[1] = cells * static_cast<unsigned long long>(K);  // mf += n0() per cell
            out->counters[2] = cells;                                       // ifft += 1 per cell
        }
        out->retain_threshold = retain;
        const PeakSlot b = *reinterpret_cast<const PeakSlot*>(hb + L.slots);
        out->argmax = b.idx;
        out->argmax_value[0] = b.re;
        out->argmax_value[1] = b.im;
        out->n_candidates = count;
        out->cand_index = static_cast<uint64_t*>(xmalloc(count * sizeof(uint64_t)));
        out->cand_value = static_cast<double*>(xmalloc(2 * count * sizeof(double)));
        if (count && count <= std::min(kSmallCand, cap)) {
            std::memcpy(out->cand_index, hb + L.idx, count * sizeof(uint64_t));
            std::memcpy(out->cand_value, hb + L.val, count * sizeof(double2));
        } else if (count) {
            CandSortBufs bufs{w.k0, w.k1, w.v0, w.v1, w.vo, w.tmp};
            sort_candidates(cand.p, count, cells * static_cast<unsigned long long>(R), 1, M / 2, M, bufs,
                            out->cand_index, out->cand_value, st);
        }
        if (keep_dense) {
            const float2* h = w.dense_h.p;
            out->dense_stored = 1;
            out->dense_count = nd;
            out->dense = static_cast<double*>(xmalloc(2 * nd * sizeof(double)));
            for (size_t i = 0; i < nd; ++i) {
                out->dense[2 * i] = h[i].x;
                out->dense[2 * i + 1] = h[i].y;
            }
        }
    } catch (...) {
        ltci_cuda_free_map(out);
        throw;
    }
    return out;
}

}  // namespace

// Per-row best over several peak-slot arrays (coarse-cell shards): the same
// magnitude (mag2f) and lowest-flat-index tie-break as the kernels' CAS publish.
__global__ void merge_peaks_kernel(const PeakSlot* __restrict__ in, int n_maps, int n_rows,
                                   PeakSlot* __restrict__ out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        PeakSlot b = in[r];
        float bm = b.idx == ~0ull ? -1.0f : mag2f(b.re, b.im);
        for (int k = 1; k < n_maps; ++k) {
            const PeakSlot c = in[static_cast<size_t>(k) * n_rows + r];
            if (c.idx == ~0ull) continue;
            const float cm = mag2f(c.re, c.im);
            if (cm > bm || (cm == bm && c.idx < b.idx)) {
                b = c;
                bm = cm;
            }
        }
        out[r] = b;
    }
}

// fd_grft on a device-resident complex64 cube (the Monte-Carlo driver, pd.cu);
// throws ltcib::Status-like errors through the same guarded() wrappers
ltci_detection_map* ltcib_fd_grft_device(const float2* d_cube, const ltci_radar& rp, const ltci_single_space& s,
                                         const ltci_options* opt) {
    try {
        return single_scale_run(LTCI_FD_GRFT, nullptr, d_cube, rp, s, opt);
    } catch (const Error& e) {
        throw ltcib::CubeError(e.code, e.msg);  // status-carrying error across translation units
    }
}

extern "C" {

int ltci_cuda_measure_fp32_peak(int device, double* tflops) {
    return guarded([&] {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(LTCI_NO_DEVICE, "ltci_cuda: no CUDA device available");
        DeviceGuard dg(device);
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        DevBuf<float> out;
        out.ensure(256);
        const int blocks = sms * 8, iters = 4096;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        ffma_peak_kernel<<<blocks, 256>>>(out.p, 64, 0.999f, 1e-4f);  // warm-up
        CK(cudaEventRecord(e0));
        ffma_peak_kernel<<<blocks, 256>>>(out.p, iters, 0.999f, 1e-4f);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * 256;
        *tflops = flops / (ms * 1e-3) / 1e12;
    });
}

const char* ltci_cuda_last_error(void) { return g_err.c_str(); }
int ltci_cuda_version(void) { return 100; }

void ltci_cuda_free_map(ltci_detection_map* m) {
    if (!m) return;
    std::free(m->cand_index);
    std::free(m->cand_value);
    std::free(m->dense);
    std::free(m->peak_index);
    std::free(m->peak_value);
    std::free(m);
}

int ltci_cuda_fd_grft(const double* cube, const ltci_radar* cube_params, const ltci_single_space* space,
                      const ltci_options* opt, ltci_detection_map** out) {
    return guarded([&] {
        if (!cube || !cube_params || !space || !out) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        *out = single_scale_run(LTCI_FD_GRFT, cube, nullptr, *cube_params, *space, opt);
    });
}

int ltci_cuda_td_grft(const double* cube, const ltci_radar* cube_params, const ltci_single_space* space,
                      const ltci_options* opt, ltci_detection_map** out) {
    return guarded([&] {
        if (!cube || !cube_params || !space || !out) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        *out = single_scale_run(LTCI_TD_GRFT, cube, nullptr, *cube_params, *space, opt);
    });
}

// kt_mfp (proj/src/detectors.cpp:266-326) is the dual-scale keystone cascade
// with one fine cell: per (folding number, acceleration) cell gift(KtRm) then
// gft({c2}) -- the preDFM factor of mgift carries the whole c2 t^2 phase when
// the fine offset is zero -- over the full Doppler axis; the flat index
// ((q, c2), r, j) is ds_kt_mfp's with a fine axis of size one.
int ltci_cuda_kt_mfp(const double* cube, const ltci_radar* cube_params, const ltci_ambiguity* amb,
                     const ltci_single_space* space, const ltci_options* opt, ltci_detection_map** out) {
    return guarded([&] {
        if (!cube || !cube_params || !amb || !space || !out) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        check_same_params(*cube_params, space->radar);
        if (space->order != 2) fail(LTCI_INVALID_ARGUMENT, "kt_mfp: needs a P = 2 search space");
        ltci_dual_space d{};
        d.radar = space->radar;
        d.order = 2;
        d.coarse[0] = ltci_grid{0.0, 1.0, 1};  // unused by the keystone variant
        d.coarse[1] = space->c[1];
        d.fine[0] = ltci_grid{0.0, 1.0, 1};
        d.fine[1] = ltci_grid{0.0, 1.0, 1};    // the single fine cell: zero offset
        for (int p = 0; p < 2; ++p) {
            d.rm_step[p] = space->rm_step[p];
            d.dfm_step[p] = space->dfm_step[p];
            d.alpha[p] = space->alpha[p];
        }
        d.kappa = 1.0;
        d.roi_first = space->roi_first;
        d.roi_last = space->roi_last;
        ltci_detection_map* m = nullptr;
        const int rc = detect(cube, cube_params, amb, &d, opt, LTCI_VARIANT_KTMFP, &m);
        if (rc != LTCI_OK) throw Error{rc, g_err};
        const unsigned long long cells =
            static_cast<unsigned long long>(amb->q_max - amb->q_min + 1) * static_cast<unsigned long long>(space->c[1].count);
        const int R = space->roi_last - space->roi_first + 1;
        m->kind = LTCI_KT_MFP;
        m->n_axes = 4;
        m->axes[0] = ltci_axis{LTCI_AXIS_FOLDING, 0, amb->q_max - amb->q_min + 1};
        m->axes[1] = ltci_axis{LTCI_AXIS_HIGHER, 2, space->c[1].count};
        m->axes[2] = ltci_axis{LTCI_AXIS_RANGE, 0, R};
        m->axes[3] = ltci_axis{LTCI_AXIS_DOPPLER, 0, cube_params->M};
        m->counters[0] = 1;                                                      // kt
        m->counters[1] = cells * static_cast<unsigned long long>(cube_params->K);  // mf += n0() per cell
        m->counters[2] = cells * static_cast<unsigned long long>(cube_params->M);  // ifft += M per cell
        m->counters[3] = cells * static_cast<unsigned long long>(R);               // fft += R per cell
        *out = m;
    });
}

int ltci_cuda_ds_grft(const double* cube, const ltci_radar* cube_params, const ltci_dual_space* space,
                      const ltci_options* opt, ltci_detection_map** out) {
    return detect(cube, cube_params, nullptr, space, opt, LTCI_VARIANT_GRFT, out);
}

int ltci_cuda_ds_kt_mfp(const double* cube, const ltci_radar* cube_params, const ltci_ambiguity* amb,
                        const ltci_dual_space* space, const ltci_options* opt, ltci_detection_map** out) {
    return detect(cube, cube_params, amb, space, opt, LTCI_VARIANT_KTMFP, out);
}

// detection_threshold (proj/src/detectors.cpp:483-489) -- host arithmetic
double ltci_cuda_detection_threshold(const ltci_radar* p, double sigma2, double pfa, int bins, int* status) {
    double out = 0.0;
    int rc = guarded([&] {
        if (!(pfa > 0.0) || !(pfa < 1.0)) fail(LTCI_INVALID_ARGUMENT, "detection_threshold: pfa must be in (0, 1)");
        if (sigma2 < 0) fail(LTCI_INVALID_ARGUMENT, "detection_threshold: sigma2 must be >= 0");
        if (bins == 0) bins = p->K;
        out = std::sqrt(-static_cast<double>(p->M) * bins * sigma2 * std::log(pfa));
    });
    if (status) *status = rc;
    return out;
}

int ltci_cuda_keystone(const double* cube, const ltci_radar* p, int taps, double* out) {
    return guarded([&] {
        validate_radar(*p);
        if (taps < 2) fail(LTCI_INVALID_ARGUMENT, "keystone: need at least 2 taps");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(LTCI_NO_DEVICE, "ltci_cuda: no CUDA device available");
        const size_t n = static_cast<size_t>(p->K) * p->M;
        DevBuf<double2> f64;
        DevBuf<float2> a, b;
        f64.ensure(n);
        a.ensure(n);
        b.ensure(n);
        CK(cudaMemcpy(f64.p, cube, n * sizeof(double2), cudaMemcpyHostToDevice));
        f64_to_c64_kernel<<<256, 256>>>(f64.p, a.p, n);
        KeystoneArgs ka{a.p, b.p, p->K, p->M, taps, p->fc, p->delta_f};
        launch_keystone(ka, nullptr);
        std::vector<float2> h(n);
        CK(cudaMemcpy(h.data(), b.p, n * sizeof(float2), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i) {
            out[2 * i] = h[i].x;
            out[2 * i + 1] = h[i].y;
        }
    });
}

int ltci_cuda_range_fft(const double* range_cube, const ltci_radar* p, double* out) {
    return guarded([&] {
        if (!range_cube || !p || !out) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        validate_radar(*p);
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(LTCI_NO_DEVICE, "ltci_cuda: no CUDA device available");
        const size_t n = static_cast<size_t>(p->K) * p->M;
        DevBuf<double2> f64;
        DevBuf<float2> b;
        f64.ensure(n);
        b.ensure(n);
        CK(cudaMemcpy(f64.p, range_cube, n * sizeof(double2), cudaMemcpyHostToDevice));
        launch_range_fft(f64.p, true, b.p, p->K, p->M, nullptr);
        std::vector<float2> h(n);
        CK(cudaMemcpy(h.data(), b.p, n * sizeof(float2), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i) {
            out[2 * i] = h[i].x;
            out[2 * i + 1] = h[i].y;
        }
    });
}

int ltci_cuda_range_fft_device(const void* d_in, void* d_out, const ltci_radar* p, void* stream) {
    return guarded([&] {
        if (!d_in || !d_out || !p) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        validate_radar(*p);
        launch_range_fft(d_in, false, static_cast<float2*>(d_out), p->K, p->M, static_cast<cudaStream_t>(stream));
    });
}

int ltci_cuda_keystone_device(const void* d_in, void* d_out, const ltci_radar* p, int taps, void* stream) {
    return guarded([&] {
        if (!d_in || !d_out || !p) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        validate_radar(*p);
        if (taps < 2) fail(LTCI_INVALID_ARGUMENT, "keystone: need at least 2 taps");
        KeystoneArgs ka{static_cast<const float2*>(d_in), static_cast<float2*>(d_out), p->K, p->M, taps, p->fc,
                        p->delta_f};
        launch_keystone(ka, static_cast<cudaStream_t>(stream));
    });
}

// mgift through K1 with a single coarse cell and the full range axis.
int ltci_cuda_mgift(const double* cube, const ltci_radar* p, const double* ctilde, int n_ctilde, int variant,
                    double* out) {
    return guarded([&] {
        validate_radar(*p);
        check_supported(*p);
        if (variant == LTCI_VARIANT_KTMFP && n_ctilde != 2) fail(LTCI_INVALID_ARGUMENT, "build_mf: KtRm needs [q, c2]");
        if (variant == LTCI_VARIANT_GRFT && (n_ctilde < 1 || n_ctilde > 4))
            fail(LTCI_INVALID_ARGUMENT, "build_mf: RM needs c1..cP");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(LTCI_NO_DEVICE, "ltci_cuda: no CUDA device available");
        const int K = p->K, M = p->M;
        const size_t n = static_cast<size_t>(K) * M;
        DevBuf<double2> f64;
        DevBuf<float2> a, X;
        DevBuf<double> cpar;
        f64.ensure(n);
        a.ensure(n);
        X.ensure(n);
        cpar.ensure(4);
        double cp4[4] = {0, 0, 0, 0};
        for (int i = 0; i < n_ctilde; ++i) cp4[i] = ctilde[i];
        CK(cudaMemcpy(cpar.p, cp4, sizeof(cp4), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(f64.p, cube, n * sizeof(double2), cudaMemcpyHostToDevice));
        f64_to_c64_kernel<<<256, 256>>>(f64.p, a.p, n);
        CoarseArgs ca{};
        ca.cube = a.p;
        ca.cparams = cpar.p;
        ca.X = X.p;
        ca.c_begin = 0;
        ca.c_count = 1;
        ca.K = K;
        ca.M = M;
        ca.P = variant == LTCI_VARIANT_GRFT ? n_ctilde : 2;
        ca.variant = variant;
        ca.n_base = 0;
        ca.R_slice = K;
        ca.inv_prf = 1.0 / p->PRF;
        ca.inv_dR = 1.0 / dR_of(*p);
        ca.two_over_lambda = 2.0 / lambda_of(*p);
        ca.Va = va_of(*p);
        ca.kt_b = -(4.0 * kPi / kC) * p->delta_f * p->delta_f / p->fc;
        radix_plan(K, ca.radix, &ca.npass);
        GatherStage gs;
        if (gather_selected(K, M, false, 1)) {  // one cell: only when LTCI_COARSE=gather forces it
            gs.init(K, M, {variant == LTCI_VARIANT_KTMFP ? cp4[0] : 0.0}, 1, 1, 1);
            gs.build(ca, nullptr);
            GatherArgs ga = gs.args(ca);
            ga.c_begin = 0;
            ga.c_count = 1;
            launch_gather_weights(ga, nullptr);
            launch_gather_cells(ga, nullptr);
        } else {
            launch_coarse(ca, coarse_pg(K, M), nullptr);
        }
        std::vector<float2> h(n);
        CK(cudaMemcpy(h.data(), X.p, n * sizeof(float2), cudaMemcpyDeviceToHost));
        // X[n][m] -> RangePulseCube data[n + K*m]
        for (int m = 0; m < M; ++m)
            for (int r = 0; r < K; ++r) {
                out[2 * (r + static_cast<size_t>(K) * m)] = h[static_cast<size_t>(r) * M + m].x;
                out[2 * (r + static_cast<size_t>(K) * m) + 1] = h[static_cast<size_t>(r) * M + m].y;
            }
    });
}

// gft through the fine kernel: one "coarse cell", one fine cell with the
// caller's higher-order values, full Doppler axis, dense output.
int ltci_cuda_gft(const double* rows, const ltci_radar* p, const double* fine_higher, int n_fine, int roi_first,
                  int roi_last, double* out) {
    return guarded([&] {
        validate_radar(*p);
        check_supported(*p);
        const int R = roi_last - roi_first + 1;
        if (R <= 0 || roi_first < 0 || roi_last >= p->K) fail(LTCI_INVALID_ARGUMENT, "gft: empty or out-of-range roi");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(LTCI_NO_DEVICE, "ltci_cuda: no CUDA device available");
        const int K = p->K, M = p->M;
        // rows[n + K*m] -> X[r][m] in complex64
        std::vector<float2> hx(static_cast<size_t>(R) * M);
        for (int r = 0; r < R; ++r)
            for (int m = 0; m < M; ++m) {
                const size_t src = 2 * (static_cast<size_t>(roi_first + r) + static_cast<size_t>(K) * m);
                hx[static_cast<size_t>(r) * M + m] = make_float2(static_cast<float>(rows[src]), static_cast<float>(rows[src + 1]));
            }
        const double lam = lambda_of(*p);
        std::vector<float2> h0(M), hs(M, make_float2(1.f, 0.f));
        for (int m = 0; m < M; ++m) {
            const double t = static_cast<double>(m + 1) / p->PRF;
            double s = 0, tp = t;
            for (int i = 0; i < n_fine; ++i) {
                tp *= t;
                s += fine_higher[i] * tp;
            }
            h0[m] = phase_lambda(s, lam);
        }
        DevBuf<float2> X, H0, HS, dense;
        DevBuf<PeakSlot> slots;
        DevBuf<CandRec> cand;
        DevBuf<unsigned long long> cnt;
        X.ensure(hx.size());
        H0.ensure(M);
        HS.ensure(M);
        dense.ensure(static_cast<size_t>(R) * M);
        slots.ensure(R);
        cand.ensure(1);
        cnt.ensure(1);
        CK(cudaMemcpy(X.p, hx.data(), hx.size() * sizeof(float2), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(H0.p, h0.data(), M * sizeof(float2), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(HS.p, hs.data(), M * sizeof(float2), cudaMemcpyHostToDevice));
        CK(cudaMemset(cnt.p, 0, sizeof(unsigned long long)));
        CK(cudaMemset(slots.p, 0, R * sizeof(PeakSlot)));
        FineArgs fa{};
        fa.X = X.p;
        fa.H0 = H0.p;
        fa.Hstep = HS.p;
        fa.slots = slots.p;
        fa.cand = cand.p;
        fa.cand_count = cnt.p;
        fa.dense = dense.p;
        fa.cand_cap = 0;
        fa.c_begin = 0;
        fa.F = 1;
        fa.R_total = R;
        fa.rows = R;
        fa.R_slice = R;
        fa.row_begin = 0;
        fa.D = M;
        fa.dop_first = 0;
        fa.kA = M / 2 - 1;
        fa.kB = M / 2;
        fa.n_outer = 1;
        fa.n_inner = 1;
        fa.n_split = 1;
        fa.chunk = 1;
        fa.retain2 = INFINITY;
        launch_fine_m(fa, M, true, nullptr);
        std::vector<float2> hd(static_cast<size_t>(R) * M);
        CK(cudaMemcpy(hd.data(), dense.p, hd.size() * sizeof(float2), cudaMemcpyDeviceToHost));
        // dense[r*M + j] -> map data[r + R*j] with the recentring twiddle
        for (int r = 0; r < R; ++r)
            for (int j = 0; j < M; ++j) {
                const float2 v = hd[static_cast<size_t>(r) * M + j];
                const double ang = 2.0 * kPi * (j - M / 2) / M;
                const double c = std::cos(ang), s = std::sin(ang);
                const size_t o = 2 * (static_cast<size_t>(r) + static_cast<size_t>(R) * j);
                out[o] = v.x * c - v.y * s;
                out[o + 1] = v.x * s + v.y * c;
            }
    });
}

int ltci_cuda_pool_idle(int device, int64_t* engines, int64_t* fd_workspaces) {
    return guarded([&] {
        if (device < 0) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: bad device ordinal");
        if (engines) *engines = static_cast<int64_t>(engine_pool().idle_count(device));
        if (fd_workspaces) *fd_workspaces = static_cast<int64_t>(fd_pool().idle_count(device));
    });
}

int ltci_engine_create(const ltci_radar* p, const ltci_dual_space* space, const ltci_ambiguity* amb, int variant,
                       const ltci_options* opt, int row_begin, int row_end, ltci_engine** out) {
    return guarded([&] {
        if (!p || !space || !out) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        auto* e = new ltci_engine();
        try {
            e->pl = make_plan(*p, *space, amb, variant, opt, row_begin, row_end);
            e->device = opt ? opt->device : 0;
            engine_init(e);
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    });
}

void ltci_engine_destroy(ltci_engine* e) {
    if (!e) return;
    {
        DeviceGuard dg(e->device);
        for (auto& x : e->ev) cudaEventDestroy(x);
        e->ev.clear();
        for (int i = 0; i < 2; ++i) {
            if (e->stage[i]) cudaFreeHost(e->stage[i]);
            if (e->stage_ev[i]) cudaEventDestroy(e->stage_ev[i]);
        }
        delete e;
    }
}

int ltci_engine_run_device(ltci_engine* e, const void* d_cube_c64, void* stream) {
    return guarded([&] {
        if (!e || !d_cube_c64) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        run_device_impl(e, static_cast<const float2*>(d_cube_c64), static_cast<cudaStream_t>(stream));
    });
}

int ltci_engine_run_host(ltci_engine* e, const double* cube, void* stream) {
    return guarded([&] {
        if (!e || !cube) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        DeviceGuard dg(e->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        upload_host_cube(e, cube, st);
        run_device_impl(e, e->cube_c64.p, st);
        e->launches += 1;  // conversion kernel
    });
}

// configs[3] front end: a range-pulse (fast-time) cube goes through K0
// (range_fft, reference proj/src/signal_model.cpp:97-107) into the engine's
// own freq-pulse buffer, then the cascade runs on it.
int ltci_engine_run_range_device(ltci_engine* e, const void* d_range_c64, void* stream) {
    return guarded([&] {
        if (!e || !d_range_c64) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        DeviceGuard dg(e->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const size_t n = static_cast<size_t>(e->pl.rp.K) * e->pl.rp.M;
        e->cube_c64.ensure(n);
        launch_range_fft(d_range_c64, false, e->cube_c64.p, e->pl.rp.K, e->pl.rp.M, st);
        run_device_impl(e, e->cube_c64.p, st);
        e->launches += 1;  // K0
    });
}

int ltci_engine_run_range_host(ltci_engine* e, const double* range_cube, void* stream) {
    return guarded([&] {
        if (!e || !range_cube) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        DeviceGuard dg(e->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const size_t n = static_cast<size_t>(e->pl.rp.K) * e->pl.rp.M;
        e->cube_f64.ensure(n);
        e->cube_c64.ensure(n);
        h2d_cube(e->cube_f64.p, range_cube, n, e->stager, st);
        // the f64 -> c64 conversion is folded into K0's loads
        launch_range_fft(e->cube_f64.p, true, e->cube_c64.p, e->pl.rp.K, e->pl.rp.M, st);
        run_device_impl(e, e->cube_c64.p, st);
        e->launches += 1;  // K0
    });
}

// The wire path: file -> two pinned staging blocks ->
// async H2D into the f64 echo buffer, the fread of block i+1 overlapping the
// DMA of block i; then f64 -> c64 on the device and the detector run.
int ltci_engine_run_file(ltci_engine* e, const char* path, void* stream) {
    return guarded([&] {
        if (!e || !path) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        ltcib::CubeReader rd;
        rd.open(path);
        if (rd.h.domain != 0)  // CubeFile::to_freq_cube (proj/src/cube_io.cpp:48-52)
            fail(LTCI_CONDITION_VIOLATED, "cube file holds range-pulse data, not freq-pulse");
        check_same_params(rd.h.radar, e->pl.rp);
        DeviceGuard dg(e->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const size_t n = static_cast<size_t>(e->pl.rp.K) * e->pl.rp.M;
        e->cube_f64.ensure(n);
        e->cube_c64.ensure(n);
        const size_t block = 4u << 20;  // doubles per staging block (32 MiB)
        if (!e->stage[0]) {
            for (int i = 0; i < 2; ++i) {
                CK(cudaHostAlloc(reinterpret_cast<void**>(&e->stage[i]), block * sizeof(double), cudaHostAllocDefault));
                CK(cudaEventCreateWithFlags(&e->stage_ev[i], cudaEventDisableTiming));
            }
            e->stage_doubles = block;
        }
        double* dst = reinterpret_cast<double*>(e->cube_f64.p);
        const size_t total = 2 * n;
        int b = 0;
        for (size_t off = 0, i = 0; off < total; off += e->stage_doubles, ++i, b ^= 1) {
            const size_t m = std::min(e->stage_doubles, total - off);
            // block b's previous DMA -- possibly queued by an earlier run_file call
            // behind that call's kernels -- must be done before it is refilled
            CK(cudaEventSynchronize(e->stage_ev[b]));
            rd.read(e->stage[b], m);
            CK(cudaMemcpyAsync(dst + off, e->stage[b], m * sizeof(double), cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(e->stage_ev[b], st));
        }
        const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 8));
        f64_to_c64_kernel<<<blocks, 256, 0, st>>>(e->cube_f64.p, e->cube_c64.p, n);
        CK(cudaGetLastError());
        run_device_impl(e, e->cube_c64.p, st);
        e->launches += 1;  // conversion kernel
    });
}

int ltci_engine_result(ltci_engine* e, void* stream, ltci_detection_map** out) {
    return guarded([&] {
        if (!e || !out) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        if (!e->ran) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: engine has not run");
        *out = assemble(e, static_cast<cudaStream_t>(stream));
    });
}

int ltci_engine_peaks_device(ltci_engine* e, void** d_ptr, int32_t* n_rows) {
    return guarded([&] {
        if (!e || !d_ptr || !n_rows) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        *d_ptr = e->slots.p;
        *n_rows = e->pl.R_slice;
    });
}

int ltci_engine_stats(ltci_engine* e, int64_t* launches, double* fine_ms, double* coarse_ms, double* keystone_ms) {
    return guarded([&] {
        if (!e) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        if (launches) *launches = e->launches;
        if (fine_ms) *fine_ms = e->fine_ms;
        if (coarse_ms) *coarse_ms = e->coarse_ms;
        if (keystone_ms) *keystone_ms = e->keystone_ms;
    });
}

int ltci_engine_set_timing(ltci_engine* e, int enable) {
    return guarded([&] {
        if (!e) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        e->timing = enable != 0;
    });
}

int ltci_engine_fine_path(ltci_engine* e, int32_t* path, int32_t* terms) {
    return guarded([&] {
        if (!e) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        if (path) *path = e->use_tc ? (e->tc_terms == 1 ? LTCI_FINE_TC_FAST : LTCI_FINE_TC_DENSE) : LTCI_FINE_FFT_CUDA_CORE;
        if (terms) *terms = e->use_tc ? e->tc_terms : 0;
    });
}

int ltci_engine_coarse_path(ltci_engine* e, int32_t* path) {
    return guarded([&] {
        if (!e || !path) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        *path = e->use_gather ? LTCI_COARSE_GATHER : LTCI_COARSE_TRANSFORM;
    });
}

int ltci_engine_work(ltci_engine* e, uint64_t* hypotheses, uint64_t* integrations) {
    return guarded([&] {
        if (!e) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        const Plan& pl = e->pl;
        const unsigned long long cc = std::min(e->c_hi, pl.coarse_cells) - e->c_lo;
        const unsigned long long H = cc * pl.fine_cells * pl.R_slice * pl.D;
        if (hypotheses) *hypotheses = H;
        if (integrations) *integrations = H * static_cast<unsigned long long>(pl.rp.M);
    });
}

int ltci_engine_set_coarse_slice(ltci_engine* e, uint64_t c_begin, uint64_t c_end) {
    return guarded([&] {
        if (!e) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: null argument");
        if (c_end == ~0ull) c_end = e->pl.coarse_cells;  // "to the end"
        if (c_begin >= c_end || c_end > e->pl.coarse_cells)
            fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: coarse slice must satisfy 0 <= begin < end <= coarse cells");
        e->c_lo = c_begin;
        e->c_hi = c_end;
    });
}

int ltci_cuda_merge_peaks(const void* d_slots, int n_maps, int n_rows, void* d_out, void* stream) {
    return guarded([&] {
        if (!d_slots || !d_out || n_maps < 1 || n_rows < 0) fail(LTCI_INVALID_ARGUMENT, "ltci_cuda: bad merge");
        if (n_rows == 0) return;
        const int blocks = std::min(148 * 4, (n_rows + 255) / 256);
        merge_peaks_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            static_cast<const PeakSlot*>(d_slots), n_maps, n_rows, static_cast<PeakSlot*>(d_out));
        CK(cudaGetLastError());
    });
}

}  // extern "C"
