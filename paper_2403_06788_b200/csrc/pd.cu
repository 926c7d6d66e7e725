// pd.cu -- batched Monte-Carlo detection probability.
//
//   synthesize_cube   proj/src/signal_model.cpp:32-51   -> synth_kernel (FP64)
//   add_noise         proj/src/signal_model.cpp:53-60   -> noise_kernel (FP64)
//   GaussianRng       proj/src/rng.cpp:8-43
//   run_pd            proj/src/bench.cpp:72-124         -> ltci_cuda_run_pd
//   build_spaces      proj/src/bench.cpp:13-21, search_space.cpp:15-116
//
// GaussianRng is splitmix64 (state += gamma, then a mix) feeding Box-Muller
// pairs, and add_noise draws (re, im) of element i from normal() calls 2i and
// 2i+1, i.e. uniforms u1 = U(mix(seed + (2i+1) gamma)), u2 = U(mix(seed +
// (2i+2) gamma)): re = r cos a, im = r sin a with r = sqrt(-2 ln u1),
// a = 2 pi u2.  The stream is counter-based, so every element is generated
// independently on the device; the FP64 math library differs from glibc by
// at most an ulp or two, far below the complex64 rounding every detector
// input goes through.  Each trial's noisy cube is formed on the device
// (clean FP64 + noise, rounded to complex64) and searched there; only the
// retained candidate list comes back for the reference's success test.

#include <algorithm>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ltci_cuda.h"
#include "cube_io.hpp"

namespace ltcib {

constexpr double kPiD = 3.14159265358979323846;
constexpr double kCD = 3.0e8;

__device__ __forceinline__ unsigned long long sm64_mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double sm64_uniform(unsigned long long seed, unsigned long long k) {
    // k-th draw (k >= 1) of splitmix64 started at `seed`, as GaussianRng::uniform01: (0, 1]
    const unsigned long long z = sm64_mix(seed + k * 0x9e3779b97f4a7c15ULL);
    return (static_cast<double>(z >> 11) + 1.0) * 0x1.0p-53;
}

// out[i] = clean[i] + CN(0, sigma2) draw i (FP64); optional complex64 rounding
__global__ void noise_kernel(const double2* __restrict__ clean, size_t n, double sigma2, unsigned long long seed,
                             double2* __restrict__ out_f64, float2* __restrict__ out_c64) {
    const double s = sqrt(sigma2 / 2.0);
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double2 v = clean ? clean[i] : make_double2(0.0, 0.0);
        if (sigma2 > 0.0) {
            const double u1 = sm64_uniform(seed, 2 * i + 1);
            const double u2 = sm64_uniform(seed, 2 * i + 2);
            const double r = sqrt(-2.0 * log(u1));
            const double a = 2.0 * kPiD * u2;
            double sn, cs;
            sincos(a, &sn, &cs);
            v.x += s * (r * cs);
            v.y += s * (r * sn);
        }
        if (out_f64) out_f64[i] = v;
        if (out_c64) out_c64[i] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
    }
}

// synthesize_cube: y[g row, m] = sum_t A_t exp(j (-4 pi / c) (f_g + fc) R_t(t_m)) inside
// the occupied band g in [-K_valid/2, K_valid/2), zero outside
__global__ void synth_kernel(ltci_radar p, int nt, const ltci_target* __restrict__ tg, double2* __restrict__ out) {
    const size_t n = static_cast<size_t>(p.K) * p.M;
    const double c4pi = -4.0 * kPiD / kCD;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % static_cast<size_t>(p.K));
        const int m = static_cast<int>(i / static_cast<size_t>(p.K));
        const int g = r < p.K / 2 ? r : r - p.K;  // row_of_index inverse
        double2 acc = make_double2(0.0, 0.0);
        if (g >= -p.K_valid / 2 && g < p.K_valid / 2) {
            const double tm = static_cast<double>(m + 1) / p.PRF;
            const double fk = p.delta_f * static_cast<double>(g);
            for (int t = 0; t < nt; ++t) {
                double range = 0.0;  // MotionParams::slant_range (Horner, highest order first)
                for (int k = tg[t].order; k >= 0; --k) range = range * tm + tg[t].c[k];
                double sn, cs;
                sincos(c4pi * (fk + p.fc) * range, &sn, &cs);
                acc.x += tg[t].amp[0] * cs - tg[t].amp[1] * sn;
                acc.y += tg[t].amp[0] * sn + tg[t].amp[1] * cs;
            }
        }
        out[i] = acc;
    }
}

}  // namespace ltcib

// engine.cu / detection.cpp internals used here
ltci_detection_map* ltcib_fd_grft_device(const float2* d_cube, const ltci_radar& rp, const ltci_single_space& s,
                                         const ltci_options* opt);
bool ltcib_detection_success(const ltci_detection_map* map, const ltci_dual_space* ds, const ltci_single_space* ss,
                             const ltci_ambiguity* amb, const ltci_target& truth);
void ltcib_set_last_error(const char* msg);

namespace {

using ltcib::CubeError;

[[noreturn]] void pd_fail(int code, const std::string& m) { throw CubeError(code, m); }

void pd_ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        pd_fail(e == cudaErrorMemoryAllocation ? LTCI_BAD_ALLOC : LTCI_RUNTIME_ERROR,
                std::string(what) + ": " + cudaGetErrorString(e));
}
#define PD_CK(x) pd_ck((x), #x)

void pd_rc(int rc) {
    if (rc != LTCI_OK) pd_fail(rc, ltci_cuda_last_error());
}

template <typename F>
int pd_guarded(F&& f) {
    try {
        f();
        return LTCI_OK;
    } catch (const CubeError& e) {
        ltcib_set_last_error(e.what());
        return e.code;
    } catch (const std::invalid_argument& e) {
        ltcib_set_last_error(e.what());
        return LTCI_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        ltcib_set_last_error("run_pd: allocation failed");
        return LTCI_BAD_ALLOC;
    } catch (const std::exception& e) {
        ltcib_set_last_error(e.what());
        return LTCI_RUNTIME_ERROR;
    }
}

template <typename T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { PD_CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

int grid_for(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16)); }

// ---- search-space builders (proj/src/search_space.cpp:15-116) -------------
constexpr double kC = ltcib::kCD;

double T_of(const ltci_radar& r) { return static_cast<double>(r.M) / r.PRF; }

void step_sizes(const ltci_radar& r, int P, const double* alpha, double* rm, double* dfm) {
    if (P < 1 || P > LTCI_MAX_ORDER) throw std::invalid_argument("step_sizes: P must be in 1..4");
    double sum = 0;
    for (int p = 0; p < P; ++p) {
        if (!(alpha[p] > 0.0) || alpha[p] > 1.0)
            throw std::invalid_argument("step_sizes: each alpha_p must be in (0, 1]");
        sum += alpha[p];
    }
    if (std::abs(sum - 1.0) > 1e-12) throw std::invalid_argument("step_sizes: alpha weights must sum to 1");
    double tp = 1.0;
    for (int p = 0; p < P; ++p) {
        tp *= T_of(r);
        rm[p] = alpha[p] * kC / (2.0 * r.fs * tp);
        dfm[p] = alpha[p] * kC / (2.0 * r.fc * tp);
    }
}

// span_grid (search_space.cpp:51-65)
ltci_grid span_grid(double lo, double hi, double step, bool cover) {
    if (!(hi >= lo)) throw std::invalid_argument("grid bounds: min must be <= max");
    if (!(step > 0)) throw std::invalid_argument("grid step must be positive");
    const double span = hi - lo;
    const int count = cover ? std::max(0, static_cast<int>(std::ceil(span / step - 0.5 - 1e-9))) + 1
                            : static_cast<int>(std::floor(span / step + 1e-9)) + 1;
    if (count < 1) throw std::invalid_argument("grid is empty");
    return ltci_grid{lo, step, count};
}

ltci_single_space build_single(const ltci_scenario& sc, int roi_first, int roi_last) {
    ltci_single_space s{};
    s.radar = sc.radar;
    s.order = sc.P;
    step_sizes(sc.radar, sc.P, sc.alpha, s.rm_step, s.dfm_step);
    for (int p = 0; p < sc.P; ++p) {
        s.alpha[p] = sc.alpha[p];
        s.c[p] = span_grid(sc.bound_lo[p], sc.bound_hi[p], s.dfm_step[p], false);
    }
    s.roi_first = roi_first;
    s.roi_last = roi_last;
    return s;
}

// build_dual_scale (search_space.cpp:82-109)
ltci_dual_space build_dual(const ltci_scenario& sc) {
    const ltci_radar& r = sc.radar;
    const double ratio = (r.fc / r.fs) / static_cast<double>(r.M);
    if (ratio > 1.0)
        pd_fail(LTCI_CONDITION_VIOLATED, "dual-scale space requires (fc/fs)/M <= 1, got " + std::to_string(ratio));
    ltci_dual_space s{};
    s.radar = r;
    s.order = sc.P;
    step_sizes(r, sc.P, sc.alpha, s.rm_step, s.dfm_step);
    s.kappa = 1.0 - r.Br / (2.0 * r.fc);
    for (int p = 0; p < sc.P; ++p) {
        s.alpha[p] = sc.alpha[p];
        s.coarse[p] = span_grid(sc.bound_lo[p], sc.bound_hi[p], s.rm_step[p], true);
        const int half = static_cast<int>(std::floor(s.rm_step[p] / s.dfm_step[p] / 2.0 + 1e-9));
        s.fine[p] = ltci_grid{-s.dfm_step[p] * static_cast<double>(half), s.dfm_step[p], 2 * half + 1};
    }
    s.roi_first = sc.roi_first;
    s.roi_last = sc.roi_last;
    return s;
}

// build_ambiguity / split_velocity (search_space.cpp:111-116,149-157)
ltci_ambiguity build_amb(const ltci_scenario& sc) {
    const double va = (kC / sc.radar.fc) * sc.radar.PRF / 2.0;
    return ltci_ambiguity{static_cast<int32_t>(std::floor(sc.bound_lo[0] / va + 0.5)),
                          static_cast<int32_t>(std::floor(sc.bound_hi[0] / va + 0.5))};
}

// wilson_interval (bench.cpp:60-68)
void wilson(int successes, int n, double& lo, double& hi) {
    const double z = 1.959963984540054;
    const double phat = static_cast<double>(successes) / n;
    const double z2n = z * z / n;
    const double center = (phat + z2n / 2.0) / (1.0 + z2n);
    const double half = z * std::sqrt(phat * (1.0 - phat) / n + z2n / (4.0 * n)) / (1.0 + z2n);
    lo = std::max(0.0, center - half);
    hi = std::min(1.0, center + half);
}

// GaussianRng::derive_seed (rng.cpp:38-41)
uint64_t derive_seed(uint64_t seed, uint64_t index) {
    uint64_t s = seed ^ (0x632be59bd9b4e019ULL * (index + 1));
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void synth_device(const ltci_radar& r, int nt, const ltci_target* targets, double2* d_out, cudaStream_t st) {
    if (nt < 0 || nt > LTCI_MAX_TARGETS) throw std::invalid_argument("synthesize: 0..8 targets");
    for (int t = 0; t < nt; ++t)
        if (targets[t].order < 0 || targets[t].order > LTCI_MAX_ORDER)
            throw std::invalid_argument("synthesize: target order must be in 0..4");
    Dev<ltci_target> d_tg(std::max(nt, 1));
    if (nt) PD_CK(cudaMemcpyAsync(d_tg.p, targets, nt * sizeof(ltci_target), cudaMemcpyHostToDevice, st));
    const size_t n = static_cast<size_t>(r.K) * r.M;
    ltcib::synth_kernel<<<grid_for(n), 256, 0, st>>>(r, nt, d_tg.p, d_out);
    PD_CK(cudaGetLastError());
    PD_CK(cudaStreamSynchronize(st));
}

void check_radar(const ltci_radar* p) {
    if (!p) throw std::invalid_argument("null radar");
    if (p->K <= 0 || p->M <= 0 || (p->K & (p->K - 1)) || (p->M & (p->M - 1)))
        throw std::invalid_argument("RadarParams: M and K must be powers of two");
}

struct MapFree {
    void operator()(ltci_detection_map* m) const { ltci_cuda_free_map(m); }
};
struct EngineFree {
    void operator()(ltci_engine* e) const { ltci_engine_destroy(e); }
};

}  // namespace

extern "C" int ltci_cuda_synthesize(const ltci_radar* p, int n_targets, const ltci_target* targets, double* out) {
    return pd_guarded([&] {
        check_radar(p);
        if (!out || (n_targets && !targets)) throw std::invalid_argument("synthesize: null argument");
        const size_t n = static_cast<size_t>(p->K) * p->M;
        Dev<double2> d(n);
        synth_device(*p, n_targets, targets, d.p, nullptr);
        PD_CK(cudaMemcpy(out, d.p, n * sizeof(double2), cudaMemcpyDeviceToHost));
    });
}

extern "C" int ltci_cuda_add_noise(const double* cube, const ltci_radar* p, double sigma2, uint64_t seed,
                                   double* out) {
    return pd_guarded([&] {
        check_radar(p);
        if (!cube || !out) throw std::invalid_argument("add_noise: null argument");
        if (sigma2 < 0) throw std::invalid_argument("add_noise: sigma2 must be >= 0");
        const size_t n = static_cast<size_t>(p->K) * p->M;
        Dev<double2> d_in(n), d_out(n);
        PD_CK(cudaMemcpy(d_in.p, cube, n * sizeof(double2), cudaMemcpyHostToDevice));
        ltcib::noise_kernel<<<grid_for(n), 256>>>(d_in.p, n, sigma2, seed, d_out.p, nullptr);
        PD_CK(cudaGetLastError());
        PD_CK(cudaMemcpy(out, d_out.p, n * sizeof(double2), cudaMemcpyDeviceToHost));
    });
}

extern "C" int ltci_cuda_run_pd(const ltci_scenario* scp, ltci_pd_point* out) {
    return pd_guarded([&] {
        if (!scp || !out) throw std::invalid_argument("run_pd: null argument");
        const ltci_scenario& sc = *scp;
        check_radar(&sc.radar);
        if (sc.trials < 1) throw std::invalid_argument("run_pd: trials must be >= 1");
        if (sc.n_targets < 1 || sc.n_targets > LTCI_MAX_TARGETS)
            throw std::invalid_argument("run_pd: scenario needs a target");
        if (sc.n_snr < 0 || sc.n_snr > LTCI_MAX_SNR) throw std::invalid_argument("run_pd: 0..64 SNR points");
        if (sc.n_detectors < 1 || sc.n_detectors > 5) throw std::invalid_argument("run_pd: 1..5 detectors");
        for (int d = 0; d < sc.n_detectors; ++d)
            if (sc.detectors[d] != LTCI_FD_GRFT && sc.detectors[d] != LTCI_DS_GRFT &&
                sc.detectors[d] != LTCI_DS_KT_MFP)
                throw std::invalid_argument("run_pd: detector not built on the GPU (fd_grft, ds_grft, ds_kt_mfp)");
        struct DeviceRestore {  // the caller's current device is left as it was
            int prev = 0;
            explicit DeviceRestore(int dev) {
                cudaGetDevice(&prev);
                if (dev != prev) PD_CK(cudaSetDevice(dev));
            }
            ~DeviceRestore() { cudaSetDevice(prev); }
        } device_restore(sc.device);

        // build_spaces (bench.cpp:13-21)
        const ltci_single_space single = build_single(sc, 0, sc.radar.K - 1);
        const ltci_dual_space dual = build_dual(sc);
        const ltci_ambiguity amb = build_amb(sc);
        int st_thr = 0;
        const double gamma = ltci_cuda_detection_threshold(&sc.radar, sc.sigma2, sc.pfa, 0, &st_thr);
        pd_rc(st_thr);

        ltci_options opt{};
        opt.retain_threshold = gamma;
        opt.threads = 1;
        opt.keystone_taps = sc.keystone_taps > 0 ? sc.keystone_taps : 8;
        opt.fine_path = LTCI_FINE_AUTO;
        opt.device = sc.device;

        // kLanes (engine set, stream, noisy buffer) triples: trial t runs on lane
        // t % kLanes, so while the host assembles one trial's candidates and runs
        // the success test, the next trials are already queued on the device.
        // One engine per dual-scale detector and lane, reused by every trial.
        constexpr int kLanes = 3;
        struct Lane {
            std::vector<std::unique_ptr<ltci_engine, EngineFree>> eng;
            cudaStream_t st = nullptr;
            int trial = -1;  // trial in flight on this lane
        };
        std::vector<Lane> lanes(kLanes);
        for (auto& ln : lanes) {
            PD_CK(cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking));
            ln.eng.resize(sc.n_detectors);
            for (int d = 0; d < sc.n_detectors; ++d) {
                if (sc.detectors[d] == LTCI_FD_GRFT) continue;
                ltci_engine* e = nullptr;
                const bool kt = sc.detectors[d] == LTCI_DS_KT_MFP;
                pd_rc(ltci_engine_create(&sc.radar, &dual, kt ? &amb : nullptr,
                                         kt ? LTCI_VARIANT_KTMFP : LTCI_VARIANT_GRFT, &opt, 0, -1, &e));
                ln.eng[d].reset(e);
            }
        }
        struct StreamFree {
            std::vector<Lane>* l;
            ~StreamFree() {
                for (auto& ln : *l)
                    if (ln.st) cudaStreamDestroy(ln.st);
            }
        } stream_free{&lanes};

        const size_t n = static_cast<size_t>(sc.radar.K) * sc.radar.M;
        Dev<double2> clean(n);
        std::vector<std::unique_ptr<Dev<float2>>> noisy;
        for (int l = 0; l < kLanes; ++l) noisy.emplace_back(new Dev<float2>(n));
        cudaStream_t st = nullptr;
        const ltci_target& truth = sc.targets[0];
        for (int pt = 0; pt < sc.n_snr; ++pt) {
            // a1_for_snr (bench.cpp:25-27): pulse-compressed SNR 10 log10(K_valid |A1|^2 / sigma2)
            const double a1 = std::sqrt(sc.sigma2 * std::pow(10.0, sc.snr_db[pt] / 10.0) / sc.radar.K_valid);
            std::vector<ltci_target> scaled(sc.targets, sc.targets + sc.n_targets);
            for (auto& t : scaled) {
                t.amp[0] *= a1;
                t.amp[1] *= a1;
            }
            synth_device(sc.radar, sc.n_targets, scaled.data(), clean.p, st);
            std::vector<int> wins(sc.n_detectors, 0);
            // FD-GRFT runs synchronously on the legacy stream; it waits for the lane's noise kernel
            auto collect = [&](int l) {
                Lane& ln = lanes[l];
                for (int d = 0; d < sc.n_detectors; ++d) {
                    std::unique_ptr<ltci_detection_map, MapFree> map;
                    if (sc.detectors[d] == LTCI_FD_GRFT) {
                        PD_CK(cudaStreamSynchronize(ln.st));
                        map.reset(ltcib_fd_grft_device(noisy[l]->p, sc.radar, single, &opt));
                    } else {
                        ltci_detection_map* m = nullptr;
                        pd_rc(ltci_engine_result(ln.eng[d].get(), ln.st, &m));
                        map.reset(m);
                    }
                    const bool kt = sc.detectors[d] == LTCI_DS_KT_MFP;
                    const bool ok = sc.detectors[d] == LTCI_FD_GRFT
                                        ? ltcib_detection_success(map.get(), nullptr, &single, nullptr, truth)
                                        : ltcib_detection_success(map.get(), &dual, nullptr, kt ? &amb : nullptr, truth);
                    wins[d] += ok ? 1 : 0;
                }
                ln.trial = -1;
            };
            for (int trial = 0; trial < sc.trials; ++trial) {
                const int l = trial % kLanes;
                if (lanes[l].trial >= 0) collect(l);
                const uint64_t seed =
                    derive_seed(sc.seed, static_cast<uint64_t>(pt) * static_cast<uint64_t>(sc.trials) + trial);
                ltcib::noise_kernel<<<grid_for(n), 256, 0, lanes[l].st>>>(clean.p, n, sc.sigma2, seed, nullptr,
                                                                          noisy[l]->p);
                PD_CK(cudaGetLastError());
                for (int d = 0; d < sc.n_detectors; ++d)
                    if (sc.detectors[d] != LTCI_FD_GRFT)
                        pd_rc(ltci_engine_run_device(lanes[l].eng[d].get(), noisy[l]->p, lanes[l].st));
                lanes[l].trial = trial;
            }
            for (int k = 0; k < kLanes; ++k) {
                const int l = (sc.trials + k) % kLanes;  // oldest first
                if (lanes[l].trial >= 0) collect(l);
            }
            for (int d = 0; d < sc.n_detectors; ++d) {
                ltci_pd_point& o = out[d * sc.n_snr + pt];
                o.snr_db = sc.snr_db[pt];
                o.trials = sc.trials;
                o.pd = static_cast<double>(wins[d]) / sc.trials;
                wilson(wins[d], sc.trials, o.ci_lo, o.ci_hi);
            }
        }
    });
}
