// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A C-ABI shim over the *unmodified* reference library (compiled from
// /root/reference/proj/src/*.cpp with the namespace renamed to ltci_ref, see
// oracle/Makefile).  It lets the Python tests, the golden-vector generator and
// bench.py's cpu_baseline / --impl reference leg call the reference's own
// code path with the same POD plan structs the CUDA library takes
// (include/ltci_cuda.h).  Only tests/, __graft_entry__.smoke() and bench.py's
// CPU legs load it.
//
// Each entry point names the reference function it forwards to.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "ltci/bench.hpp"
#include "ltci/cube_io.hpp"
#include "ltci/detection.hpp"
#include "ltci/detectors.hpp"
#include "ltci/parallel.hpp"
#include "ltci/rng.hpp"
#include "ltci/signal_model.hpp"
#include "ltci/transforms.hpp"
#include "ltci_cuda.h"

namespace R = ltci_ref;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
    g_err = what ? what : "";
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LTCI_OK;
    } catch (const R::ConditionViolated& e) {
        return fail(LTCI_CONDITION_VIOLATED, e.what());
    } catch (const R::IoError& e) {
        return fail(LTCI_IO_ERROR, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(LTCI_INVALID_ARGUMENT, e.what());
    } catch (const std::out_of_range& e) {
        return fail(LTCI_OUT_OF_RANGE, e.what());
    } catch (const std::bad_alloc& e) {
        return fail(LTCI_BAD_ALLOC, e.what());
    } catch (const std::exception& e) {
        return fail(LTCI_RUNTIME_ERROR, e.what());
    }
}

R::RadarParams radar_of(const ltci_radar& r) {
    R::RadarParams p;
    p.fc = r.fc;
    p.fs = r.fs;
    p.Br = r.Br;
    p.delta_f = r.delta_f;
    p.PRF = r.PRF;
    p.M = r.M;
    p.K = r.K;
    p.K_valid = r.K_valid;
    return p;
}

void radar_to(const R::RadarParams& p, ltci_radar* r) {
    r->fc = p.fc;
    r->fs = p.fs;
    r->Br = p.Br;
    r->delta_f = p.delta_f;
    r->PRF = p.PRF;
    r->M = p.M;
    r->K = p.K;
    r->K_valid = p.K_valid;
}

R::Grid grid_of(const ltci_grid& g) {
    R::Grid out;
    out.start = g.start;
    out.step = g.step;
    out.count = g.count;
    return out;
}

ltci_grid grid_to(const R::Grid& g) { return ltci_grid{g.start, g.step, g.count}; }

R::DualScaleSpace space_of(const ltci_dual_space& s) {
    R::DualScaleSpace d;
    d.params = radar_of(s.radar);
    for (int p = 0; p < s.order; ++p) {
        d.coarse.push_back(grid_of(s.coarse[p]));
        d.fine.push_back(grid_of(s.fine[p]));
        d.steps.rm.push_back(s.rm_step[p]);
        d.steps.dfm.push_back(s.dfm_step[p]);
        d.steps.alpha.push_back(s.alpha[p]);
    }
    d.kappa = s.kappa;
    d.roi.first = s.roi_first;
    d.roi.last = s.roi_last;
    return d;
}

R::SingleScaleSpace single_of(const ltci_single_space& s) {
    R::SingleScaleSpace d;
    d.params = radar_of(s.radar);
    for (int p = 0; p < s.order; ++p) {
        d.c.push_back(grid_of(s.c[p]));
        d.steps.rm.push_back(s.rm_step[p]);
        d.steps.dfm.push_back(s.dfm_step[p]);
        d.steps.alpha.push_back(s.alpha[p]);
    }
    d.roi.first = s.roi_first;
    d.roi.last = s.roi_last;
    return d;
}

void single_to(const R::SingleScaleSpace& d, ltci_single_space* s) {
    std::memset(s, 0, sizeof(*s));
    radar_to(d.params, &s->radar);
    s->order = d.order();
    for (int p = 0; p < d.order() && p < LTCI_MAX_ORDER; ++p) {
        s->c[p] = grid_to(d.c[p]);
        s->rm_step[p] = d.steps.rm[p];
        s->dfm_step[p] = d.steps.dfm[p];
        s->alpha[p] = d.steps.alpha[p];
    }
    s->roi_first = d.roi.first;
    s->roi_last = d.roi.last;
}

void space_to(const R::DualScaleSpace& d, ltci_dual_space* s) {
    std::memset(s, 0, sizeof(*s));
    radar_to(d.params, &s->radar);
    s->order = d.order();
    for (int p = 0; p < d.order() && p < LTCI_MAX_ORDER; ++p) {
        s->coarse[p] = grid_to(d.coarse[p]);
        s->fine[p] = grid_to(d.fine[p]);
        s->rm_step[p] = d.steps.rm[p];
        s->dfm_step[p] = d.steps.dfm[p];
        s->alpha[p] = d.steps.alpha[p];
    }
    s->kappa = d.kappa;
    s->roi_first = d.roi.first;
    s->roi_last = d.roi.last;
}

R::DetectorOptions options_of(const ltci_options* o) {
    R::DetectorOptions opt;
    if (o) {
        opt.retain_threshold = o->retain_threshold;
        opt.keep_dense = o->keep_dense != 0;
        opt.threads = o->threads;
        opt.keystone_taps = o->keystone_taps > 0 ? o->keystone_taps : 8;
        opt.trajectory = static_cast<R::TrajectoryPolicy>(o->trajectory);
    }
    return opt;
}

R::FreqPulseCube cube_of(const double* data, const R::RadarParams& p) {
    R::FreqPulseCube cube(p);
    const std::size_t n = static_cast<std::size_t>(p.K) * p.M;
    for (std::size_t i = 0; i < n; ++i) cube.data[i] = R::cplx(data[2 * i], data[2 * i + 1]);
    return cube;
}

template <typename T>
T* alloc_array(std::size_t n) {
    if (n == 0) return nullptr;
    T* p = static_cast<T*>(std::malloc(n * sizeof(T)));
    if (!p) throw std::bad_alloc();
    return p;
}

ltci_detection_map* map_to(const R::DetectionMap& m) {
    auto* out = static_cast<ltci_detection_map*>(std::calloc(1, sizeof(ltci_detection_map)));
    if (!out) throw std::bad_alloc();
    out->kind = static_cast<int32_t>(m.kind);
    out->n_axes = static_cast<int32_t>(m.axes.size());
    for (std::size_t i = 0; i < m.axes.size() && i < LTCI_MAX_AXES; ++i)
        out->axes[i] = ltci_axis{static_cast<int32_t>(m.axes[i].role), m.axes[i].order, m.axes[i].size};
    out->counters[0] = m.counters.kt;
    out->counters[1] = m.counters.mf;
    out->counters[2] = m.counters.ifft;
    out->counters[3] = m.counters.fft;
    out->retain_threshold = m.retain_threshold;
    out->doppler_first = m.doppler_first;
    out->argmax = m.argmax;
    out->argmax_value[0] = m.argmax_value.real();
    out->argmax_value[1] = m.argmax_value.imag();
    out->n_candidates = m.candidates.size();
    out->cand_index = alloc_array<uint64_t>(m.candidates.size());
    out->cand_value = alloc_array<double>(2 * m.candidates.size());
    for (std::size_t i = 0; i < m.candidates.size(); ++i) {
        out->cand_index[i] = m.candidates[i].first;
        out->cand_value[2 * i] = m.candidates[i].second.real();
        out->cand_value[2 * i + 1] = m.candidates[i].second.imag();
    }
    out->dense_stored = m.dense_stored ? 1 : 0;
    out->dense_count = m.dense.size();
    out->dense = alloc_array<double>(2 * m.dense.size());
    for (std::size_t i = 0; i < m.dense.size(); ++i) {
        out->dense[2 * i] = m.dense[i].real();
        out->dense[2 * i + 1] = m.dense[i].imag();
    }
    return out;
}

void copy_out(const std::vector<R::cplx>& v, double* out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[2 * i] = v[i].real();
        out[2 * i + 1] = v[i].imag();
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_free_map(ltci_detection_map* m) {
    if (!m) return;
    std::free(m->cand_index);
    std::free(m->cand_value);
    std::free(m->dense);
    std::free(m->peak_index);
    std::free(m->peak_value);
    std::free(m);
}

// RadarParams::create (proj/src/radar_params.cpp:10-28)
int ref_radar_create(double fc, double fs, double br, double prf, int M, int K, int k_valid,
                     ltci_radar* out) {
    return guarded([&] { radar_to(R::RadarParams::create(fc, fs, br, prf, M, K, k_valid), out); });
}

// build_dual_scale (proj/src/search_space.cpp:82-109)
int ref_build_dual_scale(const ltci_radar* r, int P, const double* lo, const double* hi,
                         const double* alpha, int roi_first, int roi_last, ltci_dual_space* out) {
    return guarded([&] {
        std::vector<R::Bounds> b;
        for (int p = 0; p < P; ++p) b.push_back(R::Bounds{lo[p], hi[p]});
        std::vector<double> a(alpha, alpha + P);
        space_to(R::build_dual_scale(radar_of(*r), P, b, a, R::RangeRoi{roi_first, roi_last}), out);
    });
}

// build_ambiguity (proj/src/search_space.cpp:111-116)
int ref_build_ambiguity(const ltci_radar* r, double vlo, double vhi, ltci_ambiguity* out) {
    return guarded([&] {
        R::AmbiguitySpace a = R::build_ambiguity(radar_of(*r), R::Bounds{vlo, vhi});
        out->q_min = a.q_min;
        out->q_max = a.q_max;
    });
}

// synthesize_cube + add_noise (proj/src/signal_model.cpp:37-65); coeffs holds
// n_coef motion coefficients c0..c_{n_coef-1} per target.
int ref_synthesize(const ltci_radar* r, int n_targets, const double* amp, const double* coeffs,
                   int n_coef, double sigma2, uint64_t seed, double* out) {
    return guarded([&] {
        R::RadarParams p = radar_of(*r);
        std::vector<R::Target> targets;
        for (int t = 0; t < n_targets; ++t) {
            std::vector<double> c(coeffs + t * n_coef, coeffs + (t + 1) * n_coef);
            targets.push_back(R::Target{R::cplx(amp[2 * t], amp[2 * t + 1]), R::MotionParams(c)});
        }
        R::FreqPulseCube cube = R::synthesize_cube(p, targets);
        if (sigma2 > 0) cube = R::add_noise(cube, sigma2, seed);
        copy_out(cube.data, out);
    });
}

// GaussianRng stream (proj/src/rng.cpp) for pinning the product's numpy port
int ref_rng_circular(uint64_t seed, double variance, int n, double* out) {
    return guarded([&] {
        R::GaussianRng rng(seed);
        for (int i = 0; i < n; ++i) {
            R::cplx v = rng.circular_normal(variance);
            out[2 * i] = v.real();
            out[2 * i + 1] = v.imag();
        }
    });
}

uint64_t ref_derive_seed(uint64_t seed, uint64_t index) { return R::GaussianRng::derive_seed(seed, index); }

// ds_grft (proj/src/detectors.cpp:414-449)
int ref_ds_grft(const double* cube, const ltci_radar* r, const ltci_dual_space* s,
                const ltci_options* o, ltci_detection_map** out) {
    return guarded([&] {
        R::FreqPulseCube c = cube_of(cube, radar_of(*r));
        *out = map_to(R::ds_grft(c, space_of(*s), options_of(o)));
    });
}

// ds_kt_mfp (proj/src/detectors.cpp:451-481)
int ref_ds_kt_mfp(const double* cube, const ltci_radar* r, const ltci_ambiguity* a,
                  const ltci_dual_space* s, const ltci_options* o, ltci_detection_map** out) {
    return guarded([&] {
        R::FreqPulseCube c = cube_of(cube, radar_of(*r));
        R::AmbiguitySpace amb;
        amb.q_min = a->q_min;
        amb.q_max = a->q_max;
        *out = map_to(R::ds_kt_mfp(c, amb, space_of(*s), options_of(o)));
    });
}

// keystone (proj/src/transforms.cpp:96-130)
int ref_keystone(const double* cube, const ltci_radar* r, int taps, double* out) {
    return guarded([&] { copy_out(R::keystone(cube_of(cube, radar_of(*r)), taps).data, out); });
}

// range_fft / range_ifft (proj/src/signal_model.cpp:85-107)
int ref_range_fft(const double* cube, const ltci_radar* r, double* out) {
    return guarded([&] {
        const R::RadarParams p = radar_of(*r);
        R::RangePulseCube c(p);
        std::memcpy(c.data.data(), cube, c.data.size() * sizeof(R::cplx));
        copy_out(R::range_fft(c).data, out);
    });
}

int ref_range_ifft(const double* cube, const ltci_radar* r, double* out) {
    return guarded([&] { copy_out(R::range_ifft(cube_of(cube, radar_of(*r))).data, out); });
}

// mgift (proj/src/transforms.cpp:157-173)
int ref_mgift(const double* cube, const ltci_radar* r, const double* ctilde, int n, int variant,
              double* out) {
    return guarded([&] {
        std::vector<double> c(ctilde, ctilde + n);
        R::DetectorVariant v = variant == LTCI_VARIANT_KTMFP ? R::DetectorVariant::KtMfp
                                                             : R::DetectorVariant::Grft;
        copy_out(R::mgift(cube_of(cube, radar_of(*r)), c, v).data, out);
    });
}

// gft (proj/src/transforms.cpp:180-214); rows is an N0 x M range-pulse cube
int ref_gft(const double* rows, const ltci_radar* r, const double* fine, int n_fine, int roi_first,
            int roi_last, double* out) {
    return guarded([&] {
        R::RadarParams p = radar_of(*r);
        R::RangePulseCube rp(p);
        const std::size_t n = static_cast<std::size_t>(p.K) * p.M;
        for (std::size_t i = 0; i < n; ++i) rp.data[i] = R::cplx(rows[2 * i], rows[2 * i + 1]);
        std::vector<double> f(fine, fine + n_fine);
        copy_out(R::gft(rp, f, R::RangeRoi{roi_first, roi_last}).data, out);
    });
}

// fd_grft_point / kt_mfp_point (proj/src/detectors.cpp:491-537)
int ref_fd_grft_point(const double* cube, const ltci_radar* r, const double* ctilde, int n,
                      int range_bin, double* out) {
    return guarded([&] {
        std::vector<double> c(ctilde, ctilde + n);
        R::cplx v = R::fd_grft_point(cube_of(cube, radar_of(*r)), c, range_bin);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

int ref_kt_mfp_point(const double* keystoned, const ltci_radar* r, int q, double c2, int range_bin,
                     int doppler_bin, double* out) {
    return guarded([&] {
        R::cplx v = R::kt_mfp_point(cube_of(keystoned, radar_of(*r)), q, c2, range_bin, doppler_bin);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

// detection_threshold (proj/src/detectors.cpp:483-489)
int ref_detection_threshold(const ltci_radar* r, double sigma2, double pfa, int bins, double* out) {
    return guarded([&] { *out = R::detection_threshold(radar_of(*r), sigma2, pfa, bins); });
}

// Per ROI range cell peak map of the dual-scale cascade, computed with the
// reference's own public kernels in the control flow of run_dual_scale
// (proj/src/detectors.cpp:356-407): per coarse cell mgift once, per fine cell
// gft, then every (row, Doppler-in-window) cell is reduced per row with the
// UnitScan tie-break (magnitude desc, flat index asc; detectors.cpp:23-31).
// The reference itself has no per-row output; this only restates its loop.
int ref_peak_map(const double* cube, const ltci_radar* r, const ltci_ambiguity* a,
                 const ltci_dual_space* s, int variant, int taps, int threads, uint64_t* peak_idx,
                 double* peak_val) {
    return guarded([&] {
        R::RadarParams p = radar_of(*r);
        R::DualScaleSpace space = space_of(*s);
        R::FreqPulseCube input = cube_of(cube, p);
        const bool kt = variant == LTCI_VARIANT_KTMFP;
        const int M = p.M;
        const int Rn = space.roi.count();
        std::vector<R::Grid> coarse_axes, fine_axes;
        int dop_first = 0, dop_count = M;
        R::AmbiguitySpace amb;
        if (kt) {
            amb.q_min = a->q_min;
            amb.q_max = a->q_max;
            coarse_axes = {space.coarse[1]};
            fine_axes = {space.fine[1]};
            input = R::keystone(input, taps > 0 ? taps : 8);
        } else {
            double dop_bin = p.Va() / M;
            int keep = static_cast<int>(std::ceil(space.kappa * space.steps.rm[0] / 2.0 / dop_bin - 1e-9));
            keep = std::min(keep, M / 2 - 1);
            coarse_axes = space.coarse;
            for (int ord = 2; ord <= space.order(); ++ord) fine_axes.push_back(space.fine[ord - 1]);
            dop_first = M / 2 - keep;
            dop_count = 2 * keep + 1;
        }
        std::uint64_t coarse_cells = 1, fine_cells = 1;
        for (const R::Grid& g : coarse_axes) coarse_cells *= static_cast<std::uint64_t>(g.count);
        if (kt) coarse_cells *= static_cast<std::uint64_t>(amb.count());
        for (const R::Grid& g : fine_axes) fine_cells *= static_cast<std::uint64_t>(g.count);

        struct Best {
            double mag = -1;
            std::uint64_t idx = 0;
            R::cplx val;
        };
        std::vector<std::vector<Best>> per_unit(coarse_cells, std::vector<Best>(Rn));
        R::parallel_for(coarse_cells, threads, [&](std::size_t cidx) {
            std::uint64_t rem = cidx;
            std::vector<int> ci(coarse_axes.size());
            for (std::size_t i = coarse_axes.size(); i-- > 0;) {
                ci[i] = static_cast<int>(rem % static_cast<std::uint64_t>(coarse_axes[i].count));
                rem /= static_cast<std::uint64_t>(coarse_axes[i].count);
            }
            std::vector<double> coarse_vals;
            if (kt) {
                coarse_vals = {static_cast<double>(amb.q_of(static_cast<int>(rem))),
                               coarse_axes[0].value(ci[0])};
            } else {
                for (std::size_t i = 0; i < coarse_axes.size(); ++i)
                    coarse_vals.push_back(coarse_axes[i].value(ci[i]));
            }
            R::RangePulseCube mg = R::mgift(input, coarse_vals,
                                            kt ? R::DetectorVariant::KtMfp : R::DetectorVariant::Grft);
            std::vector<Best>& best = per_unit[cidx];
            for (std::uint64_t fidx = 0; fidx < fine_cells; ++fidx) {
                std::uint64_t frem = fidx;
                std::vector<int> fi(fine_axes.size());
                for (std::size_t i = fine_axes.size(); i-- > 0;) {
                    fi[i] = static_cast<int>(frem % static_cast<std::uint64_t>(fine_axes[i].count));
                    frem /= static_cast<std::uint64_t>(fine_axes[i].count);
                }
                std::vector<double> fine_scaled(fine_axes.size());
                for (std::size_t i = 0; i < fine_axes.size(); ++i)
                    fine_scaled[i] = space.kappa * fine_axes[i].value(fi[i]);
                R::RangeDopplerMap rd = R::gft(mg, fine_scaled, space.roi);
                std::uint64_t base = (cidx * fine_cells + fidx) * static_cast<std::uint64_t>(Rn) * dop_count;
                for (int rr = 0; rr < Rn; ++rr)
                    for (int j = 0; j < dop_count; ++j) {
                        std::uint64_t idx = base + static_cast<std::uint64_t>(rr) * dop_count + j;
                        R::cplx v = rd.at(rr, dop_first + j);
                        double m = std::abs(v);
                        if (m > best[rr].mag || (m == best[rr].mag && idx < best[rr].idx)) {
                            best[rr].mag = m;
                            best[rr].idx = idx;
                            best[rr].val = v;
                        }
                    }
            }
        });
        for (int rr = 0; rr < Rn; ++rr) {
            Best b;
            for (std::uint64_t c = 0; c < coarse_cells; ++c) {
                const Best& u = per_unit[c][rr];
                if (u.mag > b.mag || (u.mag == b.mag && u.idx < b.idx)) b = u;
            }
            peak_idx[rr] = b.idx;
            peak_val[2 * rr] = b.val.real();
            peak_val[2 * rr + 1] = b.val.imag();
        }
    });
}

// extract_detections (proj/src/detection.cpp:158-244) on a map given as a
// candidate list; returns up to max_out detections as
// (statistic, c0, c1, c2, c3, flat index) rows.
int ref_extract_ds(const ltci_detection_map* m, const ltci_dual_space* s, const ltci_ambiguity* a,
                   double gamma, int max_out, double* rows, int* n_out) {
    return guarded([&] {
        R::DetectionMap map;
        map.kind = static_cast<R::DetectorKind>(m->kind);
        map.params = radar_of(s->radar);
        for (int i = 0; i < m->n_axes; ++i)
            map.axes.push_back(R::AxisDesc{static_cast<R::AxisDesc::Role>(m->axes[i].role),
                                           m->axes[i].order, m->axes[i].size});
        map.retain_threshold = m->retain_threshold;
        map.doppler_first = m->doppler_first;
        map.dual = space_of(*s);
        if (a) {
            R::AmbiguitySpace amb;
            amb.q_min = a->q_min;
            amb.q_max = a->q_max;
            map.amb = amb;
        }
        for (std::uint64_t i = 0; i < m->n_candidates; ++i)
            map.candidates.emplace_back(m->cand_index[i],
                                        R::cplx(m->cand_value[2 * i], m->cand_value[2 * i + 1]));
        std::vector<R::Detection> dets = R::extract_detections(map, gamma);
        int n = std::min<int>(max_out, static_cast<int>(dets.size()));
        for (int i = 0; i < n; ++i) {
            double* row = rows + 6 * i;
            row[0] = dets[i].statistic;
            for (int k = 0; k < 4; ++k)
                row[1 + k] = k < static_cast<int>(dets[i].estimate.c.size()) ? dets[i].estimate.c[k] : 0.0;
            row[5] = static_cast<double>(map.encode(dets[i].cell));
        }
        *n_out = static_cast<int>(dets.size());
    });
}

// write_cube_file (proj/src/cube_io.cpp:66-119) of a CubeFile built field by field
int ref_write_cube_file(const char* path, const ltci_cube_header* h, const double* data) {
    return guarded([&] {
        R::CubeFile f;
        f.domain = static_cast<std::uint8_t>(h->domain);
        f.params = radar_of(h->radar);
        f.sigma2 = h->sigma2;
        const std::size_t n = static_cast<std::size_t>(h->radar.K) * h->radar.M;
        f.data.resize(n);
        for (std::size_t i = 0; i < n; ++i) f.data[i] = R::cplx(data[2 * i], data[2 * i + 1]);
        R::write_cube_file(path, f);
    });
}

// read_cube_file (proj/src/cube_io.cpp:121-179)
int ref_read_cube_file(const char* path, ltci_cube_header* h, double* out, uint64_t cap) {
    return guarded([&] {
        R::CubeFile f = R::read_cube_file(path);
        h->domain = f.domain;
        radar_to(f.params, &h->radar);
        h->sigma2 = f.sigma2;
        if (cap < 2 * f.data.size()) throw std::invalid_argument("ref_read_cube_file: buffer too small");
        copy_out(f.data, out);
    });
}

// build_single_scale (proj/src/search_space.cpp:69-79)
int ref_build_single_scale(const ltci_radar* r, int P, const double* lo, const double* hi, const double* alpha,
                           int roi_first, int roi_last, ltci_single_space* out) {
    return guarded([&] {
        std::vector<R::Bounds> b(P);
        for (int p = 0; p < P; ++p) b[p] = R::Bounds{lo[p], hi[p]};
        std::vector<double> al(alpha, alpha + P);
        single_to(R::build_single_scale(radar_of(*r), P, b, al, R::RangeRoi{roi_first, roi_last}), out);
    });
}

// fd_grft (proj/src/detectors.cpp:105-197)
int ref_fd_grft(const double* cube, const ltci_radar* r, const ltci_single_space* s, const ltci_options* o,
                ltci_detection_map** out) {
    return guarded([&] {
        R::FreqPulseCube c = cube_of(cube, radar_of(*r));
        *out = map_to(R::fd_grft(c, single_of(*s), options_of(o)));
    });
}

// td_grft (proj/src/detectors.cpp:199-264): range-pulse cube in, std::out_of_range under the Error policy
int ref_td_grft(const double* cube, const ltci_radar* r, const ltci_single_space* s, const ltci_options* o,
                ltci_detection_map** out) {
    return guarded([&] {
        R::RangePulseCube c(radar_of(*r));
        const std::size_t n = static_cast<std::size_t>(r->K) * r->M;
        for (std::size_t i = 0; i < n; ++i) c.data[i] = R::cplx(cube[2 * i], cube[2 * i + 1]);
        *out = map_to(R::td_grft(c, single_of(*s), options_of(o)));
    });
}

// kt_mfp (proj/src/detectors.cpp:266-326)
int ref_kt_mfp(const double* cube, const ltci_radar* r, const ltci_ambiguity* a, const ltci_single_space* s,
               const ltci_options* o, ltci_detection_map** out) {
    return guarded([&] {
        R::FreqPulseCube c = cube_of(cube, radar_of(*r));
        R::AmbiguitySpace amb;
        amb.q_min = a->q_min;
        amb.q_max = a->q_max;
        *out = map_to(R::kt_mfp(c, amb, single_of(*s), options_of(o)));
    });
}

// extract_detections (proj/src/detection.cpp:158-244) on a single-scale map
int ref_extract_single(const ltci_detection_map* m, const ltci_single_space* s, double gamma, int max_out,
                       double* rows, int* n_out) {
    return guarded([&] {
        R::DetectionMap map;
        map.kind = static_cast<R::DetectorKind>(m->kind);
        map.params = radar_of(s->radar);
        for (int i = 0; i < m->n_axes; ++i)
            map.axes.push_back(R::AxisDesc{static_cast<R::AxisDesc::Role>(m->axes[i].role),
                                           m->axes[i].order, m->axes[i].size});
        map.retain_threshold = m->retain_threshold;
        map.single = single_of(*s);
        for (std::uint64_t i = 0; i < m->n_candidates; ++i)
            map.candidates.emplace_back(m->cand_index[i],
                                        R::cplx(m->cand_value[2 * i], m->cand_value[2 * i + 1]));
        std::vector<R::Detection> dets = R::extract_detections(map, gamma);
        int n = std::min<int>(max_out, static_cast<int>(dets.size()));
        for (int i = 0; i < n; ++i) {
            double* row = rows + 6 * i;
            row[0] = dets[i].statistic;
            for (int k = 0; k < 4; ++k)
                row[1 + k] = k < static_cast<int>(dets[i].estimate.c.size()) ? dets[i].estimate.c[k] : 0.0;
            row[5] = static_cast<double>(map.encode(dets[i].cell));
        }
        *n_out = static_cast<int>(dets.size());
    });
}

// run_pd (proj/src/bench.cpp:72-124) on a Scenario built field by field
int ref_run_pd(const ltci_scenario* sc, int threads, ltci_pd_point* out) {
    return guarded([&] {
        R::Scenario s;
        s.params = radar_of(sc->radar);
        for (int t = 0; t < sc->n_targets; ++t) {
            const ltci_target& tg = sc->targets[t];
            std::vector<double> c(tg.c, tg.c + tg.order + 1);
            s.targets.push_back(R::Target{R::cplx(tg.amp[0], tg.amp[1]), R::MotionParams(c)});
        }
        s.snr_db.assign(sc->snr_db, sc->snr_db + sc->n_snr);
        s.trials = sc->trials;
        s.pfa = sc->pfa;
        s.sigma2 = sc->sigma2;
        s.seed = sc->seed;
        for (int d = 0; d < sc->n_detectors; ++d) s.detectors.push_back(static_cast<R::DetectorKind>(sc->detectors[d]));
        s.P = sc->P;
        for (int p = 0; p < sc->P; ++p) {
            s.bounds.push_back(R::Bounds{sc->bound_lo[p], sc->bound_hi[p]});
            s.alpha.push_back(sc->alpha[p]);
        }
        s.roi = R::RangeRoi{sc->roi_first, sc->roi_last};
        s.keystone_taps = sc->keystone_taps;
        s.threads = threads;
        std::vector<R::PdCurve> curves = R::run_pd(s);
        for (std::size_t d = 0; d < curves.size(); ++d)
            for (std::size_t i = 0; i < curves[d].points.size(); ++i) {
                const R::PdPoint& q = curves[d].points[i];
                out[d * sc->n_snr + i] = ltci_pd_point{q.snr_db, q.pd, q.trials, q.ci_lo, q.ci_hi};
            }
    });
}

int ref_resolve_threads(int requested) { return R::resolve_threads(requested); }

}  // extern "C"
