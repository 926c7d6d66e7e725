// dropin.cpp -- ltci::ds_grft / ltci::ds_kt_mfp / ltci::fd_grft / ltci::td_grft / ltci::kt_mfp on the
// B200 (libltci_b200.so): the five detectors of proj/include/ltci/detectors.hpp.
//
// Same signatures, argument meaning and exceptions as the reference
// (proj/include/ltci/detectors.hpp:42-48, proj/src/detectors.cpp:414-481):
// std::invalid_argument for radar mismatch / order / ROI problems,
// std::bad_alloc when the retained cells cannot be held, std::runtime_error
// for device failures.  The body marshals the reference types into the POD
// plan of ltci_cuda.h, runs the CUDA engine, and copies the library-owned
// result into a DetectionMap returned by value.

#include <cstring>
#include <new>

#include "ltci_b200/ltci.hpp"
#include "ltci_cuda.h"

namespace {

ltci_radar to_c(const ltci::RadarParams& p) {
    ltci_radar r;
    r.fc = p.fc;
    r.fs = p.fs;
    r.Br = p.Br;
    r.delta_f = p.delta_f;
    r.PRF = p.PRF;
    r.M = p.M;
    r.K = p.K;
    r.K_valid = p.K_valid;
    return r;
}

ltci_dual_space to_c(const ltci::DualScaleSpace& s) {
    ltci_dual_space d;
    std::memset(&d, 0, sizeof(d));
    d.radar = to_c(s.params);
    if (s.coarse.size() > LTCI_MAX_ORDER || s.fine.size() != s.coarse.size())
        throw std::invalid_argument("ds detector: space order must be 1..4 with matching fine grids");
    d.order = static_cast<int32_t>(s.coarse.size());
    for (int p = 0; p < d.order; ++p) {
        d.coarse[p] = ltci_grid{s.coarse[p].start, s.coarse[p].step, s.coarse[p].count};
        d.fine[p] = ltci_grid{s.fine[p].start, s.fine[p].step, s.fine[p].count};
        d.rm_step[p] = p < static_cast<int>(s.steps.rm.size()) ? s.steps.rm[p] : 0.0;
        d.dfm_step[p] = p < static_cast<int>(s.steps.dfm.size()) ? s.steps.dfm[p] : 0.0;
        d.alpha[p] = p < static_cast<int>(s.steps.alpha.size()) ? s.steps.alpha[p] : 0.0;
    }
    if (s.steps.rm.empty()) throw std::invalid_argument("ds detector: space has no step sizes");
    d.kappa = s.kappa;
    d.roi_first = s.roi.first;
    d.roi_last = s.roi.last;
    return d;
}

ltci_single_space to_c(const ltci::SingleScaleSpace& s) {
    ltci_single_space d;
    std::memset(&d, 0, sizeof(d));
    d.radar = to_c(s.params);
    if (s.c.empty() || s.c.size() > LTCI_MAX_ORDER) throw std::invalid_argument("fd_grft: space order must be 1..4");
    d.order = static_cast<int32_t>(s.c.size());
    for (int p = 0; p < d.order; ++p) {
        d.c[p] = ltci_grid{s.c[p].start, s.c[p].step, s.c[p].count};
        d.rm_step[p] = p < static_cast<int>(s.steps.rm.size()) ? s.steps.rm[p] : 0.0;
        d.dfm_step[p] = p < static_cast<int>(s.steps.dfm.size()) ? s.steps.dfm[p] : 0.0;
        d.alpha[p] = p < static_cast<int>(s.steps.alpha.size()) ? s.steps.alpha[p] : 0.0;
    }
    d.roi_first = s.roi.first;
    d.roi_last = s.roi.last;
    return d;
}

ltci_options to_c(const ltci::DetectorOptions& o) {
    ltci_options c;
    std::memset(&c, 0, sizeof(c));
    c.retain_threshold = o.retain_threshold;
    c.keep_dense = o.keep_dense ? 1 : 0;
    c.threads = o.threads;
    c.keystone_taps = o.keystone_taps;
    c.trajectory = static_cast<int32_t>(o.trajectory);
    c.fine_path = LTCI_FINE_AUTO;
    c.device = 0;
    return c;
}

[[noreturn]] void rethrow(int rc) {
    const char* msg = ltci_cuda_last_error();
    switch (rc) {
        case LTCI_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case LTCI_CONDITION_VIOLATED: throw ltci::ConditionViolated(msg);
        case LTCI_BAD_ALLOC: throw std::bad_alloc();
        case LTCI_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

struct MapGuard {
    ltci_detection_map* m = nullptr;
    ~MapGuard() { ltci_cuda_free_map(m); }
};

ltci::DetectionMap to_cpp(const ltci_detection_map& c, const ltci::RadarParams& params) {
    ltci::DetectionMap m;
    m.kind = static_cast<ltci::DetectorKind>(c.kind);
    m.params = params;
    for (int i = 0; i < c.n_axes; ++i)
        m.axes.push_back(ltci::AxisDesc{static_cast<ltci::AxisDesc::Role>(c.axes[i].role), c.axes[i].order,
                                        c.axes[i].size});
    m.counters.kt = c.counters[0];
    m.counters.mf = c.counters[1];
    m.counters.ifft = c.counters[2];
    m.counters.fft = c.counters[3];
    m.retain_threshold = c.retain_threshold;
    m.doppler_first = c.doppler_first;
    m.argmax = c.argmax;
    m.argmax_value = ltci::cplx(c.argmax_value[0], c.argmax_value[1]);
    m.candidates.reserve(c.n_candidates);
    for (std::uint64_t i = 0; i < c.n_candidates; ++i)
        m.candidates.emplace_back(c.cand_index[i], ltci::cplx(c.cand_value[2 * i], c.cand_value[2 * i + 1]));
    m.dense_stored = c.dense_stored != 0;
    if (m.dense_stored) {
        m.dense.resize(c.dense_count);
        for (std::uint64_t i = 0; i < c.dense_count; ++i) m.dense[i] = ltci::cplx(c.dense[2 * i], c.dense[2 * i + 1]);
    }
    return m;
}

}  // namespace

namespace ltci {

DetectionMap ds_grft(const FreqPulseCube& cube, const DualScaleSpace& space, const DetectorOptions& opt) {
    return ltci_b200::ds_grft_with_peaks(cube, space, opt, nullptr);
}

// proj/src/detectors.cpp:105-197
DetectionMap fd_grft(const FreqPulseCube& cube, const SingleScaleSpace& space, const DetectorOptions& opt) {
    const ltci_radar r = to_c(cube.params);
    const ltci_single_space s = to_c(space);
    const ltci_options o = to_c(opt);
    MapGuard g;
    const std::size_t n = static_cast<std::size_t>(cube.params.K) * cube.params.M;
    if (cube.data.size() != n) throw std::invalid_argument("detector: cube data size does not match K*M");
    const int rc = ltci_cuda_fd_grft(reinterpret_cast<const double*>(cube.data.data()), &r, &s, &o, &g.m);
    if (rc != LTCI_OK) rethrow(rc);
    DetectionMap m = to_cpp(*g.m, cube.params);
    m.single = space;
    return m;
}

// proj/src/detectors.cpp:199-264
DetectionMap td_grft(const RangePulseCube& cube, const SingleScaleSpace& space, const DetectorOptions& opt) {
    const ltci_radar r = to_c(cube.params);
    const ltci_single_space s = to_c(space);
    const ltci_options o = to_c(opt);
    MapGuard g;
    const std::size_t n = static_cast<std::size_t>(cube.params.K) * cube.params.M;
    if (cube.data.size() != n) throw std::invalid_argument("detector: cube data size does not match K*M");
    const int rc = ltci_cuda_td_grft(reinterpret_cast<const double*>(cube.data.data()), &r, &s, &o, &g.m);
    if (rc != LTCI_OK) rethrow(rc);
    DetectionMap m = to_cpp(*g.m, cube.params);
    m.single = space;
    return m;
}

// proj/src/detectors.cpp:266-326
DetectionMap kt_mfp(const FreqPulseCube& cube, const AmbiguitySpace& amb, const SingleScaleSpace& space,
                    const DetectorOptions& opt) {
    const ltci_radar r = to_c(cube.params);
    if (space.c.size() != 2) throw std::invalid_argument("kt_mfp: needs a P = 2 search space");
    const ltci_single_space s = to_c(space);
    const ltci_options o = to_c(opt);
    const ltci_ambiguity a{amb.q_min, amb.q_max};
    MapGuard g;
    const std::size_t n = static_cast<std::size_t>(cube.params.K) * cube.params.M;
    if (cube.data.size() != n) throw std::invalid_argument("detector: cube data size does not match K*M");
    const int rc = ltci_cuda_kt_mfp(reinterpret_cast<const double*>(cube.data.data()), &r, &a, &s, &o, &g.m);
    if (rc != LTCI_OK) rethrow(rc);
    DetectionMap m = to_cpp(*g.m, cube.params);
    m.single = space;
    m.amb = amb;
    return m;
}

DetectionMap ds_kt_mfp(const FreqPulseCube& cube, const AmbiguitySpace& amb, const DualScaleSpace& space,
                       const DetectorOptions& opt) {
    const ltci_radar r = to_c(cube.params);
    const ltci_dual_space s = to_c(space);
    const ltci_options o = to_c(opt);
    const ltci_ambiguity a{amb.q_min, amb.q_max};
    MapGuard g;
    const std::size_t n = static_cast<std::size_t>(cube.params.K) * cube.params.M;
    if (cube.data.size() != n) throw std::invalid_argument("detector: cube data size does not match K*M");
    const int rc = ltci_cuda_ds_kt_mfp(reinterpret_cast<const double*>(cube.data.data()), &r, &a, &s, &o, &g.m);
    if (rc != LTCI_OK) rethrow(rc);
    DetectionMap m = to_cpp(*g.m, cube.params);
    m.dual = space;
    m.amb = amb;
    return m;
}

}  // namespace ltci

namespace ltci_b200 {

ltci::DetectionMap ds_grft_with_peaks(const ltci::FreqPulseCube& cube, const ltci::DualScaleSpace& space,
                                      const ltci::DetectorOptions& opt, PeakMap* peaks) {
    const ltci_radar r = to_c(cube.params);
    const ltci_dual_space s = to_c(space);
    const ltci_options o = to_c(opt);
    MapGuard g;
    const std::size_t n = static_cast<std::size_t>(cube.params.K) * cube.params.M;
    if (cube.data.size() != n) throw std::invalid_argument("detector: cube data size does not match K*M");
    const int rc = ltci_cuda_ds_grft(reinterpret_cast<const double*>(cube.data.data()), &r, &s, &o, &g.m);
    if (rc != LTCI_OK) rethrow(rc);
    ltci::DetectionMap m = to_cpp(*g.m, cube.params);
    m.dual = space;
    if (peaks) {
        peaks->index.assign(g.m->peak_index, g.m->peak_index + g.m->n_rows);
        peaks->value.resize(g.m->n_rows);
        for (int i = 0; i < g.m->n_rows; ++i)
            peaks->value[i] = ltci::cplx(g.m->peak_value[2 * i], g.m->peak_value[2 * i + 1]);
    }
    return m;
}

}  // namespace ltci_b200
