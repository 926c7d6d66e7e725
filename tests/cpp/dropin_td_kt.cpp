// C++ callers of the drop-in's ltci::td_grft / ltci::kt_mfp (libltci_b200.so):
// the marshalling of RangePulseCube / SingleScaleSpace / DetectorOptions, the
// map returned by value, and the exception types -- checked against the same
// searches through the C-ABI (ltci_cuda_td_grft / ltci_cuda_kt_mfp), which the
// Python tests pin to the reference.  Built and run by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "ltci_b200/ltci.hpp"
#include "ltci_cuda.h"

namespace {

int fails = 0;
#define CHECK(cond)                                              \
    do {                                                         \
        if (!(cond)) {                                           \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
            ++fails;                                             \
        }                                                        \
    } while (0)

ltci::RadarParams radar() {
    ltci::RadarParams p;
    p.fc = 3e9;
    p.fs = 20e6;
    p.PRF = 1000.0;
    p.M = 64;
    p.K = 128;
    p.delta_f = p.fs / p.K;
    p.K_valid = p.K;
    p.Br = p.delta_f * p.K_valid;
    return p;
}

ltci_radar to_c(const ltci::RadarParams& p) {
    return ltci_radar{p.fc, p.fs, p.Br, p.delta_f, p.PRF, p.M, p.K, p.K_valid};
}

// a deterministic full-band cube (splitmix-style hash): values in [-1, 1)
std::vector<ltci::cplx> noise(const ltci::RadarParams& p) {
    std::vector<ltci::cplx> d(static_cast<std::size_t>(p.K) * p.M);
    std::uint64_t s = 0x9E3779B97F4A7C15ull;
    auto next = [&] {
        s += 0x9E3779B97F4A7C15ull;
        std::uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        return static_cast<double>(z >> 11) / 9007199254740992.0 * 2.0 - 1.0;
    };
    for (auto& v : d) v = ltci::cplx(static_cast<float>(next()), static_cast<float>(next()));
    return d;
}

ltci::SingleScaleSpace space(const ltci::RadarParams& p, double vmax, int nv, double amax, int na) {
    ltci::SingleScaleSpace s;
    s.params = p;
    s.steps.rm = {p.delta_R() / p.T(), p.delta_R() / (p.T() * p.T())};
    s.steps.dfm = {p.lambda() / (2 * p.T()), p.lambda() / (p.T() * p.T())};
    s.steps.alpha = {0.5, 0.5};
    s.c = {ltci::Grid{-vmax, 2 * vmax / (nv - 1), nv}, ltci::Grid{-amax, na > 1 ? 2 * amax / (na - 1) : 1.0, na}};
    s.roi = ltci::RangeRoi{3, p.K - 4};
    return s;
}

ltci_single_space to_c(const ltci::SingleScaleSpace& s) {
    ltci_single_space d;
    std::memset(&d, 0, sizeof(d));
    d.radar = to_c(s.params);
    d.order = static_cast<int>(s.c.size());
    for (int i = 0; i < d.order; ++i) {
        d.c[i] = ltci_grid{s.c[i].start, s.c[i].step, s.c[i].count};
        d.rm_step[i] = s.steps.rm[i];
        d.dfm_step[i] = s.steps.dfm[i];
        d.alpha[i] = s.steps.alpha[i];
    }
    d.roi_first = s.roi.first;
    d.roi_last = s.roi.last;
    return d;
}

void same_map(const ltci::DetectionMap& m, const ltci_detection_map& c, ltci::DetectorKind kind) {
    CHECK(m.kind == kind);
    CHECK(static_cast<int>(m.axes.size()) == c.n_axes);
    for (int i = 0; i < c.n_axes && i < static_cast<int>(m.axes.size()); ++i)
        CHECK(static_cast<int>(m.axes[i].role) == c.axes[i].role && m.axes[i].order == c.axes[i].order &&
              m.axes[i].size == c.axes[i].size);
    CHECK(m.counters.kt == c.counters[0] && m.counters.mf == c.counters[1] && m.counters.ifft == c.counters[2] &&
          m.counters.fft == c.counters[3]);
    CHECK(m.argmax == c.argmax);
    CHECK(m.argmax_value == ltci::cplx(c.argmax_value[0], c.argmax_value[1]));
    CHECK(m.candidates.size() == c.n_candidates && c.n_candidates > 0);
    for (std::size_t i = 0; i < m.candidates.size() && i < c.n_candidates; ++i)
        CHECK(m.candidates[i].first == c.cand_index[i] &&
              m.candidates[i].second == ltci::cplx(c.cand_value[2 * i], c.cand_value[2 * i + 1]));
    CHECK(m.dense_stored && m.dense.size() == c.dense_count);
    for (std::size_t i = 0; i < m.dense.size() && i < c.dense_count; i += 97)
        CHECK(m.dense[i] == ltci::cplx(c.dense[2 * i], c.dense[2 * i + 1]));
}

}  // namespace

int main() {
    const ltci::RadarParams p = radar();
    // ---- td_grft: wrap policy, dense + candidates, against the C-ABI
    ltci::RangePulseCube rc{p, noise(p)};
    ltci::SingleScaleSpace s = space(p, 2000.0, 41, 40.0, 5);  // +-17 range cells over the CPI: leaves the cube
    ltci::DetectorOptions o;
    o.retain_threshold = 9.0;
    o.keep_dense = true;
    o.trajectory = ltci::TrajectoryPolicy::Wrap;
    const ltci::DetectionMap m = ltci::td_grft(rc, s, o);
    CHECK(m.single.has_value() && m.single->c.size() == 2);
    {
        const ltci_radar r = to_c(p);
        const ltci_single_space cs = to_c(s);
        ltci_options co{};
        co.retain_threshold = o.retain_threshold;
        co.keep_dense = 1;
        co.keystone_taps = 8;
        co.trajectory = 1;
        ltci_detection_map* cm = nullptr;
        CHECK(ltci_cuda_td_grft(reinterpret_cast<const double*>(rc.data.data()), &r, &cs, &co, &cm) == LTCI_OK);
        if (cm) same_map(m, *cm, ltci::DetectorKind::TdGrft);
        ltci_cuda_free_map(cm);
    }
    // ---- td_grft: the Error policy raises std::out_of_range with the reference's message
    o.trajectory = ltci::TrajectoryPolicy::Error;
    bool thrown = false;
    try {
        ltci::td_grft(rc, s, o);
    } catch (const std::out_of_range& e) {
        thrown = std::strstr(e.what(), "trajectory leaves the cube") != nullptr;
    }
    CHECK(thrown);
    // ---- kt_mfp: against the C-ABI; a P = 1 space is std::invalid_argument
    ltci::FreqPulseCube fc{p, noise(p)};
    ltci::AmbiguitySpace amb{-1, 1};
    ltci::SingleScaleSpace sk = space(p, 10.0, 3, 30.0, 4);
    o.trajectory = ltci::TrajectoryPolicy::ZeroOutside;
    o.retain_threshold = 25.0;
    const ltci::DetectionMap k = ltci::kt_mfp(fc, amb, sk, o);
    CHECK(k.amb.has_value() && k.amb->q_min == -1 && k.counters.kt == 1);
    {
        const ltci_radar r = to_c(p);
        const ltci_single_space cs = to_c(sk);
        const ltci_ambiguity ca{amb.q_min, amb.q_max};
        ltci_options co{};
        co.retain_threshold = o.retain_threshold;
        co.keep_dense = 1;
        co.keystone_taps = 8;
        ltci_detection_map* cm = nullptr;
        CHECK(ltci_cuda_kt_mfp(reinterpret_cast<const double*>(fc.data.data()), &r, &ca, &cs, &co, &cm) == LTCI_OK);
        if (cm) same_map(k, *cm, ltci::DetectorKind::KtMfp);
        ltci_cuda_free_map(cm);
    }
    thrown = false;
    try {
        ltci::SingleScaleSpace s1 = sk;
        s1.c.resize(1);
        ltci::kt_mfp(fc, amb, s1, o);
    } catch (const std::invalid_argument&) {
        thrown = true;
    }
    CHECK(thrown);
    std::printf(fails ? "dropin td/kt: %d failures\n" : "dropin td/kt: ok\n", fails);
    return fails ? 1 : 0;
}
