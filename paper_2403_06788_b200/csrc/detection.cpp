// detection.cpp -- the consumer of the detection map: cell -> motion estimate
// and local-maximum extraction with ridge-chained duplicate merging, for the
// dual-scale maps this library produces.
//
//   detection_from_cell  reference proj/src/detection.cpp:124-153
//   estimate_cell_sizes  reference proj/src/detection.cpp:55-83
//   extract_detections   reference proj/src/detection.cpp:158-244
//
// Host C++ over the (sorted, sparse) candidate list: the map is already
// reduced on the GPU to cells above the retention threshold.  Orders and
// tie-breaks follow the reference so that, given the same candidates, the
// detections are identical (tests/test_detections.py).

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ltci_cuda.h"

namespace {

constexpr double kC = 3.0e8;

struct Ctx {
    const ltci_detection_map* map;
    const ltci_dual_space* s;      // DS maps
    const ltci_single_space* ss;   // FD maps
    const ltci_ambiguity* amb;
    int M;
    double dR, va;
};

std::vector<int> decode(const ltci_detection_map& m, uint64_t idx) {
    std::vector<int> cell(m.n_axes);
    for (int i = m.n_axes - 1; i >= 0; --i) {
        cell[i] = static_cast<int>(idx % static_cast<uint64_t>(m.axes[i].size));
        idx /= static_cast<uint64_t>(m.axes[i].size);
    }
    return cell;
}

uint64_t encode(const ltci_detection_map& m, const std::vector<int>& cell) {
    uint64_t idx = 0;
    for (int i = 0; i < m.n_axes; ++i) idx = idx * static_cast<uint64_t>(m.axes[i].size) + cell[i];
    return idx;
}

int axis_index(const ltci_detection_map& m, int role, int order = 0) {
    for (int i = 0; i < m.n_axes; ++i)
        if (m.axes[i].role == role && m.axes[i].order == order) return i;
    return -1;
}

double grid_value(const ltci_grid& g, int i) { return g.start + g.step * static_cast<double>(i); }

ltci_detection from_cell(const Ctx& x, const std::vector<int>& cell, double re, double im, uint64_t idx) {
    const ltci_detection_map& m = *x.map;
    ltci_detection d;
    std::memset(&d, 0, sizeof(d));
    d.statistic = std::hypot(re, im);
    d.flat_index = idx;
    if (m.kind == LTCI_FD_GRFT) {
        // detection.cpp:101-111: c0 = n dR, c_p = grid value of the order-p axis
        const ltci_single_space& ss = *x.ss;
        const int n = cell[axis_index(m, LTCI_AXIS_RANGE)] + ss.roi_first;
        d.n_coef = ss.order + 1;
        d.c[0] = n * x.dR;
        for (int ord = 1; ord <= ss.order; ++ord)
            d.c[ord] = grid_value(ss.c[ord - 1],
                                  cell[axis_index(m, ord == 1 ? LTCI_AXIS_VELOCITY : LTCI_AXIS_HIGHER, ord)]);
        return d;
    }
    const ltci_dual_space& s = *x.s;
    const int n = cell[axis_index(m, LTCI_AXIS_RANGE)] + s.roi_first;
    const int jd = cell[axis_index(m, LTCI_AXIS_DOPPLER)];
    if (m.kind == LTCI_DS_GRFT) {
        const double vd = (static_cast<double>(m.doppler_first + jd) - x.M / 2.0) * x.va / x.M;
        d.n_coef = s.order + 1;
        d.c[0] = n * x.dR;
        d.c[1] = grid_value(s.coarse[0], cell[axis_index(m, LTCI_AXIS_COARSE, 1)]) + vd / s.kappa;
        // fine grids store unscaled values; the search used kappa*value (detection.cpp:136-141)
        for (int ord = 2; ord <= s.order; ++ord)
            d.c[ord] = grid_value(s.coarse[ord - 1], cell[axis_index(m, LTCI_AXIS_COARSE, ord)]) +
                       grid_value(s.fine[ord - 1], cell[axis_index(m, LTCI_AXIS_FINE, ord)]);
    } else {
        const double vd = (static_cast<double>(jd) - x.M / 2.0) * x.va / x.M;
        const int q = x.amb->q_min + cell[axis_index(m, LTCI_AXIS_FOLDING)];
        d.n_coef = 3;
        d.c[0] = n * x.dR;
        d.c[1] = q * x.va + vd;
        d.c[2] = grid_value(s.coarse[1], cell[axis_index(m, LTCI_AXIS_COARSE, 2)]) +
                 grid_value(s.fine[1], cell[axis_index(m, LTCI_AXIS_FINE, 2)]);
        d.has_q = 1;
        d.q = q;
        d.baseband_velocity = vd;
    }
    return d;
}

}  // namespace

void ltcib_set_last_error(const char* msg);  // engine.cu: backs ltci_cuda_last_error()

namespace {

int extract_impl(const Ctx& x, double gamma, ltci_detection* out, int max_out, int* n_out, double cs_vel) {
    const ltci_detection_map* map = x.map;
    try {
        if (gamma < 0) throw std::invalid_argument("extract_detections: gamma must be >= 0");
        if (gamma < map->retain_threshold)
            throw std::invalid_argument("extract_detections: gamma below the map's retention threshold");

        // Local-max test only needs neighbours above gamma: anything dropped by
        // retention is below the candidate under test (detection.cpp:165-168).
        std::unordered_map<uint64_t, double> mag;
        mag.reserve(map->n_candidates * 2);
        for (uint64_t i = 0; i < map->n_candidates; ++i)
            mag.emplace(map->cand_index[i], std::hypot(map->cand_value[2 * i], map->cand_value[2 * i + 1]));

        std::vector<int> local_axes;
        for (int i = 0; i < map->n_axes; ++i) {
            const int r = map->axes[i].role;
            const bool local = r == LTCI_AXIS_RANGE || r == LTCI_AXIS_DOPPLER || r == LTCI_AXIS_VELOCITY ||
                               (r == LTCI_AXIS_HIGHER && map->axes[i].order == 2) ||
                               (r == LTCI_AXIS_FINE && map->axes[i].order == 2);
            if (local) local_axes.push_back(i);
        }
        const int L = static_cast<int>(local_axes.size());
        int total = 1;
        for (int i = 0; i < L; ++i) total *= 3;

        std::vector<ltci_detection> raw;
        for (uint64_t i = 0; i < map->n_candidates; ++i) {
            const uint64_t idx = map->cand_index[i];
            const double re = map->cand_value[2 * i], im = map->cand_value[2 * i + 1];
            const double m = std::hypot(re, im);
            if (!(m > gamma)) continue;
            const std::vector<int> cell = decode(*map, idx);
            std::vector<int> nb = cell;
            bool is_max = true;
            for (int code = 0; code < total && is_max; ++code) {
                int c = code;
                bool center = true, valid = true;
                for (int a = 0; a < L; ++a) {
                    const int step = c % 3 - 1;
                    c /= 3;
                    const int ai = local_axes[a];
                    const int v = cell[ai] + step;
                    if (step != 0) center = false;
                    if (v < 0 || v >= map->axes[ai].size) valid = false;
                    nb[ai] = v;
                }
                if (center || !valid) continue;
                const uint64_t nidx = encode(*map, nb);
                auto it = mag.find(nidx);
                if (it == mag.end()) continue;
                if (it->second > m || (it->second == m && nidx < idx)) is_max = false;
            }
            if (is_max) raw.push_back(from_cell(x, cell, re, im, idx));
        }

        // cluster merge along the range/velocity ridge (detection.cpp:209-243)
        const double cs_range = x.dR;
        std::sort(raw.begin(), raw.end(), [](const ltci_detection& a, const ltci_detection& b) {
            if (a.statistic != b.statistic) return a.statistic > b.statistic;
            return a.flat_index < b.flat_index;
        });
        std::vector<ltci_detection> reps;
        std::vector<std::vector<ltci_detection>> clusters;
        for (const ltci_detection& d : raw) {
            bool joined = false;
            for (size_t c = 0; c < clusters.size() && !joined; ++c) {
                for (const ltci_detection& mem : clusters[c]) {
                    bool near = std::abs(d.c[0] - mem.c[0]) <= cs_range * 1.01;
                    if (near && d.n_coef >= 2) near = std::abs(d.c[1] - mem.c[1]) <= cs_vel * 2.01;
                    if (near) {
                        clusters[c].push_back(d);
                        joined = true;
                        break;
                    }
                }
            }
            if (!joined) {
                clusters.push_back({d});
                reps.push_back(d);
            }
        }
        *n_out = static_cast<int>(reps.size());
        for (int i = 0; i < std::min<int>(max_out, static_cast<int>(reps.size())); ++i) out[i] = reps[i];
        return LTCI_OK;
    } catch (const std::invalid_argument& e) {
        ltcib_set_last_error(e.what());
        return LTCI_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        ltcib_set_last_error("extract_detections: allocation failed");
        return LTCI_BAD_ALLOC;
    } catch (const std::exception& e) {
        ltcib_set_last_error(e.what());
        return LTCI_RUNTIME_ERROR;
    }
}

}  // namespace

// detection_success (proj/src/bench.cpp:30-46): some retained cell estimates the
// truth within one cell on every axis (cell sizes of estimate_cell_sizes,
// detection.cpp:55-79).  Used by the Monte-Carlo driver (pd.cu).
bool ltcib_detection_success(const ltci_detection_map* map, const ltci_dual_space* ds, const ltci_single_space* ss,
                             const ltci_ambiguity* amb, const ltci_target& truth) {
    const ltci_radar& r = ds ? ds->radar : ss->radar;
    const double va = (kC / r.fc) * r.PRF / 2.0;
    Ctx x{map, ds, ss, amb, r.M, kC / (2.0 * r.fs), va};
    const double cs_range = x.dR;
    double cs_vel = 0.0, cs_acc = 0.0;
    if (map->kind == LTCI_FD_GRFT) {
        cs_vel = ss->c[0].step;
        if (ss->order >= 2) cs_acc = ss->c[1].step;
    } else if (map->kind == LTCI_DS_GRFT) {
        cs_vel = (va / r.M) / ds->kappa;
        if (ds->order >= 2) cs_acc = ds->fine[1].step;
    } else {
        cs_vel = va / r.M;
        cs_acc = ds->fine[1].step;
    }
    for (uint64_t i = 0; i < map->n_candidates; ++i) {
        const ltci_detection d =
            from_cell(x, decode(*map, map->cand_index[i]), map->cand_value[2 * i], map->cand_value[2 * i + 1],
                      map->cand_index[i]);
        if (std::abs(d.c[0] - truth.c[0]) > cs_range * 1.0001) continue;
        if (truth.order >= 1 && std::abs(d.c[1] - truth.c[1]) > cs_vel * 1.0001) continue;
        if (truth.order >= 2 && d.n_coef - 1 >= 2 && std::abs(d.c[2] - truth.c[2]) > cs_acc * 1.0001) continue;
        return true;
    }
    return false;
}

extern "C" int ltci_cuda_extract_detections(const ltci_detection_map* map, const ltci_dual_space* space,
                                            const ltci_ambiguity* amb, double gamma, ltci_detection* out,
                                            int max_out, int* n_out) {
    if (!map || !space || !n_out) {
        ltcib_set_last_error("extract_detections: null argument");
        return LTCI_INVALID_ARGUMENT;
    }
    if (map->kind != LTCI_DS_GRFT && map->kind != LTCI_DS_KT_MFP) {
        ltcib_set_last_error("extract_detections: dual-scale map expected (use _single for FD-GRFT)");
        return LTCI_INVALID_ARGUMENT;
    }
    if (map->kind == LTCI_DS_KT_MFP && !amb) {
        ltcib_set_last_error("extract_detections: ambiguity needed");
        return LTCI_INVALID_ARGUMENT;
    }
    const double va = (kC / space->radar.fc) * space->radar.PRF / 2.0;
    Ctx x{map, space, nullptr, amb, space->radar.M, kC / (2.0 * space->radar.fs), va};
    // estimate_cell_sizes (detection.cpp:55-79)
    const double cs_vel = map->kind == LTCI_DS_GRFT ? (va / x.M) / space->kappa : va / x.M;
    return extract_impl(x, gamma, out, max_out, n_out, cs_vel);
}

extern "C" int ltci_cuda_extract_detections_single(const ltci_detection_map* map, const ltci_single_space* space,
                                                   double gamma, ltci_detection* out, int max_out, int* n_out) {
    if (!map || !space || !n_out) {
        ltcib_set_last_error("extract_detections: null argument");
        return LTCI_INVALID_ARGUMENT;
    }
    if (map->kind != LTCI_FD_GRFT) {
        ltcib_set_last_error("extract_detections_single: FD-GRFT map expected");
        return LTCI_INVALID_ARGUMENT;
    }
    const double va = (kC / space->radar.fc) * space->radar.PRF / 2.0;
    Ctx x{map, nullptr, space, nullptr, space->radar.M, kC / (2.0 * space->radar.fs), va};
    return extract_impl(x, gamma, out, max_out, n_out, space->c[0].step);  // detection.cpp:59-63
}
