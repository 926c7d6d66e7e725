// ltci_b200/ltci.hpp -- C++ face of the B200 drop-in.
//
// Declares, layout-compatible with the reference library, the types that
// cross the reference detector API, so that code compiled against the
// reference headers links unchanged against libltci_b200.so:
//   ltci::ds_grft   (reference proj/include/ltci/detectors.hpp:42-43)
//   ltci::ds_kt_mfp (reference proj/include/ltci/detectors.hpp:47-48)
// Member order and types follow proj/include/ltci/{common,radar_params,
// motion,cube,search_space,detection,detectors}.hpp; only the members that
// the two detectors read or fill carry behaviour here.  The bodies call the
// C-ABI in ltci_cuda.h and rethrow its status codes as the reference's
// exception types.
#pragma once

#include <complex>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace ltci {

using cplx = std::complex<double>;
inline constexpr double kPi = 3.14159265358979323846;
inline constexpr double kSpeedOfLight = 3.0e8;

// (fc/fs)/M > 1 and similar applicability failures (common.hpp:17-20)
class ConditionViolated : public std::runtime_error {
public:
    explicit ConditionViolated(const std::string& msg) : std::runtime_error(msg) {}
};

struct RadarParams {
    double fc = 0, fs = 0, Br = 0, delta_f = 0, PRF = 0;
    int M = 0, K = 0, K_valid = 0;

    double lambda() const { return kSpeedOfLight / fc; }
    double T() const { return static_cast<double>(M) / PRF; }
    double Va() const { return lambda() * PRF / 2.0; }
    double delta_R() const { return kSpeedOfLight / (2.0 * fs); }
    double slow_time(int m) const { return static_cast<double>(m + 1) / PRF; }
    int n0() const { return K; }
};

struct Grid {
    double start = 0, step = 0;
    int count = 0;
    double value(int i) const { return start + step * static_cast<double>(i); }
};

struct Bounds {
    double lo = 0, hi = 0;
};

struct RangeRoi {
    int first = 0, last = 0;
    int count() const { return last - first + 1; }
};

struct StepSizes {
    std::vector<double> rm, dfm, alpha;
};

struct SingleScaleSpace {
    RadarParams params;
    StepSizes steps;
    std::vector<Grid> c;
    RangeRoi roi;
};

struct DualScaleSpace {
    RadarParams params;
    StepSizes steps;
    std::vector<Grid> coarse, fine;
    double kappa = 1.0;
    RangeRoi roi;
    int order() const { return static_cast<int>(coarse.size()); }
};

struct AmbiguitySpace {
    int q_min = 0, q_max = 0;
    int count() const { return q_max - q_min + 1; }
};

struct FreqPulseCube {
    RadarParams params;
    std::vector<cplx> data;  // sample (k, m) at data[k + K*m]
};

// range-pulse cube (proj/include/ltci/cube.hpp:30-47): sample (n, m) at data[n + K*m]
struct RangePulseCube {
    RadarParams params;
    std::vector<cplx> data;
};

enum class TrajectoryPolicy { ZeroOutside, Wrap, Error };

struct DetectorOptions {
    double retain_threshold = 0.0;
    bool keep_dense = false;
    int threads = 1;
    int keystone_taps = 8;
    TrajectoryPolicy trajectory = TrajectoryPolicy::ZeroOutside;
};

enum class DetectorKind { FdGrft, TdGrft, KtMfp, DsGrft, DsKtMfp };

struct OpCounters {
    std::uint64_t kt = 0, mf = 0, ifft = 0, fft = 0;
};

struct AxisDesc {
    enum class Role { Range, Velocity, Higher, Doppler, Coarse, Fine, Folding };
    Role role;
    int order;
    int size;
};

struct DetectionMap {
    DetectorKind kind = DetectorKind::FdGrft;
    RadarParams params;
    std::vector<AxisDesc> axes;
    OpCounters counters;
    double retain_threshold = 0.0;
    std::vector<std::pair<std::uint64_t, cplx>> candidates;  // sorted by index
    bool dense_stored = false;
    std::vector<cplx> dense;
    std::uint64_t argmax = 0;
    cplx argmax_value{0.0, 0.0};
    std::optional<SingleScaleSpace> single;
    std::optional<DualScaleSpace> dual;
    std::optional<AmbiguitySpace> amb;
    int doppler_first = 0;
};

// proj/include/ltci/detectors.hpp:25-26
DetectionMap fd_grft(const FreqPulseCube& cube, const SingleScaleSpace& space, const DetectorOptions& opt = {});
// proj/include/ltci/detectors.hpp:29-31 (std::out_of_range under TrajectoryPolicy::Error)
DetectionMap td_grft(const RangePulseCube& cube, const SingleScaleSpace& space, const DetectorOptions& opt = {});
// proj/include/ltci/detectors.hpp:33-37
DetectionMap kt_mfp(const FreqPulseCube& cube, const AmbiguitySpace& amb, const SingleScaleSpace& space,
                    const DetectorOptions& opt = {});
DetectionMap ds_grft(const FreqPulseCube& cube, const DualScaleSpace& space, const DetectorOptions& opt = {});
DetectionMap ds_kt_mfp(const FreqPulseCube& cube, const AmbiguitySpace& amb, const DualScaleSpace& space,
                       const DetectorOptions& opt = {});

}  // namespace ltci

namespace ltci_b200 {

// Per ROI range cell: the strongest hypothesis over every coarse, fine and
// Doppler cell (ties to the lowest flat index).  No reference counterpart;
// this is the map the multi-GPU path gathers.
struct PeakMap {
    std::vector<std::uint64_t> index;
    std::vector<ltci::cplx> value;
};

ltci::DetectionMap ds_grft_with_peaks(const ltci::FreqPulseCube& cube, const ltci::DualScaleSpace& space,
                                      const ltci::DetectorOptions& opt, PeakMap* peaks);

}  // namespace ltci_b200
