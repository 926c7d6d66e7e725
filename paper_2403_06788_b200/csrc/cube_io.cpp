// cube_io.cpp -- the reference's "LTCI" cube container behind the C-ABI
// (SURVEY.md §8(f) rank 4).
//
//   header layout + CubeFile   proj/include/ltci/cube_io.hpp:9-30
//   write_cube_file            proj/src/cube_io.cpp:66-119 (temp file + rename)
//   read_cube_file             proj/src/cube_io.cpp:121-179
//   RadarParams::create        proj/src/radar_params.cpp:10-45
//
// The header is assembled bytewise (little-endian on any host, as the
// reference); the payload is moved in large blocks, byte-swapped only on a
// big-endian host.  Error messages are the reference's.

#include "cube_io.hpp"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

namespace ltcib {
namespace {

constexpr std::uint32_t kVersion = 1;
constexpr bool kLittle = __BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__;

void put_u32(unsigned char* p, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
}

void put_f64(unsigned char* p, double v) {
    std::uint64_t b;
    std::memcpy(&b, &v, 8);
    for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>((b >> (8 * i)) & 0xff);
}

std::uint32_t get_u32(const unsigned char* p) {
    std::uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<std::uint32_t>(p[i]) << (8 * i);
    return v;
}

double get_f64(const unsigned char* p) {
    std::uint64_t b = 0;
    for (int i = 0; i < 8; ++i) b |= static_cast<std::uint64_t>(p[i]) << (8 * i);
    double v;
    std::memcpy(&v, &b, 8);
    return v;
}

void swap_doubles(double* d, std::uint64_t n) {
    for (std::uint64_t i = 0; i < n; ++i) {
        std::uint64_t b;
        std::memcpy(&b, d + i, 8);
        b = __builtin_bswap64(b);
        std::memcpy(d + i, &b, 8);
    }
}

bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }

[[noreturn]] void io_fail(const std::string& m) { throw CubeError(LTCI_IO_ERROR, m); }

}  // namespace

ltci_radar radar_create(double fc, double fs, double br, double prf, int M, int K, int k_valid) {
    ltci_radar p{};
    p.fc = fc;
    p.fs = fs;
    p.PRF = prf;
    p.M = M;
    p.K = K;
    p.delta_f = fs / static_cast<double>(K);
    if (k_valid == 0) {
        k_valid = static_cast<int>(std::lround(br / p.delta_f));
        if (k_valid % 2 != 0) --k_valid;
        if (k_valid < 2) k_valid = 2;
        if (k_valid > K) k_valid = K;
    }
    p.K_valid = k_valid;
    p.Br = p.delta_f * static_cast<double>(k_valid);
    if (!(p.fc > 0) || !(p.fs > 0) || !(p.Br > 0) || !(p.PRF > 0) || p.M <= 0 || p.K <= 0)
        throw std::invalid_argument("RadarParams: fc, fs, Br, PRF, M, K must be positive");
    if (!is_pow2(p.M) || !is_pow2(p.K)) throw std::invalid_argument("RadarParams: M and K must be powers of two");
    if (p.fs < p.Br) throw std::invalid_argument("RadarParams: fs must be >= Br (Nyquist)");
    if (p.K_valid <= 0 || p.K_valid > p.K || p.K_valid % 2 != 0)
        throw std::invalid_argument("RadarParams: K_valid must be even and in (0, K]");
    if (std::abs(p.delta_f * p.K_valid - p.Br) > 1e-6 * p.Br)
        throw std::invalid_argument("RadarParams: Br must equal K_valid * delta_f");
    if (std::abs(p.delta_f * p.K - p.fs) > 1e-6 * p.fs)
        throw std::invalid_argument("RadarParams: delta_f must equal fs / K");
    return p;
}

void CubeReader::open(const std::string& p) {
    path = p;
    f = std::fopen(p.c_str(), "rb");
    if (!f) io_fail("cannot open " + p);
    unsigned char hd[kCubeHeaderSize];
    if (std::fread(hd, 1, kCubeHeaderSize, f) != kCubeHeaderSize) io_fail(p + ": truncated header");
    if (std::memcmp(hd, "LTCI", 4) != 0) io_fail(p + ": bad magic, not a cube file");
    const std::uint32_t version = get_u32(hd + 4);
    if (version != kVersion) io_fail(p + ": unsupported version " + std::to_string(version));
    h.domain = hd[8];
    const std::uint32_t K = get_u32(hd + 9), M = get_u32(hd + 13), K_valid = get_u32(hd + 17);
    const double fc = get_f64(hd + 21), fs = get_f64(hd + 29), br = get_f64(hd + 37), prf = get_f64(hd + 45);
    h.sigma2 = get_f64(hd + 53);
    if (h.domain > 1) io_fail(p + ": unknown domain flag");
    try {
        h.radar = radar_create(fc, fs, br, prf, static_cast<int>(M), static_cast<int>(K), static_cast<int>(K_valid));
    } catch (const std::invalid_argument& e) {
        io_fail(p + ": invalid parameters: " + e.what());
    }
    count = static_cast<std::uint64_t>(K) * M;
    // payload length decided up front (same outcome as reading it, no 2x buffer)
    const long here = std::ftell(f);
    if (here < 0 || std::fseek(f, 0, SEEK_END) != 0) io_fail(p + ": truncated payload");
    const long end = std::ftell(f);
    if (std::fseek(f, here, SEEK_SET) != 0) io_fail(p + ": truncated payload");
    const std::uint64_t avail = end > here ? static_cast<std::uint64_t>(end - here) : 0;
    if (avail < count * 16) io_fail(p + ": truncated payload");
    if (avail > count * 16) io_fail(p + ": trailing bytes after payload");
}

void CubeReader::read(double* dst, std::uint64_t n_doubles) {
    if (std::fread(dst, sizeof(double), n_doubles, f) != n_doubles) io_fail(path + ": truncated payload");
    if (!kLittle) swap_doubles(dst, n_doubles);
}

}  // namespace ltcib

void ltcib_set_last_error(const char* msg);  // engine.cu: backs ltci_cuda_last_error()

namespace {

template <typename F>
int io_guarded(F&& f) {
    try {
        f();
        return LTCI_OK;
    } catch (const ltcib::CubeError& e) {
        ltcib_set_last_error(e.what());
        return e.code;
    } catch (const std::invalid_argument& e) {
        ltcib_set_last_error(e.what());
        return LTCI_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        ltcib_set_last_error("cube file: allocation failed");
        return LTCI_BAD_ALLOC;
    } catch (const std::exception& e) {
        ltcib_set_last_error(e.what());
        return LTCI_RUNTIME_ERROR;
    }
}

}  // namespace

extern "C" int ltci_cuda_cube_file_info(const char* path, ltci_cube_header* out) {
    return io_guarded([&] {
        if (!path || !out) throw std::invalid_argument("cube file: null argument");
        ltcib::CubeReader r;
        r.open(path);
        *out = r.h;
    });
}

extern "C" int ltci_cuda_cube_file_read(const char* path, ltci_cube_header* hdr, double* out,
                                        uint64_t capacity_doubles) {
    return io_guarded([&] {
        if (!path || !hdr || !out) throw std::invalid_argument("cube file: null argument");
        ltcib::CubeReader r;
        r.open(path);
        if (capacity_doubles < 2 * r.count) throw std::invalid_argument("cube file: output buffer too small");
        r.read(out, 2 * r.count);
        *hdr = r.h;
    });
}

extern "C" int ltci_cuda_cube_file_write(const char* path, const ltci_cube_header* hdr, const double* data) {
    return io_guarded([&] {
        if (!path || !hdr || !data) throw std::invalid_argument("cube file: null argument");
        const ltci_radar& p = hdr->radar;
        if (p.K <= 0 || p.M <= 0) throw std::invalid_argument("write_cube_file: payload size does not match K*M");
        unsigned char hd[ltcib::kCubeHeaderSize];
        std::memcpy(hd, "LTCI", 4);
        ltcib::put_u32(hd + 4, ltcib::kVersion);
        hd[8] = static_cast<unsigned char>(hdr->domain);
        ltcib::put_u32(hd + 9, static_cast<std::uint32_t>(p.K));
        ltcib::put_u32(hd + 13, static_cast<std::uint32_t>(p.M));
        ltcib::put_u32(hd + 17, static_cast<std::uint32_t>(p.K_valid));
        ltcib::put_f64(hd + 21, p.fc);
        ltcib::put_f64(hd + 29, p.fs);
        ltcib::put_f64(hd + 37, p.Br);
        ltcib::put_f64(hd + 45, p.PRF);
        ltcib::put_f64(hd + 53, hdr->sigma2);

        const std::string tmp = std::string(path) + ".tmp";
        std::FILE* f = std::fopen(tmp.c_str(), "wb");
        if (!f) ltcib::io_fail("cannot open " + tmp + " for writing");
        bool ok = std::fwrite(hd, 1, sizeof(hd), f) == sizeof(hd);
        const std::uint64_t n = 2ull * static_cast<std::uint64_t>(p.K) * p.M;
        if (ltcib::kLittle) {
            ok = ok && std::fwrite(data, sizeof(double), n, f) == n;
        } else {
            std::vector<double> blk(1 << 16);
            for (std::uint64_t i = 0; i < n && ok; i += blk.size()) {
                const std::uint64_t m = std::min<std::uint64_t>(blk.size(), n - i);
                std::memcpy(blk.data(), data + i, m * 8);
                ltcib::swap_doubles(blk.data(), m);
                ok = std::fwrite(blk.data(), sizeof(double), m, f) == m;
            }
        }
        ok = std::fclose(f) == 0 && ok;
        if (!ok) {
            std::remove(tmp.c_str());
            ltcib::io_fail("failed writing " + tmp);
        }
        if (std::rename(tmp.c_str(), path) != 0) {
            const std::string why = std::strerror(errno);
            std::remove(tmp.c_str());
            ltcib::io_fail("cannot rename " + tmp + " to " + path + ": " + why);
        }
    });
}
