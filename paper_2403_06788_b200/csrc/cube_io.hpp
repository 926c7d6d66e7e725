// cube_io.hpp -- internal: the "LTCI" cube container,
// shared by cube_io.cpp (the C-ABI file functions) and engine.cu (the
// file -> pinned staging -> device wire path).
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/ltci_cuda.h"

namespace ltcib {

// Carries an LTCI_* status code (LTCI_IO_ERROR for ltci::IoError).
struct CubeError : std::runtime_error {
    int code;
    CubeError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

constexpr std::size_t kCubeHeaderSize = 4 + 4 + 1 + 3 * 4 + 5 * 8;  // 61 bytes

// An open cube file positioned at the payload.  open() performs every check of
// read_cube_file (proj/src/cube_io.cpp:121-170) that does not need the payload
// bytes themselves, in the reference's order, including "truncated payload" and
// "trailing bytes after payload" (decided from the file length).
struct CubeReader {
    std::FILE* f = nullptr;
    std::string path;
    ltci_cube_header h{};
    std::uint64_t count = 0;  // complex samples = K * M
    void open(const std::string& p);
    // next n_doubles payload doubles (host byte order) into dst
    void read(double* dst, std::uint64_t n_doubles);
    ~CubeReader() {
        if (f) std::fclose(f);
    }
};

// RadarParams::create (proj/src/radar_params.cpp:10-45); throws std::invalid_argument
ltci_radar radar_create(double fc, double fs, double br, double prf, int M, int K, int k_valid);

}  // namespace ltcib
