// fscan/io.hpp — scan files of the reference (proj/include/fscan/io.hpp:15-16,
// proj/src/io.cpp:84-131), same declarations and errors (std::runtime_error
// naming the path), plus a batch reader that fills one float32 buffer from
// many files concurrently for the batched GPU entry points (fscan_io.h).
#pragma once

#include <string>
#include <vector>

#include "fscan/types.hpp"

namespace fscan {

void write_scan(const std::string& path, const ScanGrid& scan);
ScanGrid read_scan(const std::string& path);

/// Added: reads every file (all of one grid size) into out (resized to
/// paths.size() * n * n floats, row-major per scan); returns the common spec
/// (delta of the first file). Throws std::runtime_error on the first bad file.
GridSpec read_scans_f32(const std::vector<std::string>& paths, std::vector<float>& out, int threads = 0);

}  // namespace fscan
