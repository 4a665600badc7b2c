// fscn_io.cpp — .fscn batch ingestion (include/fscan_io.h). File format of
// proj/src/io.cpp:84-131; many files read concurrently into one host buffer.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fscan/io.hpp"
#include "fscan_io.h"

namespace {

constexpr char kMagic[4] = {'F', 'S', 'C', 'N'};

struct Header {
    uint32_t n = 0;
    float delta = 0.0f;
};

void put(char* err, size_t len, const std::string& msg) {
    if (err && len) std::snprintf(err, len, "%s", msg.c_str());
}

// Opens `path` and reads/validates the 16-byte header; returns an error text
// (empty on success) with the reference's wording (io.cpp:104-118).
std::string open_checked(const char* path, FILE** fp, Header* h) {
    *fp = std::fopen(path, "rb");
    if (!*fp) return std::string(path) + ": cannot open";
    char magic[4];
    uint32_t reserved = 0;
    const bool ok = std::fread(magic, 1, 4, *fp) == 4 && std::fread(&h->n, 4, 1, *fp) == 1 &&
                    std::fread(&h->delta, 4, 1, *fp) == 1 && std::fread(&reserved, 4, 1, *fp) == 1;
    if (!ok || std::memcmp(magic, kMagic, 4) != 0) return std::string(path) + ": not a scan file (bad magic)";
    if (h->n == 0 || h->n > (1u << 15)) return std::string(path) + ": implausible grid size in header";
    if (!(h->delta > 0.0f)) return std::string(path) + ": GridSpec: delta must be positive";
    return "";
}

}  // namespace

extern "C" {

fscan_status fscan_fscn_read_header(const char* path, int* n, double* delta, char* err, size_t len) {
    if (!path || !n || !delta) return FSCAN_ERR_INVALID_ARGUMENT;
    FILE* fp = nullptr;
    Header h;
    const std::string e = open_checked(path, &fp, &h);
    if (fp) std::fclose(fp);
    if (!e.empty()) {
        put(err, len, e);
        return FSCAN_ERR_IO;
    }
    *n = (int)h.n;
    *delta = (double)h.delta;
    return FSCAN_OK;
}

fscan_status fscan_fscn_read_batch(const char* const* paths, int count, int n, float* out, double* deltas,
                                   int threads, char* err, size_t len) {
    if (count < 0 || n < 1 || (count > 0 && (!paths || !out))) return FSCAN_ERR_INVALID_ARGUMENT;
    if (count == 0) return FSCAN_OK;
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = std::min(threads, count);
    const size_t nn = (size_t)n * n;
    std::atomic<int> next{0};
    std::mutex mu;
    int first_bad = count;
    std::string first_err;
    auto worker = [&] {
        for (int i = next++; i < count; i = next++) {
            FILE* fp = nullptr;
            Header h;
            std::string e = open_checked(paths[i], &fp, &h);
            if (e.empty() && (int)h.n != n)
                e = std::string(paths[i]) + ": grid size " + std::to_string(h.n) + " != " + std::to_string(n);
            if (e.empty() && std::fread(out + i * nn, sizeof(float), nn, fp) != nn)
                e = std::string(paths[i]) + ": truncated scan data";
            if (fp) std::fclose(fp);
            if (e.empty()) {
                if (deltas) deltas[i] = (double)h.delta;
                continue;
            }
            std::lock_guard<std::mutex> g(mu);
            if (i < first_bad) {  // report the first failing file in list order
                first_bad = i;
                first_err = e;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (std::thread& t : pool) t.join();
    if (first_bad < count) {
        put(err, len, first_err);
        return FSCAN_ERR_IO;
    }
    return FSCAN_OK;
}

fscan_status fscan_fscn_write(const char* path, const float* grid, int n, double delta, char* err, size_t len) {
    if (!path || !grid || n < 1 || !(delta > 0.0)) return FSCAN_ERR_INVALID_ARGUMENT;
    FILE* fp = std::fopen(path, "wb");
    if (!fp) {
        put(err, len, std::string(path) + ": cannot open for writing");
        return FSCAN_ERR_IO;
    }
    const uint32_t un = (uint32_t)n, reserved = 0;
    const float d = (float)delta;
    const size_t nn = (size_t)n * n;
    const bool ok = std::fwrite(kMagic, 1, 4, fp) == 4 && std::fwrite(&un, 4, 1, fp) == 1 &&
                    std::fwrite(&d, 4, 1, fp) == 1 && std::fwrite(&reserved, 4, 1, fp) == 1 &&
                    std::fwrite(grid, sizeof(float), nn, fp) == nn;
    const bool closed = std::fclose(fp) == 0;
    if (!ok || !closed) {
        put(err, len, std::string(path) + ": write failed");
        return FSCAN_ERR_IO;
    }
    return FSCAN_OK;
}

}  // extern "C"

// ---- C++ drop-in (fscan/io.hpp) ----
namespace fscan {

void write_scan(const std::string& path, const ScanGrid& scan) {
    std::vector<float> v(scan.values.size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = static_cast<float>(scan.values[i]);
    char err[512] = {0};
    if (fscan_fscn_write(path.c_str(), v.data(), scan.spec.n, scan.spec.delta, err, sizeof err) != FSCAN_OK)
        throw std::runtime_error(err[0] ? err : (path + ": cannot open for writing"));
}

ScanGrid read_scan(const std::string& path) {
    int n = 0;
    double delta = 0.0;
    char err[512] = {0};
    if (fscan_fscn_read_header(path.c_str(), &n, &delta, err, sizeof err) != FSCAN_OK) throw std::runtime_error(err);
    std::vector<float> v((size_t)n * n);
    const char* p = path.c_str();
    if (fscan_fscn_read_batch(&p, 1, n, v.data(), nullptr, 1, err, sizeof err) != FSCAN_OK)
        throw std::runtime_error(err);
    Array2D values(n, n);
    for (size_t i = 0; i < v.size(); ++i) values[i] = v[i];
    return ScanGrid(GridSpec{n, delta}, std::move(values));
}

GridSpec read_scans_f32(const std::vector<std::string>& paths, std::vector<float>& out, int threads) {
    if (paths.empty()) {
        out.clear();
        return GridSpec{};
    }
    int n = 0;
    double delta = 0.0;
    char err[512] = {0};
    if (fscan_fscn_read_header(paths[0].c_str(), &n, &delta, err, sizeof err) != FSCAN_OK)
        throw std::runtime_error(err);
    std::vector<const char*> ps;
    for (const std::string& s : paths) ps.push_back(s.c_str());
    out.resize(paths.size() * (size_t)n * n);
    if (fscan_fscn_read_batch(ps.data(), (int)ps.size(), n, out.data(), nullptr, threads, err, sizeof err) != FSCAN_OK)
        throw std::runtime_error(err);
    return GridSpec{n, delta};
}

}  // namespace fscan
