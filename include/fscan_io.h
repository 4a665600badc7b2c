/*
 * fscan_io.h — native scan-file ingestion for the B200 path.
 *
 * The reference stores scans as .fscn files (proj/src/io.cpp:84-131:
 * "FSCN" magic, uint32 n, float32 delta, uint32 reserved, then n*n float32
 * row-major) and its odometry command reads a directory of them one by one
 * (proj/tools/main.cpp:104-122). Here a batch of files is read by a thread
 * pool straight into one caller-provided host buffer (pinned by the caller
 * for full-speed H2D copies), ready for fscan_match_batch_host /
 * fscan_odometry_batch. Error texts follow read_scan (io.cpp:104-131).
 */
#ifndef FSCAN_IO_H
#define FSCAN_IO_H

#include <stddef.h>

#include "fscan_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Header of one file: grid side and delta (FSCAN_ERR_IO on a missing,
 * malformed or implausible file). */
fscan_status fscan_fscn_read_header(const char* path, int* n, double* delta, char* err, size_t err_len);

/* Reads `count` files, each an n x n grid, into out[i * n * n]; deltas (may be
 * NULL) receives each file's delta. threads <= 0: one per hardware thread.
 * Every file is checked (magic, size == n, complete payload); the first
 * failure is reported with its path. */
fscan_status fscan_fscn_read_batch(const char* const* paths, int count, int n, float* out, double* deltas,
                                   int threads, char* err, size_t err_len);

/* write_scan (io.cpp:84-101): one n x n float32 grid. */
fscan_status fscan_fscn_write(const char* path, const float* grid, int n, double delta, char* err,
                              size_t err_len);

#ifdef __cplusplus
}
#endif

#endif
