// GPU linear scan: scan_truth (workload.cpp:56-71) and distance_histogram
// (workload.cpp:133-151) over device-resident rows.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace fclsh_b200 {

struct ScanArgs {
    const uint64_t* rows = nullptr; // device [n][words]
    uint64_t n = 0;
    const uint64_t* qrows = nullptr; // device [nq][words]
    uint64_t nq = 0;
    uint64_t dims = 0;
    uint32_t words = 0;
    uint32_t radius = 0;
};

// Grow-only device workspace; results live until the next call.
struct ScanState {
    int device = 0;
    DevBuf count, offsets, wide, id_tmp, dist_tmp, id, dist, query, hist, sample_idx, cub_tmp;
};

struct ScanOutput {
    uint64_t nq = 0, total = 0;
    uint32_t *d_query = nullptr, *d_id = nullptr, *d_dist = nullptr;
    uint64_t* d_offsets = nullptr;
};

// Every (query, point, distance) with distance <= radius, ordered by (query, point).
ScanOutput scan_truth_device(ScanState& st, const ScanArgs& a, cudaStream_t s);
// counts[dims + 1]: all pairs (sample_per_query == 0 or >= n), else the
// reference's sampled pairs (Rng(seed).stream("histogram").below(n)).
void distance_histogram_device(ScanState& st, const ScanArgs& a, uint64_t sample_per_query, uint64_t seed,
                               uint64_t* counts, cudaStream_t s);

} // namespace fclsh_b200
