// Multi-GPU result assembly. Points are sharded across
// ranks in contiguous id ranges (rank r owns ids [off_r, off_r + n_r)), every
// rank answers the whole query batch on its shard, and rank 0 receives every
// rank's (query, id, distance) triples plus their per-query offsets through
// NCCL (paper_1602_02620_b200/cluster.py). Because shard id ranges increase
// with the rank, the global (query, id) order is: for each query, rank 0's
// run, then rank 1's, ... -- this kernel places every run at its final spot.
// Counters (collisions, candidates, found) are per-shard additive (every
// posting and every id lives in exactly one shard) and are summed by an
// all-reduce, not here.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace fclsh_b200 {

namespace {

// Warp per (rank, query): copies rank r's run for query q to its place.
__global__ void k_merge_shards(uint32_t world, uint64_t nq, const uint64_t* __restrict__ offsets, // [world][nq+1]
                               const uint32_t* __restrict__ triples, uint64_t cap,                // [world][3][cap]
                               const uint64_t* __restrict__ out_offsets,                           // [nq+1]
                               uint32_t* __restrict__ out, uint64_t out_cap) {                      // [3][out_cap]
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t items = uint64_t(world) * nq;
    for (uint64_t w = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); w < items; w += warps) {
        const uint32_t r = uint32_t(w / nq);
        const uint64_t q = w % nq;
        const uint64_t* off_r = offsets + uint64_t(r) * (nq + 1);
        const uint64_t beg = off_r[q], cnt = off_r[q + 1] - beg;
        if (cnt == 0) continue;
        uint64_t dst = out_offsets[q];
        for (uint32_t rr = 0; rr < r; ++rr) {
            const uint64_t* o = offsets + uint64_t(rr) * (nq + 1);
            dst += o[q + 1] - o[q];
        }
        const uint32_t* src = triples + uint64_t(r) * 3 * cap;
        for (uint64_t k = lane; k < cnt; k += 32) {
            out[dst + k] = src[beg + k];
            out[out_cap + dst + k] = src[cap + beg + k];
            out[2 * out_cap + dst + k] = src[2 * cap + beg + k];
        }
    }
}

// out_offsets[q] = sum over ranks of offsets_r[q] (exclusive per-query start)
__global__ void k_sum_offsets(uint32_t world, uint64_t nq, const uint64_t* __restrict__ offsets,
                              uint64_t* __restrict__ out_offsets) {
    for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q <= nq; q += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t s = 0;
        for (uint32_t r = 0; r < world; ++r) s += offsets[uint64_t(r) * (nq + 1) + q];
        out_offsets[q] = s;
    }
}

} // namespace

void merge_shards(uint32_t world, uint64_t nq, const uint64_t* d_offsets, const uint32_t* d_triples, uint64_t cap,
                  uint32_t* d_out, uint64_t out_cap, uint64_t* d_out_offsets, cudaStream_t s, int device) {
    const unsigned g1 = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((nq + 256) / 256, uint64_t(sm_count(device)) * 8)));
    k_sum_offsets<<<g1, 256, 0, s>>>(world, nq, d_offsets, d_out_offsets);
    FCLSH_LAUNCHED();
    const uint64_t items = uint64_t(world) * nq;
    if (items == 0) return;
    const unsigned g2 = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((items * 32 + 255) / 256,
                                                                         uint64_t(sm_count(device)) * 8)));
    k_merge_shards<<<g2, 256, 0, s>>>(world, nq, d_offsets, d_triples, cap, d_out_offsets, d_out, out_cap);
    FCLSH_LAUNCHED();
}

} // namespace fclsh_b200
