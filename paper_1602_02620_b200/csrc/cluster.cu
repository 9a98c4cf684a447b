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
#include "cluster.hpp"

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

// ------------------------------------------------------------------------
// fclsh_cluster's merge (cluster.hpp): S result sources -- the shards of one
// device, or every rank's packed result on the root -- into one result,
// warp per query. Per query the sources' runs are concatenated in source
// order (= ascending id ranges, so the output is in (query, id) order) and
// the counters are summed (exactly additive across shards).

namespace fclsh_b200 {

namespace {

__global__ void __launch_bounds__(256) k_merge_sources(const MergeSrcs srcs, uint32_t S, uint64_t nq, MergeDst dst) {
    constexpr unsigned kAll = 0xffffffffu;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t q = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); q < nq; q += warps) {
        unsigned long long base = 0, coll = 0, cand = 0, found = 0, end_all = 0;
        unsigned long long cnt[2] = {0, 0}, beg[2] = {0, 0};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t s = lane + 32 * h;
            if (s < S) {
                const MergeSrc& m = srcs.s[s];
                beg[h] = m.off[q];
                cnt[h] = m.off[q + 1] - beg[h];
                base += beg[h];
                coll += m.coll[q];
                cand += m.cand[q];
                found += m.found[q];
                if (q + 1 == nq) end_all += m.off[nq];
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            base += __shfl_xor_sync(kAll, base, o);
            coll += __shfl_xor_sync(kAll, coll, o);
            cand += __shfl_xor_sync(kAll, cand, o);
            found += __shfl_xor_sync(kAll, found, o);
            end_all += __shfl_xor_sync(kAll, end_all, o);
        }
        if (lane == 0) {
            dst.off[q] = base;
            dst.coll[q] = coll;
            dst.cand[q] = cand;
            dst.found[q] = found;
            if (q + 1 == nq) dst.off[nq] = end_all;
        }
        // exclusive prefix of the run lengths in source order
        unsigned long long carry = base;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            unsigned long long x = cnt[h];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(kAll, x, o);
                if (lane >= uint32_t(o)) x += y;
            }
            const unsigned long long start = carry + x - cnt[h];
            carry += __shfl_sync(kAll, x, 31);
            // copy every source's run, one source at a time, lanes over its entries
            for (uint32_t k = 0; k < 32; ++k) {
                const uint32_t s = k + 32 * h;
                if (s >= S) break;
                const unsigned long long c = __shfl_sync(kAll, cnt[h], k);
                if (c == 0) continue;
                const unsigned long long st = __shfl_sync(kAll, start, k);
                const unsigned long long b = __shfl_sync(kAll, beg[h], k);
                const MergeSrc& m = srcs.s[s];
                FCLSH_DCHECK(s < S);
                for (unsigned long long j = lane; j < c; j += 32) {
                    dst.q[st + j] = uint32_t(q);
                    dst.id[st + j] = m.id[b + j];
                    dst.dist[st + j] = m.dist[b + j];
                }
            }
        }
    }
}

} // namespace

void merge_sources(const MergeSrcs& srcs, uint32_t S, uint64_t nq, const MergeDst& dst, cudaStream_t s, int device) {
    if (S == 0 || S > kMaxMergeSources) throw UsageError("merge: 1 to 64 sources");
    if (nq == 0) {
        FCLSH_CUDA(cudaMemsetAsync(dst.off, 0, 8, s));
        return;
    }
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((nq * 32 + 255) / 256,
                                                                          uint64_t(sm_count(device)) * 8)));
    k_merge_sources<<<grid, 256, 0, s>>>(srcs, S, nq, dst);
    FCLSH_LAUNCHED();
}

} // namespace fclsh_b200
