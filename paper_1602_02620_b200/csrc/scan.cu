// GPU linear scan: scan_truth (workload.cpp:56-71) and
// distance_histogram (workload.cpp:133-151) over device rows -- a second,
// exhaustive oracle for results at full config scale, and the reference's
// `linear` method.
//
// A CTA holds a tile of QT query rows in shared memory and streams data
// rows; a thread compares one data row (words in registers) with every query
// of the tile: XOR + popcount per word. The data is re-read once per query
// tile (rows stream from HBM, the tile from shared memory). scan_truth runs
// a count pass, a scan of the per-query counts, a write pass (per-query
// cursors) and a segmented sort of each query's ids, so the output is ordered
// by (query, point) exactly like the reference's double loop.

#include "scan.hpp"

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace fclsh_b200 {

namespace {

constexpr int kQT = 32;      // queries per tile (shared memory)
constexpr int kRegWords = 8; // rows of <= 512 bits are held in registers

enum Mode { kCount = 0, kWrite = 1, kHist = 2 };

template <int MODE, int RW>
__global__ void __launch_bounds__(256) k_scan_pairs(const uint64_t* __restrict__ rows, uint64_t n,
                                                    const uint64_t* __restrict__ qrows, uint64_t nq, uint32_t words,
                                                    uint32_t radius, uint32_t* __restrict__ qcount,
                                                    const unsigned long long* __restrict__ qoff,
                                                    uint32_t* __restrict__ out_id, uint32_t* __restrict__ out_dist,
                                                    unsigned long long* __restrict__ hist, uint32_t nbins) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* qs = reinterpret_cast<uint64_t*>(smem);                      // kQT x words
    unsigned int* hs = reinterpret_cast<unsigned int*>(qs + kQT * words);  // nbins (kHist)
    const uint64_t q0 = uint64_t(blockIdx.y) * kQT;
    const uint32_t qt = uint32_t(nq - q0 < uint64_t(kQT) ? nq - q0 : uint64_t(kQT));
    for (uint32_t i = threadIdx.x; i < qt * words; i += blockDim.x) qs[i] = qrows[q0 * words + i];
    if constexpr (MODE == kHist)
        for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) hs[i] = 0;
    __syncthreads();
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t* row = rows + r * words;
        uint64_t w[RW > 0 ? RW : 1];
        if constexpr (RW > 0) {
#pragma unroll
            for (int k = 0; k < RW; ++k) w[k] = k < int(words) ? __ldg(row + k) : 0ull;
        }
        for (uint32_t j = 0; j < qt; ++j) {
            const uint64_t* q = qs + j * words;
            uint32_t d = 0;
            if constexpr (RW > 0) {
#pragma unroll
                for (int k = 0; k < RW; ++k)
                    if (k < int(words)) d += __popcll(w[k] ^ q[k]);
            } else {
                for (uint32_t k = 0; k < words; ++k) d += __popcll(__ldg(row + k) ^ q[k]);
            }
            if constexpr (MODE == kHist) {
                atomicAdd(hs + d, 1u);
            } else if (d <= radius) {
                if constexpr (MODE == kCount) {
                    atomicAdd(qcount + q0 + j, 1u);
                } else {
                    const unsigned long long pos = qoff[q0 + j] + atomicAdd(qcount + q0 + j, 1u);
                    out_id[pos] = uint32_t(r);
                    out_dist[pos] = d;
                }
            }
        }
    }
    if constexpr (MODE == kHist) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x)
            if (hs[i]) atomicAdd(hist + i, (unsigned long long)hs[i]);
    }
}

// Sampled histogram: pair k = (query k / s, point idx[k]).
__global__ void k_hist_sampled(const uint64_t* __restrict__ rows, const uint64_t* __restrict__ qrows, uint64_t nq,
                               uint64_t s, const uint64_t* __restrict__ idx, uint32_t words,
                               unsigned long long* __restrict__ hist) {
    const uint64_t pairs = nq * s;
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < pairs;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t* a = rows + idx[k] * words;
        const uint64_t* b = qrows + (k / s) * words;
        uint32_t d = 0;
        for (uint32_t w = 0; w < words; ++w) d += __popcll(__ldg(a + w) ^ __ldg(b + w));
        atomicAdd(hist + d, 1ull);
    }
}

__global__ void k_widen(const uint32_t* __restrict__ a, unsigned long long* __restrict__ b, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        b[i] = a[i];
}

unsigned grid_of(uint64_t work, int device) {
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, uint64_t(sm_count(device)) * 8)));
}

__global__ void k_fill_query(uint64_t nq, const unsigned long long* __restrict__ off, uint32_t* __restrict__ out_q) {
    for (uint64_t q = blockIdx.x; q < nq; q += gridDim.x)
        for (uint64_t k = off[q] + threadIdx.x; k < off[q + 1]; k += blockDim.x) out_q[k] = uint32_t(q);
}

template <int MODE>
void launch_pairs(const ScanArgs& a, uint32_t* qcount, const unsigned long long* qoff, uint32_t* out_id,
                  uint32_t* out_dist, unsigned long long* hist, uint32_t nbins, cudaStream_t s, int device) {
    const size_t smem = size_t(kQT) * a.words * 8 + (MODE == kHist ? size_t(nbins) * 4 : 0);
    const uint64_t tiles = (a.nq + kQT - 1) / kQT;
    if (tiles > 65535) throw UsageError("scan: too many queries in one call (split the batch)");
    auto kern = a.words <= kRegWords ? k_scan_pairs<MODE, kRegWords> : k_scan_pairs<MODE, 0>;
    const int per_sm = resident_ctas(kern, 256, smem, device);
    if (per_sm < 1) throw ResourceError("scan: rows too wide for a shared-memory query tile");
    // data blocks x query tiles, about 4 waves of CTAs in all
    const uint64_t want = uint64_t(per_sm) * sm_count(device) * 4;
    const uint64_t bx = std::max<uint64_t>(1, std::min<uint64_t>((a.n + 255) / 256, (want + tiles - 1) / tiles));
    kern<<<dim3(unsigned(bx), unsigned(tiles)), 256, smem, s>>>(a.rows, a.n, a.qrows, a.nq, a.words, a.radius,
                                                               qcount, qoff, out_id, out_dist, hist, nbins);
    FCLSH_LAUNCHED();
}

} // namespace

ScanOutput scan_truth_device(ScanState& st, const ScanArgs& a, cudaStream_t s) {
    if (a.n >= (uint64_t(1) << 32)) throw UsageError("scan: point ids must fit 32 bits");
    ScanOutput o;
    o.nq = a.nq;
    FCLSH_CUDA(cudaSetDevice(st.device));
    auto* cnt = static_cast<uint32_t*>(st.count.ensure(std::max<uint64_t>(1, a.nq + 1) * 4));
    auto* off = static_cast<unsigned long long*>(st.offsets.ensure((a.nq + 1) * 8));
    auto* wide = static_cast<unsigned long long*>(st.wide.ensure((a.nq + 1) * 8));
    if (a.nq == 0) {
        FCLSH_CUDA(cudaMemsetAsync(off, 0, 8, s));
        o.d_offsets = reinterpret_cast<uint64_t*>(off);
        return o;
    }
    // pass 1: matches per query
    FCLSH_CUDA(cudaMemsetAsync(cnt, 0, (a.nq + 1) * 4, s));
    if (a.n) launch_pairs<kCount>(a, cnt, nullptr, nullptr, nullptr, nullptr, 0, s, st.device);
    // offsets (64-bit): widen the counts, exclusive scan
    {
        k_widen<<<grid_of(a.nq + 1, st.device), 256, 0, s>>>(cnt, wide, a.nq + 1);
        FCLSH_LAUNCHED();
        size_t tb = 0;
        FCLSH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, wide, off, a.nq + 1, s));
        FCLSH_CUDA(cub::DeviceScan::ExclusiveSum(st.cub_tmp.ensure(tb), tb, wide, off, a.nq + 1, s));
    }
    unsigned long long total = 0;
    FCLSH_CUDA(cudaMemcpyAsync(&total, off + a.nq, 8, cudaMemcpyDeviceToHost, s));
    FCLSH_CUDA(cudaStreamSynchronize(s));
    o.total = total;
    const uint64_t cap = std::max<uint64_t>(1, total);
    auto* id0 = static_cast<uint32_t*>(st.id_tmp.ensure(cap * 4));
    auto* d0 = static_cast<uint32_t*>(st.dist_tmp.ensure(cap * 4));
    auto* id1 = static_cast<uint32_t*>(st.id.ensure(cap * 4));
    auto* d1 = static_cast<uint32_t*>(st.dist.ensure(cap * 4));
    auto* oq = static_cast<uint32_t*>(st.query.ensure(cap * 4));
    if (total) {
        // pass 2: write each match at its query's offset + cursor
        FCLSH_CUDA(cudaMemsetAsync(cnt, 0, (a.nq + 1) * 4, s));
        launch_pairs<kWrite>(a, cnt, off, id0, d0, nullptr, 0, s, st.device);
        // ascending ids within each query
        size_t sb = 0;
        FCLSH_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, sb, id0, id1, d0, d1, int64_t(total), int64_t(a.nq),
                                                       off, off + 1, s));
        FCLSH_CUDA(cub::DeviceSegmentedSort::SortPairs(st.cub_tmp.ensure(sb), sb, id0, id1, d0, d1, int64_t(total),
                                                       int64_t(a.nq), off, off + 1, s));
        k_fill_query<<<unsigned(std::min<uint64_t>(a.nq, 65535)), 128, 0, s>>>(a.nq, off, oq);
        FCLSH_LAUNCHED();
    }
    o.d_query = oq;
    o.d_id = id1;
    o.d_dist = d1;
    o.d_offsets = reinterpret_cast<uint64_t*>(off);
    return o;
}

void distance_histogram_device(ScanState& st, const ScanArgs& a, uint64_t sample_per_query, uint64_t seed,
                               uint64_t* counts, cudaStream_t s) {
    FCLSH_CUDA(cudaSetDevice(st.device));
    const uint32_t nbins = uint32_t(a.dims + 1);
    auto* hist = static_cast<unsigned long long*>(st.hist.ensure(uint64_t(nbins) * 8));
    FCLSH_CUDA(cudaMemsetAsync(hist, 0, uint64_t(nbins) * 8, s));
    if (a.nq && a.n) {
        if (sample_per_query == 0 || sample_per_query >= a.n) {
            launch_pairs<kHist>(a, nullptr, nullptr, nullptr, nullptr, hist, nbins, s, st.device);
        } else {
            // the reference's draws: Rng(seed).stream("histogram").below(n), query-major
            Rng rng = Rng(seed).stream("histogram");
            std::vector<uint64_t> idx(a.nq * sample_per_query);
            for (auto& v : idx) v = rng.below(a.n);
            auto* didx = static_cast<uint64_t*>(st.sample_idx.ensure(idx.size() * 8));
            FCLSH_CUDA(cudaMemcpyAsync(didx, idx.data(), idx.size() * 8, cudaMemcpyHostToDevice, s));
            const uint64_t pairs = idx.size();
            k_hist_sampled<<<grid_of(pairs, st.device), 256, 0, s>>>(a.rows, a.qrows, a.nq, sample_per_query, didx, a.words, hist);
            FCLSH_LAUNCHED();
            FCLSH_CUDA(cudaStreamSynchronize(s)); // idx lives on the host stack
        }
    }
    FCLSH_CUDA(cudaMemcpyAsync(counts, hist, uint64_t(nbins) * 8, cudaMemcpyDeviceToHost, s));
    FCLSH_CUDA(cudaStreamSynchronize(s));
}

} // namespace fclsh_b200
