// Multi-GPU sharded index behind fclsh_cluster_* (include/fclsh_gpu.h).
//
// Points are sharded in contiguous id ranges over world x shards_per_rank
// shards (shard g owns ids [g*n/S, (g+1)*n/S), balanced); every shard is a
// DeviceIndex built with the same families (they depend on (d, r, seed) only,
// index.cpp:83-88) and the shard's id offset. One member per GPU: either one
// process drives every GPU (fclsh_cluster_create, ncclCommInitAll) or each
// process drives its own (fclsh_cluster_create_rank, ncclCommInitRank -- one
// process per GPU under torchrun). A batch:
//   1. the root (rank 0) holds the query rows; ncclBroadcast to every member;
//   2. every shard answers the batch concurrently (one stream per shard);
//   3. each member merges its shards' results (k_merge_sources): per query
//      the shards' runs in shard order, counters summed -- shard id ranges
//      increase with the shard number, so this is (query, id) order, and
//      every posting and id lives in exactly one shard, so the counters are
//      the single index's (the reference's query_r_nn, index.cpp:157-188);
//   4. members send their packed result to the root (ncclAllGather of the
//      totals, then grouped ncclSend / ncclRecv), and the root merges the
//      ranks' results the same way.
// NCCL is loaded at run time (dlopen: the copy torch already mapped, else
// the system libnccl.so.2) and only for world > 1 (or FCLSH_CLUSTER_NCCL=1).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "index.cuh"

namespace fclsh_b200 {

// ------------------------------------------------------------- merge kernel
constexpr uint32_t kMaxMergeSources = 64;
struct MergeSrc {
    const unsigned long long *off, *coll, *cand, *found; // [nq+1], [nq] x 3
    const uint32_t *id, *dist;                           // [off[nq]]
};
struct MergeSrcs {
    MergeSrc s[kMaxMergeSources];
};
struct MergeDst {
    unsigned long long *off, *coll, *cand, *found;
    uint32_t *q, *id, *dist;
};
void merge_sources(const MergeSrcs& srcs, uint32_t S, uint64_t nq, const MergeDst& dst, cudaStream_t s, int device);

// Packed result of one member: [off (nq+1) | coll nq | cand nq | found nq]
// u64, then [q | id | dist] u32 x total. One contiguous block, one ncclSend.
struct Packed {
    static uint64_t words64(uint64_t nq) { return 4 * nq + 1; }
    static uint64_t bytes(uint64_t nq, uint64_t total) {
        return (words64(nq) * 8 + 3 * total * 4 + 7) & ~uint64_t(7);
    }
    static MergeDst dst(void* p, uint64_t nq, uint64_t total) {
        auto* w = static_cast<unsigned long long*>(p);
        auto* t = reinterpret_cast<uint32_t*>(w + words64(nq));
        return MergeDst{w, w + nq + 1, w + 2 * nq + 1, w + 3 * nq + 1, t, t + total, t + 2 * total};
    }
    static MergeSrc src(const void* p, uint64_t nq, uint64_t total) {
        const MergeDst d = dst(const_cast<void*>(p), nq, total);
        return MergeSrc{d.off, d.coll, d.cand, d.found, d.id, d.dist};
    }
};

// ------------------------------------------------------------------ cluster
struct ClusterShard {
    std::unique_ptr<DeviceIndex> ix;
    uint64_t begin = 0, end = 0; // global ids (before the cluster's id offset)
    QueryOutput out;
};

struct ClusterMember {
    int device = 0;
    uint32_t rank = 0;
    void* comm = nullptr; // ncclComm_t (world > 1)
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    std::vector<ClusterShard> shards;
    DevBuf q_rows;       // the broadcast batch
    DevBuf packed;       // this member's merged result (packed)
    DevBuf recv;         // root: every other rank's packed result
    DevBuf out;          // root: the final merged result (packed)
    DevBuf totals;       // u64 [world] (all-gathered batch totals)
    unsigned long long* h_totals = nullptr; // pinned mirror
    uint64_t total = 0;  // this member's batch total
    ~ClusterMember();
};

struct ClusterResult {
    uint64_t nq = 0, total = 0;
    // device pointers on the root's device (valid until the next batch)
    const unsigned long long *off = nullptr, *coll = nullptr, *cand = nullptr, *found = nullptr;
    const uint32_t *q = nullptr, *id = nullptr, *dist = nullptr;
    int device = 0;
    cudaStream_t stream = nullptr; // the root member's stream (results complete in its order)
    bool root = false;             // false: this process holds no result (rank != 0)
    const ClusterShard* single = nullptr; // one shard in all: its own output (host fast path)
};

struct Cluster {
    uint32_t world = 1;           // ranks (one per GPU)
    uint32_t shards_per_rank = 1;
    bool use_nccl = false;
    std::vector<std::unique_ptr<ClusterMember>> members; // the ranks this process drives
    bool built = false;
    uint64_t n = 0, dims = 0, id_offset = 0;
    uint32_t radius = 0, row_words = 0;
    double build_ms = 0;
    std::mutex mu;

    uint32_t total_shards() const { return world * shards_per_rank; }
    ClusterMember* root() const; // the rank-0 member if this process drives it
    ~Cluster();
};

// Creation: single process over `devices` (ncclCommInitAll when > 1), or one
// rank of a multi-process cluster (ncclCommInitRank with the root's id).
std::unique_ptr<Cluster> cluster_create(const int* devices, uint32_t ndev, uint32_t shards_per_rank);
std::unique_ptr<Cluster> cluster_create_rank(const unsigned char* uid, uint32_t world, uint32_t rank, int device,
                                             uint32_t shards_per_rank);
void cluster_unique_id(unsigned char* uid); // 128 bytes (ncclGetUniqueId)

// rows: every point (rows_global) or only this process's contiguous range.
void cluster_build(Cluster& cl, const uint64_t* rows, bool rows_on_device, bool rows_global, uint64_t n,
                   uint64_t dims, uint32_t radius, const Plan& plan, uint64_t rng_seed,
                   const IndexBuildOptions& opt);

// One batch over the whole cluster (collective: every process calls it).
// q_rows: host or device (q_on_device) rows on the root; ignored elsewhere.
// stream: the caller's stream on the root's device (device rows are read
// after it, results are ordered before it); may be null.
ClusterResult cluster_query(Cluster& cl, const uint64_t* q_rows, bool q_on_device, uint64_t nq, uint32_t radius,
                            cudaStream_t stream);

} // namespace fclsh_b200
