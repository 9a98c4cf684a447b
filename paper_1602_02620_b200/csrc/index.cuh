// K2 table build and K3-K5 query (reference: build_index, index.cpp:49-119;
// PostingTable, posting.cpp:9-21; query_r_nn, index.cpp:125-188).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "common.cuh"
#include "hash.cuh"
#include "host.hpp"

namespace fclsh_b200 {

constexpr int kLayoutAuto = 0;
constexpr int kLayoutCsr = 1;
constexpr int kLayoutBuckets = 2;
constexpr int kMethodCovering = 0;
constexpr int kMethodClassic = 2; // Method::classic (index.hpp:22)

// Device layout of one shard's index. An entry is
// u64 (key << 32 | id) when prime < 2^32, else {u64 key, u64 id}.
//   rows     n x W u64          the shard's points (verify reads them)
//   kLayoutBuckets (default):
//     entries  T x 2^bb x 4     per table, open-addressed buckets of four
//                               entries, home bucket key >> shift, linear
//                               probing, load <= 50%, empty = all-ones
//   kLayoutCsr (memory-tight):
//     entries  T x n            per table, (key, id) sorted by (key, id)
//     dir      T x (D + 1) u32  CSR offsets of D = 2^b key cells
//                               (cell = key >> shift)
struct DeviceIndex {
    int device = 0;
    cudaStream_t stream = nullptr;
    Plan plan;
    uint32_t radius = 0;
    uint64_t n = 0, dims = 0;
    uint32_t row_words = 0;
    uint64_t prime = 0;
    bool wide = false;        // 16-byte entries (prime >= 2^32)
    uint64_t tables = 0;      // T
    int layout = 0;           // kLayoutCsr or kLayoutBuckets
    uint64_t nbuckets = 0;    // buckets per table (kLayoutBuckets)
    uint32_t dir_bits = 0;    // b (kLayoutCsr)
    uint32_t key_shift = 0;   // cell / home bucket = (key * key_scale) >> key_shift
    uint64_t key_scale = 0;   // floor(2^64 / prime)
    uint64_t id_offset = 0;
    double build_ms = 0;
    int method = kMethodCovering;
    std::unique_ptr<DeviceFamilySet> fs;
    DevBuf rows, entries, dir;
    // per-table key filter (buckets layout, index.cu): filter_words 32-bit
    // words per table, bit floor(key * 32 * filter_words / P) set iff
    // some posting of the table maps there; 0 words: no filter
    DevBuf filter;
    uint32_t filter_words = 0;
    bool l2_persist = false; // holds a share of the device's persisting-L2 limit (restored by the last holder)

    // query workspace (grow-only)
    DevBuf q_rows, q_keys, r_start, r_count, counters, coll_off, coll_sel, fill, cand, cand_sorted, src_pos,
        res_tmp_id, res_tmp_dist, res2_id, res2_dist, res_cta_id, res_cta_dist, overflow, overflow2, overflow_cnt,
        out_q, out_id, out_dist, cub_tmp;
    // mapped pinned words k_compact publishes {total, hand-over counts, seq} to;
    // the batch sequence number is counted on the device (pub_seq_dev)
    unsigned long long* h_pub = nullptr;
    unsigned long long* d_pub = nullptr;
    unsigned long long pub_seq = 0;
    DevBuf pub_seq_dev, cub_tmp2;
    // the common path as a CUDA graph, keyed by shape + buffers (index.cu)
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t gsrc = nullptr;          // the captured graph gexec was instantiated from (owns gprologue)
    cudaGraphNode_t gprologue = nullptr; // the batch prologue's kernel node (its HostDest patched per launch)
    std::vector<const void*> gkey, gpending;
    uint64_t gkernels = 0;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr; // caller-stream fork / join
    // side branch of a batch: the HostDest descriptor's H2D copy (beside the hash)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    uint64_t last_total = 0;
    uint64_t last_dense = 0;    // queries the CTA-per-query kernel served
    uint64_t last_overflow = 0; // queries that took the general path
    double t_hash_ms = 0, t_probe_ms = 0, t_verify_ms = 0;
    // device time of the last query per stage: hash (S1), fused warp-per-query
    // probe+dedup+verify (S2+S3), the CTA-per-query kernel for the dense
    // queries the warp kernel hands over, found scan, compaction, general path
    // for what is left (+ its rescan / recompaction; includes one host sync)
    static constexpr int kStages = 6;
    double stage_ms[kStages] = {};
    cudaEvent_t ev[kStages + 1] = {};
    bool stages_pending = false;
    // per-stage events cost ~4 us each in a replayed graph: off by default,
    // the batch total (batch_ms) is always measured
    bool stage_timing = false, stages_timed = false;
    double batch_ms = 0;
    // the batch between query_enqueue and query_finish
    struct Pending {
        bool active = false;
        uint64_t nq = 0;
        uint32_t radius = 0;
        const uint64_t* d_q = nullptr;
        bool host_cnt = false, dense_all = false;
        uint64_t dest_cap = 0;
        unsigned long long seq = 0;
        cudaStream_t caller = nullptr; // joined after the batch (null: none)
    } pending;
    void collect_stages(); // waits for the last batch, fills stage_ms / t_*_ms (-1 = not measured)

    ~DeviceIndex();
    uint64_t cells() const { return uint64_t(1) << dir_bits; }
    uint64_t entry_bytes() const { return wide ? 16 : 8; }
    uint64_t device_bytes() const { return rows.bytes + entries.bytes + dir.bytes; }
};

// Raises the device's persisting-L2 limit to cover `bytes` (the key filter)
// for as long as some index holds it; the last release restores the limit
// found by the first acquire.
bool l2_persist_acquire(int device, uint64_t bytes);
void l2_persist_release(int device);

struct IndexBuildOptions {
    uint64_t prime = kMersenne61;
    bool include_zero_column = false;
    uint64_t table_budget = kDefaultTableBudget;
    int device = 0;
    uint64_t id_offset = 0;
    int directory_bits = 0;
    int layout = kLayoutAuto;
    uint64_t mem_budget = 0; // device bytes this build may take (0: the free memory); picks the layout
    // Method (index.hpp:22): covering_batch (= covering_reference: identical
    // buckets) or classic bit sampling with IndexOptions::delta / k_override /
    // tables_override (index.hpp:29-32; 0 = unset)
    int method = kMethodCovering;
    double delta = 0.1;
    uint32_t k_override = 0;
    uint64_t tables_override = 0;
};

// build_index(data, covering_batch, radius, plan, Rng(rng_seed), opt).
std::unique_ptr<DeviceIndex> build_index(const uint64_t* rows, bool rows_on_device, uint64_t n,
                                         uint64_t dims, uint32_t radius, const Plan& plan,
                                         uint64_t rng_seed, const IndexBuildOptions& opt);

struct QueryOutput {
    uint64_t nq = 0, total = 0;
    uint32_t *d_query = nullptr, *d_id = nullptr, *d_dist = nullptr;
    uint64_t *d_offsets = nullptr, *d_coll = nullptr, *d_cand = nullptr, *d_found = nullptr;
    // host_counters: the batch kernel wrote [offsets | collisions | candidates
    // | found] into HostDest::counters; host_results: also query / id /
    // distance into the HostDest arrays (total <= cap). Otherwise those are
    // in the device buffers above.
    bool host_counters = false, host_results = false;
};

// Mapped pinned host destination (device-usable pointers) that the batch's
// compaction kernel writes directly, overlapping the transfer with its own
// work: counters = 4 x (nq + 1) words, q / id / distance = cap entries each.
struct HostDest {
    unsigned long long* counters;
    uint32_t* q;
    uint32_t* id;
    uint32_t* dist;
    unsigned long long cap;
};

// query_r_nn for nq device rows; results in index-owned device buffers.
// Split in two so that several indexes (the shards of a cluster) run their
// batches concurrently: query_enqueue queues the batch on the index's stream
// (after the work already queued on `stream`) and returns at once;
// query_finish waits for the batch's published total, runs the general path
// if any query needs it, joins `stream` and returns the outputs. One batch in
// flight per index. query_device = both.
// dest (optional): mapped pinned host destination the batch writes directly.
// hash_src (optional): the same rows in mapped pinned host memory (device
// view); the hash kernel reads them there and writes d_q as it goes, so no
// separate host-to-device copy of the batch is needed.
void query_enqueue(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, cudaStream_t stream,
                   const HostDest* dest = nullptr, const uint64_t* hash_src = nullptr);
QueryOutput query_finish(DeviceIndex& ix);
QueryOutput query_device(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, cudaStream_t stream,
                         const HostDest* dest = nullptr, const uint64_t* hash_src = nullptr);

// query_c_r_nn (index.cpp:190-235) for nq device rows: d_counters [nq][3]
// {collisions, candidates, found}, d_best [nq][2] {id, distance} (all-ones
// when nothing was retrieved). posting_budget < 0: the default 3L. Synchronous.
void query_c_device(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, int64_t posting_budget,
                    uint64_t* d_counters, uint32_t* d_best, cudaStream_t stream);

} // namespace fclsh_b200
