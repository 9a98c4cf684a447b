// fclsh_gpu.hpp -- header-only C++ adapter over the C-ABI (fclsh_gpu.h),
// shaped like the reference library so a reference caller switches by
// changing a namespace.
//
//   reference (proj/include/fclsh/...)          this adapter (fclsh::gpu)
//   build_covering_family(d, r, rng, opt)  ->   build_covering_family(d, r, seed, prime)
//   hash_batch_into(f, q, out, scratch)    ->   hash_batch(f, rows, n, words) (many rows)
//   make_plan(d, r, c, n, rng, force, b)   ->   make_plan(d, r, c, n, seed, force, b)
//   build_index(data, method, r, plan,     ->   build_index(rows, n, d, r, plan, seed, opt)
//               rng, opt)
//   query_r_nn(index, q, r, scratch)       ->   Index::query_r_nn(rows, nq, r)   (batched)
//   UsageError / DataError / ResourceError ->   same names, same meaning
//
// Exceptions carry the library's message; the class follows the C-ABI code
// (2 usage, 3 data, 4 resource, 5 CUDA runtime).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fclsh_gpu.h"

namespace fclsh::gpu {

struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ResourceError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(int rc) {
    if (rc == FCLSH_OK) return;
    const std::string msg = fclsh_last_error();
    switch (rc) {
    case FCLSH_ERR_USAGE: throw UsageError(msg);
    case FCLSH_ERR_DATA: throw DataError(msg);
    case FCLSH_ERR_RESOURCE: throw ResourceError(msg);
    case FCLSH_ERR_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
    }
}

inline constexpr uint64_t kMersenne61 = FCLSH_PRIME_M61;
inline constexpr uint64_t kMersenne31 = FCLSH_PRIME_M31;

class CoveringFamily {
public:
    explicit CoveringFamily(fclsh_family* h) : h_(h, fclsh_family_destroy) { check(fclsh_family_info_get(h, &info_)); }
    uint64_t dims() const { return info_.dims; }
    uint32_t radius() const { return info_.radius; }
    uint64_t prime() const { return info_.prime; }
    uint64_t table_count() const { return info_.tables; }
    std::vector<uint32_t> mapping() const {
        std::vector<uint32_t> m(info_.dims);
        check(fclsh_family_export(h_.get(), m.data(), nullptr));
        return m;
    }
    std::vector<uint64_t> seeds() const {
        std::vector<uint64_t> s(info_.dims);
        check(fclsh_family_export(h_.get(), nullptr, s.data()));
        return s;
    }
    const fclsh_family* handle() const { return h_.get(); }

private:
    std::shared_ptr<fclsh_family> h_;
    fclsh_family_info info_{};
};

inline CoveringFamily build_covering_family(uint64_t dims, uint32_t radius, uint64_t rng_seed,
                                            uint64_t prime = kMersenne61, bool include_zero_column = false,
                                            int32_t kind = FCLSH_KIND_AUTO) {
    fclsh_family* h = nullptr;
    check(fclsh_family_build(dims, radius, kind, rng_seed, prime, include_zero_column ? 1 : 0, &h));
    return CoveringFamily(h);
}

inline CoveringFamily make_covering_family(uint64_t dims, uint32_t radius, int32_t kind,
                                           const std::vector<uint32_t>& mapping, const std::vector<uint64_t>& seeds,
                                           uint64_t prime = kMersenne61) {
    if (mapping.size() != dims || seeds.size() != dims)
        throw UsageError("covering family: mapping/seeds must have one entry per dimension");
    fclsh_family* h = nullptr;
    check(fclsh_family_make(dims, radius, kind, mapping.data(), seeds.data(), prime, &h));
    return CoveringFamily(h);
}

// hash_batch_into for n rows (rows: n x words u64, BitVector word layout);
// returns n x L keys, point-major.
inline std::vector<uint64_t> hash_batch(const CoveringFamily& f, const uint64_t* rows, uint64_t n,
                                        uint32_t words, int device = 0) {
    std::vector<uint64_t> keys(n * f.table_count());
    check(fclsh_hash_batch_host(f.handle(), rows, n, words, keys.data(), 8, device));
    return keys;
}

class PreprocessPlan {
public:
    explicit PreprocessPlan(fclsh_plan* h) : h_(h, fclsh_plan_destroy) { check(fclsh_plan_info_get(h, &info_)); }
    const fclsh_plan_info& info() const { return info_; }
    const fclsh_plan* handle() const { return h_.get(); }

private:
    std::shared_ptr<fclsh_plan> h_;
    fclsh_plan_info info_{};
};

inline PreprocessPlan make_plan(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t rng_seed,
                                const fclsh_plan_override* force = nullptr,
                                uint64_t table_budget = FCLSH_DEFAULT_TABLE_BUDGET) {
    fclsh_plan* h = nullptr;
    check(fclsh_plan_make(dims, radius, c, n, rng_seed, force, table_budget, &h));
    return PreprocessPlan(h);
}

struct RnnBatch { // query_r_nn for every row of a batch
    std::vector<uint32_t> query, id, distance; // sorted by (query, id)
    std::vector<uint64_t> offsets;             // nq + 1
    std::vector<uint64_t> collisions, candidates, found;
};

class Index {
public:
    explicit Index(fclsh_index* h) : h_(h, fclsh_index_destroy) { check(fclsh_index_info_get(h, &info_)); }
    uint64_t table_count() const { return info_.table_count; }
    uint64_t entry_count() const { return info_.entry_count; }

    RnnBatch query_r_nn(const uint64_t* q_rows, uint64_t nq, uint32_t radius) {
        fclsh_result* r = nullptr;
        check(fclsh_query(h_.get(), q_rows, nq, radius, &r));
        return to_batch(r, nq);
    }

    // the host result block -> vectors (frees the block)
    static RnnBatch to_batch(fclsh_result* r, uint64_t nq) {
        std::unique_ptr<fclsh_result, void (*)(fclsh_result*)> guard(r, fclsh_result_free);
        RnnBatch b;
        if (!r) return b;
        b.query.assign(r->query, r->query + r->total);
        b.id.assign(r->id, r->id + r->total);
        b.distance.assign(r->distance, r->distance + r->total);
        b.offsets.assign(r->offsets, r->offsets + nq + 1);
        b.collisions.assign(r->collisions, r->collisions + nq);
        b.candidates.assign(r->candidates, r->candidates + nq);
        b.found.assign(r->found, r->found + nq);
        return b;
    }

private:
    std::shared_ptr<fclsh_index> h_;
    fclsh_index_info info_{};
};

// build_index(data, Method, radius, plan, rng, IndexOptions) with every option
// (fclsh_index_options_default, then set prime / method / delta / ...)
inline Index build_index(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius, const PreprocessPlan& plan,
                         uint64_t rng_seed, const fclsh_index_options& o) {
    fclsh_index* h = nullptr;
    check(fclsh_index_build(rows, 0, n, dims, radius, plan.handle(), rng_seed, &o, &h));
    return Index(h);
}

inline Index build_index(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius, const PreprocessPlan& plan,
                         uint64_t rng_seed, uint64_t prime = kMersenne61, int device = 0) {
    fclsh_index_options o;
    fclsh_index_options_default(&o);
    o.prime = prime;
    o.device = device;
    return build_index(rows, n, dims, radius, plan, rng_seed, o);
}

// Method::classic (index.cpp:65-76): bit sampling over the identity plan
inline Index build_classic_index(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius,
                                 const PreprocessPlan& plan, uint64_t rng_seed, uint64_t prime = kMersenne61,
                                 double delta = 0.1, uint32_t k_override = 0, uint64_t tables_override = 0) {
    fclsh_index_options o;
    fclsh_index_options_default(&o);
    o.prime = prime;
    o.method = FCLSH_METHOD_CLASSIC;
    o.delta = delta;
    o.k_override = k_override;
    o.tables_override = tables_override;
    return build_index(rows, n, dims, radius, plan, rng_seed, o);
}

// A point-sharded index over several GPUs (or several shards on one GPU):
// the same query_r_nn results as one Index over all points (fclsh_cluster_*).
class Cluster {
public:
    // this process drives `devices`, shards_per_device shards each
    Cluster(const std::vector<int>& devices, uint32_t shards_per_device) : h_(nullptr, fclsh_cluster_destroy) {
        fclsh_cluster* h = nullptr;
        check(fclsh_cluster_create(devices.data(), uint32_t(devices.size()), shards_per_device, &h));
        h_.reset(h, fclsh_cluster_destroy);
    }
    // one rank of a multi-process cluster (id from rank 0's unique_id())
    Cluster(const unsigned char* id, uint32_t world, uint32_t rank, int device, uint32_t shards_per_rank)
        : h_(nullptr, fclsh_cluster_destroy) {
        fclsh_cluster* h = nullptr;
        check(fclsh_cluster_create_rank(id, world, rank, device, shards_per_rank, &h));
        h_.reset(h, fclsh_cluster_destroy);
    }
    static std::vector<unsigned char> unique_id() {
        std::vector<unsigned char> id(FCLSH_CLUSTER_ID_BYTES);
        check(fclsh_cluster_unique_id(id.data()));
        return id;
    }
    void build(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius, const PreprocessPlan& plan,
               uint64_t rng_seed, uint64_t prime = kMersenne61, bool local_rows = false) {
        fclsh_index_options o;
        fclsh_index_options_default(&o);
        o.prime = prime;
        check(fclsh_cluster_build(h_.get(), rows, 0, local_rows ? FCLSH_ROWS_LOCAL : FCLSH_ROWS_GLOBAL, n, dims,
                                  radius, plan.handle(), rng_seed, &o));
    }
    fclsh_cluster_info info() const {
        fclsh_cluster_info i{};
        check(fclsh_cluster_info_get(h_.get(), &i));
        return i;
    }
    // collective; the merged result on rank 0 (empty elsewhere)
    RnnBatch query_r_nn(const uint64_t* q_rows, uint64_t nq, uint32_t radius) {
        fclsh_result* r = nullptr;
        check(fclsh_cluster_query(h_.get(), q_rows, nq, radius, &r));
        return Index::to_batch(r, nq);
    }

private:
    std::shared_ptr<fclsh_cluster> h_;
};

} // namespace fclsh::gpu
