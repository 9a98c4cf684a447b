// C-ABI of libfclsh_b200.so (include/fclsh_gpu.h). Every entry point maps the
// reference's exceptions to return codes (errors.hpp:8-29) and records the
// message for fclsh_last_error().

#include "../../include/fclsh_gpu.h"

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "common.cuh"
#include "hash.cuh"
#include "host.hpp"
#include "dataset.hpp"
#include "index.cuh"
#include "scan.hpp"
#include "cluster.hpp"

namespace fclsh_b200 {
void gen_bernoulli(uint64_t seed, uint64_t row0, uint64_t n, uint64_t dims, uint64_t* rows, int threads);
void gen_clustered(uint64_t seed, uint64_t centres, uint64_t row0, uint64_t n, uint64_t dims, double flip_p,
                   uint64_t* rows, int threads);
void gen_planted(uint64_t seed, const uint64_t* data, uint64_t n, uint64_t dims, uint64_t nq, uint32_t kmax,
                 uint64_t* qrows, uint32_t* src_out);

void merge_shards(uint32_t world, uint64_t nq, const uint64_t* d_offsets, const uint32_t* d_triples, uint64_t cap,
                  uint32_t* d_out, uint64_t out_cap, uint64_t* d_out_offsets, cudaStream_t s, int device);

uint64_t& launch_counter() {
    static thread_local uint64_t c = 0;
    return c;
}

int resident_ctas_impl(const void* kern, int threads, size_t smem, int device) {
    struct Key {
        const void* k;
        int threads;
        size_t smem;
        int device;
        bool operator<(const Key& o) const {
            if (k != o.k) return k < o.k;
            if (threads != o.threads) return threads < o.threads;
            if (smem != o.smem) return smem < o.smem;
            return device < o.device;
        }
    };
    static std::mutex mu;
    static std::map<Key, int> cache;
    static std::map<std::pair<const void*, int>, size_t> limit; // dynamic-smem limit set so far
    const Key key{kern, threads, smem, device};
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    // the limit only ever grows: a smaller launch must not lower it under a
    // larger one that is already cached
    size_t& lim = limit[{kern, device}];
    if (smem > lim) {
        FCLSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        lim = smem;
    }
    int per_sm = 0;
    FCLSH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    cache[key] = per_sm;
    return per_sm;
}
} // namespace fclsh_b200

using namespace fclsh_b200;

struct fclsh_family {
    Family f;
    std::mutex mu;
    std::map<int, std::unique_ptr<DeviceFamilySet>> dev;
    DeviceFamilySet& on(int device) {
        std::lock_guard<std::mutex> lk(mu);
        auto& slot = dev[device];
        if (!slot) slot = make_device_family_set(f, device);
        return *slot;
    }
};

struct fclsh_plan {
    Plan p;
};

struct fclsh_dataset {
    HostDataset ds;
};

struct fclsh_scan {
    ScanState st;
};

struct fclsh_cluster {
    std::unique_ptr<Cluster> cl;
    DevBuf q_host_rows; // one-shard fast path: device staging for the host call
};

struct fclsh_index {
    std::unique_ptr<DeviceIndex> ix;
    DevBuf q_host_rows; // device staging for fclsh_query
    // Calls on one handle serialize (the header's contract): the query entry
    // points share the index's scratch, result buffers, captured graph and
    // publish handshake, so concurrent callers take turns here.
    mutable std::mutex mu;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return FCLSH_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host memory exhausted";
        return FCLSH_ERR_RESOURCE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FCLSH_ERR_OTHER;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw UsageError(std::string(what) + " must not be NULL");
}

// fclsh_query results live in pinned blocks (device-to-host copies run at
// full speed, no staging) recycled through this pool, so a steady stream of
// batches does not pay cudaHostAlloc per call. A block starts with a header
// {magic, capacity}; fclsh_result_free hands it back.
constexpr size_t kResultHeader = 64;
constexpr uint64_t kResultMagic = 0x66636c7368726573ull; // "fclshres"
class PinnedPool {
  public:
    void* take(size_t bytes) {
        size_t cap = 4096;
        while (cap < bytes) cap <<= 1;
        void* p = nullptr;
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto it = free_.find(cap);
            if (it != free_.end()) {
                p = it->second;
                free_.erase(it);
                cached_ -= cap;
            }
        }
        if (!p) {
            // mapped: the batch kernel writes results straight into the block
            if (cudaHostAlloc(&p, cap, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                throw ResourceError("query: pinned host memory for the result exhausted");
            }
            void* d = nullptr;
            if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) {
                cudaGetLastError();
                d = nullptr;
            }
            static_cast<uint64_t*>(p)[2] = reinterpret_cast<uintptr_t>(d);
        }
        static_cast<uint64_t*>(p)[0] = kResultMagic;
        static_cast<uint64_t*>(p)[1] = cap;
        return p;
    }
    // device-usable address of a pointer into a block (null: not mapped)
    template <typename T>
    static T* device_view(void* blk, T* host) {
        const uint64_t d = static_cast<uint64_t*>(blk)[2];
        if (!d) return nullptr;
        return reinterpret_cast<T*>(d + (reinterpret_cast<unsigned char*>(host) - static_cast<unsigned char*>(blk)));
    }
    void give(void* blk) {
        auto* h = static_cast<uint64_t*>(blk);
        if (h[0] != kResultMagic) return; // not ours: leave it alone
        const size_t cap = h[1];
        h[0] = 0;
        std::lock_guard<std::mutex> lk(mu_);
        if (cached_ + cap <= (size_t(256) << 20)) {
            free_.emplace(cap, blk);
            cached_ += cap;
        } else {
            cudaFreeHost(blk);
        }
    }

  private:
    std::mutex mu_;
    std::multimap<size_t, void*> free_;
    size_t cached_ = 0;
};

PinnedPool& pinned_pool() {
    static PinnedPool* pool = new PinnedPool; // never destroyed: CUDA may be torn down first at exit
    return *pool;
}

// One pinned block per result: [header | fclsh_result | offsets | collisions
// | candidates | found | id | distance | query], room for `ids` triples.
fclsh_result* new_result(uint64_t nq, uint64_t ids, unsigned char** blk_out) {
    const uint64_t qb = (nq + 1) * 8;
    const uint64_t tb = std::max<uint64_t>(1, ids) * 4;
    const size_t bytes = kResultHeader + sizeof(fclsh_result) + 4 * qb + 3 * (tb + 16);
    unsigned char* blk = static_cast<unsigned char*>(pinned_pool().take(bytes));
    fclsh_result* r = reinterpret_cast<fclsh_result*>(blk + kResultHeader);
    std::memset(r, 0, sizeof(fclsh_result));
    unsigned char* p = blk + kResultHeader + ((sizeof(fclsh_result) + 15) & ~size_t(15));
    r->nq = nq;
    r->offsets = reinterpret_cast<uint64_t*>(p); // device layout: offsets | collisions | candidates | found
    r->collisions = r->offsets + (nq + 1);
    r->candidates = r->offsets + 2 * (nq + 1);
    r->found = r->offsets + 3 * (nq + 1);
    p += 4 * qb;
    r->id = reinterpret_cast<uint32_t*>(p);
    r->distance = reinterpret_cast<uint32_t*>(p + ((tb + 15) & ~uint64_t(15)));
    r->query = reinterpret_cast<uint32_t*>(p + 2 * ((tb + 15) & ~uint64_t(15)));
    r->time_hash_ms = r->time_probe_ms = r->time_verify_ms = -1;
    if (blk_out) *blk_out = blk;
    return r;
}

// query_r_nn for host rows on one index, host result out (fclsh_query and
// the one-shard cluster): see fclsh_query in the header.
fclsh_result* query_host(DeviceIndex& ix, DevBuf& staging, const uint64_t* q_rows, uint64_t nq, uint32_t radius) {
    FCLSH_CUDA(cudaSetDevice(ix.device));
    const uint64_t W = ix.row_words;
    uint64_t* dq = static_cast<uint64_t*>(staging.ensure(std::max<uint64_t>(1, nq) * W * 8));
    // Rows in pinned (page-locked, device-mapped) host memory are hashed
    // in place: the hash kernel reads them over PCIe and writes the
    // device copy the verify reads, so the batch has no separate H2D
    // copy. Pageable rows: one cudaMemcpyAsync. FCLSH_NO_ZERO_COPY=1: copy always.
    const uint64_t* hsrc = nullptr;
    static const bool no_zc = getenv("FCLSH_NO_ZERO_COPY") != nullptr;
    if (nq && !no_zc) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, q_rows) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer)
            hsrc = static_cast<const uint64_t*>(pa.devicePointer);
        cudaGetLastError();
    }
    if (nq && !hsrc) FCLSH_CUDA(cudaMemcpyAsync(dq, q_rows, nq * W * 8, cudaMemcpyHostToDevice, ix.stream));
    // one pinned block per result: [header | fclsh_result | counters | id | distance | query].
    // Sized for a guess of the result count, so the counters can be read
    // back while the batch runs; a larger total takes a larger block.
    const uint64_t qb = (nq + 1) * 8;
    cudaStream_t s = ix.stream;
    unsigned char* blk = nullptr;
    fclsh_result* r = nullptr;
    uint64_t cap = 0;
    auto layout = [&](uint64_t ids) {
        r = new_result(nq, ids, &blk);
        cap = ids;
    };
    layout(std::max<uint64_t>(1024, ix.last_total + ix.last_total / 4));
    // the batch kernel writes counters and results straight into the block
    HostDest dest{PinnedPool::device_view(blk, reinterpret_cast<unsigned long long*>(r->offsets)),
                  PinnedPool::device_view(blk, r->query), PinnedPool::device_view(blk, r->id),
                  PinnedPool::device_view(blk, r->distance), cap};
    QueryOutput o;
    try {
        static const bool no_dest = getenv("FCLSH_NO_HOST_DEST") != nullptr; // A/B: D2H copies instead
        o = query_device(ix, dq, nq, radius, s, dest.counters && !no_dest ? &dest : nullptr, hsrc);
    } catch (...) {
        cudaStreamSynchronize(s);
        pinned_pool().give(blk);
        throw;
    }
    bool copies = false;
    const bool grew = o.total > cap;
    if (grew) { // more results than the guess: a larger block
        pinned_pool().give(blk); // (no copy or kernel targets it any more: the batch was published)
        layout(o.total);
    }
    if (!o.host_counters || grew) {
        FCLSH_CUDA(cudaMemcpyAsync(r->offsets, o.d_offsets, 4 * qb, cudaMemcpyDeviceToHost, s));
        copies = true;
    }
    r->total = o.total;
    if (o.total && (!o.host_results || grew)) {
        FCLSH_CUDA(cudaMemcpyAsync(r->query, o.d_query, o.total * 4, cudaMemcpyDeviceToHost, s));
        FCLSH_CUDA(cudaMemcpyAsync(r->id, o.d_id, o.total * 4, cudaMemcpyDeviceToHost, s));
        FCLSH_CUDA(cudaMemcpyAsync(r->distance, o.d_dist, o.total * 4, cudaMemcpyDeviceToHost, s));
        copies = true;
    }
    if (copies) stream_spin_wait(s);
    r->time_hash_ms = r->time_probe_ms = r->time_verify_ms = -1; // stage timing off: not measured
    if (ix.stage_timing) {
        ix.collect_stages();
        r->time_hash_ms = ix.t_hash_ms;
        r->time_probe_ms = ix.t_probe_ms;
        r->time_verify_ms = ix.t_verify_ms;
    }
    return r;
}

} // namespace

extern "C" {

const char* fclsh_version(void) { return "fclsh_b200 0.1 (sm_100a)"; }
const char* fclsh_last_error(void) { return g_err.c_str(); }

int fclsh_device_count(int* out) {
    return guarded([&] {
        need(out, "out");
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *out = c;
    });
}

uint64_t fclsh_rng_stream(uint64_t seed, const char* label) { return Rng(seed).stream(label ? label : "").seed(); }
uint64_t fclsh_rng_stream_index(uint64_t seed, const char* label, uint64_t index) {
    return Rng(seed).stream(label ? label : "", index).seed();
}

int fclsh_family_build(uint64_t dims, uint32_t radius, int32_t kind, uint64_t rng_seed, uint64_t prime,
                       int include_zero_column, fclsh_family** out) {
    return guarded([&] {
        need(out, "out");
        if (kind < -1 || kind > 1) throw UsageError("covering family: unknown construction kind");
        auto h = std::make_unique<fclsh_family>();
        h->f = build_family(dims, radius, kind, rng_seed, prime, include_zero_column != 0);
        *out = h.release();
    });
}

int fclsh_family_make(uint64_t dims, uint32_t radius, int32_t kind, const uint32_t* mapping,
                      const uint64_t* seeds, uint64_t prime, fclsh_family** out) {
    return guarded([&] {
        need(out, "out");
        if (kind != 0 && kind != 1) throw UsageError("covering family: unknown construction kind");
        if (dims && (!mapping || !seeds)) throw UsageError("covering family: mapping/seeds must have one entry per dimension");
        auto h = std::make_unique<fclsh_family>();
        h->f = make_family(dims, radius, static_cast<Kind>(kind), std::vector<uint32_t>(mapping, mapping + dims),
                           std::vector<uint64_t>(seeds, seeds + dims), prime);
        *out = h.release();
    });
}

int fclsh_family_info_get(const fclsh_family* f, fclsh_family_info* out) {
    return guarded([&] {
        need(f, "family");
        need(out, "out");
        out->dims = f->f.dims;
        out->radius = f->f.radius;
        out->kind = static_cast<int32_t>(f->f.kind);
        out->prime = f->f.prime;
        out->tables = f->f.tables();
    });
}

int fclsh_family_export(const fclsh_family* f, uint32_t* mapping, uint64_t* seeds) {
    return guarded([&] {
        need(f, "family");
        if (mapping) std::memcpy(mapping, f->f.mapping.data(), f->f.dims * 4);
        if (seeds) std::memcpy(seeds, f->f.seeds.data(), f->f.dims * 8);
    });
}

void fclsh_family_destroy(fclsh_family* f) { delete f; }

int fclsh_hash_batch(const fclsh_family* fc, const uint64_t* d_rows, uint64_t n, uint32_t row_words, void* d_keys,
                     uint32_t key_bytes, uint64_t key_stride, int32_t layout, int device, void* stream) {
    return guarded([&] {
        need(fc, "family");
        auto* f = const_cast<fclsh_family*>(fc);
        if (row_words != (f->f.dims + 63) / 64) throw UsageError("hash: vector width does not match the family");
        if (n && (!d_rows || !d_keys)) throw UsageError("hash: NULL buffer");
        FCLSH_CUDA(cudaSetDevice(device));
        hash_rows(f->on(device), d_rows, n, d_keys, key_bytes, key_stride, layout,
                  static_cast<cudaStream_t>(stream));
    });
}

int fclsh_hash_batch_host(const fclsh_family* fc, const uint64_t* rows, uint64_t n, uint32_t row_words, void* keys,
                          uint32_t key_bytes, int device) {
    return guarded([&] {
        need(fc, "family");
        auto* f = const_cast<fclsh_family*>(fc);
        if (row_words != (f->f.dims + 63) / 64) throw UsageError("hash: vector width does not match the family");
        if (n == 0) return;
        need(rows, "rows");
        need(keys, "keys");
        FCLSH_CUDA(cudaSetDevice(device));
        DeviceFamilySet& fs = f->on(device);
        DevBuf dr, dk;
        const uint64_t L = f->f.tables();
        dr.ensure(n * row_words * 8);
        dk.ensure(n * L * key_bytes);
        FCLSH_CUDA(cudaMemcpy(dr.p, rows, n * row_words * 8, cudaMemcpyHostToDevice));
        hash_rows(fs, dr.as<uint64_t>(), n, dk.p, key_bytes, L, kLayoutPointMajor, nullptr);
        FCLSH_CUDA(cudaMemcpy(keys, dk.p, n * L * key_bytes, cudaMemcpyDeviceToHost));
    });
}

int fclsh_plan_make(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t rng_seed,
                    const fclsh_plan_override* force, uint64_t table_budget, fclsh_plan** out) {
    return guarded([&] {
        need(out, "out");
        PlanOverride ov{};
        if (force) {
            if (force->kind < 0 || force->kind > 2) throw UsageError("plan: unknown plan kind");
            ov = PlanOverride{static_cast<PlanKind>(force->kind), force->t};
        }
        auto h = std::make_unique<fclsh_plan>();
        h->p = make_plan(dims, radius, c, n, rng_seed, force ? &ov : nullptr, table_budget);
        *out = h.release();
    });
}

int fclsh_plan_info_get(const fclsh_plan* p, fclsh_plan_info* out) {
    return guarded([&] {
        need(p, "plan");
        need(out, "out");
        out->kind = static_cast<int32_t>(p->p.kind);
        out->dims = p->p.dims;
        out->radius = p->p.radius;
        out->t = p->p.t;
        out->per_part_radius = p->p.per_part_radius;
        out->part_count = p->p.part_count();
        out->table_count = p->p.table_count();
    });
}

int fclsh_plan_export(const fclsh_plan* p, uint32_t* permutation, uint64_t* parts) {
    return guarded([&] {
        need(p, "plan");
        if (permutation && !p->p.permutation.empty())
            std::memcpy(permutation, p->p.permutation.data(), p->p.permutation.size() * 4);
        if (parts)
            for (size_t i = 0; i < p->p.parts.size(); ++i) {
                parts[2 * i] = p->p.parts[i].first;
                parts[2 * i + 1] = p->p.parts[i].second;
            }
    });
}

void fclsh_plan_destroy(fclsh_plan* p) { delete p; }

void fclsh_index_options_default(fclsh_index_options* o) {
    if (!o) return;
    o->prime = FCLSH_PRIME_M61;
    o->include_zero_column = 0;
    o->table_budget = FCLSH_DEFAULT_TABLE_BUDGET;
    o->device = 0;
    o->id_offset = 0;
    o->directory_bits = 0;
    o->layout = FCLSH_TABLES_AUTO;
    o->method = FCLSH_METHOD_COVERING;
    o->delta = 0.1;
    o->k_override = 0;
    o->tables_override = 0;
}

int fclsh_index_build(const uint64_t* rows, int rows_on_device, uint64_t n, uint64_t dims, uint32_t radius,
                      const fclsh_plan* plan, uint64_t rng_seed, const fclsh_index_options* opt, fclsh_index** out) {
    return guarded([&] {
        need(out, "out");
        need(plan, "plan");
        if (n) need(rows, "rows");
        fclsh_index_options o;
        fclsh_index_options_default(&o);
        if (opt) o = *opt;
        IndexBuildOptions bo;
        bo.prime = o.prime;
        bo.include_zero_column = o.include_zero_column != 0;
        bo.table_budget = o.table_budget;
        bo.device = o.device;
        bo.id_offset = o.id_offset;
        bo.directory_bits = o.directory_bits;
        bo.layout = o.layout;
        bo.method = o.method;
        bo.delta = o.delta;
        bo.k_override = o.k_override;
        bo.tables_override = o.tables_override;
        auto h = std::make_unique<fclsh_index>();
        h->ix = build_index(rows, rows_on_device != 0, n, dims, radius, plan->p, rng_seed, bo);
        *out = h.release();
    });
}

int fclsh_index_info_get(const fclsh_index* ix, fclsh_index_info* out) {
    return guarded([&] {
        need(ix, "index");
        need(out, "out");
        const DeviceIndex& d = *ix->ix;
        out->n = d.n;
        out->dims = d.dims;
        out->radius = d.radius;
        out->table_count = d.tables;
        out->entry_count = d.tables * d.n;
        out->directory_bits = d.dir_bits;
        out->device_bytes = d.device_bytes();
        out->build_ms = d.build_ms;
        out->layout = d.layout;
        out->buckets_per_table = d.nbuckets;
        out->method = d.method;
        out->classic_k = d.fs->classic ? d.fs->cls_k : 0;
    });
}

int fclsh_index_family(const fclsh_index* ix, uint32_t part, fclsh_family** out) {
    return guarded([&] {
        need(ix, "index");
        need(out, "out");
        if (ix->ix->fs->classic) throw UsageError("index: a classic index holds a bit-sampling family");
        if (part >= ix->ix->fs->parts) throw UsageError("index: part out of range");
        auto h = std::make_unique<fclsh_family>();
        h->f = ix->ix->fs->families[part];
        *out = h.release();
    });
}

int fclsh_index_bitsample_family(const fclsh_index* ix, uint32_t* positions, uint64_t* seeds) {
    return guarded([&] {
        need(ix, "index");
        if (!ix->ix->fs->classic) throw UsageError("index: not a classic index");
        const BitSampleFamily& f = ix->ix->fs->classic_family;
        if (positions) std::memcpy(positions, f.positions.data(), f.positions.size() * 4);
        if (seeds) std::memcpy(seeds, f.seeds.data(), f.seeds.size() * 8);
    });
}

void fclsh_index_destroy(fclsh_index* ix) { delete ix; }

int fclsh_choose_k(uint64_t dims, uint32_t radius, uint64_t tables, double delta, uint32_t* out) {
    return guarded([&] {
        need(out, "out");
        *out = choose_k(dims, radius, tables, delta);
    });
}

int fclsh_bitsample_family_build(uint64_t dims, uint32_t k, uint64_t tables, uint64_t rng_seed, uint64_t prime,
                                 uint32_t* positions, uint64_t* seeds) {
    return guarded([&] {
        const BitSampleFamily f = build_bit_sample_family(dims, k, tables, rng_seed, prime);
        if (positions) std::memcpy(positions, f.positions.data(), f.positions.size() * 4);
        if (seeds) std::memcpy(seeds, f.seeds.data(), f.seeds.size() * 8);
    });
}

int fclsh_hash_tables_batch(uint64_t dims, uint32_t k, uint64_t tables, const uint32_t* positions,
                            const uint64_t* seeds, uint64_t prime, const uint64_t* rows, uint64_t n, uint64_t* keys,
                            int device) {
    return guarded([&] {
        if (dims == 0) throw UsageError("bit sample family: dims must be positive");
        if (k == 0) throw UsageError("bit sample family: k must be >= 1");
        if (tables == 0) throw UsageError("bit sample family: need at least one table");
        if (prime < 3 || prime % 2 == 0) throw UsageError("bit sample family: prime must be odd and > 2");
        need(positions, "positions");
        need(seeds, "seeds");
        BitSampleFamily f;
        f.dims = dims;
        f.k = k;
        f.tables = tables;
        f.prime = prime;
        f.positions.assign(positions, positions + tables * uint64_t(k));
        f.seeds.assign(seeds, seeds + tables * uint64_t(k));
        for (uint32_t p : f.positions)
            if (p >= dims) throw UsageError("bit sample family: position out of range");
        if (n == 0) return;
        need(rows, "rows");
        need(keys, "keys");
        FCLSH_CUDA(cudaSetDevice(device));
        auto fs = make_device_classic_set(f, device);
        const uint64_t W = (dims + 63) / 64;
        DevBuf dr, dk;
        dr.ensure(n * W * 8);
        dk.ensure(n * tables * 8);
        FCLSH_CUDA(cudaMemcpy(dr.p, rows, n * W * 8, cudaMemcpyHostToDevice));
        hash_rows(*fs, dr.as<uint64_t>(), n, dk.p, 8, tables, kLayoutPointMajor, nullptr);
        FCLSH_CUDA(cudaMemcpy(keys, dk.p, n * tables * 8, cudaMemcpyDeviceToHost));
    });
}

int fclsh_query(fclsh_index* ixh, const uint64_t* q_rows, uint64_t nq, uint32_t radius, fclsh_result** out) {
    return guarded([&] {
        need(ixh, "index");
        need(out, "out");
        if (nq) need(q_rows, "q_rows");
        std::lock_guard<std::mutex> lk(ixh->mu);
        *out = query_host(*ixh->ix, ixh->q_host_rows, q_rows, nq, radius);
    });
}

void fclsh_result_free(fclsh_result* r) {
    if (!r) return;
    pinned_pool().give(reinterpret_cast<unsigned char*>(r) - kResultHeader);
}

int fclsh_query_c_r_nn(fclsh_index* ixh, const uint64_t* q_rows, uint64_t nq, uint32_t radius,
                       int64_t posting_budget, uint64_t* counters, uint32_t* best) {
    return guarded([&] {
        need(ixh, "index");
        if (nq) {
            need(q_rows, "q_rows");
            need(counters, "counters");
            need(best, "best");
        }
        std::lock_guard<std::mutex> lk(ixh->mu);
        DeviceIndex& ix = *ixh->ix;
        FCLSH_CUDA(cudaSetDevice(ix.device));
        const uint64_t W = ix.row_words;
        uint64_t* dq = static_cast<uint64_t*>(ixh->q_host_rows.ensure(std::max<uint64_t>(1, nq) * W * 8));
        DevBuf out;
        auto* dc = static_cast<uint64_t*>(out.ensure(std::max<uint64_t>(1, nq) * 32));
        auto* db = reinterpret_cast<uint32_t*>(dc + 3 * nq);
        if (nq) FCLSH_CUDA(cudaMemcpyAsync(dq, q_rows, nq * W * 8, cudaMemcpyHostToDevice, ix.stream));
        query_c_device(ix, dq, nq, radius, posting_budget, dc, db, ix.stream);
        if (nq) {
            FCLSH_CUDA(cudaMemcpyAsync(counters, dc, nq * 24, cudaMemcpyDeviceToHost, ix.stream));
            FCLSH_CUDA(cudaMemcpyAsync(best, db, nq * 8, cudaMemcpyDeviceToHost, ix.stream));
            FCLSH_CUDA(cudaStreamSynchronize(ix.stream));
        }
    });
}

int fclsh_query_device(fclsh_index* ixh, const uint64_t* d_q_rows, uint64_t nq, uint32_t radius, void* stream,
                       fclsh_device_result* out) {
    return guarded([&] {
        need(ixh, "index");
        need(out, "out");
        if (nq) need(d_q_rows, "d_q_rows");
        std::lock_guard<std::mutex> lk(ixh->mu);
        QueryOutput o = query_device(*ixh->ix, d_q_rows, nq, radius, static_cast<cudaStream_t>(stream));
        out->nq = nq;
        out->total = o.total;
        out->d_query = o.d_query;
        out->d_id = o.d_id;
        out->d_distance = o.d_dist;
        out->d_offsets = o.d_offsets;
        out->d_collisions = o.d_coll;
        out->d_candidates = o.d_cand;
        out->d_found = o.d_found;
    });
}

int fclsh_result_copy_device(const fclsh_device_result* r, uint32_t* d_triples, uint64_t cap, uint64_t* d_offsets,
                             uint64_t* d_counters, int device, void* stream) {
    return guarded([&] {
        need(r, "result");
        if (d_triples && cap < r->total) throw UsageError("result copy: cap below the triple count");
        FCLSH_CUDA(cudaSetDevice(device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const uint64_t t = r->total, nq = r->nq;
        if (d_triples && t) {
            FCLSH_CUDA(cudaMemcpyAsync(d_triples, r->d_query, t * 4, cudaMemcpyDeviceToDevice, s));
            FCLSH_CUDA(cudaMemcpyAsync(d_triples + cap, r->d_id, t * 4, cudaMemcpyDeviceToDevice, s));
            FCLSH_CUDA(cudaMemcpyAsync(d_triples + 2 * cap, r->d_distance, t * 4, cudaMemcpyDeviceToDevice, s));
        }
        if (d_offsets) FCLSH_CUDA(cudaMemcpyAsync(d_offsets, r->d_offsets, (nq + 1) * 8, cudaMemcpyDeviceToDevice, s));
        if (d_counters && nq) {
            FCLSH_CUDA(cudaMemcpyAsync(d_counters, r->d_collisions, nq * 8, cudaMemcpyDeviceToDevice, s));
            FCLSH_CUDA(cudaMemcpyAsync(d_counters + nq, r->d_candidates, nq * 8, cudaMemcpyDeviceToDevice, s));
            FCLSH_CUDA(cudaMemcpyAsync(d_counters + 2 * nq, r->d_found, nq * 8, cudaMemcpyDeviceToDevice, s));
        }
    });
}

int fclsh_merge_shards(uint32_t world, uint64_t nq, const uint64_t* d_offsets, const uint32_t* d_triples, uint64_t cap,
                       uint32_t* d_out, uint64_t out_cap, uint64_t* d_out_offsets, int device, void* stream) {
    return guarded([&] {
        if (world == 0) throw UsageError("merge: world must be >= 1");
        need(d_offsets, "d_offsets");
        need(d_out_offsets, "d_out_offsets");
        FCLSH_CUDA(cudaSetDevice(device));
        merge_shards(world, nq, d_offsets, d_triples, cap, d_out, out_cap, d_out_offsets,
                     static_cast<cudaStream_t>(stream), device);
    });
}

int fclsh_query_stage_ms(const fclsh_index* ix, double* ms, int n) {
    if (!ix || (!ms && n > 0)) {
        g_err = "fclsh_query_stage_ms: NULL argument";
        return -FCLSH_ERR_USAGE;
    }
    const int k = std::min(n, DeviceIndex::kStages);
    std::lock_guard<std::mutex> lk(ix->mu);
    const int rc = guarded([&] { ix->ix->collect_stages(); });
    if (rc != FCLSH_OK) return -rc;
    for (int i = 0; i < k; ++i) ms[i] = ix->ix->stage_ms[i];
    return k;
}

int fclsh_query_stage_timing(fclsh_index* ix, int enable) {
    if (!ix) {
        g_err = "fclsh_query_stage_timing: NULL index";
        return FCLSH_ERR_USAGE;
    }
    std::lock_guard<std::mutex> lk(ix->mu);
    ix->ix->stage_timing = enable != 0;
    return FCLSH_OK;
}

int fclsh_query_batch_ms(const fclsh_index* ix, double* ms) {
    if (!ix || !ms) {
        g_err = "fclsh_query_batch_ms: NULL argument";
        return FCLSH_ERR_USAGE;
    }
    std::lock_guard<std::mutex> lk(ix->mu);
    return guarded([&] {
        ix->ix->collect_stages();
        *ms = ix->ix->batch_ms;
    });
}

int fclsh_query_path_counts(const fclsh_index* ix, uint64_t* dense, uint64_t* general) {
    if (!ix) {
        g_err = "fclsh_query_path_counts: NULL index";
        return -FCLSH_ERR_USAGE;
    }
    std::lock_guard<std::mutex> lk(ix->mu);
    if (dense) *dense = ix->ix->last_dense;
    if (general) *general = ix->ix->last_overflow;
    return 0;
}

int fclsh_dataset_load(const char* path, fclsh_dataset** out) {
    return guarded([&] {
        need(path, "path");
        need(out, "out");
        auto h = std::make_unique<fclsh_dataset>();
        h->ds = load_dataset(path);
        *out = h.release();
    });
}

int fclsh_dataset_info_get(const fclsh_dataset* ds, uint64_t* n, uint64_t* dims, int32_t* format,
                           const uint64_t** rows) {
    return guarded([&] {
        need(ds, "dataset");
        if (n) *n = ds->ds.n;
        if (dims) *dims = ds->ds.dims;
        if (format) *format = ds->ds.format;
        if (rows) *rows = ds->ds.rows;
    });
}

int fclsh_dataset_upload(const fclsh_dataset* ds, uint64_t* d_rows, int device, void* stream) {
    return guarded([&] {
        need(ds, "dataset");
        const uint64_t bytes = ds->ds.n * ds->ds.words() * 8;
        if (!bytes) return;
        need(d_rows, "d_rows");
        FCLSH_CUDA(cudaSetDevice(device));
        FCLSH_CUDA(cudaMemcpyAsync(d_rows, ds->ds.rows, bytes, cudaMemcpyHostToDevice,
                                   static_cast<cudaStream_t>(stream)));
    });
}

void fclsh_dataset_destroy(fclsh_dataset* ds) { delete ds; }

int fclsh_dataset_save(const char* path, const uint64_t* rows, uint64_t n, uint64_t dims, int32_t format) {
    return guarded([&] {
        need(path, "path");
        if (n) need(rows, "rows");
        save_dataset(path, rows, n, dims, format);
    });
}

int fclsh_scan_create(int device, fclsh_scan** out) {
    return guarded([&] {
        need(out, "out");
        auto h = std::make_unique<fclsh_scan>();
        h->st.device = device;
        *out = h.release();
    });
}

void fclsh_scan_destroy(fclsh_scan* sc) { delete sc; }

int fclsh_scan_truth(fclsh_scan* sc, const uint64_t* d_rows, uint64_t n, const uint64_t* d_q_rows, uint64_t nq,
                     uint64_t dims, uint32_t radius, void* stream, fclsh_device_result* out) {
    return guarded([&] {
        need(sc, "scan");
        need(out, "out");
        if (dims == 0) throw UsageError("scan: zero width");
        if (n) need(d_rows, "d_rows");
        if (nq) need(d_q_rows, "d_q_rows");
        ScanArgs a;
        a.rows = d_rows;
        a.n = n;
        a.qrows = d_q_rows;
        a.nq = nq;
        a.dims = dims;
        a.words = uint32_t((dims + 63) / 64);
        a.radius = radius;
        const ScanOutput o = scan_truth_device(sc->st, a, static_cast<cudaStream_t>(stream));
        std::memset(out, 0, sizeof(*out));
        out->nq = o.nq;
        out->total = o.total;
        out->d_query = o.d_query;
        out->d_id = o.d_id;
        out->d_distance = o.d_dist;
        out->d_offsets = o.d_offsets;
    });
}

int fclsh_distance_histogram(fclsh_scan* sc, const uint64_t* d_rows, uint64_t n, const uint64_t* d_q_rows,
                             uint64_t nq, uint64_t dims, uint64_t sample_per_query, uint64_t seed, void* stream,
                             uint64_t* counts) {
    return guarded([&] {
        need(sc, "scan");
        need(counts, "counts");
        if (dims == 0) throw UsageError("histogram: zero width");
        if (n) need(d_rows, "d_rows");
        if (nq) need(d_q_rows, "d_q_rows");
        ScanArgs a;
        a.rows = d_rows;
        a.n = n;
        a.qrows = d_q_rows;
        a.nq = nq;
        a.dims = dims;
        a.words = uint32_t((dims + 63) / 64);
        distance_histogram_device(sc->st, a, sample_per_query, seed, counts, static_cast<cudaStream_t>(stream));
    });
}

/* ------------------------------------------------------------- cluster -- */

int fclsh_cluster_unique_id(unsigned char* id) {
    return guarded([&] {
        need(id, "id");
        cluster_unique_id(id);
    });
}

int fclsh_cluster_create(const int* devices, uint32_t ndev, uint32_t shards_per_device, fclsh_cluster** out) {
    return guarded([&] {
        need(out, "out");
        if (ndev) need(devices, "devices");
        auto h = std::make_unique<fclsh_cluster>();
        h->cl = cluster_create(devices, ndev, shards_per_device);
        *out = h.release();
    });
}

int fclsh_cluster_create_rank(const unsigned char* id, uint32_t world, uint32_t rank, int device,
                              uint32_t shards_per_rank, fclsh_cluster** out) {
    return guarded([&] {
        need(out, "out");
        if (world > 1) need(id, "id");
        static const unsigned char zero[FCLSH_CLUSTER_ID_BYTES] = {};
        auto h = std::make_unique<fclsh_cluster>();
        h->cl = cluster_create_rank(id ? id : zero, world, rank, device, shards_per_rank);
        *out = h.release();
    });
}

int fclsh_cluster_build(fclsh_cluster* ch, const uint64_t* rows, int rows_on_device, int rows_scope, uint64_t n,
                        uint64_t dims, uint32_t radius, const fclsh_plan* plan, uint64_t rng_seed,
                        const fclsh_index_options* opt) {
    return guarded([&] {
        need(ch, "cluster");
        need(plan, "plan");
        if (n) need(rows, "rows");
        if (rows_scope != FCLSH_ROWS_GLOBAL && rows_scope != FCLSH_ROWS_LOCAL)
            throw UsageError("cluster: unknown rows scope");
        if (dims != plan->p.dims) throw UsageError("index: dataset width does not match the plan");
        if (n == 0) throw UsageError("index: empty dataset");
        fclsh_index_options o;
        fclsh_index_options_default(&o);
        if (opt) o = *opt;
        IndexBuildOptions bo;
        bo.prime = o.prime;
        bo.include_zero_column = o.include_zero_column != 0;
        bo.table_budget = o.table_budget;
        bo.device = o.device;
        bo.id_offset = o.id_offset;
        bo.directory_bits = o.directory_bits;
        bo.layout = o.layout;
        bo.method = o.method;
        bo.delta = o.delta;
        bo.k_override = o.k_override;
        bo.tables_override = o.tables_override;
        cluster_build(*ch->cl, rows, rows_on_device != 0, rows_scope == FCLSH_ROWS_GLOBAL, n, dims, radius, plan->p,
                      rng_seed, bo);
    });
}

int fclsh_cluster_info_get(const fclsh_cluster* ch, fclsh_cluster_info* out) {
    return guarded([&] {
        need(ch, "cluster");
        need(out, "out");
        const Cluster& c = *ch->cl;
        std::memset(out, 0, sizeof(*out));
        out->world = c.world;
        out->rank = c.members.front()->rank;
        out->local_ranks = uint32_t(c.members.size());
        out->shards_per_rank = c.shards_per_rank;
        out->total_shards = c.total_shards();
        out->device = c.members.front()->device;
        out->uses_nccl = c.use_nccl ? 1 : 0;
        out->n = c.n;
        out->dims = c.dims;
        out->radius = c.radius;
        out->build_ms = c.build_ms;
        for (auto& m : c.members)
            for (auto& sh : m->shards) {
                out->table_count = sh.ix->tables;
                out->local_entry_count += sh.ix->tables * sh.ix->n;
                out->local_device_bytes += sh.ix->device_bytes();
                out->local_points += sh.ix->n;
                if (sh.ix->layout == kLayoutBuckets) ++out->local_bucket_shards;
            }
    });
}

int fclsh_cluster_query(fclsh_cluster* ch, const uint64_t* q_rows, uint64_t nq, uint32_t radius,
                        fclsh_result** out) {
    return guarded([&] {
        need(ch, "cluster");
        need(out, "out");
        *out = nullptr;
        Cluster& c = *ch->cl;
        ClusterMember* R = c.root();
        if (nq && R) need(q_rows, "q_rows");
        if (c.world == 1 && c.shards_per_rank == 1 && c.built) {
            // one shard in all: the index's own host path (zero-copy rows,
            // results written into the host block by the batch)
            std::lock_guard<std::mutex> lk(c.mu);
            *out = query_host(*R->shards[0].ix, ch->q_host_rows, q_rows, nq, radius);
            return;
        }
        const ClusterResult res = cluster_query(c, q_rows, false, nq, radius, nullptr);
        if (!res.root) return; // this process holds no result (rank != 0)
        FCLSH_CUDA(cudaSetDevice(res.device));
        unsigned char* blk = nullptr;
        fclsh_result* r = new_result(nq, res.total, &blk);
        cudaStream_t s = res.stream;
        try {
            FCLSH_CUDA(cudaMemcpyAsync(r->offsets, res.off, (nq + 1) * 8, cudaMemcpyDeviceToHost, s));
            if (nq) {
                FCLSH_CUDA(cudaMemcpyAsync(r->collisions, res.coll, nq * 8, cudaMemcpyDeviceToHost, s));
                FCLSH_CUDA(cudaMemcpyAsync(r->candidates, res.cand, nq * 8, cudaMemcpyDeviceToHost, s));
                FCLSH_CUDA(cudaMemcpyAsync(r->found, res.found, nq * 8, cudaMemcpyDeviceToHost, s));
            }
            if (res.total) {
                FCLSH_CUDA(cudaMemcpyAsync(r->query, res.q, res.total * 4, cudaMemcpyDeviceToHost, s));
                FCLSH_CUDA(cudaMemcpyAsync(r->id, res.id, res.total * 4, cudaMemcpyDeviceToHost, s));
                FCLSH_CUDA(cudaMemcpyAsync(r->distance, res.dist, res.total * 4, cudaMemcpyDeviceToHost, s));
            }
            stream_spin_wait(s);
        } catch (...) {
            cudaStreamSynchronize(s);
            pinned_pool().give(blk);
            throw;
        }
        r->total = res.total;
        *out = r;
    });
}

int fclsh_cluster_query_device(fclsh_cluster* ch, const uint64_t* d_q_rows, uint64_t nq, uint32_t radius,
                               void* stream, fclsh_device_result* out) {
    return guarded([&] {
        need(ch, "cluster");
        need(out, "out");
        std::memset(out, 0, sizeof(*out));
        Cluster& c = *ch->cl;
        if (nq && c.root()) need(d_q_rows, "d_q_rows");
        const ClusterResult res = cluster_query(c, d_q_rows, true, nq, radius, static_cast<cudaStream_t>(stream));
        if (!res.root) return;
        out->nq = nq;
        out->total = res.total;
        out->d_query = const_cast<uint32_t*>(res.q);
        out->d_id = const_cast<uint32_t*>(res.id);
        out->d_distance = const_cast<uint32_t*>(res.dist);
        out->d_offsets = reinterpret_cast<uint64_t*>(const_cast<unsigned long long*>(res.off));
        out->d_collisions = reinterpret_cast<uint64_t*>(const_cast<unsigned long long*>(res.coll));
        out->d_candidates = reinterpret_cast<uint64_t*>(const_cast<unsigned long long*>(res.cand));
        out->d_found = reinterpret_cast<uint64_t*>(const_cast<unsigned long long*>(res.found));
    });
}

int fclsh_cluster_stage_timing(fclsh_cluster* ch, int enable) {
    return guarded([&] {
        need(ch, "cluster");
        std::lock_guard<std::mutex> lk(ch->cl->mu);
        for (auto& m : ch->cl->members)
            for (auto& sh : m->shards) sh.ix->stage_timing = enable != 0;
    });
}

namespace {
DeviceIndex& local_shard(const fclsh_cluster* ch, uint32_t k) {
    for (auto& m : ch->cl->members) {
        if (k < m->shards.size()) return *m->shards[k].ix;
        k -= uint32_t(m->shards.size());
    }
    throw UsageError("cluster: shard out of range");
}
} // namespace

int fclsh_cluster_stage_ms(const fclsh_cluster* ch, uint32_t shard, double* ms, int n) {
    if (!ch || (!ms && n > 0)) {
        g_err = "fclsh_cluster_stage_ms: NULL argument";
        return -FCLSH_ERR_USAGE;
    }
    std::lock_guard<std::mutex> lk(ch->cl->mu);
    int k = 0;
    const int rc = guarded([&] {
        DeviceIndex& ix = local_shard(ch, shard);
        ix.collect_stages();
        k = std::min(n, DeviceIndex::kStages);
        for (int i = 0; i < k; ++i) ms[i] = ix.stage_ms[i];
    });
    return rc == FCLSH_OK ? k : -rc;
}

int fclsh_cluster_path_counts(const fclsh_cluster* ch, uint32_t shard, uint64_t* dense, uint64_t* general) {
    if (!ch) {
        g_err = "fclsh_cluster_path_counts: NULL cluster";
        return -FCLSH_ERR_USAGE;
    }
    std::lock_guard<std::mutex> lk(ch->cl->mu);
    return -guarded([&] {
        DeviceIndex& ix = local_shard(ch, shard);
        if (dense) *dense = ix.last_dense;
        if (general) *general = ix.last_overflow;
    });
}

void fclsh_cluster_destroy(fclsh_cluster* c) { delete c; }

uint64_t fclsh_launch_count(void) { return launch_counter(); }
void fclsh_launch_count_reset(void) { launch_counter() = 0; }

int fclsh_gen_bernoulli(uint64_t seed, uint64_t row0, uint64_t n, uint64_t dims, uint64_t* rows, int threads) {
    return guarded([&] {
        if (dims == 0) throw UsageError("gen: dims must be positive");
        if (n) need(rows, "rows");
        gen_bernoulli(seed, row0, n, dims, rows, threads);
    });
}

int fclsh_gen_clustered(uint64_t seed, uint64_t centres, uint64_t row0, uint64_t n, uint64_t dims, double flip_p,
                        uint64_t* rows, int threads) {
    return guarded([&] {
        if (dims == 0) throw UsageError("gen: dims must be positive");
        if (centres == 0) throw UsageError("gen: need at least one centre");
        if (!(flip_p >= 0.0 && flip_p <= 1.0)) throw UsageError("gen: flip probability out of [0, 1]");
        if (n) need(rows, "rows");
        gen_clustered(seed, centres, row0, n, dims, flip_p, rows, threads);
    });
}

int fclsh_gen_planted(uint64_t seed, const uint64_t* data, uint64_t n, uint64_t dims, uint64_t nq, uint32_t kmax,
                      uint64_t* qrows, uint32_t* src_out) {
    return guarded([&] {
        if (dims == 0) throw UsageError("gen: dims must be positive");
        if (n == 0) throw UsageError("gen: data size must be positive");
        if (kmax > dims) throw UsageError("gen: planted distance exceeds dims");
        need(data, "data");
        if (nq) need(qrows, "qrows");
        gen_planted(seed, data, n, dims, nq, kmax, qrows, src_out);
    });
}

} // extern "C"
