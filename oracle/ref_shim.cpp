// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (the 12 files of
// /root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libfclsh_ref.so). It lets the Python test-suite and the
// bench's CPU-baseline / `--impl reference` arm call the reference's own
// functions on plain buffers:
//
//   ref_build_family   -> fclsh::build_covering_family   (covering.cpp:40-80)
//   ref_hash_batch     -> fclsh::hash_batch_into          (covering.cpp:169-182)
//                         fclsh::hash_reference_into      (covering.cpp:150-161)
//   ref_make_plan      -> fclsh::make_plan                (transform.cpp:32-113)
//   ref_index_build    -> fclsh::build_index              (index.cpp:49-119)
//   ref_index_query    -> fclsh::query_r_nn               (index.cpp:157-188)
//   ref_index_query_c  -> fclsh::query_c_r_nn             (index.cpp:190-235)
//   ref_scan_truth     -> fclsh::scan_truth               (workload.cpp:56-71)
//   ref_distance_histogram -> fclsh::distance_histogram   (workload.cpp:133-151)
//   ref_run_experiment -> fclsh::run_experiment + write_metrics (bench.cpp:64-170)
//   ref_dataset_save / ref_dataset_load -> fclsh::save_dataset[_text] /
//                         fclsh::load_dataset             (dataset.cpp:82-111)
//   ref_fht_mod / ref_batch_hash_kernel -> hadamard.cpp:51-72
//   ref_choose_k / ref_bitsample_family / ref_hash_tables -> classic.cpp:10-63
//   ref_index_build_classic -> fclsh::build_index(Method::classic) (index.cpp:65-76)
//
// Rows cross the boundary as row-major uint64 words, bit i of a row in word
// i/64 at offset i%64 (the BitVector layout, bitvec.hpp:13-19).
//
// The only non-reference logic here is threading: T host threads each run
// the reference function on a disjoint slice (the functions are pure /
// const-safe), and `ref_index_build` with threads > 1
// builds the IndexSet with the very same per-part families, hash calls and
// PostingTable::finalize as build_index, only with the table sorts spread
// over threads (threads == 1 calls build_index itself).

#include "fclsh/bench.hpp"
#include "fclsh/bitvec.hpp"
#include "fclsh/classic.hpp"
#include "fclsh/covering.hpp"
#include "fclsh/dataset.hpp"
#include "fclsh/errors.hpp"
#include "fclsh/hadamard.hpp"
#include "fclsh/index.hpp"
#include "fclsh/rng.hpp"
#include "fclsh/transform.hpp"
#include "fclsh/workload.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

using namespace fclsh;

namespace {

thread_local std::string g_err;

int fail_code(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const UsageError*>(&e)) return 2;
    if (dynamic_cast<const DataError*>(&e)) return 3;
    if (dynamic_cast<const ResourceError*>(&e)) return 4;
    return 1;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

BitVector row_to_bits(const uint64_t* row, size_t dims) {
    BitVector v(dims);
    size_t words = (dims + 63) / 64;
    for (size_t w = 0; w < words; ++w) {
        uint64_t bits = row[w];
        while (bits) {
            unsigned tz = static_cast<unsigned>(__builtin_ctzll(bits));
            size_t i = w * 64 + tz;
            if (i < dims) v.set(i, true);
            bits &= bits - 1;
        }
    }
    return v;
}

Dataset rows_to_dataset(const uint64_t* rows, uint64_t n, uint64_t dims, int threads) {
    Dataset ds;
    ds.dims = dims;
    ds.points.resize(n);
    size_t words = (dims + 63) / 64;
    int T = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
        pool.emplace_back([&, t] {
            for (uint64_t i = t; i < n; i += T) ds.points[i] = row_to_bits(rows + i * words, dims);
        });
    }
    for (auto& th : pool) th.join();
    return ds;
}

template <typename F>
void parallel_for(uint64_t n, int threads, F&& f) {
    int T = std::max(1, threads);
    if (T == 1 || n < 2) {
        for (uint64_t i = 0; i < n; ++i) f(i, 0);
        return;
    }
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
        pool.emplace_back([&, t] {
            for (;;) {
                uint64_t i = next.fetch_add(1);
                if (i >= n) break;
                f(i, t);
            }
        });
    }
    for (auto& th : pool) th.join();
}

ConstructionKind kind_of(int k) { return k == 1 ? ConstructionKind::specific : ConstructionKind::general; }

struct RefIndex {
    Dataset data;
    PreprocessPlan plan;
    IndexSet index;
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

uint64_t ref_rng_stream(uint64_t seed, const char* label) { return Rng(seed).stream(label).seed(); }

uint64_t ref_rng_stream_idx(uint64_t seed, const char* label, uint64_t idx) {
    return Rng(seed).stream(label, idx).seed();
}

// Draws `count` next_u64 values of Rng(seed) (checks the MT19937-64 restatement).
void ref_rng_draw(uint64_t seed, uint64_t count, uint64_t* out) {
    Rng r(seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

void ref_rng_below(uint64_t seed, uint64_t bound, uint64_t count, uint64_t* out) {
    Rng r(seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = r.below(bound);
}

// kind: -1 = derive from widths (covering.cpp:74-80), 0 = general, 1 = specific.
int ref_build_family(uint64_t dims, uint32_t radius, int kind, uint64_t seed, uint64_t prime,
                     int include_zero, uint32_t* mapping, uint64_t* seeds, int* kind_out) {
    return guarded([&] {
        Rng rng(seed);
        CoveringOptions opt;
        opt.prime = prime;
        opt.include_zero_column = include_zero != 0;
        CoveringFamily f = kind < 0 ? build_covering_family(dims, radius, rng, opt)
                                    : build_covering_family(dims, radius, kind_of(kind), rng, opt);
        std::copy(f.mapping.begin(), f.mapping.end(), mapping);
        std::copy(f.seeds.begin(), f.seeds.end(), seeds);
        *kind_out = f.kind == ConstructionKind::specific ? 1 : 0;
    });
}

// out is n x L (L = 2^(radius+1)-1), point-major. reference_path selects
// hash_reference_into (bcLSH) instead of hash_batch_into (fcLSH).
// *elapsed gets the wall time of the hashing loop alone.
int ref_hash_batch(uint64_t dims, uint32_t radius, int kind, const uint32_t* mapping,
                   const uint64_t* seeds, uint64_t prime, const uint64_t* rows, uint64_t n,
                   uint64_t* out, int threads, int reference_path, double* elapsed) {
    return guarded([&] {
        CoveringFamily f = make_covering_family(
            dims, radius, kind_of(kind), std::vector<uint32_t>(mapping, mapping + dims),
            std::vector<uint64_t>(seeds, seeds + dims), prime);
        Dataset ds = rows_to_dataset(rows, n, dims, threads);
        size_t L = f.table_count();
        int T = std::max(1, threads);
        std::vector<std::vector<uint64_t>> scratch(T);
        double t0 = now_s();
        parallel_for(n, T, [&](uint64_t i, int t) {
            std::span<uint64_t> o(out + i * L, L);
            if (reference_path)
                hash_reference_into(f, ds[i], o);
            else
                hash_batch_into(f, ds[i], o, scratch[t]);
        });
        if (elapsed) *elapsed = now_s() - t0;
    });
}

int ref_fht_mod(uint64_t* v, uint64_t n, uint64_t p) {
    return guarded([&] { fht_mod_in_place(std::span<uint64_t>(v, n), p); });
}

int ref_fht(int64_t* v, uint64_t n) {
    return guarded([&] { fht_in_place(std::span<int64_t>(v, n)); });
}

int ref_batch_hash_kernel(uint64_t* t, uint64_t n, uint64_t l1, uint64_t p) {
    return guarded([&] { batch_hash_kernel(std::span<uint64_t>(t, n), l1, p); });
}

// plan_kind: 0 identity, 1 replicate, 2 partition. perm gets dims entries
// (partition only), parts gets 2*t entries (begin, end).
int ref_make_plan(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t seed,
                  int has_override, int okind, uint32_t ot, uint64_t budget, int* kind,
                  uint32_t* t, uint32_t* per_part_radius, uint32_t* perm, uint64_t* parts) {
    return guarded([&] {
        Rng rng(seed);
        std::optional<PlanOverride> ov;
        if (has_override) ov = PlanOverride{static_cast<PlanKind>(okind), ot};
        PreprocessPlan p = make_plan(dims, radius, c, n, rng, ov, budget);
        *kind = static_cast<int>(p.kind);
        *t = p.t;
        *per_part_radius = p.per_part_radius;
        if (p.kind == PlanKind::partition) {
            std::copy(p.permutation.begin(), p.permutation.end(), perm);
            for (size_t i = 0; i < p.parts.size(); ++i) {
                parts[2 * i] = p.parts[i].first;
                parts[2 * i + 1] = p.parts[i].second;
            }
        }
    });
}

// Builds make_plan(dims, radius, c, n, Rng(plan_seed), override) and then
// build_index(data, covering_batch, radius, plan, Rng(index_seed), {prime, ...}).
void* ref_index_build(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius,
                      uint64_t plan_seed, int has_override, int okind, uint32_t ot, double c,
                      uint64_t index_seed, uint64_t prime, int include_zero, uint64_t budget,
                      int threads, double* elapsed, int* code) {
    RefIndex* h = nullptr;
    *code = guarded([&] {
        auto idx = std::make_unique<RefIndex>();
        idx->data = rows_to_dataset(rows, n, dims, threads);
        Rng plan_rng(plan_seed);
        std::optional<PlanOverride> ov;
        if (has_override) ov = PlanOverride{static_cast<PlanKind>(okind), ot};
        idx->plan = make_plan(dims, radius, c, n, plan_rng, ov, budget);
        IndexOptions opt;
        opt.prime = prime;
        opt.include_zero_column = include_zero != 0;
        opt.table_budget = budget;
        Rng rng(index_seed);
        double t0 = now_s();
        if (threads <= 1) {
            idx->index = build_index(idx->data, Method::covering_batch, radius, idx->plan, rng, opt);
        } else {
            // Same construction as build_index (index.cpp:49-119), sorts spread over threads.
            IndexSet& index = idx->index;
            if (n == 0) throw UsageError("index: empty dataset");
            if (idx->data.dims != idx->plan.dims)
                throw UsageError("index: dataset width does not match the plan");
            if (radius != idx->plan.radius) throw UsageError("index: radius does not match the plan");
            if (plan_table_count(idx->plan) > opt.table_budget)
                throw ResourceError("index: table count exceeds the budget");
            index.data = &idx->data;
            index.method = Method::covering_batch;
            index.radius = radius;
            index.plan = idx->plan;
            size_t P = idx->plan.part_count();
            index.parts.resize(P);
            CoveringOptions copt;
            copt.prime = opt.prime;
            copt.include_zero_column = opt.include_zero_column;
            for (size_t p = 0; p < P; ++p) {
                Rng fr = rng.stream("family", p);
                index.parts[p].family =
                    build_covering_family(idx->plan.part_dims(p), idx->plan.per_part_radius, fr, copt);
                index.parts[p].tables.resize(std::get<CoveringFamily>(index.parts[p].family).table_count());
            }
            // hash: keys[p][id][v]
            std::vector<std::vector<uint64_t>> keys(P);
            for (size_t p = 0; p < P; ++p)
                keys[p].resize(n * index.parts[p].tables.size());
            std::vector<std::vector<uint64_t>> scratch(threads);
            parallel_for(n, threads, [&](uint64_t id, int t) {
                std::vector<BitVector> views = apply_plan(idx->plan, idx->data[id]);
                for (size_t p = 0; p < P; ++p) {
                    const auto& f = std::get<CoveringFamily>(index.parts[p].family);
                    size_t L = f.table_count();
                    hash_batch_into(f, views[p], std::span<uint64_t>(keys[p].data() + id * L, L),
                                    scratch[t]);
                }
            });
            std::vector<std::pair<size_t, size_t>> tabs;
            for (size_t p = 0; p < P; ++p)
                for (size_t v = 0; v < index.parts[p].tables.size(); ++v) tabs.emplace_back(p, v);
            parallel_for(tabs.size(), threads, [&](uint64_t k, int) {
                auto [p, v] = tabs[k];
                auto& table = index.parts[p].tables[v];
                size_t L = index.parts[p].tables.size();
                table.reserve(n);
                for (uint64_t id = 0; id < n; ++id)
                    table.add(keys[p][id * L + v], static_cast<uint32_t>(id));
                table.finalize();
            });
        }
        if (elapsed) *elapsed = now_s() - t0;
        h = idx.release();
    });
    return h;
}

void ref_index_destroy(void* h) { delete static_cast<RefIndex*>(h); }

uint64_t ref_index_table_count(void* h) { return static_cast<RefIndex*>(h)->index.table_count(); }
uint64_t ref_index_entry_count(void* h) { return static_cast<RefIndex*>(h)->index.entry_count(); }

// Exports part p's family (mapping/seeds of length part_dims(p)).
int ref_index_family(void* h, uint32_t p, uint32_t* mapping, uint64_t* seeds, uint64_t* dims,
                     uint32_t* radius, int* kind) {
    return guarded([&] {
        auto* idx = static_cast<RefIndex*>(h);
        const auto& f = std::get<CoveringFamily>(idx->index.parts.at(p).family);
        if (mapping) std::copy(f.mapping.begin(), f.mapping.end(), mapping);
        if (seeds) std::copy(f.seeds.begin(), f.seeds.end(), seeds);
        *dims = f.dims;
        *radius = f.radius;
        *kind = f.kind == ConstructionKind::specific ? 1 : 0;
    });
}

// query_r_nn for every query row. counters: nq x 3 (collisions, candidates,
// found); offsets: nq+1; *ids_out: malloc'd concatenation of every query's
// ascending id list (free with ref_free). *elapsed: wall time of the
// query_r_nn calls alone.
int ref_index_query(void* h, const uint64_t* qrows, uint64_t nq, uint32_t radius, int threads,
                    uint64_t* counters, uint64_t* offsets, uint32_t** ids_out, double* elapsed) {
    return guarded([&] {
        auto* idx = static_cast<RefIndex*>(h);
        Dataset qs = rows_to_dataset(qrows, nq, idx->data.dims, threads);
        int T = std::max(1, threads);
        std::vector<QueryScratch> scratch(T);
        std::vector<std::vector<uint32_t>> res(nq);
        double t0 = now_s();
        parallel_for(nq, T, [&](uint64_t q, int t) {
            RnnResult r = query_r_nn(idx->index, qs[q], radius, scratch[t]);
            counters[3 * q + 0] = r.report.collisions;
            counters[3 * q + 1] = r.report.candidates;
            counters[3 * q + 2] = r.report.found;
            res[q] = std::move(r.ids);
        });
        if (elapsed) *elapsed = now_s() - t0;
        uint64_t total = 0;
        for (uint64_t q = 0; q < nq; ++q) {
            offsets[q] = total;
            total += res[q].size();
        }
        offsets[nq] = total;
        uint32_t* ids = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(1, total) * 4));
        for (uint64_t q = 0; q < nq; ++q)
            std::copy(res[q].begin(), res[q].end(), ids + offsets[q]);
        *ids_out = ids;
    });
}

// query_c_r_nn (index.cpp:190-235) for nq rows: counters[3*q] =
// {collisions, candidates, found}, best[2*q] = {id, distance} or
// {UINT32_MAX, UINT32_MAX} when nothing was retrieved. budget < 0: default 3L.
int ref_index_query_c(void* h, const uint64_t* qrows, uint64_t nq, uint32_t radius, int64_t budget, int threads,
                      uint64_t* counters, uint32_t* best) {
    return guarded([&] {
        auto* idx = static_cast<RefIndex*>(h);
        Dataset qs = rows_to_dataset(qrows, nq, idx->data.dims, threads);
        int T = std::max(1, threads);
        std::vector<QueryScratch> scratch(T);
        std::optional<uint64_t> b;
        if (budget >= 0) b = uint64_t(budget);
        parallel_for(nq, T, [&](uint64_t q, int t) {
            CrnnResult r = query_c_r_nn(idx->index, qs[q], radius, scratch[t], b);
            counters[3 * q + 0] = r.report.collisions;
            counters[3 * q + 1] = r.report.candidates;
            counters[3 * q + 2] = r.report.found;
            best[2 * q] = r.id ? *r.id : UINT32_MAX;
            best[2 * q + 1] = r.id ? r.distance : UINT32_MAX;
        });
    });
}

// scan_truth over query slices on T threads; *triples_out: malloc'd
// (query, point, distance) u32 triples sorted by (query, point).
int ref_scan_truth(const uint64_t* rows, uint64_t n, const uint64_t* qrows, uint64_t nq,
                   uint64_t dims, uint32_t radius, int threads, uint32_t** triples_out,
                   uint64_t* count) {
    return guarded([&] {
        Dataset data = rows_to_dataset(rows, n, dims, threads);
        int T = std::max(1, threads);
        uint64_t chunk = std::max<uint64_t>(1, (nq + 4 * T - 1) / (4 * T));
        uint64_t nchunks = (nq + chunk - 1) / chunk;
        std::vector<std::vector<TruthEntry>> parts(nchunks);
        parallel_for(nchunks, T, [&](uint64_t c, int) {
            Dataset qs;
            qs.dims = dims;
            uint64_t b = c * chunk, e = std::min(nq, b + chunk);
            for (uint64_t q = b; q < e; ++q)
                qs.points.push_back(row_to_bits(qrows + q * ((dims + 63) / 64), dims));
            GroundTruth g = scan_truth(data, qs, radius);
            for (auto& te : g.entries) te.query += static_cast<uint32_t>(b);
            parts[c] = std::move(g.entries);
        });
        uint64_t total = 0;
        for (auto& p : parts) total += p.size();
        uint32_t* out = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(1, total) * 12));
        uint64_t k = 0;
        for (auto& p : parts)
            for (auto& te : p) {
                out[3 * k] = te.query;
                out[3 * k + 1] = te.point;
                out[3 * k + 2] = te.distance;
                ++k;
            }
        *triples_out = out;
        *count = total;
    });
}

// distance_histogram(data, queries, sample_per_query, seed): counts[dims + 1].
int ref_distance_histogram(const uint64_t* rows, uint64_t n, const uint64_t* qrows, uint64_t nq, uint64_t dims,
                           uint64_t sample_per_query, uint64_t seed, uint64_t* counts) {
    return guarded([&] {
        Dataset data = rows_to_dataset(rows, n, dims, 8);
        Dataset qs = rows_to_dataset(qrows, nq, dims, 8);
        std::vector<uint64_t> c = distance_histogram(data, qs, sample_per_query, seed);
        std::copy(c.begin(), c.end(), counts);
    });
}

// save_dataset (text == 0, FCL1) or save_dataset_text (text != 0).
int ref_dataset_save(const char* path, const uint64_t* rows, uint64_t n, uint64_t dims, int text) {
    return guarded([&] {
        Dataset ds = rows_to_dataset(rows, n, dims, 1);
        if (text)
            save_dataset_text(ds, path);
        else
            save_dataset(ds, path);
    });
}

// load_dataset; *rows_out: malloc'd [n][ceil(dims/64)] words.
int ref_dataset_load(const char* path, uint64_t* n, uint64_t* dims, uint64_t** rows_out) {
    return guarded([&] {
        Dataset ds = load_dataset(path);
        const size_t W = (ds.dims + 63) / 64;
        uint64_t* out = static_cast<uint64_t*>(std::calloc(std::max<size_t>(1, ds.size() * W), 8));
        for (size_t i = 0; i < ds.size(); ++i)
            std::copy(ds[i].words().begin(), ds[i].words().end(), out + i * W);
        *n = ds.size();
        *dims = ds.dims;
        *rows_out = out;
    });
}

// run_experiment(data, queries, truth, cfg): one row of 12 doubles per query
// {query_id, radius, collisions, candidates, found, true_near, precision,
// recall, s1_us, s2_us, s3_us, 0}; csv_out is unused.
int ref_run_experiment(const uint64_t* rows, uint64_t n, const uint64_t* qrows, uint64_t nq, uint64_t dims,
                       const uint32_t* truth, uint64_t ntruth, uint32_t truth_radius, const char* method,
                       uint32_t radius, double c, int override_kind, uint32_t override_t, uint64_t seed,
                       uint32_t repeats, int fresh_seeds, uint64_t prime, double* out, char** csv_out) {
    return guarded([&] {
        Dataset data = rows_to_dataset(rows, n, dims, 8);
        Dataset qs = rows_to_dataset(qrows, nq, dims, 8);
        GroundTruth g;
        g.radius = truth_radius;
        for (uint64_t k = 0; k < ntruth; ++k)
            g.entries.push_back(TruthEntry{truth[3 * k], truth[3 * k + 1], truth[3 * k + 2]});
        ExperimentConfig cfg;
        cfg.method = method;
        cfg.radius = radius;
        cfg.c = c;
        if (override_kind >= 0) cfg.plan_override = PlanOverride{static_cast<PlanKind>(override_kind), override_t};
        cfg.seed = seed;
        cfg.repeats = repeats;
        cfg.fresh_seeds = fresh_seeds != 0;
        cfg.prime = prime;
        std::vector<MetricsRow> res = run_experiment(data, qs, g, cfg);
        for (size_t i = 0; i < res.size(); ++i) {
            const MetricsRow& r = res[i];
            double* o = out + 12 * i;
            o[0] = r.query_id;
            o[1] = r.radius;
            o[2] = r.collisions;
            o[3] = r.candidates;
            o[4] = r.found;
            o[5] = r.true_near;
            o[6] = r.precision;
            o[7] = r.recall;
            o[8] = r.time_s1_us;
            o[9] = r.time_s2_us;
            o[10] = r.time_s3_us;
            o[11] = 0;
        }
        // (write_metrics needs iostreams, which crash when this statically
        // linked libstdc++ shares a process with another one: the CSV comes
        // from oracle/_ref/ref_write_metrics instead)
        (void)csv_out;
    });
}

// ---------------------------------------------------------- classic.cpp
int ref_choose_k(uint64_t dims, uint32_t radius, uint64_t tables, double delta, uint32_t* out) {
    return guarded([&] { *out = choose_k(dims, radius, tables, delta); });
}

// build_bit_sample_family(dims, k, tables, Rng(seed), prime): positions / seeds [tables * k]
int ref_bitsample_family(uint64_t dims, uint32_t k, uint64_t tables, uint64_t seed, uint64_t prime,
                         uint32_t* positions, uint64_t* seeds) {
    return guarded([&] {
        Rng rng(seed);
        BitSampleFamily f = build_bit_sample_family(dims, k, tables, rng, prime);
        std::copy(f.positions.begin(), f.positions.end(), positions);
        std::copy(f.seeds.begin(), f.seeds.end(), seeds);
    });
}

// hash_tables_into for every row: out [n][tables]
int ref_hash_tables(uint64_t dims, uint32_t k, uint64_t tables, const uint32_t* positions, const uint64_t* seeds,
                    uint64_t prime, const uint64_t* rows, uint64_t n, uint64_t* out, int threads) {
    return guarded([&] {
        BitSampleFamily f;
        f.dims = dims;
        f.k = k;
        f.tables = tables;
        f.prime = prime;
        f.positions.assign(positions, positions + tables * k);
        f.seeds.assign(seeds, seeds + tables * k);
        Dataset ds = rows_to_dataset(rows, n, dims, threads);
        parallel_for(n, threads, [&](uint64_t i, int) {
            hash_tables_into(f, ds[i], std::span<uint64_t>(out + i * tables, tables));
        });
    });
}

// make_plan(dims, radius, c, n, Rng(plan_seed), identity) + build_index(data,
// Method::classic, radius, plan, Rng(index_seed), {prime, budget, delta,
// k_override, tables_override}) -- single-threaded, the reference's own.
void* ref_index_build_classic(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius, uint64_t plan_seed,
                              double c, uint64_t index_seed, uint64_t prime, uint64_t budget, double delta,
                              uint32_t k_override, uint64_t tables_override, int* code) {
    RefIndex* h = nullptr;
    *code = guarded([&] {
        auto idx = std::make_unique<RefIndex>();
        idx->data = rows_to_dataset(rows, n, dims, 8);
        Rng plan_rng(plan_seed);
        idx->plan = make_plan(dims, radius, c, n, plan_rng, PlanOverride{PlanKind::identity, 1}, budget);
        IndexOptions opt;
        opt.prime = prime;
        opt.table_budget = budget;
        opt.delta = delta;
        if (k_override) opt.k_override = k_override;
        if (tables_override) opt.tables_override = tables_override;
        Rng rng(index_seed);
        idx->index = build_index(idx->data, Method::classic, radius, idx->plan, rng, opt);
        h = idx.release();
    });
    return h;
}

} // extern "C"
