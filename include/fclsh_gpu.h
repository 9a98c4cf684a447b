/*
 * fclsh_gpu.h -- C-ABI of the B200-native fcLSH engine (libfclsh_b200.so).
 *
 * Drop-in boundary for the reference library's hot path (arXiv 1602.02620
 * reference, /root/reference/proj). The reference has no FFI of its own: its
 * interface is the C++ API listed next to each entry point below. This ABI
 * restates that API over plain pointers, sizes and opaque handles, batched
 * (one call hashes / queries many rows) because per-row calls would be
 * launch-bound on a GPU. No torch or CUDA types appear in the signatures;
 * streams travel as `void*` (a cudaStream_t, NULL = the library's own).
 *
 * Conventions
 *  - Rows are row-major uint64 words, bit i of a row in word i/64 at offset
 *    i%64, padding bits zero: exactly BitVector's layout (bitvec.hpp:13-19).
 *    For d % 64 == 0 an FCL1 file row is byte-identical (dataset.hpp:20-23).
 *  - An `Rng&` argument of the reference is passed as the Rng's 64-bit seed:
 *    every consumer on this path derives its draws through Rng::stream(),
 *    which depends on the seed alone (rng.cpp:31-37).
 *  - Return codes mirror the reference's exception classes and CLI exit
 *    codes (errors.hpp:8-29, tools/fclsh.cpp:302-318):
 *      0 ok, 2 UsageError, 3 DataError, 4 ResourceError,
 *      5 CUDA runtime failure (no reference counterpart; the reference never
 *        touches a device), 1 any other failure.
 *    fclsh_last_error() returns the message of the last failure on the
 *    calling thread, with the reference's wording where one exists.
 *  - Device (`d_`) pointers must be device memory on the handle's device.
 *  - Handles are bound to one device; calls on one handle serialize (the
 *    library locks each handle: concurrent callers take turns). Distinct
 *    handles may be driven from distinct host threads. Device result
 *    pointers returned by a handle stay valid until its next query.
 */
#ifndef FCLSH_GPU_H
#define FCLSH_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCLSH_OK 0
#define FCLSH_ERR_OTHER 1
#define FCLSH_ERR_USAGE 2
#define FCLSH_ERR_DATA 3
#define FCLSH_ERR_RESOURCE 4
#define FCLSH_ERR_CUDA 5

/* ConstructionKind (covering.hpp:21) and PlanKind (transform.hpp:24). */
#define FCLSH_KIND_AUTO (-1)
#define FCLSH_KIND_GENERAL 0
#define FCLSH_KIND_SPECIFIC 1
#define FCLSH_PLAN_IDENTITY 0
#define FCLSH_PLAN_REPLICATE 1
#define FCLSH_PLAN_PARTITION 2

/* Key layouts of fclsh_hash_batch. */
#define FCLSH_LAYOUT_TABLE_MAJOR 0 /* key[(part*L + v-1)*key_stride + row] */
#define FCLSH_LAYOUT_POINT_MAJOR 1 /* key[row*key_stride + part*L + v-1]  */

/* kMersenne61 (modmath.hpp:10) and the 32-bit-key field 2^31-1. */
#define FCLSH_PRIME_M61 ((uint64_t)0x1FFFFFFFFFFFFFFFull)
#define FCLSH_PRIME_M31 ((uint64_t)0x7FFFFFFFull)
/* kDefaultTableBudget (transform.hpp:52) */
#define FCLSH_DEFAULT_TABLE_BUDGET ((uint64_t)1 << 21)

const char* fclsh_version(void);
const char* fclsh_last_error(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
int fclsh_device_count(int* out);

/* ------------------------------------------------------------------ Rng ---
 * Rng(seed).stream(label) / .stream(label, index) seeds (rng.cpp:31-37). */
uint64_t fclsh_rng_stream(uint64_t seed, const char* label);
uint64_t fclsh_rng_stream_index(uint64_t seed, const char* label, uint64_t index);

/* ---------------------------------------------------------------- family ---
 * An r-covering family over one view (covering.hpp:34-43). */
typedef struct fclsh_family fclsh_family;

typedef struct {
    uint64_t dims;
    uint32_t radius;
    int32_t kind;    /* FCLSH_KIND_* (never AUTO once built) */
    uint64_t prime;
    uint64_t tables; /* 2^(radius+1) - 1 */
} fclsh_family_info;

/* build_covering_family(dims, radius[, kind], Rng(rng_seed), {prime, include_zero_column})
 * (covering.hpp:55-60, covering.cpp:40-80). kind = FCLSH_KIND_AUTO derives it
 * from the widths (covering.cpp:74-80). */
int fclsh_family_build(uint64_t dims, uint32_t radius, int32_t kind, uint64_t rng_seed,
                       uint64_t prime, int include_zero_column, fclsh_family** out);
/* make_covering_family(dims, radius, kind, mapping, seeds, prime)
 * (covering.hpp:62-66, covering.cpp:84-111): explicit, validated. */
int fclsh_family_make(uint64_t dims, uint32_t radius, int32_t kind, const uint32_t* mapping,
                      const uint64_t* seeds, uint64_t prime, fclsh_family** out);
int fclsh_family_info_get(const fclsh_family* f, fclsh_family_info* out);
/* Copies mapping[dims] / seeds[dims] out (either may be NULL). */
int fclsh_family_export(const fclsh_family* f, uint32_t* mapping, uint64_t* seeds);
void fclsh_family_destroy(fclsh_family* f);

/* hash_batch_into for n rows at once (covering.hpp:83-84, covering.cpp:169-182):
 * keys of row i, table v (1..L) = h[v]; canonical residues mod prime.
 * key_bytes: 4 (prime < 2^32) or 8. key_stride in keys (>= n for TABLE_MAJOR,
 * >= L for POINT_MAJOR). Device buffers; asynchronous on `stream`. */
int fclsh_hash_batch(const fclsh_family* f, const uint64_t* d_rows, uint64_t n,
                     uint32_t row_words, void* d_keys, uint32_t key_bytes, uint64_t key_stride,
                     int32_t layout, int device, void* stream);
/* Same from host buffers (copies in, hashes, copies out; synchronous).
 * keys is point-major [n][L]. */
int fclsh_hash_batch_host(const fclsh_family* f, const uint64_t* rows, uint64_t n,
                          uint32_t row_words, void* keys, uint32_t key_bytes, int device);

/* ------------------------------------------------------ classic family ---
 * Bit-sampling LSH, the paper's classic baseline (classic.hpp:15-50). */
/* choose_k(dims, radius, tables, delta) (classic.cpp:10-23). */
int fclsh_choose_k(uint64_t dims, uint32_t radius, uint64_t tables, double delta, uint32_t* out);
/* build_bit_sample_family(dims, k, tables, Rng(rng_seed), prime)
 * (classic.cpp:25-46): positions / seeds [tables * k]. */
int fclsh_bitsample_family_build(uint64_t dims, uint32_t k, uint64_t tables, uint64_t rng_seed, uint64_t prime,
                                 uint32_t* positions, uint64_t* seeds);
/* hash_tables_into (classic.cpp:48-63) for n host rows on the device:
 * keys [n][tables] (u64), synchronous. */
int fclsh_hash_tables_batch(uint64_t dims, uint32_t k, uint64_t tables, const uint32_t* positions,
                            const uint64_t* seeds, uint64_t prime, const uint64_t* rows, uint64_t n, uint64_t* keys,
                            int device);

/* ------------------------------------------------------------------ plan ---
 * PreprocessPlan (transform.hpp:26-44) */
typedef struct fclsh_plan fclsh_plan;

typedef struct {
    int32_t kind; /* FCLSH_PLAN_* */
    uint32_t t;
} fclsh_plan_override;

typedef struct {
    int32_t kind;
    uint64_t dims;
    uint32_t radius;
    uint32_t t;
    uint32_t per_part_radius;
    uint32_t part_count;
    uint64_t table_count; /* plan_table_count (transform.cpp:155-158) */
} fclsh_plan_info;

/* make_plan(dims, radius, c, n, Rng(rng_seed), force, table_budget)
 * (transform.hpp:57-59, transform.cpp:32-113). force may be NULL. */
int fclsh_plan_make(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t rng_seed,
                    const fclsh_plan_override* force, uint64_t table_budget, fclsh_plan** out);
int fclsh_plan_info_get(const fclsh_plan* p, fclsh_plan_info* out);
/* permutation[dims] and parts[2*t] (begin, end) of a partition plan. */
int fclsh_plan_export(const fclsh_plan* p, uint32_t* permutation, uint64_t* parts);
void fclsh_plan_destroy(fclsh_plan* p);

/* ----------------------------------------------------------------- index ---
 * IndexSet (index.hpp:42-52), built on one device. Owns a device copy of
 * the rows (needed by the verify pass) and every table. */
typedef struct fclsh_index fclsh_index;

typedef struct {
    uint64_t prime;              /* IndexOptions::prime (index.hpp:25) */
    int32_t include_zero_column; /* IndexOptions::include_zero_column */
    uint64_t table_budget;       /* IndexOptions::table_budget */
    int32_t device;              /* CUDA device ordinal */
    uint64_t id_offset;          /* added to every reported id (shards) */
    int32_t directory_bits;      /* CSR layout: 0 = automatic */
    int32_t layout;              /* FCLSH_TABLES_* */
    int32_t method;              /* FCLSH_METHOD_* (Method, index.hpp:22) */
    double delta;                /* IndexOptions::delta (classic; default 0.1) */
    uint32_t k_override;         /* IndexOptions::k_override (classic; 0 = unset) */
    uint64_t tables_override;    /* IndexOptions::tables_override (classic; 0 = unset) */
} fclsh_index_options;

/* Method (index.hpp:22). COVERING = covering_batch; covering_reference
 * (bcLSH) builds identical buckets (index.hpp:17-22), so it is COVERING too.
 * CLASSIC = bit-sampling LSH (classic.hpp) over the identity plan. */
#define FCLSH_METHOD_COVERING 0
#define FCLSH_METHOD_CLASSIC 2

/* Device table layouts (same query results):
 * BUCKETS  open-addressed buckets of four postings, one random 32-byte read
 *          per probe, ~16 bytes per posting (default when it fits);
 * CSR      the reference's sorted posting array + a key-cell directory, two
 *          random reads per probe, ~10 bytes per posting. */
#define FCLSH_TABLES_AUTO 0
#define FCLSH_TABLES_CSR 1
#define FCLSH_TABLES_BUCKETS 2

void fclsh_index_options_default(fclsh_index_options* o);

/* build_index(data, Method::covering_batch, radius, plan, Rng(rng_seed), opt)
 * (index.hpp:70-71, index.cpp:49-119). rows: n x row_words words, host
 * memory (rows_on_device = 0) or device memory on opt->device (1). */
int fclsh_index_build(const uint64_t* rows, int rows_on_device, uint64_t n, uint64_t dims,
                      uint32_t radius, const fclsh_plan* plan, uint64_t rng_seed,
                      const fclsh_index_options* opt, fclsh_index** out);
typedef struct {
    uint64_t n;
    uint64_t dims;
    uint32_t radius;
    uint64_t table_count; /* IndexSet::table_count (index.cpp:20-24) */
    uint64_t entry_count; /* IndexSet::entry_count (index.cpp:26-31) */
    uint32_t directory_bits;
    uint64_t device_bytes;
    double build_ms; /* device time of the last build, CUDA events */
    int32_t layout;  /* FCLSH_TABLES_CSR or FCLSH_TABLES_BUCKETS */
    uint64_t buckets_per_table;
    int32_t method;     /* FCLSH_METHOD_* */
    uint32_t classic_k; /* bits sampled per table (classic) */
} fclsh_index_info;
int fclsh_index_info_get(const fclsh_index* ix, fclsh_index_info* out);
/* Part p's family (a new handle the caller destroys; covering indexes). */
int fclsh_index_family(const fclsh_index* ix, uint32_t part, fclsh_family** out);
/* A classic index's bit-sampling family: positions / seeds [tables * k]
 * (either may be NULL). */
int fclsh_index_bitsample_family(const fclsh_index* ix, uint32_t* positions, uint64_t* seeds);
void fclsh_index_destroy(fclsh_index* ix);

/* ----------------------------------------------------------------- query ---
 * query_r_nn (index.hpp:78-79, index.cpp:157-188) for nq rows at once.
 * Result triples (query, id, distance) are sorted by (query, id); per-query
 * QueryReport counters (report.hpp:14-21) equal the reference's exactly. */
typedef struct {
    uint64_t nq;
    uint64_t total;      /* number of triples */
    uint32_t* query;     /* [total] */
    uint32_t* id;        /* [total], id_offset applied */
    uint32_t* distance;  /* [total] */
    uint64_t* offsets;   /* [nq+1]: query q owns triples [offsets[q], offsets[q+1]) */
    uint64_t* collisions;/* [nq] */
    uint64_t* candidates;/* [nq] */
    uint64_t* found;     /* [nq] */
    double time_hash_ms, time_probe_ms, time_verify_ms; /* S1 / S2 / S3, CUDA events; -1 unless
                                                            fclsh_query_stage_timing is on */
} fclsh_result;

/* Host rows in, host result out (the library allocates; free with
 * fclsh_result_free). Synchronous. q_rows may be pinned (page-locked) host
 * memory for a full-speed upload. The result is one mapped pinned block (its
 * arrays are slices of it) taken from a pool that fclsh_result_free refills;
 * the batch's kernels write the counters and results into it directly, as
 * they complete (D2H copies only when the total outgrows the block). */
int fclsh_query(fclsh_index* ix, const uint64_t* q_rows, uint64_t nq, uint32_t radius,
                fclsh_result** out);
void fclsh_result_free(fclsh_result* r);

/* Device-resident variant: q rows already on the device, results stay in
 * index-owned device buffers that live until the next query on `ix`.
 * Pointers returned are device pointers. The work runs on the index's own
 * stream, ordered after the work already queued on `stream` and before
 * anything queued on `stream` afterwards (event fork/join; NULL = no join).
 * The call returns once `total` is known (the device publishes it to mapped
 * host memory); the output arrays complete in `stream` order. A batch shape
 * seen twice in a row is replayed as one CUDA graph. */
typedef struct {
    uint64_t nq;
    uint64_t total;
    uint32_t* d_query;
    uint32_t* d_id;
    uint32_t* d_distance;
    uint64_t* d_offsets;    /* [nq+1] */
    uint64_t* d_collisions; /* [nq] */
    uint64_t* d_candidates; /* [nq] */
    uint64_t* d_found;      /* [nq] */
} fclsh_device_result;
int fclsh_query_device(fclsh_index* ix, const uint64_t* d_q_rows, uint64_t nq, uint32_t radius,
                       void* stream, fclsh_device_result* out);

/* query_c_r_nn (index.hpp:90-93, index.cpp:190-235) for nq host rows:
 * walk the buckets in table order and stop after posting_budget postings
 * (< 0: the reference's default 3L), return the closest point retrieved
 * (ties: the lowest id). counters[nq][3] = {collisions, candidates, found},
 * best[nq][2] = {id (+ id_offset), distance}, both UINT32_MAX when nothing
 * was retrieved. Any budget (budgets above 12288 distinct ids, or a cut
 * bucket above 4096 postings, run from a global-memory id set). Synchronous. */
int fclsh_query_c_r_nn(fclsh_index* ix, const uint64_t* q_rows, uint64_t nq, uint32_t radius,
                       int64_t posting_budget, uint64_t* counters, uint32_t* best);

/* Copies a device result into caller device buffers (all on `device`):
 * d_triples [3][cap] (rows: query, id, distance; cap >= r->total),
 * d_offsets [nq+1], d_counters [3][nq] (rows: collisions, candidates, found).
 * Any output pointer may be NULL. Asynchronous on `stream`. */
int fclsh_result_copy_device(const fclsh_device_result* r, uint32_t* d_triples, uint64_t cap,
                             uint64_t* d_offsets, uint64_t* d_counters, int device, void* stream);

/* Multi-GPU result assembly (points sharded by contiguous id ranges in rank
 * order): given every rank's offsets [world][nq+1] and triples
 * [world][3][cap], writes the merged triples, ordered by (query, id), to
 * d_out [3][out_cap] and their per-query offsets to d_out_offsets [nq+1].
 * out_cap >= total over ranks. Asynchronous on `stream`. */
int fclsh_merge_shards(uint32_t world, uint64_t nq, const uint64_t* d_offsets, const uint32_t* d_triples,
                       uint64_t cap, uint32_t* d_out, uint64_t out_cap, uint64_t* d_out_offsets, int device,
                       void* stream);

/* Device time (CUDA events, ms) of each stage of the last query on ix:
 * [0] hash (S1) [1] fused probe + dedup + verify (S2+S3, warp per query)
 * [2] the same fused, CTA per query, for the dense queries [1] handed over
 * [3] found scan [4] compaction [5] general path for queries that
 * overflowed both (with its rescan/recompaction; includes the host round
 * trip that discovers them). Writes min(n, 6) values; returns the number
 * written (negative on error). */
int fclsh_query_stage_ms(const fclsh_index* ix, double* ms, int n);

/* Per-stage timing (the events of fclsh_query_stage_ms, the batch total of
 * fclsh_query_batch_ms and the time_*_ms fields of fclsh_result) is off by
 * default: each event costs ~4 us of device time in a replayed batch. Off,
 * those values are -1. */
int fclsh_query_stage_timing(fclsh_index* ix, int enable);
/* Device time (ms) of the last query batch on ix, hash to compaction (-1
 * unless stage timing was on for it). */
int fclsh_query_batch_ms(const fclsh_index* ix, double* ms);

/* How the last query on ix was served: *dense = queries handed from the
 * warp-per-query kernel to the CTA-per-query kernel, *general = queries
 * that went on to the general (sort-based) path. Either pointer may be
 * NULL. Returns 0 or a negative error code. */
int fclsh_query_path_counts(const fclsh_index* ix, uint64_t* dense, uint64_t* general);

/* --------------------------------------------------------------- dataset ---
 * The reference's containers (dataset.hpp:20-31; load_dataset /
 * save_dataset / save_dataset_text, dataset.cpp:82-111), read into the row
 * layout above. FCL1 rows are byte-identical to it for d % 64 == 0, so the
 * file body is read with one fread into pinned host memory; upload copies it
 * to the device at full speed. Errors and messages follow the reference
 * (truncation, dirty padding bits, trailing bytes, text width / characters:
 * DataError; unopenable path: UsageError). */
#define FCLSH_DATASET_FCL1 1
#define FCLSH_DATASET_TEXT 2
typedef struct fclsh_dataset fclsh_dataset;
/* load_dataset: sniffs the "FCL1" magic, else parses text. */
int fclsh_dataset_load(const char* path, fclsh_dataset** out);
/* n, dims, format and the host rows [n][ceil(dims/64)] (valid until destroy);
 * any output may be NULL. */
int fclsh_dataset_info_get(const fclsh_dataset* ds, uint64_t* n, uint64_t* dims, int32_t* format,
                           const uint64_t** rows);
/* Copies the rows to d_rows (n * ceil(dims/64) words on `device`), async on stream. */
int fclsh_dataset_upload(const fclsh_dataset* ds, uint64_t* d_rows, int device, void* stream);
void fclsh_dataset_destroy(fclsh_dataset* ds);
/* save_dataset (FCLSH_DATASET_FCL1) / save_dataset_text (FCLSH_DATASET_TEXT)
 * of host rows [n][ceil(dims/64)] (padding bits are written as zero). */
int fclsh_dataset_save(const char* path, const uint64_t* rows, uint64_t n, uint64_t dims, int32_t format);

/* ----------------------------------------------------------- linear scan ---
 * scan_truth (workload.cpp:56-71) and distance_histogram
 * (workload.cpp:133-151) on device rows: an exhaustive second oracle at full
 * config scale and the reference's `linear` method. A scan handle owns its
 * device workspace; results live until its next call. */
typedef struct fclsh_scan fclsh_scan;
int fclsh_scan_create(int device, fclsh_scan** out);
void fclsh_scan_destroy(fclsh_scan* sc);
/* Every (query, point, distance) with distance <= radius, ordered by
 * (query, point); out's counter pointers are NULL. Synchronous (the total
 * sizes the output). */
int fclsh_scan_truth(fclsh_scan* sc, const uint64_t* d_rows, uint64_t n, const uint64_t* d_q_rows, uint64_t nq,
                     uint64_t dims, uint32_t radius, void* stream, fclsh_device_result* out);
/* counts[dims + 1] (host): every pair if sample_per_query is 0 or >= n, else
 * sample_per_query points per query drawn as the reference draws them
 * (Rng(seed).stream("histogram").below(n), query-major). Synchronous. */
int fclsh_distance_histogram(fclsh_scan* sc, const uint64_t* d_rows, uint64_t n, const uint64_t* d_q_rows,
                             uint64_t nq, uint64_t dims, uint64_t sample_per_query, uint64_t seed, void* stream,
                             uint64_t* counts);

/* --------------------------------------------------------------- cluster ---
 * A point-sharded index over the GPUs of one box (the
 * reference is single-process and single-threaded, so this has
 * no reference counterpart beyond query_r_nn's results). The n points are cut
 * into world x shards_per_rank contiguous, balanced id ranges (shard g owns
 * [g*n/S, (g+1)*n/S)); each shard is an index (fclsh_index_build semantics,
 * the same plan, seed and families, ids offset by the shard start), rank r
 * holds shards [r*spr, (r+1)*spr) on its GPU. A query batch is broadcast
 * from rank 0 (ncclBroadcast), answered by every shard concurrently, merged
 * per GPU, sent to rank 0 (ncclAllGather of the totals, grouped
 * ncclSend/ncclRecv) and merged there: triples in (query, id) order and
 * counters summed, i.e. exactly fclsh_query's result on one index over all
 * points (every posting and id lives in one shard). NCCL (libnccl.so.2) is
 * loaded at run time, only when world > 1 (FCLSH_CLUSTER_NCCL=1: also at 1).
 *
 * Two ways to form one:
 *  - fclsh_cluster_create: this process drives ndev GPUs (ncclCommInitAll);
 *    shards_per_device >= 1, so S shards fit on fewer GPUs (S = 8 on one GPU
 *    runs the 8-GPU layout on a single device);
 *  - fclsh_cluster_create_rank: one process per GPU (torchrun): rank 0 calls
 *    fclsh_cluster_unique_id, sends the id to the others out of band, and
 *    every rank calls this with it (ncclCommInitRank).
 * Build and query are collective: every process calls them, in the same
 * order. Calls on one handle serialize. At most 64 shards in all. */
typedef struct fclsh_cluster fclsh_cluster;
#define FCLSH_CLUSTER_ID_BYTES 128
#define FCLSH_ROWS_GLOBAL 0 /* rows = all n points */
#define FCLSH_ROWS_LOCAL 1  /* rows = only the contiguous range of this process's shards */

int fclsh_cluster_unique_id(unsigned char* id /* [FCLSH_CLUSTER_ID_BYTES] */);
int fclsh_cluster_create(const int* devices, uint32_t ndev, uint32_t shards_per_device, fclsh_cluster** out);
int fclsh_cluster_create_rank(const unsigned char* id, uint32_t world, uint32_t rank, int device,
                              uint32_t shards_per_rank, fclsh_cluster** out);
/* build_index over the sharded points (index.hpp:70-71). opt->device is
 * ignored (each rank builds on its own GPU); opt->id_offset is added to every
 * id. rows: host memory, or device memory (rows_on_device) readable from every
 * GPU of this process. */
int fclsh_cluster_build(fclsh_cluster* cl, const uint64_t* rows, int rows_on_device, int rows_scope, uint64_t n,
                        uint64_t dims, uint32_t radius, const fclsh_plan* plan, uint64_t rng_seed,
                        const fclsh_index_options* opt);
typedef struct {
    uint32_t world;           /* ranks (GPUs) */
    uint32_t rank;            /* rank of this handle's first GPU */
    uint32_t local_ranks;     /* GPUs this process drives */
    uint32_t shards_per_rank;
    uint32_t total_shards;
    int32_t device;           /* this handle's first GPU */
    int32_t uses_nccl;
    uint64_t n, dims;
    uint32_t radius;
    uint64_t table_count;        /* per shard */
    uint64_t local_points;       /* points held by this process */
    uint64_t local_entry_count;  /* postings held by this process */
    uint64_t local_device_bytes;
    uint32_t local_bucket_shards; /* shards in the bucket layout (the rest: CSR) */
    double build_ms;              /* slowest rank's device build time */
} fclsh_cluster_info;
int fclsh_cluster_info_get(const fclsh_cluster* cl, fclsh_cluster_info* out);
/* query_r_nn over the whole cluster, host rows in (read on rank 0 only), host
 * result out on rank 0 (*out = NULL on the other ranks); free with
 * fclsh_result_free. Synchronous. */
int fclsh_cluster_query(fclsh_cluster* cl, const uint64_t* q_rows, uint64_t nq, uint32_t radius,
                        fclsh_result** out);
/* Device rows in (on rank 0's GPU), device result on rank 0's GPU valid until
 * the next batch (all-zero *out on other ranks). `stream` is a stream on this
 * process's first GPU: the batch starts after the work queued on it and the
 * results are ordered before what is queued on it afterwards. */
int fclsh_cluster_query_device(fclsh_cluster* cl, const uint64_t* d_q_rows, uint64_t nq, uint32_t radius,
                               void* stream, fclsh_device_result* out);
/* Per-shard stage timing (fclsh_query_stage_timing / _stage_ms /
 * _path_counts of the shard indexes this process holds, numbered in rank then
 * shard order from 0). */
int fclsh_cluster_stage_timing(fclsh_cluster* cl, int enable);
int fclsh_cluster_stage_ms(const fclsh_cluster* cl, uint32_t local_shard, double* ms, int n);
int fclsh_cluster_path_counts(const fclsh_cluster* cl, uint32_t local_shard, uint64_t* dense, uint64_t* general);
void fclsh_cluster_destroy(fclsh_cluster* cl);

/* Number of kernels the library launched on this thread since the last
 * reset (launch accounting for the bench). */
uint64_t fclsh_launch_count(void);
void fclsh_launch_count_reset(void);

/* ------------------------------------------------------------- workloads ---
 * Seeded synthetic inputs of the BASELINE configs. Host
 * buffers, multithreaded, counter-based (deterministic for any thread count):
 * rows [row0, row0 + n) of one unbounded stream, so each rank of a cluster
 * generates just its own slice of a global dataset.
 *   bernoulli: n rows of d i.i.d. Bernoulli(0.5) bits.
 *   clustered: centres rows of Bernoulli(0.5) bits; each of n rows copies a
 *              uniformly drawn centre and flips each bit w.p. flip_p.
 *   planted:   nq queries, each a uniformly drawn data row with k flipped
 *              distinct positions, k uniform in [0, kmax]; src_out gets the
 *              source row id (may be NULL).                                */
int fclsh_gen_bernoulli(uint64_t seed, uint64_t row0, uint64_t n, uint64_t dims, uint64_t* rows, int threads);
int fclsh_gen_clustered(uint64_t seed, uint64_t centres, uint64_t row0, uint64_t n, uint64_t dims, double flip_p,
                        uint64_t* rows, int threads);
int fclsh_gen_planted(uint64_t seed, const uint64_t* data, uint64_t n, uint64_t dims, uint64_t nq,
                      uint32_t kmax, uint64_t* qrows, uint32_t* src_out);

#ifdef __cplusplus
}
#endif

#endif /* FCLSH_GPU_H */
