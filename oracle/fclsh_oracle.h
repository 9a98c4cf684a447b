/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the fcLSH hot path.
 *
 * A plain-C restatement of the reference algorithm (arXiv 1602.02620
 * reference library under /root/reference/proj). Only tests/, the smoke
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * legs may load it, and only as the checker. The product library
 * (paper_1602_02620_b200/) never links, loads or calls it.
 *
 * Parity pin: tests/test_oracle_pin.py checks every function here against
 * the compiled reference (oracle/_ref/libfclsh_ref.so, built from the
 * reference's own sources by oracle/Makefile) and against the golden values
 * restated from the reference's unit tests (test_hadamard.cpp,
 * test_covering.cpp, test_transform.cpp, test_index.cpp).
 *
 * Row layout everywhere: row-major uint64 words, bit i of a row in word i/64
 * at offset i%64, padding bits zero (bitvec.hpp:13-19).
 */
#ifndef FCLSH_ORACLE_H
#define FCLSH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
void orc_free(void* p);

/* rng.cpp:9-14 */
uint64_t orc_splitmix64(uint64_t x);
/* rng.cpp:31-37 -- seed of Rng(seed).stream(label[, idx]) */
uint64_t orc_rng_stream(uint64_t seed, const char* label);
uint64_t orc_rng_stream_idx(uint64_t seed, const char* label, uint64_t idx);

typedef struct {
    uint64_t mt[312];
    int mti;
} orc_rng;

/* rng.cpp:29 -- Rng(seed) seeds std::mt19937_64 with splitmix64(seed) */
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);                     /* rng.cpp:39 */
uint64_t orc_rng_below(orc_rng* r, uint64_t bound);    /* rng.cpp:41-50 */
void orc_rng_shuffle_u32(orc_rng* r, uint32_t* v, size_t n); /* rng.hpp:38-44 */
void orc_rng_draw(uint64_t seed, uint64_t count, uint64_t* out);

/* hadamard.cpp:51-72 */
int orc_fht_mod(uint64_t* v, uint64_t n, uint64_t p);
int orc_batch_hash_kernel(uint64_t* t, uint64_t n, uint64_t l1, uint64_t p);

/* covering.cpp:40-80 (kind -1 = derive from widths; 0 general; 1 specific) */
int orc_build_family(uint64_t dims, uint32_t radius, int kind, uint64_t seed, uint64_t prime,
                     int include_zero, uint32_t* mapping, uint64_t* seeds, int* kind_out);

/* covering.cpp:169-182 (batch) and :150-161 (per mask). out is n x L,
 * point-major, L = 2^(radius+1)-1. rows have ceil(dims/64) words. */
int orc_hash_batch(const uint32_t* mapping, const uint64_t* seeds, uint64_t dims, uint32_t radius,
                   uint64_t prime, const uint64_t* rows, uint64_t n, uint64_t* out, int threads);
int orc_hash_reference(const uint32_t* mapping, const uint64_t* seeds, uint64_t dims,
                       uint32_t radius, uint64_t prime, const uint64_t* rows, uint64_t n,
                       uint64_t* out);

/* transform.cpp:32-113; plan kind 0 identity, 1 replicate, 2 partition */
int orc_make_plan(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t seed,
                  int has_override, int okind, uint32_t ot, uint64_t budget, int* kind,
                  uint32_t* t, uint32_t* per_part_radius, uint32_t* perm, uint64_t* parts);

/* transform.cpp:115-158: view p of every row (identity: copy, replicate:
 * t copies back to back, partition: permuted slice). out rows have
 * ceil(part_dims/64) words. */
int orc_apply_plan(int kind, uint64_t dims, uint32_t t, const uint32_t* perm,
                   const uint64_t* parts, uint32_t p, const uint64_t* rows, uint64_t n,
                   uint64_t* out);

typedef struct orc_index orc_index;

/* make_plan(...) + build_index(data, covering_batch, ...) (index.cpp:49-119).
 * The index keeps its own copy of the rows. */
orc_index* orc_index_build(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius,
                           uint64_t plan_seed, int has_override, int okind, uint32_t ot, double c,
                           uint64_t index_seed, uint64_t prime, int include_zero, uint64_t budget,
                           int threads, int* code);
void orc_index_destroy(orc_index* h);
uint64_t orc_index_table_count(const orc_index* h);
/* part p's family */
int orc_index_family(const orc_index* h, uint32_t p, uint32_t* mapping, uint64_t* seeds,
                     uint64_t* dims, uint32_t* radius, int* kind);

/* query_r_nn (index.cpp:157-188) for each query row: counters nq x 3
 * (collisions, candidates, found), offsets nq+1, *ids_out malloc'd. */
int orc_index_query(const orc_index* h, const uint64_t* qrows, uint64_t nq, uint32_t radius,
                    int threads, uint64_t* counters, uint64_t* offsets, uint32_t** ids_out);

/* scan_truth (workload.cpp:56-71): (query, point, distance) sorted. */
int orc_scan_truth(const uint64_t* rows, uint64_t n, const uint64_t* qrows, uint64_t nq,
                   uint64_t dims, uint32_t radius, int threads, uint32_t** triples_out,
                   uint64_t* count);

/* BASELINE workload inputs (not reference code; identical bytes to the
 * product's fclsh_gen_*, so CPU legs never load the product library). */
void orc_gen_bernoulli(uint64_t seed, uint64_t row0, uint64_t n, uint64_t dims, uint64_t* rows, int threads);
void orc_gen_clustered(uint64_t seed, uint64_t centres, uint64_t row0, uint64_t n, uint64_t dims, double flip_p,
                       uint64_t* rows, int threads);
void orc_gen_planted(uint64_t seed, const uint64_t* data, uint64_t n, uint64_t dims, uint64_t nq, uint32_t kmax,
                     uint64_t* qrows, uint32_t* src_out);

#ifdef __cplusplus
}
#endif

#endif
