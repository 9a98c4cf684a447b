/* TEST INFRASTRUCTURE ONLY -- see fclsh_oracle.h for the contract.
 *
 * Plain-C restatement of the reference's hot path. Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Deliberately simple: sequential per point, sorted posting arrays, binary
 * search -- the same algorithm as the reference, not a fast one.
 */
#define _GNU_SOURCE
#include "fclsh_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }
void orc_free(void* p) { free(p); }

/* ---------------------------------------------------------------- rng.cpp */

uint64_t orc_splitmix64(uint64_t x) { /* rng.cpp:9-14 */
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

static uint64_t fnv1a(const char* s) { /* rng.cpp:18-25 */
    uint64_t h = 0xcbf29ce484222325ull;
    for (; *s; ++s) {
        h ^= (uint8_t)*s;
        h *= 0x100000001b3ull;
    }
    return h;
}

uint64_t orc_rng_stream(uint64_t seed, const char* label) { /* rng.cpp:31-33 */
    return orc_splitmix64(seed ^ fnv1a(label));
}

uint64_t orc_rng_stream_idx(uint64_t seed, const char* label, uint64_t idx) { /* rng.cpp:35-37 */
    return orc_splitmix64(seed ^ fnv1a(label) ^ orc_splitmix64(idx + 1));
}

/* std::mt19937_64 as the C++ standard specifies it ([rand.predef]). */
void orc_rng_init(orc_rng* r, uint64_t seed) { /* rng.cpp:29 */
    uint64_t s = orc_splitmix64(seed);
    r->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

uint64_t orc_rng_next(orc_rng* r) {
    static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
    if (r->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[i + 1] & 0x7FFFFFFFull);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag[x & 1];
        }
        for (; i < 311; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[i + 1] & 0x7FFFFFFFull);
            r->mt[i] = r->mt[i + 156 - 312] ^ (x >> 1) ^ mag[x & 1];
        }
        uint64_t x = (r->mt[311] & 0xFFFFFFFF80000000ull) | (r->mt[0] & 0x7FFFFFFFull);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag[x & 1];
        r->mti = 0;
    }
    uint64_t y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

uint64_t orc_rng_below(orc_rng* r, uint64_t bound) { /* rng.cpp:41-50 */
    uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
        x = orc_rng_next(r);
    } while (x >= limit);
    return x % bound;
}

void orc_rng_shuffle_u32(orc_rng* r, uint32_t* v, size_t n) { /* rng.hpp:38-44 */
    for (size_t i = n; i > 1; --i) {
        size_t j = (size_t)orc_rng_below(r, i);
        uint32_t tmp = v[i - 1];
        v[i - 1] = v[j];
        v[j] = tmp;
    }
}

void orc_rng_draw(uint64_t seed, uint64_t count, uint64_t* out) {
    orc_rng r;
    orc_rng_init(&r, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = orc_rng_next(&r);
}

/* ------------------------------------------------- modmath.hpp / hadamard */

static inline uint64_t add_mod(uint64_t a, uint64_t b, uint64_t p) { /* modmath.hpp:12-15 */
    uint64_t s = a + b;
    return s >= p ? s - p : s;
}
static inline uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t p) { /* modmath.hpp:17-19 */
    return a >= b ? a - b : a + p - b;
}
static inline uint64_t mul_mod(uint64_t a, uint64_t b, uint64_t p) { /* modmath.hpp:21-23 */
    return (uint64_t)(((unsigned __int128)a * b) % p);
}

static int is_pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }

int orc_fht_mod(uint64_t* v, uint64_t n, uint64_t p) { /* hadamard.cpp:51-64 */
    if (p < 3 || p % 2 == 0) return set_err(2, "fht_mod: modulus must be odd and > 2");
    if (!is_pow2(n)) return set_err(2, "fht_mod: length is not a power of two");
    for (uint64_t half = 1; half < n; half *= 2)
        for (uint64_t block = 0; block < n; block += 2 * half)
            for (uint64_t i = block; i < block + half; ++i) {
                uint64_t a = v[i], b = v[i + half];
                v[i] = add_mod(a, b, p);
                v[i + half] = sub_mod(a, b, p);
            }
    return 0;
}

int orc_batch_hash_kernel(uint64_t* t, uint64_t n, uint64_t l1, uint64_t p) { /* hadamard.cpp:66-72 */
    int rc = orc_fht_mod(t, n, p);
    if (rc) return rc;
    uint64_t half = (p + 1) / 2; /* modmath.hpp:26-29 */
    for (uint64_t i = 0; i < n; ++i) t[i] = mul_mod(half, sub_mod(l1, t[i], p), p);
    return 0;
}

/* ------------------------------------------------------------ covering.cpp */

static int check_basic(uint64_t dims, uint32_t radius, uint64_t prime) { /* covering.cpp:14-22 */
    if (dims == 0) return set_err(2, "covering family: dims must be positive");
    if (radius == 0) return set_err(2, "covering family: radius must be >= 1");
    if (radius > 20) return set_err(4, "covering family: radius exceeds the table budget (max 20)");
    if (prime < 3 || prime % 2 == 0) return set_err(2, "covering family: prime must be odd and > 2");
    return 0;
}

int orc_build_family(uint64_t dims, uint32_t radius, int kind, uint64_t seed, uint64_t prime,
                     int include_zero, uint32_t* mapping, uint64_t* seeds, int* kind_out) {
    int rc = check_basic(dims, radius, prime);
    if (rc) return rc;
    uint64_t order = 1ull << (radius + 1);
    if (kind < 0) kind = dims > order ? 0 : 1; /* covering.cpp:74-80 */
    /* covering.cpp:24-32 */
    if (kind == 1 && dims > order) return set_err(2, "covering family: specific construction needs dims <= order");
    if (kind == 0 && dims <= order) return set_err(2, "covering family: general construction needs dims > order");
    orc_rng r;
    if (kind == 0) { /* covering.cpp:53-59 */
        orc_rng_init(&r, orc_rng_stream(seed, "mapping"));
        for (uint64_t i = 0; i < dims; ++i)
            mapping[i] = include_zero ? (uint32_t)orc_rng_below(&r, order)
                                      : (uint32_t)(1 + orc_rng_below(&r, order - 1));
    } else { /* covering.cpp:60-66 */
        uint32_t* cols = (uint32_t*)malloc(order * sizeof(uint32_t));
        for (uint64_t c = 0; c < order; ++c) cols[c] = (uint32_t)c;
        orc_rng_init(&r, orc_rng_stream(seed, "permutation"));
        orc_rng_shuffle_u32(&r, cols, order);
        for (uint64_t i = 0; i < dims; ++i) mapping[i] = cols[i];
        free(cols);
    }
    orc_rng_init(&r, orc_rng_stream(seed, "seeds")); /* covering.cpp:68-69 */
    for (uint64_t i = 0; i < dims; ++i) seeds[i] = orc_rng_below(&r, prime);
    *kind_out = kind;
    return 0;
}

typedef struct {
    const uint32_t* mapping;
    const uint64_t* seeds;
    uint64_t dims, prime;
    uint32_t radius;
    const uint64_t* rows;
    uint64_t n;
    uint64_t* out;
    int tid, threads;
} hash_job;

/* covering.cpp:169-182: scatter seeds of set bits onto their columns (in
 * ascending bit order, bitvec.hpp:63-73), then batch_hash_kernel, drop h[0]. */
static void hash_one(const hash_job* j, const uint64_t* row, uint64_t* out, uint64_t* scratch) {
    uint64_t order = 1ull << (j->radius + 1);
    uint64_t words = (j->dims + 63) / 64;
    memset(scratch, 0, order * sizeof(uint64_t));
    uint64_t l1 = 0;
    for (uint64_t w = 0; w < words; ++w) {
        uint64_t bits = row[w];
        while (bits) {
            uint64_t i = w * 64 + (uint64_t)__builtin_ctzll(bits);
            bits &= bits - 1;
            if (i >= j->dims) break;
            uint64_t b = j->seeds[i];
            scratch[j->mapping[i]] = add_mod(scratch[j->mapping[i]], b, j->prime);
            l1 = add_mod(l1, b, j->prime);
        }
    }
    orc_batch_hash_kernel(scratch, order, l1, j->prime);
    memcpy(out, scratch + 1, (order - 1) * sizeof(uint64_t));
}

static void* hash_worker(void* arg) {
    hash_job* j = (hash_job*)arg;
    uint64_t order = 1ull << (j->radius + 1);
    uint64_t words = (j->dims + 63) / 64;
    uint64_t* scratch = (uint64_t*)malloc(order * sizeof(uint64_t));
    for (uint64_t i = (uint64_t)j->tid; i < j->n; i += (uint64_t)j->threads)
        hash_one(j, j->rows + i * words, j->out + i * (order - 1), scratch);
    free(scratch);
    return NULL;
}

int orc_hash_batch(const uint32_t* mapping, const uint64_t* seeds, uint64_t dims, uint32_t radius,
                   uint64_t prime, const uint64_t* rows, uint64_t n, uint64_t* out, int threads) {
    int rc = check_basic(dims, radius, prime);
    if (rc) return rc;
    if (threads < 1) threads = 1;
    hash_job* jobs = (hash_job*)calloc((size_t)threads, sizeof(hash_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        hash_job j = {mapping, seeds, dims, prime, radius, rows, n, out, t, threads};
        jobs[t] = j;
        if (threads == 1)
            hash_worker(&jobs[t]);
        else
            pthread_create(&th[t], NULL, hash_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
    return 0;
}

/* covering.cpp:34-36,150-161: out[v-1] = sum over set bits i with
 * parity(v & mapping[i]) of seeds[i], mod prime. */
int orc_hash_reference(const uint32_t* mapping, const uint64_t* seeds, uint64_t dims,
                       uint32_t radius, uint64_t prime, const uint64_t* rows, uint64_t n,
                       uint64_t* out) {
    int rc = check_basic(dims, radius, prime);
    if (rc) return rc;
    uint64_t order = 1ull << (radius + 1), words = (dims + 63) / 64;
    for (uint64_t q = 0; q < n; ++q) {
        uint64_t* o = out + q * (order - 1);
        memset(o, 0, (order - 1) * sizeof(uint64_t));
        for (uint64_t i = 0; i < dims; ++i) {
            if (!((rows[q * words + i / 64] >> (i % 64)) & 1)) continue;
            for (uint64_t v = 1; v < order; ++v)
                if (__builtin_popcountll(v & mapping[i]) & 1) o[v - 1] = add_mod(o[v - 1], seeds[i], prime);
        }
    }
    return 0;
}

/* ----------------------------------------------------------- transform.cpp */

static uint64_t tables_for_radius(uint32_t r) { return (1ull << (r + 1)) - 1; }

int orc_make_plan(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t seed,
                  int has_override, int okind, uint32_t ot, uint64_t budget, int* kind_out,
                  uint32_t* t_out, uint32_t* ppr_out, uint32_t* perm, uint64_t* parts) {
    /* transform.cpp:34-38 */
    if (dims == 0) return set_err(2, "plan: dims must be positive");
    if (radius == 0) return set_err(2, "plan: radius must be >= 1");
    if (radius >= dims) return set_err(2, "plan: radius must be below dims");
    if (c < 1.0) return set_err(2, "plan: approximation factor must be >= 1");
    if (n < 2) return set_err(2, "plan: need at least two data points");
    int kind;
    uint32_t t;
    double logn = log2((double)n), cr = c * (double)radius;
    if (has_override) { /* transform.cpp:44-50 */
        if (ot == 0) return set_err(2, "plan: override factor must be >= 1");
        if (okind == 0 && ot != 1) return set_err(2, "plan: identity override must have t = 1");
        kind = okind;
        t = ot;
    } else if (cr < logn - 1e-9) {
        kind = 1;
        t = (uint32_t)floor(logn / cr + 1e-9);
    } else if (cr > logn + 1e-9) {
        kind = 2;
        t = (uint32_t)ceil(cr / logn - 1e-9);
    } else {
        kind = 0;
        t = 1;
    }
    if (t <= 1) kind = 0;
    if (kind == 0) { /* transform.cpp:62-67 */
        if (radius > 20 || tables_for_radius(radius) > budget)
            return set_err(4, "plan: radius needs more tables than the budget allows");
        *kind_out = 0;
        *t_out = 1;
        *ppr_out = radius;
        return 0;
    }
    if (kind == 1) { /* transform.cpp:69-81 */
        while (t > 1 && ((uint64_t)t * radius > 20 || tables_for_radius(t * radius) > budget)) --t;
        if (t == 1) {
            *kind_out = 0;
            *t_out = 1;
            *ppr_out = radius;
            return 0;
        }
        *kind_out = 1;
        *t_out = t;
        *ppr_out = t * radius;
        return 0;
    }
    /* partition, transform.cpp:83-112 */
    if (t > radius) return set_err(2, "plan: cannot cut radius into that many parts");
    if (t > dims) return set_err(2, "plan: more parts than dimensions");
    uint32_t pr = radius / t;
    if (pr > 20 || (uint64_t)t * tables_for_radius(pr) > budget)
        return set_err(4, "plan: partition table count exceeds the budget");
    for (uint64_t i = 0; i < dims; ++i) perm[i] = (uint32_t)i;
    orc_rng r;
    orc_rng_init(&r, orc_rng_stream(seed, "plan-permutation"));
    orc_rng_shuffle_u32(&r, perm, dims);
    uint64_t base = dims / t, rem = dims % t, begin = 0;
    for (uint32_t p = 0; p < t; ++p) {
        uint64_t width = base + (p >= t - rem ? 1 : 0);
        parts[2 * p] = begin;
        parts[2 * p + 1] = begin + width;
        begin += width;
    }
    *kind_out = 2;
    *t_out = t;
    *ppr_out = pr;
    return 0;
}

static uint64_t view_dims(int kind, uint64_t dims, uint32_t t, const uint64_t* parts, uint32_t p) {
    if (kind == 2) return parts[2 * p + 1] - parts[2 * p];
    if (kind == 1) return dims * t;
    return dims;
}

int orc_apply_plan(int kind, uint64_t dims, uint32_t t, const uint32_t* perm,
                   const uint64_t* parts, uint32_t p, const uint64_t* rows, uint64_t n,
                   uint64_t* out) {
    uint64_t w_in = (dims + 63) / 64;
    uint64_t pd = view_dims(kind, dims, t, parts, p), w_out = (pd + 63) / 64;
    for (uint64_t q = 0; q < n; ++q) {
        const uint64_t* row = rows + q * w_in;
        uint64_t* o = out + q * w_out;
        memset(o, 0, w_out * 8);
        for (uint64_t j = 0; j < pd; ++j) {
            uint64_t src;
            if (kind == 2) src = perm[parts[2 * p] + j]; /* transform.cpp:123-135 */
            else if (kind == 1) src = j % dims;           /* transform.cpp:115-121 */
            else src = j;
            if ((row[src / 64] >> (src % 64)) & 1) o[j / 64] |= 1ull << (j % 64);
        }
    }
    return 0;
}

/* ------------------------------------------------- posting.cpp / index.cpp */

typedef struct {
    uint64_t hash;
    uint32_t id;
} entry;

static int cmp_entry(const void* a, const void* b) { /* posting.hpp:18-20 */
    const entry* x = (const entry*)a;
    const entry* y = (const entry*)b;
    if (x->hash != y->hash) return x->hash < y->hash ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

struct orc_index {
    uint64_t n, dims, words;
    uint32_t radius;
    int kind;
    uint32_t t, ppr, parts_n;
    uint32_t* perm;
    uint64_t* parts;
    uint64_t* rows;
    /* per part */
    uint64_t* fam_dims;
    uint32_t** mapping;
    uint64_t** seeds;
    int* fam_kind;
    uint64_t prime;
    uint64_t* table_base; /* first table of part p */
    uint64_t tables;
    entry** tab; /* tables x n, sorted */
};

void orc_index_destroy(orc_index* h) {
    if (!h) return;
    for (uint32_t p = 0; p < h->parts_n; ++p) {
        free(h->mapping[p]);
        free(h->seeds[p]);
    }
    if (h->tab)
        for (uint64_t t = 0; t < h->tables; ++t) free(h->tab[t]);
    free(h->tab);
    free(h->mapping);
    free(h->seeds);
    free(h->fam_dims);
    free(h->fam_kind);
    free(h->table_base);
    free(h->perm);
    free(h->parts);
    free(h->rows);
    free(h);
}

uint64_t orc_index_table_count(const orc_index* h) { return h->tables; }

int orc_index_family(const orc_index* h, uint32_t p, uint32_t* mapping, uint64_t* seeds,
                     uint64_t* dims, uint32_t* radius, int* kind) {
    if (p >= h->parts_n) return set_err(2, "part out of range");
    if (mapping) memcpy(mapping, h->mapping[p], h->fam_dims[p] * 4);
    if (seeds) memcpy(seeds, h->seeds[p], h->fam_dims[p] * 8);
    *dims = h->fam_dims[p];
    *radius = h->ppr;
    *kind = h->fam_kind[p];
    return 0;
}

typedef struct {
    orc_index* h;
    uint32_t p;
    const uint64_t* views; /* n x view words */
    uint64_t t_begin, t_end;
} build_job;

static void* build_worker(void* arg) {
    build_job* j = (build_job*)arg;
    orc_index* h = j->h;
    uint32_t p = j->p;
    uint64_t order = 1ull << (h->ppr + 1), L = order - 1;
    uint64_t vw = (h->fam_dims[p] + 63) / 64;
    uint64_t* keys = (uint64_t*)malloc(L * sizeof(uint64_t));
    uint64_t* scratch = (uint64_t*)malloc(order * sizeof(uint64_t));
    hash_job hj = {h->mapping[p], h->seeds[p], h->fam_dims[p], h->prime, h->ppr, NULL, 0, NULL, 0, 1};
    /* index.cpp:101-114 -- each worker owns the tables [t_begin, t_end) */
    for (uint64_t id = 0; id < h->n; ++id) {
        hash_one(&hj, j->views + id * vw, keys, scratch);
        for (uint64_t v = j->t_begin; v < j->t_end; ++v) {
            entry e = {keys[v], (uint32_t)id};
            h->tab[h->table_base[p] + v][id] = e;
        }
    }
    for (uint64_t v = j->t_begin; v < j->t_end; ++v) /* posting.cpp:9-12 */
        qsort(h->tab[h->table_base[p] + v], h->n, sizeof(entry), cmp_entry);
    free(keys);
    free(scratch);
    return NULL;
}

orc_index* orc_index_build(const uint64_t* rows, uint64_t n, uint64_t dims, uint32_t radius,
                           uint64_t plan_seed, int has_override, int okind, uint32_t ot, double c,
                           uint64_t index_seed, uint64_t prime, int include_zero, uint64_t budget,
                           int threads, int* code) {
    *code = 0;
    orc_index* h = (orc_index*)calloc(1, sizeof(orc_index));
    h->n = n;
    h->dims = dims;
    h->words = (dims + 63) / 64;
    h->radius = radius;
    h->prime = prime;
    h->perm = (uint32_t*)malloc((dims ? dims : 1) * 4);
    h->parts = (uint64_t*)malloc(2 * (radius + 1) * 8 + 16);
    int rc = orc_make_plan(dims, radius, c, n, plan_seed, has_override, okind, ot, budget, &h->kind,
                           &h->t, &h->ppr, h->perm, h->parts);
    if (rc) goto fail;
    /* index.cpp:51-53 */
    if (n == 0) { rc = set_err(2, "index: empty dataset"); goto fail; }
    h->parts_n = h->kind == 2 ? h->t : 1;
    uint64_t L = tables_for_radius(h->ppr);
    h->tables = h->parts_n * L;
    if (h->tables > budget) { rc = set_err(4, "index: table count exceeds the budget"); goto fail; } /* index.cpp:78-79 */
    h->rows = (uint64_t*)malloc(n * h->words * 8);
    memcpy(h->rows, rows, n * h->words * 8);
    h->fam_dims = (uint64_t*)calloc(h->parts_n, 8);
    h->fam_kind = (int*)calloc(h->parts_n, sizeof(int));
    h->mapping = (uint32_t**)calloc(h->parts_n, sizeof(uint32_t*));
    h->seeds = (uint64_t**)calloc(h->parts_n, sizeof(uint64_t*));
    h->table_base = (uint64_t*)calloc(h->parts_n, 8);
    h->tab = (entry**)calloc(h->tables, sizeof(entry*));
    for (uint32_t p = 0; p < h->parts_n; ++p) { /* index.cpp:83-88 */
        uint64_t pd = view_dims(h->kind, dims, h->t, h->parts, p);
        h->fam_dims[p] = pd;
        h->mapping[p] = (uint32_t*)malloc(pd * 4);
        h->seeds[p] = (uint64_t*)malloc(pd * 8);
        rc = orc_build_family(pd, h->ppr, -1, orc_rng_stream_idx(index_seed, "family", p), prime,
                              include_zero, h->mapping[p], h->seeds[p], &h->fam_kind[p]);
        if (rc) goto fail;
        h->table_base[p] = p * L;
    }
    for (uint64_t t = 0; t < h->tables; ++t) h->tab[t] = (entry*)malloc(n * sizeof(entry));
    if (threads < 1) threads = 1;
    for (uint32_t p = 0; p < h->parts_n; ++p) {
        uint64_t pd = h->fam_dims[p], vw = (pd + 63) / 64;
        uint64_t* views = (uint64_t*)malloc(n * vw * 8);
        orc_apply_plan(h->kind, dims, h->t, h->perm, h->parts, p, rows, n, views);
        int T = threads < (int)L ? threads : (int)L;
        build_job* jobs = (build_job*)calloc((size_t)T, sizeof(build_job));
        pthread_t* th = (pthread_t*)calloc((size_t)T, sizeof(pthread_t));
        for (int k = 0; k < T; ++k) {
            build_job j = {h, p, views, L * (uint64_t)k / (uint64_t)T, L * (uint64_t)(k + 1) / (uint64_t)T};
            jobs[k] = j;
            if (T == 1) build_worker(&jobs[k]);
            else pthread_create(&th[k], NULL, build_worker, &jobs[k]);
        }
        if (T > 1)
            for (int k = 0; k < T; ++k) pthread_join(th[k], NULL);
        free(jobs);
        free(th);
        free(views);
    }
    return h;
fail:
    *code = rc;
    orc_index_destroy(h);
    return NULL;
}

typedef struct {
    const orc_index* h;
    const uint64_t* qrows;
    uint64_t nq;
    uint32_t radius;
    uint64_t* counters;
    uint32_t** res;
    uint64_t* res_n;
    int tid, threads;
} query_job;

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

static void* query_worker(void* arg) { /* index.cpp:157-188 */
    query_job* j = (query_job*)arg;
    const orc_index* h = j->h;
    uint32_t* stamp = (uint32_t*)calloc(h->n, 4);
    uint32_t epoch = 0;
    uint64_t L = tables_for_radius(h->ppr), order = L + 1;
    uint64_t* keys = (uint64_t*)malloc(L * 8);
    uint64_t* scratch = (uint64_t*)malloc(order * 8);
    uint64_t maxw = 0;
    for (uint32_t p = 0; p < h->parts_n; ++p) {
        uint64_t w = (h->fam_dims[p] + 63) / 64;
        if (w > maxw) maxw = w;
    }
    uint64_t* view = (uint64_t*)malloc(maxw * 8);
    uint64_t cap = 64;
    uint32_t* cand = (uint32_t*)malloc(cap * 4);
    for (uint64_t q = (uint64_t)j->tid; q < j->nq; q += (uint64_t)j->threads) {
        const uint64_t* qrow = j->qrows + q * h->words;
        ++epoch; /* index.cpp:33-41 (no wrap within a worker's lifetime here) */
        uint64_t coll = 0, ncand = 0;
        for (uint32_t p = 0; p < h->parts_n; ++p) {
            orc_apply_plan(h->kind, h->dims, h->t, h->perm, h->parts, p, qrow, 1, view);
            hash_job hj = {h->mapping[p], h->seeds[p], h->fam_dims[p], h->prime, h->ppr, NULL, 0, NULL, 0, 1};
            hash_one(&hj, view, keys, scratch);
            for (uint64_t v = 0; v < L; ++v) { /* posting.cpp:14-21 */
                const entry* tb = h->tab[h->table_base[p] + v];
                uint64_t lo = 0, hi = h->n, key = keys[v];
                while (lo < hi) {
                    uint64_t mid = (lo + hi) / 2;
                    if (tb[mid].hash < key) lo = mid + 1;
                    else hi = mid;
                }
                for (uint64_t k = lo; k < h->n && tb[k].hash == key; ++k) {
                    ++coll;
                    uint32_t id = tb[k].id;
                    if (stamp[id] != epoch) { /* index.cpp:43-47 */
                        stamp[id] = epoch;
                        if (ncand == cap) {
                            cap *= 2;
                            cand = (uint32_t*)realloc(cand, cap * 4);
                        }
                        cand[ncand++] = id;
                    }
                }
            }
        }
        /* index.cpp:182-185: verify on the full original row, ids ascending */
        uint32_t* out = (uint32_t*)malloc((ncand ? ncand : 1) * 4);
        uint64_t nf = 0;
        for (uint64_t k = 0; k < ncand; ++k) {
            const uint64_t* row = h->rows + (uint64_t)cand[k] * h->words;
            uint64_t dist = 0;
            for (uint64_t w = 0; w < h->words; ++w) dist += (uint64_t)__builtin_popcountll(row[w] ^ qrow[w]);
            if (dist <= j->radius) out[nf++] = cand[k];
        }
        qsort(out, nf, 4, cmp_u32);
        j->counters[3 * q] = coll;
        j->counters[3 * q + 1] = ncand;
        j->counters[3 * q + 2] = nf;
        j->res[q] = out;
        j->res_n[q] = nf;
    }
    free(stamp);
    free(keys);
    free(scratch);
    free(view);
    free(cand);
    return NULL;
}

int orc_index_query(const orc_index* h, const uint64_t* qrows, uint64_t nq, uint32_t radius,
                    int threads, uint64_t* counters, uint64_t* offsets, uint32_t** ids_out) {
    if (radius > h->radius) return set_err(2, "query radius exceeds the index radius"); /* index.cpp:147-153 */
    if (threads < 1) threads = 1;
    uint32_t** res = (uint32_t**)calloc(nq ? nq : 1, sizeof(uint32_t*));
    uint64_t* res_n = (uint64_t*)calloc(nq ? nq : 1, 8);
    query_job* jobs = (query_job*)calloc((size_t)threads, sizeof(query_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        query_job j = {h, qrows, nq, radius, counters, res, res_n, t, threads};
        jobs[t] = j;
        if (threads == 1) query_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, query_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    uint64_t total = 0;
    for (uint64_t q = 0; q < nq; ++q) {
        offsets[q] = total;
        total += res_n[q];
    }
    offsets[nq] = total;
    uint32_t* ids = (uint32_t*)malloc((total ? total : 1) * 4);
    for (uint64_t q = 0; q < nq; ++q) {
        memcpy(ids + offsets[q], res[q], res_n[q] * 4);
        free(res[q]);
    }
    *ids_out = ids;
    free(res);
    free(res_n);
    free(jobs);
    free(th);
    return 0;
}

/* ------------------------------------------------------------ workload.cpp */

typedef struct {
    const uint64_t *rows, *qrows;
    uint64_t n, nq, words;
    uint32_t radius;
    uint32_t* buf;
    uint64_t count, cap;
    uint64_t qb, qe;
} scan_job;

static void* scan_worker(void* arg) { /* workload.cpp:56-71 */
    scan_job* j = (scan_job*)arg;
    for (uint64_t q = j->qb; q < j->qe; ++q) {
        const uint64_t* qr = j->qrows + q * j->words;
        for (uint64_t p = 0; p < j->n; ++p) {
            const uint64_t* r = j->rows + p * j->words;
            uint32_t d = 0;
            for (uint64_t w = 0; w < j->words; ++w) d += (uint32_t)__builtin_popcountll(r[w] ^ qr[w]);
            if (d <= j->radius) {
                if (j->count == j->cap) {
                    j->cap = j->cap ? 2 * j->cap : 1024;
                    j->buf = (uint32_t*)realloc(j->buf, j->cap * 12);
                }
                j->buf[3 * j->count] = (uint32_t)q;
                j->buf[3 * j->count + 1] = (uint32_t)p;
                j->buf[3 * j->count + 2] = d;
                ++j->count;
            }
        }
    }
    return NULL;
}

int orc_scan_truth(const uint64_t* rows, uint64_t n, const uint64_t* qrows, uint64_t nq,
                   uint64_t dims, uint32_t radius, int threads, uint32_t** triples_out,
                   uint64_t* count) {
    if (threads < 1) threads = 1;
    scan_job* jobs = (scan_job*)calloc((size_t)threads, sizeof(scan_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    uint64_t words = (dims + 63) / 64;
    for (int t = 0; t < threads; ++t) {
        scan_job j = {rows, qrows, n, nq, words, radius, NULL, 0, 0,
                      nq * (uint64_t)t / (uint64_t)threads, nq * (uint64_t)(t + 1) / (uint64_t)threads};
        jobs[t] = j;
        if (threads == 1) scan_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, scan_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    uint64_t total = 0;
    for (int t = 0; t < threads; ++t) total += jobs[t].count;
    uint32_t* out = (uint32_t*)malloc((total ? total : 1) * 12);
    uint64_t k = 0;
    for (int t = 0; t < threads; ++t) {
        memcpy(out + 3 * k, jobs[t].buf, jobs[t].count * 12);
        k += jobs[t].count;
        free(jobs[t].buf);
    }
    *triples_out = out;
    *count = total;
    free(jobs);
    free(th);
    return 0;
}

/* ------------------------------------------------- BASELINE workload inputs
 * Not reference code: the seeded synthetic inputs of the BASELINE configs
 * (DESIGN.md "Inputs"), restated here so that the CPU baseline and the
 * reference arm of bench.py build the identical bytes without loading the
 * product library. Counter-based: word k of a stream with key K is
 * splitmix64(K + k * gamma) (the k-th SplitMix64 output seeded with K);
 * stream keys come from the reference's labelled Rng::stream seeds.
 * tests/test_oracle_pin.py pins these bytes to the product's generators. */

static const uint64_t kGamma = 0x9e3779b97f4a7c15ull;
static inline uint64_t word_at(uint64_t key, uint64_t k) { return orc_splitmix64(key + k * kGamma); }
static inline uint64_t scale_below(uint64_t r, uint64_t bound) { /* floor(r * bound / 2^64) */
    return (uint64_t)(((unsigned __int128)r * bound) >> 64);
}

typedef struct {
    int kind; /* 0 bernoulli, 1 clustered */
    uint64_t key, kc, kf, thresh, row0, dims, words, centres, b, e;
    const uint64_t* cen;
    uint64_t* rows;
} gen_job;

static void* gen_worker(void* arg) {
    gen_job* j = (gen_job*)arg;
    const uint64_t W = j->words;
    const uint64_t tail = j->dims % 64 ? (1ull << (j->dims % 64)) - 1 : ~0ull;
    for (uint64_t i = j->b; i < j->e; ++i) {
        const uint64_t g = j->row0 + i;
        if (j->kind == 0) {
            for (uint64_t w = 0; w < W; ++w) j->rows[i * W + w] = word_at(j->key, g * W + w);
            j->rows[i * W + W - 1] &= tail;
        } else {
            const uint64_t c = scale_below(word_at(j->kc, g), j->centres);
            for (uint64_t w = 0; w < W; ++w) {
                uint64_t flips = 0;
                const uint64_t bits = j->dims - w * 64 < 64 ? j->dims - w * 64 : 64;
                for (uint64_t k = 0; k < bits; ++k)
                    if (word_at(j->kf, g * j->dims + w * 64 + k) < j->thresh) flips |= 1ull << k;
                j->rows[i * W + w] = j->cen[c * W + w] ^ flips;
            }
        }
    }
    return NULL;
}

static void gen_run(gen_job proto, uint64_t n, int threads) {
    if (threads < 1) threads = 1;
    if (n < 1024) threads = 1;
    gen_job* jobs = (gen_job*)calloc((size_t)threads, sizeof(gen_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = proto;
        jobs[t].b = n * (uint64_t)t / (uint64_t)threads;
        jobs[t].e = n * (uint64_t)(t + 1) / (uint64_t)threads;
        if (threads == 1) gen_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, gen_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

void orc_gen_bernoulli(uint64_t seed, uint64_t row0, uint64_t n, uint64_t dims, uint64_t* rows, int threads) {
    gen_job j;
    memset(&j, 0, sizeof j);
    j.kind = 0;
    j.key = orc_rng_stream(seed, "data");
    j.row0 = row0;
    j.dims = dims;
    j.words = (dims + 63) / 64;
    j.rows = rows;
    gen_run(j, n, threads);
}

void orc_gen_clustered(uint64_t seed, uint64_t centres, uint64_t row0, uint64_t n, uint64_t dims, double flip_p,
                       uint64_t* rows, int threads) {
    const uint64_t W = (dims + 63) / 64;
    uint64_t* cen = (uint64_t*)malloc((centres ? centres : 1) * W * 8);
    orc_gen_bernoulli(orc_rng_stream(seed, "centres"), 0, centres, dims, cen, threads);
    gen_job j;
    memset(&j, 0, sizeof j);
    j.kind = 1;
    j.kc = orc_rng_stream(seed, "assign");
    j.kf = orc_rng_stream(seed, "flips");
    j.thresh = flip_p >= 1.0 ? ~0ull : (uint64_t)(flip_p * 18446744073709551616.0);
    j.row0 = row0;
    j.dims = dims;
    j.words = W;
    j.centres = centres;
    j.cen = cen;
    j.rows = rows;
    gen_run(j, n, threads);
    free(cen);
}

void orc_gen_planted(uint64_t seed, const uint64_t* data, uint64_t n, uint64_t dims, uint64_t nq, uint32_t kmax,
                     uint64_t* qrows, uint32_t* src_out) {
    const uint64_t W = (dims + 63) / 64;
    const uint64_t kq = orc_rng_stream(seed, "queries");
    const uint64_t kp = orc_rng_stream(seed, "positions");
    uint32_t* pos = (uint32_t*)malloc((dims ? dims : 1) * 4);
    for (uint64_t j = 0; j < nq; ++j) {
        const uint64_t src = scale_below(word_at(kq, 2 * j), n);
        const uint64_t k = scale_below(word_at(kq, 2 * j + 1), (uint64_t)kmax + 1);
        memcpy(qrows + j * W, data + src * W, W * 8);
        for (uint64_t i = 0; i < dims; ++i) pos[i] = (uint32_t)i;
        /* k distinct positions: prefix of a Fisher-Yates shuffle */
        for (uint64_t s = 0; s < k && s < dims; ++s) {
            const uint64_t r = s + scale_below(word_at(kp, j * dims + s), dims - s);
            const uint32_t tmp = pos[s];
            pos[s] = pos[r];
            pos[r] = tmp;
            qrows[j * W + pos[s] / 64] ^= 1ull << (pos[s] % 64);
        }
        if (src_out) src_out[j] = (uint32_t)src;
    }
    free(pos);
}
