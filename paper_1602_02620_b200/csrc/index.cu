// K2 (table build) and K3-K5 (probe, dedup, verify) for sm_100a.
//
// Every table of the reference is a PostingTable: (key, id) entries sorted by
// (key, id), looked up by binary search (posting.cpp:9-21). query_r_nn walks
// every table's bucket for the query key, counts every posting it touches
// (`collisions`), keeps the first sighting of each id (`candidates`) and
// verifies those on the full row (`found`, ids ascending) (index.cpp:157-188).
// On the GPU the probe is bound by random DRAM accesses, so the device tables
// are built for one random access per probe:
//
//  kBuckets (default)  open-addressed bucket table per table: 2^bb buckets of
//      four (key, id) slots, home bucket = key >> shift (keys are uniform in
//      [0, P)), linear probing into the next bucket, filled slots always a
//      prefix of the bucket. Load <= 50%, so a probe reads one 32-byte
//      bucket (64 B for 8-byte keys) and almost never a second. Every
//      posting with key k sits in the run of full buckets starting at
//      home(k), so counts are exact.
//  kCsr  (fallback when memory is tight)  the reference's sorted array plus a
//      directory of 2^b key cells (CSR offsets): two random accesses per probe,
//      ~10 bytes per posting instead of ~16.
//
// Build: K1 writes one part's L key columns table-major, then per table
// kBuckets inserts every (key, id) with a CAS into the first free slot of its
// run; kCsr counts cells, scans, scatters and sorts each cell by (key, id).
//
// Query (all queries of a batch at once):
//   S1  K1 hashes the query rows point-major (key[q*T + t]).
//   S2+S3  k_query_fused, one warp per query: lanes probe tables lane,
//       lane+32, ... four at a time, append matching ids to a shared-memory
//       list (its length = collisions), bitonic-sort it (adjacent uniques =
//       candidates), verify with XOR+popcount (found, ids ascending) into the
//       query's result slot.
//   Queries whose list or result set overflows the fused kernel's capacity
//   go through the general path (count, scan, gather, CUB segmented sort,
//   verify); a scan of the per-query found counts and one compaction write
//   the (query, id, distance) triples ordered by (query, id).

#include "index.cuh"

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace fclsh_b200 {

namespace {

struct NarrowEntry { // key < 2^32: one u64, (key << 32 | id) orders as (key, id)
    using E = unsigned long long;
    using K = uint32_t;
    static constexpr int kBucketLoads = 2; // 32-byte bucket = 2 x 16 B
    __device__ __forceinline__ static uint64_t key(E e) { return e >> 32; }
    __device__ __forceinline__ static uint32_t id(E e) { return uint32_t(e); }
    __device__ __forceinline__ static E make(uint64_t k, uint32_t i) { return (E(k) << 32) | i; }
    __device__ __forceinline__ static bool less(E a, E b) { return a < b; }
    __device__ __forceinline__ static bool empty(E e) { return e == ~0ull; }
    // a posting of key k (k < prime <= 2^32 - 1, so an empty slot's key field 0xFFFFFFFF never
    // equals one): one 32-bit compare instead of the 64-bit empty test and key compare
    __device__ __forceinline__ static bool match(E e, uint64_t k) { return uint32_t(e >> 32) == uint32_t(k); }
    __host__ __device__ static constexpr unsigned char empty_byte() { return 0xFF; }
    // claim slot p for e; true if this thread placed it
    __device__ __forceinline__ static bool claim(E* p, E e) { return atomicCAS(p, ~0ull, e) == ~0ull; }
};

struct WideEntry { // 8-byte keys: {key, id}
    using E = ulonglong2;
    using K = uint64_t;
    static constexpr int kBucketLoads = 4; // 64-byte bucket
    __device__ __forceinline__ static uint64_t key(E e) { return e.x; }
    __device__ __forceinline__ static uint32_t id(E e) { return uint32_t(e.y); }
    __device__ __forceinline__ static E make(uint64_t k, uint32_t i) { return make_ulonglong2(k, i); }
    __device__ __forceinline__ static bool less(E a, E b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }
    __device__ __forceinline__ static bool empty(E e) { return e.x == ~0ull; }
    __device__ __forceinline__ static bool match(E e, uint64_t k) { return e.x == k; } // k < prime < 2^63
    __host__ __device__ static constexpr unsigned char empty_byte() { return 0xFF; }
    __device__ __forceinline__ static bool claim(E* p, E e) {
        if (atomicCAS(&p->x, ~0ull, e.x) != ~0ull) return false;
        p->y = e.y; // the slot is ours; nobody reads it before the build ends
        return true;
    }
};

constexpr int kSlots = 4; // per bucket
constexpr uint32_t kBuildSlab = 64; // tables per table-major slab of the bucket build
#ifndef FCLSH_SCAN_TILE_LOG
#define FCLSH_SCAN_TILE_LOG 10
#endif
#ifndef FCLSH_SCAN_SPLIT
#define FCLSH_SCAN_SPLIT 8
#endif
constexpr int kScanTileLog = FCLSH_SCAN_TILE_LOG; // queries per tile of the found scan (k_scan_compact), = its CTA size
constexpr int kScanSplit = FCLSH_SCAN_SPLIT;      // CTAs sharing one tile's copying
// The warp kernel hands out the queries past its first wave from kQCtr
// counters kQCtrStride words (256 B) apart -- CTA b draws from counter
// b % kQCtr -- instead of one: ~10k returning atomics on one address
// serialise in its L2 slice (18.7 % of the kernel's stall samples on cfg3,
// profiles/r02/ncu_k_query_warp_pf_atomic_cfg3.txt)
constexpr uint32_t kQCtr = 16, kQCtrStride = 64;
#ifndef FCLSH_FE4_MINB
#define FCLSH_FE4_MINB 5 // CTAs per SM of the cfg3 warp kernel (A/B builds: 6 same, 7-8 spill and lose 17 %)
#endif
constexpr uint64_t kCntHeader = 64 + uint64_t(kQCtr) * kQCtrStride * 4; // bytes before the tile sums
#ifndef FCLSH_FUSED_CAP
#define FCLSH_FUSED_CAP 256
#endif
#ifndef FCLSH_FUSED_U
#define FCLSH_FUSED_U 2
#endif
#ifndef FCLSH_DENSE_U
#define FCLSH_DENSE_U 2
#endif
#ifndef FCLSH_DENSE_RUN
#define FCLSH_DENSE_RUN 2
#endif
constexpr int kDenseU = FCLSH_DENSE_U;     // home buckets per thread in flight in the CTA kernel
constexpr int kDenseRun = FCLSH_DENSE_RUN; // buckets read at a time along a spilled run (CTA kernel)
constexpr int kFusedU = FCLSH_FUSED_U; // tables per lane in flight in the warp kernel
constexpr int kFusedCap = FCLSH_FUSED_CAP;
#ifndef FCLSH_WARP_U_DEFAULT
#define FCLSH_WARP_U_DEFAULT 2
#endif
constexpr int kWarpU = FCLSH_WARP_U_DEFAULT; // probes per lane in flight in k_query_warp_pf // warp-kernel id-set slots (3/4 of it: distinct ids; more: the CTA kernel)

// One bucket (4 slots) with 256-bit loads: a random probe is one L1 request
// for the narrow layout (two for wide) instead of four 64-bit ones; the
// tables are read-only while queries run (.nc). tools/rand_bench.cu measures
// the random-access ceiling this targets.
__device__ __forceinline__ void load_bucket(const unsigned long long* bp, unsigned long long (&x)[kSlots]) {
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
        : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3])
        : "l"(bp));
}
#ifndef FCLSH_BUCKET_EF
#define FCLSH_BUCKET_EF 1
#endif
// home-bucket read of the warp kernel: never reused within a batch, so with
// FCLSH_BUCKET_EF its L2 line is marked evict_first (keeps the key filter)
__device__ __forceinline__ void load_bucket_probe(const unsigned long long* bp, unsigned long long (&x)[kSlots],
                                                  uint64_t pol) {
#if FCLSH_BUCKET_EF
    asm("ld.global.nc.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
        : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3])
        : "l"(bp), "l"(pol));
#else
    (void)pol;
    load_bucket(bp, x);
#endif
}
__device__ __forceinline__ void load_bucket(const ulonglong2* bp, ulonglong2 (&x)[kSlots]) {
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
        : "=l"(x[0].x), "=l"(x[0].y), "=l"(x[1].x), "=l"(x[1].y)
        : "l"(bp));
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
        : "=l"(x[2].x), "=l"(x[2].y), "=l"(x[3].x), "=l"(x[3].y)
        : "l"(bp + 2));
}

// Hamming distance (bitvec.cpp:73-79) of a stored row and a query row with
// vector loads: vec = 4 -> 256-bit loads (W % 4 == 0, 32-B aligned rows: a
// d = 256 row is one load, one 32-B sector), 2 -> 128-bit, 1 -> 64-bit.
__device__ __forceinline__ uint32_t row_distance(const uint64_t* r, const uint64_t* q, uint32_t words, int vec) {
    uint32_t d = 0;
    if (vec == 4) {
        for (uint32_t w = 0; w < words; w += 4) {
            unsigned long long a0, a1, a2, a3, b0, b1, b2, b3;
            asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(r + w));
            asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(b0), "=l"(b1), "=l"(b2), "=l"(b3) : "l"(q + w));
            d += __popcll(a0 ^ b0) + __popcll(a1 ^ b1) + __popcll(a2 ^ b2) + __popcll(a3 ^ b3);
        }
    } else if (vec == 2) {
        for (uint32_t w = 0; w < words; w += 2) {
            const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(r + w));
            const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(q + w));
            d += __popcll(a.x ^ b.x) + __popcll(a.y ^ b.y);
        }
    } else {
        for (uint32_t w = 0; w < words; ++w) d += __popcll(__ldg(r + w) ^ __ldg(q + w));
    }
    return d;
}

// Read-only view of one shard's tables, passed by value to the kernels.
template <typename T>
struct Tables {
    const typename T::E* data; // entries (CSR) or buckets (kBuckets)
    const uint32_t* dir;       // CSR only
    uint64_t n;                // postings per table
    uint64_t cells;            // CSR cells per table
    uint64_t nbuckets;         // buckets per table
    uint32_t shift;            // CSR: cell = (key * kscale) >> shift; buckets: home bucket, the same
    uint64_t kscale;           // floor(2^64 / P): key * kscale is the key's 64-bit fraction of [0, P)
    const uint32_t* filter;    // buckets: per-table key filter (null: none)
    uint32_t filter_words;     // filter words (32 bits) per table
};

// Key filter of the bucket tables: M = 32 * filter_words bits per table
// (about one per posting); key k maps to bit floor(k * M / 2^kbits) (keys are
// uniform in [0, P)). Kept in L2 (~64 MB for cfg2) with an evict_last policy. A probe whose bit is clear has no posting, so its random
// DRAM read of the home bucket is skipped (cfg2: ~80 % of probes miss, and a
// clear bit rejects ~37 % of them). No false negatives: every inserted
// posting sets its bit.
// Publishing a batch to mapped host memory: release / acquire at system
// scope (MEMBAR.ALL.SYS) instead of __threadfence_system()'s sequentially
// consistent fence (MEMBAR.SC.SYS + an L1 invalidate). FCLSH_PUB_SC=1
// restores the SC fences (A/B).
#ifndef FCLSH_PUB_SC
#define FCLSH_PUB_SC 0
#endif
// the flag store: every earlier write of this thread (and, cumulatively,
// those ordered before them by a CTA barrier) is visible to the host first
__device__ __forceinline__ void pub_flag(unsigned long long* flag, unsigned long long seq) {
#if FCLSH_PUB_SC
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(flag) = seq;
#else
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(seq) : "memory");
#endif
}
// a CTA's arrival after its writes (acq_rel: the last arriver sees every
// other CTA's writes before it publishes)
__device__ __forceinline__ unsigned int pub_arrive(unsigned int* ctr) {
#if FCLSH_PUB_SC
    __threadfence_system();
    const unsigned int d = atomicAdd(ctr, 1u);
    __threadfence_system();
    return d;
#else
    unsigned int d;
    asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], 1;" : "=r"(d) : "l"(ctr) : "memory");
    return d;
#endif
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void load_bucket_probe(const ulonglong2* bp, ulonglong2 (&x)[kSlots], uint64_t) {
    load_bucket(bp, x);
}
__device__ __forceinline__ uint32_t ld_filter(const uint32_t* a, uint64_t pol) {
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t filter_bit(uint64_t key, uint32_t words, uint64_t kscale) {
    return uint32_t(__umul64hi(key * kscale, uint64_t(words) * 32));
}
// Home bucket (CSR: cell) of a key: the top bits of its 64-bit fraction of
// [0, P), so keys spread evenly over the buckets for any prime (a plain
// key >> s would leave part of the table empty when P is far below 2^kbits)
__host__ __device__ __forceinline__ uint64_t home_of(uint64_t key, uint64_t kscale, uint32_t shift) {
    return (key * kscale) >> shift;
}
template <typename T>
__device__ __forceinline__ uint64_t home_of(uint64_t key, const Tables<T>& tb) {
    return home_of(key, tb.kscale, tb.shift);
}
// filter test of (table t, key): one L2 word read (evict_last policy)
template <typename T>
__device__ __forceinline__ bool filter_pass(const Tables<T>& tb, uint32_t t, uint64_t key, uint64_t pol) {
    const uint32_t r = filter_bit(key, tb.filter_words, tb.kscale);
    return (ld_filter(tb.filter + uint64_t(t) * tb.filter_words + (r >> 5), pol) >> (r & 31)) & 1u;
}

// First position in [a, e) of a CSR cell (sorted by (key, id)) whose key is
// >= key. Clustered data makes some cells long (a run of one popular key),
// and every other key of that cell would otherwise scan past the run.
template <typename T>
__device__ __forceinline__ uint32_t cell_lower_bound(const typename T::E* et, uint32_t a, uint32_t e, uint64_t key) {
    while (e - a > 8) {
        const uint32_t mid = a + (e - a) / 2;
        if (T::key(et[mid]) < key)
            a = mid + 1;
        else
            e = mid;
    }
    while (a < e && T::key(et[a]) < key) ++a;
    return a;
}

// Calls on_id(id) for every posting of table t with this key; returns the count.
template <typename T, int LAYOUT, typename F>
__device__ __forceinline__ uint32_t probe_one(const Tables<T>& tb, uint32_t t, uint64_t key, F&& on_id) {
    using E = typename T::E;
    uint32_t cnt = 0;
    if constexpr (LAYOUT == kLayoutCsr) {
        const uint32_t* d = tb.dir + uint64_t(t) * (tb.cells + 1) + home_of(key, tb);
        uint32_t a = __ldg(d);
        const uint32_t e = __ldg(d + 1);
        const E* et = tb.data + uint64_t(t) * tb.n;
        a = cell_lower_bound<T>(et, a, e, key);
        while (a < e && T::key(et[a]) == key) {
            on_id(T::id(et[a]));
            ++a;
            ++cnt;
        }
    } else {
        uint64_t b = home_of(key, tb);
        const E* base = tb.data + uint64_t(t) * tb.nbuckets * kSlots;
        for (;;) {
            E s[kSlots];
            load_bucket(base + b * kSlots, s);
#pragma unroll
            for (int j = 0; j < kSlots; ++j)
                if (!T::empty(s[j]) && T::key(s[j]) == key) {
                    on_id(T::id(s[j]));
                    ++cnt;
                }
            if (T::empty(s[kSlots - 1])) break;
            b = (b + 1) & (tb.nbuckets - 1);
        }
    }
    return cnt;
}

// ----------------------------------------------------------------- build

// point-major keys [n][L] -> table-major [c][n] for the slab of tables
// [tb, tb + c), through 32 x 32 shared tiles (both sides 128-byte coalesced),
// so the inserts of a few tables read their keys contiguously instead of a
// 4-byte word out of every row's sector; slabs keep the table-major copy
// small (one slab, not all L tables: cfg4 on one GPU fits the 60 %-load
// bucket tables beside it)
template <typename K>
__global__ void __launch_bounds__(256) k_keys_table_major(const K* __restrict__ in, K* __restrict__ out, uint64_t n,
                                                          uint32_t L, uint32_t tb, uint32_t c) {
    __shared__ K tile[32][33];
    const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const uint64_t tiles_t = (c + 31) / 32, tiles = tiles_t * ((n + 31) / 32);
    for (uint64_t tl = blockIdx.x; tl < tiles; tl += gridDim.x) {
        const uint32_t t0 = uint32_t(tl % tiles_t) * 32;
        const uint64_t i0 = (tl / tiles_t) * 32;
        for (uint32_t r = ty; r < 32; r += 8) {
            const uint64_t i = i0 + r;
            const uint32_t t = t0 + tx;
            if (i < n && t < c) tile[r][tx] = in[i * L + tb + t];
        }
        __syncthreads();
        for (uint32_t r = ty; r < 32; r += 8) {
            const uint32_t t = t0 + r;
            const uint64_t i = i0 + tx;
            if (i < n && t < c) out[uint64_t(t) * n + i] = tile[tx][r];
        }
        __syncthreads();
    }
}

// keys are table-major for a slab of one part's tables starting at table
// key_t0: key of (row i, table t) at keys[(t - key_t0)*n + i]
template <typename T>
__global__ void k_bucket_insert(const typename T::K* __restrict__ keys, uint32_t key_t0, uint64_t n, uint32_t t0,
                                uint32_t tg,
                                uint32_t shift, uint64_t nbuckets, typename T::E* __restrict__ buckets,
                                uint32_t* __restrict__ filter, uint32_t filter_words, uint64_t kscale) {
    // tables [t0, t0 + tg) only: the buckets of a few tables stay in L2 while
    // their postings are inserted (all 511 at once thrash it: 43 GB of DRAM
    // reads for 8.6 GB of tables)
    const uint64_t total = n * tg;
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < total; x += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t t = t0 + uint32_t(x / n);
        const uint64_t i = x % n;
        typename T::E* bt = buckets + uint64_t(t) * nbuckets * kSlots;
        const uint64_t key = keys[uint64_t(t - key_t0) * n + i];
        const typename T::E e = T::make(key, uint32_t(i));
        if (filter) {
            const uint32_t r = filter_bit(key, filter_words, kscale);
            atomicOr(filter + uint64_t(t) * filter_words + (r >> 5), 1u << (r & 31));
        }
        uint64_t b = home_of(key, kscale, shift);
        FCLSH_DCHECK(b < nbuckets && t < t0 + tg);
        for (;;) {
            typename T::E* bp = bt + b * kSlots;
            bool done = false;
#pragma unroll
            for (int j = 0; j < kSlots && !done; ++j) done = T::claim(bp + j, e);
            if (done) break;
            b = (b + 1) & (nbuckets - 1);
        }
    }
}

// CSR build over tables [t0, t0+c) of one part; keys point-major (stride L).
template <typename K>
__global__ void k_hist(const K* __restrict__ keys, uint64_t n, uint32_t L, uint32_t t0, uint32_t c, uint32_t shift,
                       uint64_t kscale, uint64_t cells, uint32_t* __restrict__ cnt) {
    const uint64_t total = n * c;
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < total; x += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = x / c;
        const uint32_t t = uint32_t(x % c);
        atomicAdd(cnt + uint64_t(t) * (cells + 1) + home_of(uint64_t(keys[i * L + t0 + t]), kscale, shift), 1u);
    }
}

// One CTA per table: exclusive scan of cnt[0..cells] -> dir and cursor.
__global__ void __launch_bounds__(1024) k_scan_cells(const uint32_t* __restrict__ cnt, uint64_t cells,
                                                     uint32_t* __restrict__ dir, uint32_t* __restrict__ cursor) {
    using BlockScan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ uint32_t carry_s;
    const uint32_t t = blockIdx.x;
    const uint32_t* c = cnt + uint64_t(t) * (cells + 1);
    uint32_t* d = dir + uint64_t(t) * (cells + 1);
    uint32_t* u = cursor + uint64_t(t) * (cells + 1);
    uint32_t carry = 0;
    constexpr int IPT = 4;
    for (uint64_t base = 0; base < cells + 1; base += 1024 * IPT) {
        uint32_t v[IPT];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const uint64_t i = base + threadIdx.x * IPT + k;
            v[k] = i < cells + 1 ? c[i] : 0u;
        }
        uint32_t agg;
        BlockScan(tmp).ExclusiveSum(v, v, agg);
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const uint64_t i = base + threadIdx.x * IPT + k;
            if (i < cells + 1) {
                d[i] = v[k] + carry;
                u[i] = v[k] + carry;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + agg;
        __syncthreads();
        carry = carry_s;
    }
}

template <typename T, typename K>
__global__ void k_scatter(const K* __restrict__ keys, uint64_t n, uint32_t L, uint32_t t0, uint32_t c, uint32_t shift,
                          uint64_t kscale, uint64_t cells, uint32_t* __restrict__ cursor, typename T::E* __restrict__ entries) {
    const uint64_t total = n * c;
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < total; x += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = x / c;
        const uint32_t t = uint32_t(x % c);
        const uint64_t key = keys[i * L + t0 + t];
        const uint32_t pos = atomicAdd(cursor + uint64_t(t) * (cells + 1) + home_of(key, kscale, shift), 1u);
        entries[uint64_t(t) * n + pos] = T::make(key, uint32_t(i));
    }
}

constexpr uint32_t kSmallCell = 16;

// Thread per cell: insertion-sort cells up to kSmallCell entries; longer
// cells are queued for k_sort_big.
template <typename T>
__global__ void k_sort_cells(const uint32_t* __restrict__ dir, uint64_t cells, uint64_t n, uint32_t tables,
                             typename T::E* __restrict__ entries, uint2* __restrict__ big,
                             unsigned int* __restrict__ big_count) {
    using E = typename T::E;
    const uint64_t total = uint64_t(tables) * cells;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t t = uint32_t(i / cells);
        const uint64_t c = i % cells;
        const uint32_t* d = dir + uint64_t(t) * (cells + 1);
        const uint32_t b = d[c], e = d[c + 1];
        const uint32_t len = e - b;
        if (len <= 1) continue;
        if (len > kSmallCell) {
            const unsigned int slot = atomicAdd(big_count, 1u);
            big[slot] = make_uint2(t, uint32_t(c));
            continue;
        }
        E* p = entries + uint64_t(t) * n + b;
        E v[kSmallCell];
#pragma unroll
        for (uint32_t k = 0; k < kSmallCell; ++k)
            if (k < len) v[k] = p[k];
        for (uint32_t k = 1; k < len; ++k) {
            E x = v[k];
            int j = int(k) - 1;
            while (j >= 0 && T::less(x, v[j])) {
                v[j + 1] = v[j];
                --j;
            }
            v[j + 1] = x;
        }
#pragma unroll
        for (uint32_t k = 0; k < kSmallCell; ++k)
            if (k < len) p[k] = v[k];
    }
}

// Ascending-only bitonic network (every compare puts the min at the lower
// index), so positions >= len behave as +inf padding and are never touched.
template <typename T, typename Ptr>
__device__ void bitonic_sort(Ptr a, uint32_t len, uint32_t pow2) {
    for (uint32_t k = 2; k <= pow2; k <<= 1) {
        for (uint32_t i = threadIdx.x; i < pow2 / 2; i += blockDim.x) { // flip step
            const uint32_t blk = i / (k / 2), off = i % (k / 2);
            const uint32_t lo = blk * k + off, hi = blk * k + (k - 1 - off);
            if (hi < len && T::less(a[hi], a[lo])) {
                auto tmp = a[lo];
                a[lo] = a[hi];
                a[hi] = tmp;
            }
        }
        __syncthreads();
        for (uint32_t j = k / 4; j > 0; j >>= 1) { // half cleaners
            for (uint32_t i = threadIdx.x; i < pow2 / 2; i += blockDim.x) {
                const uint32_t blk = i / j, off = i % j;
                const uint32_t lo = blk * 2 * j + off, hi = lo + j;
                if (hi < len && T::less(a[hi], a[lo])) {
                    auto tmp = a[lo];
                    a[lo] = a[hi];
                    a[hi] = tmp;
                }
            }
            __syncthreads();
        }
    }
}

// 4-byte global -> shared copies in flight without registers (cp.async)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_ix() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all_ix() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T>
__global__ void __launch_bounds__(512) k_sort_big(const uint32_t* __restrict__ dir, uint64_t cells, uint64_t n,
                                                  typename T::E* __restrict__ entries, const uint2* __restrict__ big,
                                                  uint32_t cap) {
    using E = typename T::E;
    extern __shared__ __align__(16) unsigned char smem[];
    E* s = reinterpret_cast<E*>(smem);
    const uint2 bc = big[blockIdx.x];
    const uint32_t* d = dir + uint64_t(bc.x) * (cells + 1);
    const uint32_t b = d[bc.y], len = d[bc.y + 1] - b;
    E* p = entries + uint64_t(bc.x) * n + b;
    uint32_t pow2 = 1;
    while (pow2 < len) pow2 <<= 1;
    if (len <= cap) {
        for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) s[i] = p[i];
        __syncthreads();
        bitonic_sort<T>(s, len, pow2);
        for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) p[i] = s[i];
    } else {
        bitonic_sort<T>(p, len, pow2); // in global memory (very long cells only)
    }
}

// ----------------------------------------------------------------- query

// the run of bucketed table t from bucket b on (b, b+1, ... until a bucket
// with a free last slot): push every id whose key matches
template <typename T, typename F>
__device__ __forceinline__ void probe_run(const Tables<T>& tb, uint32_t t, uint64_t b, typename T::K key, F&& push) {
    using E = typename T::E;
    const E* base = tb.data + uint64_t(t) * tb.nbuckets * kSlots;
    for (;;) {
        E x[kSlots];
        load_bucket(base + b * kSlots, x);
#pragma unroll
        for (int j = 0; j < kSlots; ++j)
            if (!T::empty(x[j]) && T::key(x[j]) == key) push(T::id(x[j]));
        if (T::empty(x[kSlots - 1])) break;
        b = (b + 1) & (tb.nbuckets - 1);
    }
}

// K3+K4+K5 fused, one warp per query (the common path). Lanes probe tables
// lane, lane+32, ... (U in flight); every colliding id goes into a per-warp
// shared-memory open-addressing set of WS slots, so only distinct candidates
// are kept (cfg2: ~1.1 distinct of ~103 collisions) and no collision list is
// sorted. Lanes then verify the set's ids, the found (id, dist) pairs are
// sorted in registers (at most 32, one per lane) and written to the query's
// slots. The small footprint (WS ids per warp) leaves most of the unified
// L1/shared array to L1, which holds the lines of the probes in flight. A
// query with more than 3/4 * WS distinct candidates or more than slot_cap
// results is handed to the CTA kernel (overflow list), which then writes all
// of that query's outputs.
template <typename T, int LAYOUT, int WS, int U>
__global__ void __launch_bounds__(256) k_query_fused(
    const typename T::K* __restrict__ qkeys, uint64_t nq, uint32_t tables, const Tables<T> tb,
    const uint64_t* __restrict__ rows, const uint64_t* __restrict__ qrows, uint32_t words, uint32_t radius,
    uint32_t slot_cap, unsigned long long* __restrict__ coll_q, unsigned long long* __restrict__ cand_q,
    unsigned long long* __restrict__ found_q, unsigned long long* __restrict__ src_pos, uint32_t* __restrict__ tmp_id,
    uint32_t* __restrict__ tmp_dist, uint32_t* __restrict__ overflow, unsigned int* __restrict__ overflow_count,
    unsigned int* __restrict__ qnext, unsigned long long* __restrict__ tile_sum,
    const unsigned long long* __restrict__ desc) {
    using E = typename T::E;
    // host destination of the counters (HostDest, null: device only), written as each query completes
    static_assert((WS & (WS - 1)) == 0 && WS >= 128 && WS % 32 == 0, "set size");
    constexpr uint32_t kEmpty = 0xFFFFFFFFu;
    constexpr uint32_t kMaxD = WS / 4 * 3; // distinct ids a query may have here (set load <= 3/4 + 32)
    constexpr int kLogWS = __builtin_ctz(WS);
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned int* dcnt_s = reinterpret_cast<unsigned int*>(smem); // [8] distinct ids per warp
    uint32_t* set = reinterpret_cast<uint32_t*>(smem) + 8 + warp * WS;
    for (int k = lane; k < WS; k += 32) set[k] = kEmpty; // afterwards cleared as it is read
    pdl_trigger();
    pdl_wait(); // the batch's keys (hash kernel) are complete from here on
    // the host destination (written by the batch prologue, a PDL predecessor:
    // read only after the wait)
    unsigned long long* const hc = desc ? reinterpret_cast<unsigned long long*>(desc[0]) : nullptr;
    // queries are handed out one at a time (a warp that finishes early takes
    // the next), so the last wave does not leave most warps idle
    auto fetch = [&]() -> uint64_t {
        unsigned int v = 0;
        if (lane == 0) v = atomicAdd(qnext, 1u);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    for (uint64_t q = fetch(); q < nq; q = fetch()) {
        if (lane == 0) dcnt_s[warp] = 0;
        __syncwarp();
        const typename T::K* qk = qkeys + q * tables;
        uint32_t coll = 0; // this lane's postings
        auto push = [&](uint32_t id) {
            ++coll;
            if (dcnt_s[warp] >= kMaxD) return; // overflowing: only the count matters now
            uint32_t h = (id * 0x9E3779B1u) >> (32 - kLogWS);
            for (;;) {
                const uint32_t old = atomicCAS(set + h, kEmpty, id);
                if (old == id) return; // seen
                if (old == kEmpty) break;
                h = (h + 1) & (WS - 1);
            }
            atomicAdd(dcnt_s + warp, 1u);
        };
        for (uint32_t t0 = 0; t0 < tables; t0 += 32 * U) {
            uint64_t key[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t t = t0 + u * 32 + lane;
                key[u] = t < tables ? uint64_t(qk[t]) : 0ull;
            }
            if constexpr (LAYOUT == kLayoutCsr) {
                uint32_t s[U], e[U];
#pragma unroll
                for (int u = 0; u < U; ++u) { // U directory lookups in flight
                    const uint32_t t = t0 + u * 32 + lane;
                    if (t < tables) {
                        const uint32_t* d = tb.dir + uint64_t(t) * (tb.cells + 1) + home_of(key[u], tb);
                        s[u] = __ldg(d);
                        e[u] = __ldg(d + 1);
                    } else {
                        s[u] = e[u] = 0;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const E* et = tb.data + uint64_t(t0 + u * 32 + lane) * tb.n;
                    uint32_t a = s[u];
                    a = cell_lower_bound<T>(et, a, e[u], key[u]);
                    while (a < e[u] && T::key(et[a]) == key[u]) push(T::id(et[a++]));
                }
            } else {
                E sl[U][kSlots];
#pragma unroll
                for (int u = 0; u < U; ++u) { // U home buckets in flight
                    const uint32_t t = t0 + u * 32 + lane;
                    if (t < tables)
                        load_bucket(tb.data + (uint64_t(t) * tb.nbuckets + home_of(key[u], tb)) * kSlots, sl[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t t = t0 + u * 32 + lane;
                    if (t >= tables) continue;
#pragma unroll
                    for (int j = 0; j < kSlots; ++j)
                        if (!T::empty(sl[u][j]) && T::key(sl[u][j]) == key[u]) push(T::id(sl[u][j]));
                    if (!T::empty(sl[u][kSlots - 1])) // the run continues into the next bucket (~3 %)
                        probe_run<T>(tb, t, (home_of(key[u], tb) + 1) & (tb.nbuckets - 1), key[u], push);
                }
            }
            __syncwarp();
            // too many distinct ids: the CTA kernel redoes it (a vote keeps the exit warp-uniform)
            if (__any_sync(0xffffffffu, dcnt_s[warp] >= kMaxD)) break;
        }
        __syncwarp();
        const uint32_t nd = __shfl_sync(0xffffffffu, dcnt_s[warp], 0);
        const uint64_t m = __reduce_add_sync(0xffffffffu, coll);
        // verify the distinct ids (clearing the set behind), collect passes in slot order
        const uint64_t* qr = qrows + q * words;
        uint32_t nfound = 0;
        unsigned long long mine = ~0ull; // this lane's found (id << 32 | dist), kept for the sort
#pragma unroll 1
        for (int k0 = 0; k0 < WS; k0 += 32) {
            const uint32_t id = set[k0 + lane];
            const bool valid = id != kEmpty;
            if (valid) set[k0 + lane] = kEmpty;
            uint32_t dist = 0;
            if (valid && nd < kMaxD) {
                const uint64_t* r = rows + uint64_t(id) * words;
                for (uint32_t w = 0; w < words; ++w) dist += __popcll(__ldg(r + w) ^ __ldg(qr + w));
            }
            const bool pass = valid && nd < kMaxD && dist <= radius;
            const uint32_t bp = __ballot_sync(0xffffffffu, pass);
            if (bp) {
                // the pass of rank i among this query's passes goes to lane i
                const uint32_t pos = nfound + __popc(bp & ((1u << lane) - 1u));
                const unsigned long long e = (static_cast<unsigned long long>(id) << 32) | dist;
                for (uint32_t b = bp; b; b &= b - 1) {
                    const int src = __ffs(b) - 1;
                    const unsigned long long v = __shfl_sync(0xffffffffu, e, src);
                    const uint32_t p = __shfl_sync(0xffffffffu, pos, src);
                    if (p == uint32_t(lane)) mine = v;
                }
                nfound += __popc(bp);
            }
        }
        if (nd >= kMaxD || nfound > slot_cap || nfound > 32) {
            if (lane == 0) {
                const unsigned int at = atomicAdd(overflow_count, 1u);
                FCLSH_DCHECK(at < nq);
                overflow[at] = uint32_t(q);
                found_q[q] = 0; // written by the CTA kernel later
                src_pos[q] = 0;
            }
            continue;
        }
        // ascending ids: bitonic sort across the warp (one entry per lane, padding = +inf)
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, mine, j);
                const bool up = (lane & k) == 0;
                const bool lower = (lane & j) == 0;
                const unsigned long long lo = mine < other ? mine : other, hi = mine < other ? other : mine;
                mine = (lower == up) ? lo : hi;
            }
        }
        if (uint32_t(lane) < nfound) {
            FCLSH_DCHECK(q < nq && uint32_t(lane) < slot_cap);
            tmp_id[q * slot_cap + lane] = uint32_t(mine >> 32);
            tmp_dist[q * slot_cap + lane] = uint32_t(mine);
        }
        if (lane == 0) {
            coll_q[q] = m;
            cand_q[q] = nd;
            found_q[q] = nfound;
            if (hc) {
                hc[(nq + 1) + q] = m;
                hc[2 * (nq + 1) + q] = nd;
                hc[3 * (nq + 1) + q] = nfound;
            }
            src_pos[q] = q * slot_cap;
            if (nfound) atomicAdd(tile_sum + (q >> kScanTileLog), (unsigned long long)nfound);
        }
    }
}

// K3+K4+K5 fused, one warp per query, without shared memory: the distinct
// ids live in registers across the warp (lane k holds the k-th distinct id),
// so the whole unified L1/shared array is L1 for the lines of the probes in
// flight (rand_bench: any shared-memory carveout lowers the random-read rate
// by ~12 %). Collisions are offered to the list in warp-uniform steps, each
// lane offering at most one id per step: an offered id is compared with the
// nd listed ids (broadcast by shuffles), ids new to the list are deduplicated
// among the lanes with a match-any, and the lowest lane of each group appends
// it. Every offered id is a collision, every append a candidate (the
// reference's counters). More than 32 distinct ids or more than slot_cap
// results: the query is handed to the CTA kernel, which recomputes all of its
// outputs. The found (id << 32 | dist) are one per lane, sorted by a shuffle
// bitonic network with ~0 padding.
#ifndef FCLSH_WARP_MINB
#define FCLSH_WARP_MINB 6
#endif
template <typename T, int LAYOUT, int U>
__global__ void __launch_bounds__(256, FCLSH_WARP_MINB) k_query_warp(
    const typename T::K* __restrict__ qkeys, uint64_t nq, uint32_t tables, const Tables<T> tb,
    const uint64_t* __restrict__ rows, const uint64_t* __restrict__ qrows, uint32_t words, uint32_t radius,
    uint32_t slot_cap, unsigned long long* __restrict__ coll_q, unsigned long long* __restrict__ cand_q,
    unsigned long long* __restrict__ found_q, unsigned long long* __restrict__ src_pos, uint32_t* __restrict__ tmp_id,
    uint32_t* __restrict__ tmp_dist, uint32_t* __restrict__ overflow, unsigned int* __restrict__ overflow_count,
    unsigned int* __restrict__ qnext, unsigned long long* __restrict__ tile_sum,
    const unsigned long long* __restrict__ desc) {
    using E = typename T::E;
    constexpr unsigned kAll = 0xffffffffu;
    constexpr uint32_t kEmpty = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const uint64_t fpol = l2_evict_last_policy();
    const uint64_t bpol = l2_evict_first_policy();
    pdl_trigger();
    pdl_wait(); // the batch's keys (hash kernel) are complete from here on
    // the host destination (written by the batch prologue, a PDL predecessor:
    // read only after the wait)
    unsigned long long* const hc = desc ? reinterpret_cast<unsigned long long*>(desc[0]) : nullptr;
    auto fetch = [&]() -> uint64_t {
        unsigned int v = 0;
        if (lane == 0) v = atomicAdd(qnext, 1u);
        return __shfl_sync(kAll, v, 0);
    };
    for (uint64_t q = fetch(); q < nq; q = fetch()) {
        const typename T::K* qk = qkeys + q * tables;
        uint32_t list = kEmpty; // this lane's distinct id (lane < nd)
        uint32_t nd = 0;        // distinct ids so far (warp-uniform)
        bool over = false;      // more than 32 distinct ids (warp-uniform)
        uint32_t coll = 0;      // this lane's postings
        // one warp-uniform step: each lane offers at most one colliding id
        auto offer = [&](bool has, uint32_t id) {
            coll += has;
            if (!__any_sync(kAll, has) || over) return;
            bool seen = false;
            for (uint32_t k = 0; k < nd; ++k) seen |= __shfl_sync(kAll, list, k) == id;
            const bool fresh = has && !seen;
            const uint32_t grp = __match_any_sync(kAll, fresh ? id : kEmpty);
            const uint32_t lead = __ballot_sync(kAll, fresh && __ffs(grp) - 1 == lane);
            if (!lead) return;
            if (nd + __popc(lead) > 32) {
                over = true;
                return;
            }
            for (uint32_t b = lead; b; b &= b - 1) {
                const uint32_t v = __shfl_sync(kAll, id, __ffs(b) - 1);
                if (uint32_t(lane) == nd) list = v;
                ++nd;
            }
        };
        for (uint32_t t0 = 0; t0 < tables && !over; t0 += 32 * U) {
            uint64_t key[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t t = t0 + u * 32 + lane;
                key[u] = t < tables ? uint64_t(qk[t]) : 0ull;
            }
            if constexpr (LAYOUT == kLayoutCsr) {
                uint32_t s[U], e[U];
#pragma unroll
                for (int u = 0; u < U; ++u) { // U directory lookups in flight
                    const uint32_t t = t0 + u * 32 + lane;
                    if (t < tables) {
                        const uint32_t* d = tb.dir + uint64_t(t) * (tb.cells + 1) + home_of(key[u], tb);
                        s[u] = __ldg(d);
                        e[u] = __ldg(d + 1);
                    } else {
                        s[u] = e[u] = 0;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const E* et = tb.data + uint64_t(t0 + u * 32 + lane) * tb.n;
                    uint32_t a = cell_lower_bound<T>(et, s[u], e[u], key[u]);
                    bool has = a < e[u] && T::key(et[a]) == key[u];
                    while (__any_sync(kAll, has)) {
                        offer(has, has ? T::id(et[a]) : 0u);
                        if (has) {
                            ++a;
                            has = a < e[u] && T::key(et[a]) == key[u];
                        }
                    }
                }
            } else {
                bool pass[U];
#pragma unroll
                for (int u = 0; u < U; ++u) pass[u] = t0 + u * 32 + lane < tables;
                if (tb.filter) { // a clear filter bit: no posting has this key, no bucket read
#pragma unroll
                    for (int u = 0; u < U; ++u) pass[u] = pass[u] && filter_pass(tb, t0 + u * 32 + lane, key[u], fpol);
                }
                E sl[U][kSlots];
#pragma unroll
                for (int u = 0; u < U; ++u) { // U home buckets in flight
                    const uint32_t t = t0 + u * 32 + lane;
                    if (pass[u]) {
                        load_bucket_probe(tb.data + (uint64_t(t) * tb.nbuckets + home_of(key[u], tb)) * kSlots, sl[u],
                                          bpol);
                    } else {
#pragma unroll
                        for (int j = 0; j < kSlots; ++j) sl[u][j] = T::make(~0ull, ~0u);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool live = pass[u];
#pragma unroll
                    for (int j = 0; j < kSlots; ++j)
                        offer(live && !T::empty(sl[u][j]) && T::key(sl[u][j]) == key[u], T::id(sl[u][j]));
                    // the run continues into the next bucket (~3 %)
                    bool cont = live && !T::empty(sl[u][kSlots - 1]);
                    uint64_t b = home_of(key[u], tb) + 1;
                    const E* base = tb.data + uint64_t(t0 + u * 32 + lane) * tb.nbuckets * kSlots;
                    while (__any_sync(kAll, cont)) {
                        E x[kSlots];
#pragma unroll
                        for (int j = 0; j < kSlots; ++j) x[j] = T::make(~0ull, ~0u);
                        b &= tb.nbuckets - 1;
                        if (cont) load_bucket(base + b * kSlots, x);
#pragma unroll
                        for (int j = 0; j < kSlots; ++j)
                            offer(cont && !T::empty(x[j]) && T::key(x[j]) == key[u], T::id(x[j]));
                        cont = cont && !T::empty(x[kSlots - 1]);
                        ++b;
                    }
                }
            }
        }
        const uint64_t m = __reduce_add_sync(kAll, coll);
        // verify the listed ids, one per lane
        uint32_t dist = 0;
        if (!over && uint32_t(lane) < nd) {
            const uint64_t* r = rows + uint64_t(list) * words;
            const uint64_t* qr = qrows + q * words;
            for (uint32_t w = 0; w < words; ++w) dist += __popcll(__ldg(r + w) ^ __ldg(qr + w));
        }
        const bool pass = !over && uint32_t(lane) < nd && dist <= radius;
        const uint32_t nfound = __popc(__ballot_sync(kAll, pass));
        if (over || nfound > slot_cap) {
            if (lane == 0) {
                const unsigned int at = atomicAdd(overflow_count, 1u);
                FCLSH_DCHECK(at < nq);
                overflow[at] = uint32_t(q);
                found_q[q] = 0; // written by the CTA kernel later
                src_pos[q] = 0;
            }
            continue;
        }
        // ascending ids: bitonic sort across the warp (non-passes = +inf)
        unsigned long long mine = pass ? (static_cast<unsigned long long>(list) << 32) | dist : ~0ull;
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const unsigned long long other = __shfl_xor_sync(kAll, mine, j);
                const bool up = (lane & k) == 0;
                const bool lower = (lane & j) == 0;
                const unsigned long long lo = mine < other ? mine : other, hi = mine < other ? other : mine;
                mine = (lower == up) ? lo : hi;
            }
        }
        if (uint32_t(lane) < nfound) {
            FCLSH_DCHECK(q < nq && uint32_t(lane) < slot_cap);
            tmp_id[q * slot_cap + lane] = uint32_t(mine >> 32);
            tmp_dist[q * slot_cap + lane] = uint32_t(mine);
        }
        if (lane == 0) {
            coll_q[q] = m;
            cand_q[q] = nd;
            found_q[q] = nfound;
            if (hc) {
                hc[(nq + 1) + q] = m;
                hc[2 * (nq + 1) + q] = nd;
                hc[3 * (nq + 1) + q] = nfound;
            }
            src_pos[q] = q * slot_cap;
            if (nfound) atomicAdd(tile_sum + (q >> kScanTileLog), (unsigned long long)nfound);
        }
    }
}

// Warp per query with the probe rounds software-pipelined (buckets layout;
// the default for indexes of <= 640 tables). k_query_warp walks the tables in
// rounds of 32 x U, and every round is a chain of three dependent memory
// trips: the round's keys, their L2 filter words, then the random bucket
// reads. Here the three stages of consecutive rounds overlap: while round c's
// bucket reads are in flight the warp has already issued round c+1's filter
// words (keys loaded a round earlier) and round c+2's keys, so a round waits
// on its bucket reads only (reference loop replaced: index.cpp:169-177).
// Dedup, counters, verify and outputs are k_query_warp's.
// The covering hash of one query row inside the query kernel (fused: no
// separate hash launch, no grid-wide wait for the batch's keys). Narrow keys
// (prime < 2^32), parts of N = 32 x FE columns. Per part: the sketch
// t[c] = sum of the seeds of the set positions mapped to column c (the
// family's column lists, positions already in source-row bits), an exact
// int64 Walsh-Hadamard transform F over the warp (index bits 5.. in
// registers, bits 0..4 across lanes), and key[v] = (F[0] - F[v]) / 2 mod P
// = sum of the seeds at set positions i with popcount(v & m(i)) odd: the
// reference's h[v] (covering.cpp:150-182, hadamard.cpp:51-72). Keys go to
// the batch's key array (read back by this warp and, for handed-over
// queries, by the other query kernels); the row stays in registers, and
// rows read from mapped host memory are also copied to the device rows.
// FCLSH_TRACE builds (tools/trace_query.py; never the shipped library): the
// warp kernel stamps each query's phases -- globaltimer at start and end,
// SM clocks at the end of the hash, the probes and the verify -- into
// g_trace[q * 16 ..] (8..15: SM clocks at the end of each probe round), which the host appends to $FCLSH_TRACE_OUT per batch.
#ifdef FCLSH_TRACE
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define FCLSH_TRACE_STAMP(q, k, v) \
    do { \
        if (g_trace && lane == 0) g_trace[(q) * 16 + (k)] = (v); \
    } while (0)
// batch timeline (globaltimer, ns): the first / last stamp of each event over
// the batch's CTAs (warps for kTlWarpExit); reset per batch by the host and
// appended to $FCLSH_TL_OUT (tools/trace_query.py)
enum : int {
    kTlProEntry, kTlProExit, kTlWarpEntry, kTlWarpEntryLast, kTlWarpWait, kTlWarpExit, kTlDenseEntry, kTlDenseWait,
    kTlDenseExit, kTlCompEntry, kTlCompWait, kTlCompExit, kTlPublish, kTlCompLoaded, kTlCompScanned, kTlSlots
};
__device__ unsigned long long g_tl[16];
#define FCLSH_TL_MIN(k) \
    do { \
        if (threadIdx.x == 0) atomicMin(&g_tl[k], gtimer()); \
    } while (0)
#define FCLSH_TL_MAX(k) \
    do { \
        if (threadIdx.x == 0) atomicMax(&g_tl[k], gtimer()); \
    } while (0)
#define FCLSH_TL_MAXW(k) \
    do { \
        if ((threadIdx.x & 31) == 0) atomicMax(&g_tl[k], gtimer()); \
    } while (0)
#else
#define FCLSH_TRACE_STAMP(q, k, v) \
    do { \
    } while (0)
#define FCLSH_TL_MIN(k) \
    do { \
    } while (0)
#define FCLSH_TL_MAX(k) FCLSH_TL_MIN(k)
#define FCLSH_TL_MAXW(k) FCLSH_TL_MIN(k)
#endif

struct FusedHash {
    uint32_t parts = 0, N = 0, L = 0;
    uint64_t max_dims = 0;
    const uint32_t* col_ptr = nullptr; // [parts][N+1]
    const uint32_t* ent_pos = nullptr; // [parts][max_dims] source-row bit
    const uint64_t* ent_seed = nullptr;
    const uint64_t* ent_pk = nullptr; // [parts][max_dims] seed << 32 | source bit
    const uint64_t* ent_sk = nullptr; // [parts][max_dims] seed << 32 | column << 16 | source bit (view order)
    uint32_t sk_warp_bytes = 0;       // > 0: position-parallel sketch; per-warp scratch after the family
    uint64_t prime = 0;
    const uint64_t* hash_src = nullptr; // mapped pinned host rows (null: the device rows)
    uint32_t smem_bytes = 0; // > 0: the kernel stages col_ptr and ent_pk in shared memory (this many bytes)
};

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t ld_cg(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// family entries from shared memory (staged per CTA) or through the read-only path
template <bool SMEM>
__device__ __forceinline__ uint32_t fam_ld(const uint32_t* p) {
    if constexpr (SMEM) return *p;
    else return __ldg(p);
}
template <bool SMEM>
__device__ __forceinline__ uint64_t fam_ld(const uint64_t* p) {
    if constexpr (SMEM) return *p;
    else return __ldg(p);
}

// One part's keys in registers: key[i] = h[v] for v = lane + 32 i (v = 0 is
// no table), from the row held as word `lane` on lane `lane` (rw).
// R32 (rows of <= 16 words, d <= 1024): the row is also held as 32-bit half `lane` on lane
// `lane`, so an entry's row bit costs one 32-bit shuffle instead of a 64-bit one (two SHFLs):
// cfg3's probe kernel 90.0 -> 87.0 us (profiles/r02/ab_fused_row32.txt). A compile-time choice:
// the kernel sits at its register cap and a run-time branch here spills.
template <int FE, bool SMEM, bool R32 = false, typename K>
__device__ __forceinline__ void hash_part(const FusedHash& fh, const uint32_t* cp_all, const uint64_t* pk_all,
                                          uint32_t p, uint32_t words, uint64_t rw, int lane, K (&key)[FE]) {
    constexpr unsigned kAll = 0xffffffffu;
    const uint64_t P = fh.prime;
    const uint32_t* cp = cp_all + uint64_t(p) * (fh.N + 1);
    const uint64_t* pk = pk_all + uint64_t(p) * fh.max_dims;
    // the sketch of the lane's FE columns: every column's (seed, bit)
    // entries are loaded kBatch at a time for all FE columns at once (no
    // load waits on another: two L2 round trips per batch of kBatch * FE
    // entries instead of one per entry); a missing entry loads as 0 = seed 0
    constexpr int kBatch = 4;
    uint32_t b0[FE], cnt[FE], mx = 0;
    long long t[FE];
#pragma unroll
    for (int i = 0; i < FE; ++i) {
        const uint32_t c = uint32_t(lane) + 32u * i;
        b0[i] = fam_ld<SMEM>(cp + c);
        cnt[i] = fam_ld<SMEM>(cp + c + 1) - b0[i];
        mx = max(mx, cnt[i]);
        t[i] = 0;
    }
    const uint32_t m = __reduce_max_sync(kAll, mx); // warp-uniform trip count (the shuffles need every lane)
    uint32_t rh = 0;
    if constexpr (R32) rh = uint32_t(__shfl_sync(kAll, rw, lane >> 1) >> ((lane & 1) * 32));
    for (uint32_t k0 = 0; k0 < m; k0 += kBatch) {
        uint64_t e[FE][kBatch];
#pragma unroll
        for (int i = 0; i < FE; ++i)
#pragma unroll
            for (int k = 0; k < kBatch; ++k) e[i][k] = k0 + k < cnt[i] ? fam_ld<SMEM>(pk + b0[i] + k0 + k) : 0ull;
#pragma unroll
        for (int i = 0; i < FE; ++i)
#pragma unroll
            for (int k = 0; k < kBatch; ++k) {
                const uint32_t pos = uint32_t(e[i][k]);
                FCLSH_DCHECK((pos >> 6) < words && b0[i] + cnt[i] <= fh.max_dims);
                uint32_t w; // the 32-bit half of the row that holds bit `pos`
                if constexpr (R32) {
                    w = __shfl_sync(kAll, rh, int(pos >> 5));
                } else {
                    const uint64_t w64 = __shfl_sync(kAll, rw, int(pos >> 6));
                    w = uint32_t(w64 >> (pos & 32u));
                }
                if ((w >> (pos & 31)) & 1) t[i] += (long long)(e[i][k] >> 32);
            }
    }
#pragma unroll
    for (int h = 1; h < FE; h <<= 1) { // index bits 5.. : within the lane
#pragma unroll
        for (int i = 0; i < FE; ++i)
            if (!(i & h)) {
                const long long x = t[i], y = t[i | h];
                t[i] = x + y;
                t[i | h] = x - y;
            }
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { // index bits 0..4: across lanes
#pragma unroll
        for (int i = 0; i < FE; ++i) {
            const long long other = __shfl_xor_sync(kAll, t[i], o);
            t[i] = (lane & o) ? other - t[i] : t[i] + other;
        }
    }
    const long long l1 = __shfl_sync(kAll, t[0], 0); // F[0] = sum of the sketch
#pragma unroll
    for (int i = 0; i < FE; ++i) {
        uint64_t x = uint64_t(l1 - t[i]) >> 1;
        if (P == 0x7FFFFFFFull) {
            x = (x & P) + (x >> 31);
            x = (x & P) + (x >> 31);
            x = x >= P ? x - P : x;
        } else {
            x %= P;
        }
        key[i] = K(x);
    }
}

// hash_part with a position-parallel sketch: lane k takes view positions k,
// k + 32, ... of the part (entries seed << 32 | column << 16 | source bit,
// staged in shared memory), tests its row bit (the row staged in this warp's
// shared scratch) and adds the seed's two 16-bit halves to the column's two
// 32-bit shared accumulators (RED.ADD on shared memory: integer, so the
// order does not matter). ceil(d'/32) entries per lane instead of FE x the
// longest column list (cfg3: 8 against 32 entry slots per part and lane).
template <int FE, typename K>
__device__ __forceinline__ void hash_part_sk(const FusedHash& fh, const uint64_t* sk_all, uint32_t p,
                                             const uint32_t* row_s, uint32_t* acc, int lane, K (&key)[FE]) {
    constexpr unsigned kAll = 0xffffffffu;
    constexpr uint32_t N = 32u * FE;
    const uint64_t P = fh.prime;
    uint32_t* lo = acc;
    uint32_t* hi = acc + N;
#pragma unroll
    for (int i = 0; i < 2 * FE; ++i) acc[lane + 32 * i] = 0;
    __syncwarp();
    const uint64_t* e = sk_all + uint64_t(p) * fh.max_dims;
    const uint32_t nent = uint32_t(fh.max_dims);
#pragma unroll 4
    for (uint32_t k = lane; k < nent; k += 32) {
        const uint64_t x = e[k];
        const uint32_t pos = uint32_t(x) & 0xFFFFu, col = uint32_t(x) >> 16;
        FCLSH_DCHECK(col < N);
        if ((row_s[pos >> 5] >> (pos & 31)) & 1u) {
            const uint32_t sd = uint32_t(x >> 32);
            atomicAdd(lo + col, sd & 0xFFFFu);
            atomicAdd(hi + col, sd >> 16);
        }
    }
    __syncwarp();
    long long t[FE];
#pragma unroll
    for (int i = 0; i < FE; ++i) {
        const uint32_t c = uint32_t(lane) + 32u * i;
        t[i] = (long long)lo[c] + ((long long)hi[c] << 16);
    }
#pragma unroll
    for (int h = 1; h < FE; h <<= 1) { // index bits 5.. : within the lane
#pragma unroll
        for (int i = 0; i < FE; ++i)
            if (!(i & h)) {
                const long long x = t[i], y = t[i | h];
                t[i] = x + y;
                t[i | h] = x - y;
            }
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { // index bits 0..4: across lanes
#pragma unroll
        for (int i = 0; i < FE; ++i) {
            const long long other = __shfl_xor_sync(kAll, t[i], o);
            t[i] = (lane & o) ? other - t[i] : t[i] + other;
        }
    }
    const long long l1 = __shfl_sync(kAll, t[0], 0); // F[0] = sum of the sketch
#pragma unroll
    for (int i = 0; i < FE; ++i) {
        uint64_t x = uint64_t(l1 - t[i]) >> 1;
        if (P == 0x7FFFFFFFull) {
            x = (x & P) + (x >> 31);
            x = (x & P) + (x >> 31);
            x = x >= P ? x - P : x;
        } else {
            x %= P;
        }
        key[i] = K(x);
    }
}

// the query row into registers (word `lane` on lane `lane`); rows in mapped
// host memory are also copied to the device rows
__device__ __forceinline__ uint64_t fused_row(const FusedHash& fh, uint64_t q, uint32_t words,
                                              const uint64_t* qrows, int lane) {
    const uint64_t* src = (fh.hash_src ? fh.hash_src : qrows) + q * words;
    uint64_t rw = 0;
    if (uint32_t(lane) < words) {
        rw = src[lane];
        if (fh.hash_src) const_cast<uint64_t*>(qrows)[q * words + lane] = rw;
    }
    return rw;
}

template <int FE, bool SMEM, bool SK, bool R32 = false, typename K>
__device__ __forceinline__ void fused_hash(const FusedHash& fh, const uint32_t* cp_all, const uint64_t* pk_all,
                                           uint64_t q, uint32_t words, const uint64_t* qrows, K* keys, int lane,
                                           uint64_t& rw, uint64_t* row_s, uint32_t* acc) {
    rw = fused_row(fh, q, words, qrows, lane);
    if constexpr (SK) {
        if (uint32_t(lane) < words) row_s[lane] = rw;
        __syncwarp();
    }
    for (uint32_t p = 0; p < fh.parts; ++p) {
        K key[FE];
        if constexpr (SK)
            hash_part_sk<FE>(fh, pk_all, p, reinterpret_cast<const uint32_t*>(row_s), acc, lane, key);
        else
            hash_part<FE, SMEM, R32>(fh, cp_all, pk_all, p, words, rw, lane, key);
        K* kp = keys + uint64_t(p) * fh.L;
#pragma unroll
        for (int i = 0; i < FE; ++i) {
            const uint32_t v = uint32_t(lane) + 32u * i;
            if (v) kp[v - 1] = key[i];
        }
    }
}

// PM (with FE > 0): part-major -- a part's keys are hashed into registers
// and its tables probed straight from them (lane `lane` of round (p, i) probes
// the table of v = lane + 32 i), so the keys make no global round trip before
// the probes, and part p's probes are in flight before part p+1 is hashed;
// the keys are also stored for the hand-over kernels.
// SK (with FSM): the position-parallel sketch (hash_part_sk); the family's
// entries and every warp's row + column accumulators in shared memory.
template <typename T, int U, int MINB, int FE, bool FSM = false, bool PM = false, bool SK = false, bool R32 = false>
__global__ void __launch_bounds__(256, MINB) k_query_warp_pf(
    typename T::K* qkeys, uint64_t nq, uint32_t tables, const Tables<T> tb,
    const uint64_t* __restrict__ rows, const uint64_t* __restrict__ qrows, uint32_t words, uint32_t radius,
    uint32_t slot_cap, unsigned long long* __restrict__ coll_q, unsigned long long* __restrict__ cand_q,
    unsigned long long* __restrict__ found_q, unsigned long long* __restrict__ src_pos, uint32_t* __restrict__ tmp_id,
    uint32_t* __restrict__ tmp_dist, uint32_t* __restrict__ overflow, unsigned int* __restrict__ overflow_count,
    unsigned int* __restrict__ qnext, unsigned long long* __restrict__ tile_sum,
    const unsigned long long* __restrict__ desc, int vec_rows, const FusedHash fh) {
    using E = typename T::E;
    using K = typename T::K;
    constexpr unsigned kAll = 0xffffffffu;
    constexpr uint32_t kEmpty = 0xFFFFFFFFu;
    constexpr uint32_t kStep = 32 * U; // tables per round
    const int lane = threadIdx.x & 31;
    const uint64_t fpol = l2_evict_last_policy();
    const uint64_t bpol = l2_evict_first_policy();
    pdl_trigger();
    FCLSH_TL_MIN(kTlWarpEntry);
    FCLSH_TL_MAX(kTlWarpEntryLast);
    // FE > 0 with fh.smem_bytes: the family's column lists (read by every
    // query's hash) staged once per CTA, so a query's hash waits on no global
    // load but its row's
    extern __shared__ __align__(16) unsigned char fam_smem[];
    const uint32_t* cp_all = fh.col_ptr;
    const uint64_t* pk_all = fh.ent_pk;
    uint64_t* row_s = nullptr; // SK: this warp's row and column accumulators
    uint32_t* acc_s = nullptr;
    if constexpr (FE > 0 && FSM && SK) {
        uint64_t* sk_s = reinterpret_cast<uint64_t*>(fam_smem);
        const uint32_t nsk = fh.parts * uint32_t(fh.max_dims);
        for (uint32_t i = threadIdx.x; i < nsk; i += blockDim.x) sk_s[i] = __ldg(fh.ent_sk + i);
        unsigned char* wbase = fam_smem + size_t(nsk) * 8 + size_t(threadIdx.x >> 5) * fh.sk_warp_bytes;
        acc_s = reinterpret_cast<uint32_t*>(wbase);
        row_s = reinterpret_cast<uint64_t*>(wbase + size_t(FE) * 32 * 2 * 4);
        __syncthreads();
        pk_all = sk_s;
    } else if constexpr (FE > 0 && FSM) {
        uint64_t* pk_s = reinterpret_cast<uint64_t*>(fam_smem);
        const uint32_t npk = fh.parts * uint32_t(fh.max_dims);
        uint32_t* cp_s = reinterpret_cast<uint32_t*>(pk_s + npk);
        const uint32_t ncp = fh.parts * (fh.N + 1);
        for (uint32_t i = threadIdx.x; i < npk; i += blockDim.x) pk_s[i] = __ldg(fh.ent_pk + i);
        for (uint32_t i = threadIdx.x; i < ncp; i += blockDim.x) cp_s[i] = __ldg(fh.col_ptr + i);
        __syncthreads();
        cp_all = cp_s;
        pk_all = pk_s;
    }
    pdl_wait(); // the batch's keys (hash kernel; FE > 0: this kernel) are complete from here on
    FCLSH_TL_MIN(kTlWarpWait);
    // the host destination (written by the batch prologue, a PDL predecessor:
    // read only after the wait)
    unsigned long long* const hc = desc ? reinterpret_cast<unsigned long long*>(desc[0]) : nullptr;
    // the grid's warps take queries 0 .. warps-1 directly (no atomic storm as
    // every warp starts); later ones come from counter c = CTA % C, which
    // hands out nwarp + c, nwarp + c + C, ... The next query is claimed once
    // the current one's probes are done (the atomic's round trip overlaps its
    // verify and outputs) and read at the top of the loop.
    const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nctr = gridDim.x < kQCtr ? gridDim.x : kQCtr, cj = blockIdx.x % nctr;
    unsigned int* const my_ctr = qnext + cj * kQCtrStride;
    unsigned int claimed = 0; // lane 0: the claimed counter value
    auto claim = [&] {
        if (lane == 0) claimed = atomicAdd(my_ctr, 1u);
    };
    auto next_q = [&]() -> uint64_t {
        return nwarp + cj + uint64_t(nctr) * __shfl_sync(kAll, claimed, 0);
    };
#ifdef FCLSH_TRACE
    const unsigned long long t_entry = gtimer();
#endif
    for (uint64_t q = gwarp; q < nq; q = next_q()) {
        const K* qk = qkeys + q * tables;
        uint64_t rw = 0; // FE > 0: word `lane` of the query row
#ifdef FCLSH_TRACE
        const long long c0 = clock64();
        FCLSH_TRACE_STAMP(q, 0, gtimer());
        FCLSH_TRACE_STAMP(q, 6, t_entry);
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        FCLSH_TRACE_STAMP(q, 5, smid);
#endif
        if constexpr (FE > 0 && !PM) {
            fused_hash<FE, FSM, SK, R32>(fh, cp_all, pk_all, q, words, qrows, qkeys + q * tables, lane, rw, row_s, acc_s);
            __syncwarp(); // the keys (written across lanes) are visible to the loads below
        }
#ifdef FCLSH_TRACE
        FCLSH_TRACE_STAMP(q, 2, clock64() - c0);
#endif
        // FE > 0: the keys were written by this warp a moment ago: coherent
        // L2 loads, not the read-only path
        auto ldk = [&](uint32_t t) -> K {
            if constexpr (FE > 0) return ld_cg(qk + t);
            else return __ldg(qk + t);
        };
        uint32_t list = kEmpty; // this lane's distinct id (lane < nd)
        uint32_t nd = 0;        // distinct ids so far (warp-uniform)
        bool over = false;      // more than 32 distinct ids (warp-uniform)
        uint32_t coll = 0;      // this lane's postings
        // one warp-uniform step: each lane offers at most one colliding id
        // (counted by the caller); ids already listed -- the usual case, the
        // query's near point seen again in table after table -- cost one
        // vote, only new ones the match-any dedup and the append
        auto offer_id = [&](bool has, uint32_t id) {
            if (over) return;
            bool seen = false;
            for (uint32_t k = 0; k < nd; ++k) seen |= __shfl_sync(kAll, list, k) == id;
            const bool fresh = has && !seen;
            if (!__any_sync(kAll, fresh)) return;
            const uint32_t grp = __match_any_sync(kAll, fresh ? id : kEmpty);
            const uint32_t lead = __ballot_sync(kAll, fresh && __ffs(grp) - 1 == lane);
            if (nd + __popc(lead) > 32) {
                over = true;
                return;
            }
            for (uint32_t b = lead; b; b &= b - 1) {
                const uint32_t v = __shfl_sync(kAll, id, __ffs(b) - 1);
                if (uint32_t(lane) == nd) list = v;
                ++nd;
            }
        };
        // the postings of one bucket with this lane's key: a vote when no lane
        // has one (most probes), else one offer step per posting
        auto offer_bucket = [&](const E (&bk)[kSlots], bool live, uint64_t kk) {
            uint32_t mm = 0;
#pragma unroll
            for (int i = 0; i < kSlots; ++i) mm |= uint32_t(T::match(bk[i], kk)) << i;
            mm = live ? mm : 0u;
            coll += __popc(mm);
            while (__any_sync(kAll, mm != 0)) {
                const int i = __ffs(mm) - 1;
                const uint32_t id = i <= 0 ? T::id(bk[0]) : i == 1 ? T::id(bk[1]) : i == 2 ? T::id(bk[2]) : T::id(bk[3]);
                offer_id(mm != 0, id);
                mm &= mm - 1;
            }
        };
        // the run of full buckets after a home bucket whose last slot is taken (~3 %)
        auto probe_run = [&](bool cont, uint64_t kk, uint32_t t) {
            uint64_t b = home_of(kk, tb) + 1;
            const E* base = tb.data + uint64_t(t) * tb.nbuckets * kSlots;
            while (__any_sync(kAll, cont)) {
                E x[kSlots];
#pragma unroll
                for (int j = 0; j < kSlots; ++j) x[j] = T::make(~0ull, ~0u);
                b &= tb.nbuckets - 1;
                if (cont) load_bucket(base + b * kSlots, x);
                offer_bucket(x, cont, kk);
                cont = cont && !T::empty(x[kSlots - 1]);
                ++b;
            }
        };
        if constexpr (FE > 0 && PM) {
            rw = fused_row(fh, q, words, qrows, lane);
            if constexpr (SK) {
                if (uint32_t(lane) < words) row_s[lane] = rw;
                __syncwarp();
            }
            K* const qkw = qkeys + q * tables;
            // every part is hashed and its keys stored even once the query is
            // handed over (> 32 distinct ids): the CTA kernel probes from them
            for (uint32_t p = 0; p < fh.parts; ++p) {
                K key[FE];
                if constexpr (SK)
                    hash_part_sk<FE>(fh, pk_all, p, reinterpret_cast<const uint32_t*>(row_s), acc_s, lane, key);
                else
                    hash_part<FE, FSM>(fh, cp_all, pk_all, p, words, rw, lane, key);
                bool live[FE];
#pragma unroll
                for (int i = 0; i < FE; ++i) {
                    const uint32_t v = uint32_t(lane) + 32u * i, t = p * fh.L + v - 1;
                    if (v) qkw[t] = key[i];
                    live[i] = !over && v != 0 && (!tb.filter || filter_pass(tb, t, uint64_t(key[i]), fpol));
                }
#pragma unroll
                for (int i0 = 0; i0 < FE; i0 += U) {
                    if (over) break;
                    E sl[U][kSlots];
#pragma unroll
                    for (int u = 0; u < U; ++u) { // U home buckets in flight
                        const int i = i0 + u;
                        const uint32_t t = p * fh.L + uint32_t(lane) + 32u * i - 1;
                        if (i < FE && live[i < FE ? i : 0]) {
                            FCLSH_DCHECK(t < tables && home_of(uint64_t(key[i]), tb) < tb.nbuckets);
                            load_bucket_probe(tb.data + (uint64_t(t) * tb.nbuckets + home_of(uint64_t(key[i]), tb)) * kSlots,
                                              sl[u], bpol);
                        } else {
#pragma unroll
                            for (int j = 0; j < kSlots; ++j) sl[u][j] = T::make(~0ull, ~0u);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int i = i0 + u;
                        if (i >= FE) break;
                        const uint64_t kk = uint64_t(key[i]);
                        const bool lv = live[i];
                        offer_bucket(sl[u], lv, kk);
                        probe_run(lv && !T::empty(sl[u][kSlots - 1]), kk, p * fh.L + uint32_t(lane) + 32u * i - 1);
                    }
#ifdef FCLSH_TRACE
                    {
                        const uint32_t r = p * ((FE + U - 1) / U) + i0 / U;
                        if (r < 8) FCLSH_TRACE_STAMP(q, 8 + r, clock64() - c0);
                    }
#endif
                }
            }
        } else {
        // the pipeline: keys of rounds c, c+1, c+2 and the filter result of c+1
        K k0[U], k1[U], k2[U];
        bool p1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t t0 = u * 32 + lane, t1 = kStep + t0;
            k0[u] = t0 < tables ? ldk(t0) : K(0);
            k1[u] = t1 < tables ? ldk(t1) : K(0);
        }
        bool p0[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t t = u * 32 + lane;
            p0[u] = t < tables && (!tb.filter || filter_pass(tb, t, uint64_t(k0[u]), fpol));
        }
        for (uint32_t base_t = 0; base_t < tables && !over; base_t += kStep) {
            E sl[U][kSlots];
#pragma unroll
            for (int u = 0; u < U; ++u) { // round c: U home buckets in flight
                const uint32_t t = base_t + u * 32 + lane;
                if (p0[u]) {
                    FCLSH_DCHECK(t < tables && home_of(uint64_t(k0[u]), tb) < tb.nbuckets);
                    load_bucket_probe(tb.data + (uint64_t(t) * tb.nbuckets + home_of(uint64_t(k0[u]), tb)) * kSlots,
                                      sl[u], bpol);
                } else {
#pragma unroll
                    for (int j = 0; j < kSlots; ++j) sl[u][j] = T::make(~0ull, ~0u);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) { // round c+1: filter words; round c+2: keys
                const uint32_t t1 = base_t + kStep + u * 32 + lane, t2 = t1 + kStep;
                p1[u] = t1 < tables && (!tb.filter || filter_pass(tb, t1, uint64_t(k1[u]), fpol));
                k2[u] = t2 < tables ? ldk(t2) : K(0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t kk = uint64_t(k0[u]);
                const bool live = p0[u];
                offer_bucket(sl[u], live, kk);
                probe_run(live && !T::empty(sl[u][kSlots - 1]), kk, base_t + u * 32 + lane);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                k0[u] = k1[u];
                p0[u] = p1[u];
                k1[u] = k2[u];
            }
#ifdef FCLSH_TRACE
            if (base_t / kStep < 8) FCLSH_TRACE_STAMP(q, 8 + base_t / kStep, clock64() - c0);
#endif
        }
        } // (pipelined rounds)
        const uint64_t m = __reduce_add_sync(kAll, coll);
        claim(); // the warp's next query (read at the top of the loop)
#ifdef FCLSH_TRACE
        FCLSH_TRACE_STAMP(q, 3, clock64() - c0);
#endif
        // verify the listed ids, one per lane
        uint32_t dist = 0;
        if constexpr (FE > 0) { // the query row is in registers (word w on lane w)
            const uint64_t* r = rows + uint64_t(over || uint32_t(lane) >= nd ? 0 : list) * words;
            if (words % 4 == 0) { // 256-bit loads of the candidate row (stored rows are 32-B aligned)
                for (uint32_t w = 0; w < words; w += 4) {
                    unsigned long long a0, a1, a2, a3;
                    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                        : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3)
                        : "l"(r + w));
                    dist += __popcll(a0 ^ __shfl_sync(kAll, rw, w)) + __popcll(a1 ^ __shfl_sync(kAll, rw, w + 1)) +
                            __popcll(a2 ^ __shfl_sync(kAll, rw, w + 2)) + __popcll(a3 ^ __shfl_sync(kAll, rw, w + 3));
                }
            } else {
                for (uint32_t w = 0; w < words; ++w) dist += __popcll(__ldg(r + w) ^ __shfl_sync(kAll, rw, w));
            }
            if (over || uint32_t(lane) >= nd) dist = 0;
        } else if (!over && uint32_t(lane) < nd) {
            dist = row_distance(rows + uint64_t(list) * words, qrows + q * words, words, vec_rows);
        }
        const bool pass = !over && uint32_t(lane) < nd && dist <= radius;
        const uint32_t pass_mask = __ballot_sync(kAll, pass);
        const uint32_t nfound = __popc(pass_mask);
        if (over || nfound > slot_cap) {
            if (lane == 0) {
                const unsigned int at = atomicAdd(overflow_count, 1u);
                FCLSH_DCHECK(at < nq);
                overflow[at] = uint32_t(q);
                found_q[q] = 0; // written by the CTA kernel later
                src_pos[q] = 0;
            }
            continue;
        }
        // ascending ids: bitonic sort across the warp (non-passes = +inf); one
        // result (the usual query: its planted near point) just moves to lane 0
        unsigned long long mine = pass ? (static_cast<unsigned long long>(list) << 32) | dist : ~0ull;
        if (nfound == 1) {
            mine = __shfl_sync(kAll, mine, __ffs(pass_mask) - 1);
        } else if (nfound > 1) {
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    const unsigned long long other = __shfl_xor_sync(kAll, mine, j);
                    const bool up = (lane & k) == 0;
                    const bool lower = (lane & j) == 0;
                    const unsigned long long lo = mine < other ? mine : other, hi = mine < other ? other : mine;
                    mine = (lower == up) ? lo : hi;
                }
            }
        }
        if (uint32_t(lane) < nfound) {
            FCLSH_DCHECK(q < nq && uint32_t(lane) < slot_cap);
            tmp_id[q * slot_cap + lane] = uint32_t(mine >> 32);
            tmp_dist[q * slot_cap + lane] = uint32_t(mine);
        }
        if (lane == 0) {
            coll_q[q] = m;
            cand_q[q] = nd;
            found_q[q] = nfound;
            if (hc) {
                hc[(nq + 1) + q] = m;
                hc[2 * (nq + 1) + q] = nd;
                hc[3 * (nq + 1) + q] = nfound;
            }
            src_pos[q] = q * slot_cap;
            if (nfound) atomicAdd(tile_sum + (q >> kScanTileLog), (unsigned long long)nfound);
        }
#ifdef FCLSH_TRACE
        FCLSH_TRACE_STAMP(q, 4, clock64() - c0);
        FCLSH_TRACE_STAMP(q, 1, gtimer());
        FCLSH_TRACE_STAMP(q, 7, nd);
#endif
    }
    FCLSH_TL_MAXW(kTlWarpExit);
}

// Exclusive prefix sum of v over the CTA's threads (blockDim.x a multiple of
// 32, <= 1024); ws: 32 words of shared scratch; total = the CTA's sum.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* ws, uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= uint32_t(o)) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < nw ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= uint32_t(o)) w += y;
        }
        ws[lane] = w;
    }
    __syncthreads();
    const uint32_t excl = x - v + (wid ? ws[wid - 1] : 0u);
    total = ws[nw - 1];
    __syncthreads(); // ws may be reused
    return excl;
}

constexpr int kFlatTables = 2048; // CSR tables the CTA kernel's flattened probe phase handles
constexpr int kFlatU = 4;         // cell entries per thread in flight there
constexpr size_t kFlatSmem = size_t(kFlatTables + 2) * 4 + size_t(kFlatTables + 2) * 4 + size_t(kFlatTables) * 8 + 16;

// Dense queries (clustered data, cfg4): one CTA per query. Dedup is a
// shared-memory open-addressing id set instead of a sort of the collision
// list, so the cost follows the distinct candidates (cfg4: ~480) rather than
// the collisions (~1900). Phase 1 probes (thread per table), inserts into the
// set and lists the set slot of every new id; phase 2 verifies the listed
// candidates and appends (id << 32 | dist) to a shared found list; only that
// list is sorted (ascending ids, index.cpp:171-186). The set is cleared once
// per CTA and afterwards only at the listed slots. Queries: ovf[0 ..
// *ovf_cnt) (the warp kernel's hand-over, count read on the device), or every
// query 0 .. direct_n when ovf is null, handed out one at a time. A query with
// 3/4 * HS or more distinct candidates or more than FCAP results, or whose
// results do not fit the region, goes to the general path (ovf2), which
// recomputes all its outputs.
template <typename T, int LAYOUT, int HS, int FCAP, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_query_dense(
    const typename T::K* __restrict__ qkeys, uint32_t tables, const Tables<T> tb, const uint64_t* __restrict__ rows,
    const uint64_t* __restrict__ qrows, uint32_t words, uint32_t radius, const uint32_t* __restrict__ ovf,
    const unsigned int* __restrict__ ovf_cnt, uint32_t direct_n, unsigned long long* __restrict__ coll_q,
    unsigned long long* __restrict__ cand_q, unsigned long long* __restrict__ found_q,
    unsigned long long* __restrict__ src_pos, uint64_t src_base, uint32_t* __restrict__ res_id,
    uint32_t* __restrict__ res_dist, uint64_t res_cap, unsigned long long* __restrict__ res_cursor,
    uint32_t* __restrict__ ovf2, unsigned int* __restrict__ ovf2_cnt, unsigned int* __restrict__ qnext,
    unsigned long long* __restrict__ tile_sum, const unsigned long long* __restrict__ desc, uint64_t nq_all,
    uint32_t slot_cap, uint32_t* __restrict__ slot_id, uint32_t* __restrict__ slot_dist, int vec_rows) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* fl = reinterpret_cast<unsigned long long*>(smem); // FCAP found entries
    uint32_t* set = reinterpret_cast<uint32_t*>(fl + FCAP);                // HS ids
    constexpr uint32_t kMaxDistinct = HS / 4 * 3;
    uint16_t* clist = reinterpret_cast<uint16_t*>(set + HS); // set slot of each distinct candidate
    static_assert(HS <= 65536, "slot numbers are 16-bit");
    __shared__ unsigned int coll_s, cand_s, found_s;
    __shared__ volatile int bad_s;
    __shared__ unsigned long long base_s;
    __shared__ uint32_t scan_ws[32];
    constexpr uint32_t kEmpty = 0xFFFFFFFFu;
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    pdl_trigger();
    FCLSH_TL_MIN(kTlDenseEntry);
    pdl_wait(); // the warp kernel's hand-over list is complete from here on
    FCLSH_TL_MIN(kTlDenseWait);
    FCLSH_TL_MAX(kTlDenseExit);
    // the host destination (written by the batch prologue, a PDL predecessor:
    // read only after the wait)
    unsigned long long* const hc = desc ? reinterpret_cast<unsigned long long*>(desc[0]) : nullptr;
    const unsigned int ns = ovf ? *ovf_cnt : direct_n;
    if (blockIdx.x >= ns) return; // at most ns CTAs can get a query (usually ns == 0: nothing handed over)
    __shared__ unsigned int next_s, pf_next_s;
    // CSR, flattened: the next query's keys and directory words are fetched
    // while this query verifies (keys into f_key, cell bounds by cp.async
    // into f_start / f_off), so its directory round trips overlap this one's
    // verify and outputs (FCLSH_DENSE_PF=0 build: off, A/B)
#ifndef FCLSH_DENSE_PF
#define FCLSH_DENSE_PF 1
#endif
    const bool flat_pf = FCLSH_DENSE_PF && LAYOUT == kLayoutCsr && tables <= uint32_t(kFlatTables);
    bool pf_have = false; // this query's directory words were prefetched
    // the flattened CSR phase's per-table arrays (CSR shared memory only)
    uint32_t* const f_off = reinterpret_cast<uint32_t*>(clist + kMaxDistinct + (kMaxDistinct & 1)); // [tables + 1]
    uint32_t* const f_start = f_off + kFlatTables + 1;                                              // [tables]
    uint64_t* const f_key = reinterpret_cast<uint64_t*>(f_start + kFlatTables + (kFlatTables & 1) + 1); // [tables]
    // dynamic hand-out (query costs vary widely on clustered data); the next
    // query is claimed as the current one starts, so the atomic's round trip
    // overlaps the probes
    unsigned int claimed = 0; // thread 0
    auto fetch = [&]() -> uint32_t {
        if (tid == 0) next_s = claimed;
        __syncthreads();
        return next_s; // rewritten only after the body's barriers
    };
    if (tid == 0) claimed = atomicAdd(qnext, 1u);
    // the set is cleared once here and afterwards only where a query wrote
    for (uint32_t i = tid; i < HS; i += nt) set[i] = kEmpty;
    for (uint32_t s_ = fetch(); s_ < ns; s_ = fetch()) {
        const uint64_t q = ovf ? ovf[s_] : s_;
        if (tid == 0) {
            claimed = atomicAdd(qnext, 1u);
            coll_s = cand_s = found_s = 0;
            bad_s = 0;
        }
        __syncthreads();
        // the next query's prefetch (CSR, flattened): its keys, loaded during phase 1
        constexpr int kPf = (kFlatTables + NT - 1) / NT;
        typename T::K pf_key[kPf];
        uint32_t pf_s = 0;
        bool pf = false;
        // phase 1: probe, dedup into the set, list each new id's slot
        const typename T::K* qk = qkeys + q * tables;
        uint32_t coll = 0;
        auto insert = [&](uint32_t id) {
            if (bad_s) return; // the set holds at most kMaxDistinct + nt ids
            uint32_t h = (id * 0x9E3779B1u) >> (32 - __builtin_ctz(HS));
            for (;;) {
                const uint32_t old = atomicCAS(set + h, kEmpty, id);
                if (old == id) return; // seen
                if (old == kEmpty) break;
                h = (h + 1) & (HS - 1);
            }
            const uint32_t pos = atomicAdd(&cand_s, 1u);
            if (pos < kMaxDistinct)
                clist[pos] = uint16_t(h);
            else
                bad_s = 1;
        };
        if constexpr (LAYOUT == kLayoutBuckets && kDenseU > 1) {
            // kDenseU home buckets per thread in flight; a run that spills
            // past a full bucket is read kDenseRun adjacent buckets at a time
            // (clustered data: popular keys fill runs of many buckets, and a
            // bucket-by-bucket walk is a chain of dependent reads)
            using E = typename T::E;
            for (uint32_t t0 = tid; t0 < tables; t0 += kDenseU * nt) {
                if (bad_s) break;
                E sl[kDenseU][kSlots];
                uint64_t key[kDenseU];
                bool pass[kDenseU];
#pragma unroll
                for (int u = 0; u < kDenseU; ++u) {
                    const uint32_t t = t0 + u * nt;
                    pass[u] = t < tables;
                    key[u] = pass[u] ? uint64_t(qk[t]) : 0ull;
                }
                if (tb.filter) { // a clear filter bit: no posting has this key
                    const uint64_t fpol = l2_evict_last_policy();
#pragma unroll
                    for (int u = 0; u < kDenseU; ++u) pass[u] = pass[u] && filter_pass(tb, t0 + u * nt, key[u], fpol);
                }
#pragma unroll
                for (int u = 0; u < kDenseU; ++u) {
                    const uint32_t t = t0 + u * nt;
                    if (pass[u]) {
                        load_bucket(tb.data + (uint64_t(t) * tb.nbuckets + home_of(key[u], tb)) * kSlots, sl[u]);
                    } else {
#pragma unroll
                        for (int j = 0; j < kSlots; ++j) sl[u][j] = T::make(~0ull, ~0u);
                    }
                }
#pragma unroll
                for (int u = 0; u < kDenseU; ++u) {
#pragma unroll
                    for (int j = 0; j < kSlots; ++j)
                        if (!T::empty(sl[u][j]) && T::key(sl[u][j]) == key[u]) {
                            ++coll;
                            insert(T::id(sl[u][j]));
                        }
                    if (T::empty(sl[u][kSlots - 1])) continue;
                    const E* base = tb.data + uint64_t(t0 + u * nt) * tb.nbuckets * kSlots;
                    uint64_t b = home_of(key[u], tb) + 1;
                    for (bool cont = true; cont; b += kDenseRun) {
                        E x[kDenseRun][kSlots];
#pragma unroll
                        for (int k = 0; k < kDenseRun; ++k)
                            load_bucket(base + ((b + k) & (tb.nbuckets - 1)) * kSlots, x[k]);
#pragma unroll
                        for (int k = 0; k < kDenseRun; ++k) {
                            if (!cont) break;
#pragma unroll
                            for (int j = 0; j < kSlots; ++j)
                                if (!T::empty(x[k][j]) && T::key(x[k][j]) == key[u]) {
                                    ++coll;
                                    insert(T::id(x[k][j]));
                                }
                            cont = !T::empty(x[k][kSlots - 1]);
                        }
                    }
                }
            }
        } else if (LAYOUT == kLayoutCsr && tables <= uint32_t(kFlatTables)) {
            // CSR, flattened: the directory read of every table first (its
            // cell [s, e) and the query's key into shared memory), a block
            // scan of the cell lengths, then the CTA's threads take the
            // concatenated cells' entries j = tid, tid + nt, ... (kFlatU in
            // flight each) and keep the ones with their table's key. A
            // popular key's long cell is read by many threads at once
            // (adjacent entries, coalesced) instead of walked by one thread
            // while the CTA waits for it at the barrier.
            using E = typename T::E;
            constexpr int kPer = (kFlatTables + NT - 1) / NT; // tables per thread
            uint32_t len[kPer], loc = 0;
            const uint32_t tb0 = tid * kPer;
            if (pf_have) { // fetched during the previous query (this thread's own tables)
                cp_async_wait_all_ix();
#pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    const uint32_t t = tb0 + k;
                    len[k] = t < tables ? f_off[t] - f_start[t] : 0u;
                    loc += len[k];
                }
            } else {
                uint64_t key[kPer];
#pragma unroll
                for (int k = 0; k < kPer; ++k) key[k] = tb0 + k < tables ? uint64_t(qk[tb0 + k]) : 0ull;
#pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    const uint32_t t = tb0 + k;
                    len[k] = 0;
                    if (t < tables) {
                        FCLSH_DCHECK(home_of(key[k], tb) < tb.cells);
                        const uint32_t* d = tb.dir + uint64_t(t) * (tb.cells + 1) + home_of(key[k], tb);
                        const uint32_t a = __ldg(d), e = __ldg(d + 1);
                        f_start[t] = a;
                        f_key[t] = key[k];
                        len[k] = e - a;
                    }
                    loc += len[k];
                }
            }
            uint32_t total = 0;
            if (tid == 0) pf_next_s = claimed; // (read after the scan's barriers)
            uint32_t run = block_exclusive_scan(loc, scan_ws, total);
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                if (tb0 + k < tables) f_off[tb0 + k] = run;
                run += len[k];
            }
            if (tid == 0) f_off[tables] = total;
            __syncthreads();
            // the next query's keys (this thread's tables), in flight beside
            // the entry loads; their directory words follow after the verify
            pf_s = pf_next_s;
            pf = flat_pf && pf_s < ns;
            if (pf) {
                const uint64_t qn = ovf ? ovf[pf_s] : pf_s;
                const typename T::K* qkn = qkeys + qn * tables;
#pragma unroll
                for (int k = 0; k < kPf; ++k) pf_key[k] = tb0 + k < tables ? qkn[tb0 + k] : typename T::K(0);
            }
            for (uint32_t j0 = tid; j0 < total && !bad_s; j0 += kFlatU * nt) {
                E e[kFlatU];
                uint32_t tt[kFlatU];
#pragma unroll
                for (int u = 0; u < kFlatU; ++u) {
                    const uint32_t j = j0 + u * nt;
                    tt[u] = ~0u;
                    if (j < total) {
                        uint32_t lo = 0, hi = tables; // the table t with f_off[t] <= j < f_off[t + 1]
                        while (hi - lo > 1) {
                            const uint32_t mid = (lo + hi) >> 1;
                            if (f_off[mid] <= j)
                                lo = mid;
                            else
                                hi = mid;
                        }
                        tt[u] = lo;
                        FCLSH_DCHECK(lo < tables && f_off[lo] <= j && j < f_off[lo + 1] &&
                                     f_start[lo] + (j - f_off[lo]) < tb.n);
                        e[u] = tb.data[uint64_t(lo) * tb.n + f_start[lo] + (j - f_off[lo])];
                    }
                }
#pragma unroll
                for (int u = 0; u < kFlatU; ++u)
                    if (tt[u] != ~0u && T::key(e[u]) == f_key[tt[u]]) {
                        ++coll;
                        insert(T::id(e[u]));
                    }
            }
        } else {
            for (uint32_t t = tid; t < tables; t += nt) {
                if (bad_s) break;
                coll += probe_one<T, LAYOUT>(tb, t, uint64_t(qk[t]), insert);
            }
        }
        atomicAdd(&coll_s, coll);
        __syncthreads();
        const uint32_t ncand = cand_s;
        // phase 2: verify the distinct candidates only
        if (!bad_s) {
            const uint64_t* qr = qrows + q * words;
            for (uint32_t k = tid; k < ncand; k += nt) {
                const uint32_t id = set[clist[k]];
                const uint64_t* r = rows + uint64_t(id) * words;
                const uint32_t d = row_distance(r, qr, words, vec_rows);
                if (d <= radius) {
                    const uint32_t pos = atomicAdd(&found_s, 1u);
                    if (pos < FCAP)
                        fl[pos] = (static_cast<unsigned long long>(id) << 32) | d;
                    else
                        bad_s = 1;
                }
            }
        }
        if (pf) { // phase 1 is done with f_key / f_start / f_off: the next query's go there
#pragma unroll
            for (int k = 0; k < kPf; ++k) {
                const uint32_t t = tid * kPf + k;
                if (t < tables) {
                    const uint64_t key = uint64_t(pf_key[k]);
                    FCLSH_DCHECK(home_of(key, tb) < tb.cells);
                    const uint32_t* d = tb.dir + uint64_t(t) * (tb.cells + 1) + home_of(key, tb);
                    f_key[t] = key;
                    cp_async4(f_start + t, d);     // the cell's first entry
                    cp_async4(f_off + t, d + 1);   // and its end (phase 1 turns it into the length)
                }
            }
            cp_async_commit_ix();
        }
        pf_have = pf;
        __syncthreads();
        // clear what this query wrote (all of it when the list is incomplete)
        if (ncand <= kMaxDistinct) {
            for (uint32_t k = tid; k < ncand; k += nt) set[clist[k]] = kEmpty;
        } else {
            for (uint32_t i = tid; i < HS; i += nt) set[i] = kEmpty;
        }
        __syncthreads();
        const uint32_t nf = found_s;
        if (tid == 0) {
            bool bad = bad_s;
            base_s = 0;
            if (!bad && nf > slot_cap) {
                base_s = atomicAdd(res_cursor, (unsigned long long)nf);
                bad = base_s + nf > res_cap; // region full
            }
            if (bad) {
                ovf2[atomicAdd(ovf2_cnt, 1u)] = uint32_t(q);
                found_q[q] = 0; // written by the general path later
                src_pos[q] = 0;
                bad_s = 1;
            } else {
                coll_q[q] = coll_s;
                cand_q[q] = cand_s;
                found_q[q] = nf;
                if (hc) {
                    hc[(nq_all + 1) + q] = coll_s;
                    hc[2 * (nq_all + 1) + q] = cand_s;
                    hc[3 * (nq_all + 1) + q] = nf;
                }
                // up to slot_cap results go to the query's own slots (no bump allocation)
                src_pos[q] = nf <= slot_cap ? q * slot_cap : src_base + base_s;
                if (nf) atomicAdd(tile_sum + (q >> kScanTileLog), (unsigned long long)nf);
            }
        }
        __syncthreads();
        if (!bad_s && nf) {
            uint32_t P = 1;
            while (P < nf) P <<= 1;
            for (uint32_t i = nf + tid; i < P; i += nt) fl[i] = ~0ull;
            __syncthreads();
            bitonic_sort<NarrowEntry>(fl, P, P);
            const bool slots = nf <= slot_cap;
            FCLSH_DCHECK(slots ? q < nq_all : base_s + nf <= res_cap);
            uint32_t* const oid = slots ? slot_id + q * slot_cap : res_id + base_s;
            uint32_t* const odist = slots ? slot_dist + q * slot_cap : res_dist + base_s;
            for (uint32_t k = tid; k < nf; k += nt) {
                const unsigned long long e = fl[k];
                oid[k] = uint32_t(e >> 32);
                odist[k] = uint32_t(e);
            }
        }
        __syncthreads();
    }
}

struct NarrowIdOrder {
    __device__ __forceinline__ static bool less(uint32_t a, uint32_t b) { return a < b; }
};

// ------------------------------------------------------- Strategy 1 query

// query_c_r_nn (index.cpp:190-235), one CTA per query: walk the buckets in
// table order (part, then table; ids ascending inside a bucket) and stop
// after `budget` postings, duplicates included; count collisions, distinct
// candidates, found (<= radius), and keep the closest point retrieved, ties
// to the lowest id. The walk is order-dependent, so the CTA first counts
// every table's postings, scans the counts to find the table where the
// budget runs out, then inserts the ids of the tables before it plus the
// smallest ids of that table into a shared set, and verifies the set.
template <typename T, int LAYOUT>
__global__ void __launch_bounds__(512) k_query_c(const typename T::K* __restrict__ qkeys, uint64_t nq,
                                                 uint32_t tables, const Tables<T> tb,
                                                 const uint64_t* __restrict__ rows,
                                                 const uint64_t* __restrict__ qrows, uint32_t words, uint32_t radius,
                                                 uint64_t budget, unsigned long long* __restrict__ counters,
                                                 uint32_t* __restrict__ best, unsigned int* __restrict__ qnext,
                                                 unsigned int* __restrict__ err, uint32_t hs_log, uint32_t kcap,
                                                 uint32_t* __restrict__ gscratch, uint64_t id_offset) {
    // the id set (2^hs_log slots) and the cut table's ids (kcap) live in
    // shared memory, or, for budgets beyond it, in this CTA's slice of a
    // global scratch [set | cut ids | slot list of the inserted ids]
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t HS = 1u << hs_log;
    const uint32_t tpad = (tables + 3) & ~3u;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem); // tables: postings per table, then their prefix
    uint32_t* set;
    uint32_t* kbuf;
    uint32_t* slots = nullptr; // global mode: the slot of every inserted id (verify walks these, not the set)
    if (gscratch) {
        uint32_t* g = gscratch + uint64_t(blockIdx.x) * (uint64_t(tpad) + HS + kcap + HS / 2);
        cnt = g;
        set = g + tpad;
        kbuf = set + HS;
        slots = kbuf + kcap;
    } else {
        set = cnt + tpad;
        kbuf = set + HS;
    }
    __shared__ unsigned long long wsum[16], best_s;
    __shared__ unsigned int cand_s, found_s, cut_s, cutr_s, kn_s, next_s, bad_s;
    constexpr uint32_t kEmpty = 0xFFFFFFFFu;
    const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    for (uint32_t i = tid; i < HS; i += nt) set[i] = kEmpty;
    auto fetch = [&]() -> uint32_t {
        if (tid == 0) next_s = atomicAdd(qnext, 1u);
        __syncthreads();
        return next_s;
    };
    for (uint64_t q = fetch(); q < nq; q = fetch()) {
        const typename T::K* qk = qkeys + q * tables;
        // A: postings per table
        for (uint32_t t = tid; t < tables; t += nt) cnt[t] = probe_one<T, LAYOUT>(tb, t, uint64_t(qk[t]), [](uint32_t) {});
        if (tid == 0) {
            cand_s = found_s = kn_s = bad_s = 0;
            best_s = ~0ull;
            cut_s = tables; // no cut
            cutr_s = 0;
        }
        __syncthreads();
        // B: exclusive prefix over tables in walk order (contiguous chunk per thread)
        const uint32_t per = (tables + nt - 1) / nt, b0 = min(tables, tid * per), b1 = min(tables, b0 + per);
        unsigned long long mine = 0;
        for (uint32_t t = b0; t < b1; ++t) mine += cnt[t];
        unsigned long long x = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= uint32_t(o)) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        unsigned long long run = x - mine;
        for (uint32_t w = 0; w < wid; ++w) run += wsum[w];
        unsigned long long total = 0;
        for (uint32_t w = 0; w < (nt >> 5); ++w) total += wsum[w];
        // the table where the budget runs out: cum < budget < cum + cnt
        for (uint32_t t = b0; t < b1; ++t) {
            const uint32_t c = cnt[t];
            if (run < budget && run + c > budget) {
                cut_s = t;
                cutr_s = uint32_t(budget - run);
            }
            cnt[t] = uint32_t(run < 0xFFFFFFFFull ? run : 0xFFFFFFFFull); // now the exclusive prefix
            run += c;
        }
        __syncthreads();
        const uint32_t cut = cut_s, cutr = cutr_s;
        const unsigned long long coll = total < budget ? total : budget;
        // C: ids of the tables walked in full, and of the cut table's smallest ids
        auto insert = [&](uint32_t id) {
            uint32_t h = (id * 0x9E3779B1u) >> (32 - hs_log);
            for (;;) {
                const uint32_t old = atomicCAS(set + h, kEmpty, id);
                if (old == id) return;
                if (old == kEmpty) break;
                h = (h + 1) & (HS - 1);
            }
            const uint32_t k = atomicAdd(&cand_s, 1u);
            FCLSH_DCHECK(!slots || k < HS / 2);
            if (slots) slots[k] = h;
        };
        for (uint32_t t = tid; t < tables; t += nt) {
            const bool full = t < cut && cnt[t] < budget;
            if (full) {
                probe_one<T, LAYOUT>(tb, t, uint64_t(qk[t]), insert);
            } else if (t == cut) {
                probe_one<T, LAYOUT>(tb, t, uint64_t(qk[t]), [&](uint32_t id) {
                    const uint32_t p = atomicAdd(&kn_s, 1u);
                    if (p < kcap) kbuf[p] = id;
                    else bad_s = 1;
                });
            }
        }
        __syncthreads();
        if (cut < tables) { // the cut table: ascending ids, the first cutr of them
            const uint32_t m = min(kn_s, kcap);
            uint32_t P = 1;
            while (P < m) P <<= 1;
            for (uint32_t i = m + tid; i < P; i += nt) kbuf[i] = kEmpty;
            __syncthreads();
            bitonic_sort<NarrowIdOrder>(kbuf, P, P);
            for (uint32_t i = tid; i < cutr && i < m; i += nt) insert(kbuf[i]);
            __syncthreads();
        }
        // D: verify the distinct candidates, closest first (ties: lowest id)
        const uint64_t* qr = qrows + q * words;
        uint32_t fnd = 0;
        unsigned long long bst = ~0ull;
        const uint32_t walk = slots ? cand_s : HS; // global mode: the listed slots only
        for (uint32_t i = tid; i < walk; i += nt) {
            const uint32_t sl = slots ? slots[i] : i;
            const uint32_t id = set[sl];
            if (id == kEmpty) continue;
            set[sl] = kEmpty;
            const uint64_t* r = rows + uint64_t(id) * words;
            uint32_t d = 0;
            for (uint32_t w = 0; w < words; ++w) d += __popcll(__ldg(r + w) ^ __ldg(qr + w));
            if (d <= radius) ++fnd;
            const unsigned long long key = (static_cast<unsigned long long>(d) << 32) | id;
            bst = key < bst ? key : bst;
        }
        if (fnd) atomicAdd(&found_s, fnd);
        if (bst != ~0ull) atomicMin(&best_s, bst);
        __syncthreads();
        if (tid == 0) {
            counters[3 * q] = coll;
            counters[3 * q + 1] = cand_s;
            counters[3 * q + 2] = found_s;
            // shard ids: reported with the index's id offset, like query_r_nn's
            best[2 * q] = best_s == ~0ull ? kEmpty : uint32_t(uint32_t(best_s) + id_offset);
            best[2 * q + 1] = best_s == ~0ull ? kEmpty : uint32_t(best_s >> 32);
            if (bad_s) atomicAdd(err, 1u);
        }
        __syncthreads();
    }
}

// General path for the selected queries qsel[0..ns): per (query, table)
// counts -> per-query collision totals; scan; gather the ids; CUB segmented
// sort; verify.
template <typename T, int LAYOUT>
__global__ void k_count_sel(const typename T::K* __restrict__ qkeys, const uint32_t* __restrict__ qsel, uint64_t ns,
                            uint32_t tables, const Tables<T> tb, unsigned long long* __restrict__ coll) {
    const uint64_t total = ns * tables;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s_ = i / tables;
        const uint32_t t = uint32_t(i % tables);
        const uint64_t key = qkeys[uint64_t(qsel[s_]) * tables + t];
        const uint32_t c = probe_one<T, LAYOUT>(tb, t, key, [](uint32_t) {});
        if (c) atomicAdd(coll + s_, (unsigned long long)c);
    }
}

template <typename T, int LAYOUT>
__global__ void k_gather_sel(const typename T::K* __restrict__ qkeys, const uint32_t* __restrict__ qsel, uint64_t ns,
                             uint32_t tables, const Tables<T> tb, const unsigned long long* __restrict__ coll_off,
                             unsigned long long* __restrict__ fill, uint32_t* __restrict__ cand) {
    const uint64_t total = ns * tables;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s_ = i / tables;
        const uint32_t t = uint32_t(i % tables);
        const uint64_t key = qkeys[uint64_t(qsel[s_]) * tables + t];
        probe_one<T, LAYOUT>(tb, t, key, [&](uint32_t id) {
            const uint64_t dst = coll_off[s_] + atomicAdd(fill + s_, 1ull);
            cand[dst] = id;
        });
    }
}

// Warp per selected query over its sorted candidate list; writes the query's
// counters and its results at base_pos + coll_off[s].
__global__ void k_verify_sel(uint64_t ns, const uint32_t* __restrict__ qsel,
                             const unsigned long long* __restrict__ coll_off, const uint32_t* __restrict__ sorted,
                             const uint64_t* __restrict__ rows, const uint64_t* __restrict__ qrows, uint32_t words,
                             uint32_t radius, uint64_t base_pos, uint32_t* __restrict__ res_id,
                             uint32_t* __restrict__ res_dist, unsigned long long* __restrict__ coll_q,
                             unsigned long long* __restrict__ cand_q, unsigned long long* __restrict__ found_q,
                             unsigned long long* __restrict__ src_pos) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t s_ = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); s_ < ns; s_ += warps) {
        const uint64_t q = qsel[s_];
        const uint64_t beg = coll_off[s_], end = coll_off[s_ + 1];
        const uint64_t* qr = qrows + q * words;
        uint64_t ncand = 0, nfound = 0;
        for (uint64_t base = beg; base < end; base += 32) {
            const uint64_t k = base + lane;
            const bool valid = k < end;
            const uint32_t id = valid ? sorted[k] : 0u;
            const bool uniq = valid && (k == beg || sorted[k - 1] != id);
            uint32_t dist = 0;
            if (uniq) {
                const uint64_t* r = rows + uint64_t(id) * words;
                for (uint32_t w = 0; w < words; ++w) dist += __popcll(__ldg(r + w) ^ __ldg(qr + w));
            }
            const bool pass = uniq && dist <= radius;
            const uint32_t bu = __ballot_sync(0xffffffffu, uniq);
            const uint32_t bp = __ballot_sync(0xffffffffu, pass);
            if (pass) {
                const uint64_t pos = beg + nfound + __popc(bp & ((1u << lane) - 1u));
                res_id[pos] = id;
                res_dist[pos] = dist;
            }
            ncand += __popc(bu);
            nfound += __popc(bp);
        }
        if (lane == 0) {
            coll_q[q] = end - beg;
            cand_q[q] = ncand;
            found_q[q] = nfound;
            src_pos[q] = base_pos + beg;
        }
    }
}

// Copies every query's results (slot of the fused path, or region of the
// general path) to its place in the (query, id) ordered output.
// Result sources by src_pos: [0, tmp_len) warp-kernel slots, [tmp_len,
// tmp_len + cta_len) the CTA kernel's region, beyond: the general path.
__global__ void k_compact(uint64_t nq, const unsigned long long* __restrict__ src_pos,
                          const unsigned long long* __restrict__ res_off, const uint32_t* __restrict__ tmp_id,
                          const uint32_t* __restrict__ tmp_dist, uint64_t tmp_len, const uint32_t* __restrict__ cta_id,
                          const uint32_t* __restrict__ cta_dist, uint64_t cta_len, const uint32_t* __restrict__ tmp2_id,
                          const uint32_t* __restrict__ tmp2_dist, uint64_t id_offset, uint32_t* __restrict__ out_q,
                          uint32_t* __restrict__ out_id, uint32_t* __restrict__ out_dist,
                          unsigned long long* __restrict__ pub, unsigned long long* __restrict__ dseq,
                          const unsigned int* __restrict__ cnts) {
    const uint32_t lane = threadIdx.x & 31;
    if (pub && blockIdx.x == 0 && threadIdx.x == 0) {
        // the batch's total and hand-over counts to mapped host memory, then
        // the sequence number the host spins on (no memcpy + stream sync)
        const unsigned long long seq = *dseq + 1; // batch number (graph replays need no parameter)
        *dseq = seq;
        pub[0] = res_off[nq];
        pub[1] = cnts[0];
        pub[2] = cnts[1];
        pub_flag(pub + 3, seq);
    }
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t q = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); q < nq; q += warps) {
        const uint64_t dst = res_off[q], cnt = res_off[q + 1] - dst;
        if (cnt == 0) continue;
        uint64_t src = src_pos[q];
        const uint32_t* ti = tmp_id;
        const uint32_t* td = tmp_dist;
        if (src >= tmp_len + cta_len) {
            src -= tmp_len + cta_len;
            ti = tmp2_id;
            td = tmp2_dist;
        } else if (src >= tmp_len) {
            src -= tmp_len;
            ti = cta_id;
            td = cta_dist;
        }
        for (uint64_t k = lane; k < cnt; k += 32) {
            out_q[dst + k] = uint32_t(q);
            out_id[dst + k] = uint32_t(ti[src + k] + id_offset);
            out_dist[dst + k] = td[src + k];
        }
    }
}

// The found scan, the offsets, the compaction and the publish in one kernel
// (replaces a memset + CUB's two scan kernels + k_compact): CTA t owns the
// 1024 queries of tile t; the query kernels have added each tile's results
// to tile_sum[t], so the tile's prefix is the sum of the earlier tiles'
// sums, a block scan gives every query's offset, and one thread per result
// (its query found by a binary search over the tile's offsets) copies it.
// kScanSplit CTAs share each tile (each recomputes its scan, one writes the
// offsets). With a host destination (desc: copied from pinned memory in the
// batch, beside the hash; reading mapped host memory from every CTA costs
// ~0.35 ms) the counters and, when they fit, the results go straight into
// mapped pinned host memory, coalesced, instead of a D2H copy after the
// kernel; the last CTA to finish publishes the batch (total, overflow counts,
// sequence number) once every CTA's writes are fenced.
__global__ void __launch_bounds__(1024) k_scan_compact(
    uint64_t nq, const unsigned long long* __restrict__ found_q, const unsigned long long* __restrict__ tile_sum,
    unsigned long long* __restrict__ res_off, const unsigned long long* __restrict__ src_pos,
    const uint32_t* __restrict__ tmp_id, const uint32_t* __restrict__ tmp_dist, uint64_t tmp_len,
    const uint32_t* __restrict__ cta_id, const uint32_t* __restrict__ cta_dist, uint64_t id_offset,
    uint32_t* __restrict__ out_q, uint32_t* __restrict__ out_id, uint32_t* __restrict__ out_dist,
    unsigned long long* __restrict__ pub, unsigned long long* __restrict__ dseq, unsigned int* __restrict__ cnts,
    const unsigned long long* __restrict__ coll_q, const unsigned long long* __restrict__ cand_q,
    const unsigned long long* __restrict__ desc) {
    constexpr uint32_t TQ = 1u << kScanTileLog;
    __shared__ unsigned long long off_s[TQ + 1], src_s[TQ], wsum[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // grid: kScanSplit CTAs per tile of TQ queries, then one publisher CTA
    const uint32_t nwork = gridDim.x - 1, ntiles = nwork / kScanSplit;
    const uint32_t t = blockIdx.x / kScanSplit, part = blockIdx.x % kScanSplit;
    const uint64_t q0 = uint64_t(t) * TQ;
    const uint32_t m = blockIdx.x < nwork ? uint32_t(nq - q0 < TQ ? nq - q0 : TQ) : 0u;
    if (blockIdx.x == nwork && wid) return; // (the publisher needs one warp)
    FCLSH_TL_MIN(kTlCompEntry);
    pdl_wait(); // the query kernels' outputs are complete from here on
    FCLSH_TL_MIN(kTlCompWait);
    if (blockIdx.x == nwork) {
        // device outputs: publish as soon as the total is known (the sum of
        // the tile sums), so the host's return overlaps the compaction; the
        // caller's reads of the outputs follow this kernel in stream order. A
        // CTA of its own: the system-scope release (~1.3 us) holds up no
        // barrier of the compaction's CTAs. Host outputs: published below,
        // once every CTA's writes are visible.
        if (!pub || (desc && desc[0])) return;
        const unsigned long long seq = *dseq + 1;
        const unsigned int c0 = cnts[0], c1 = cnts[1];
        unsigned long long all = 0;
        for (uint32_t i = lane; i < ntiles; i += 32) all += tile_sum[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) all += __shfl_xor_sync(0xffffffffu, all, o);
        if (lane == 0) {
            *dseq = seq;
            pub[0] = all;
            pub[1] = c0;
            pub[2] = c1;
            pub_flag(pub + 3, seq);
            FCLSH_TL_MAX(kTlPublish);
        }
        return;
    }
    // the host destination (null counters: device buffers only), read by
    // every thread (one L1 line, no barrier)
    HostDest hd;
    hd.counters = desc ? reinterpret_cast<unsigned long long*>(desc[0]) : nullptr;
    hd.q = desc ? reinterpret_cast<uint32_t*>(desc[1]) : nullptr;
    hd.id = desc ? reinterpret_cast<uint32_t*>(desc[2]) : nullptr;
    hd.dist = desc ? reinterpret_cast<uint32_t*>(desc[3]) : nullptr;
    hd.cap = desc ? desc[4] : 0;
    // this tile's found counts and result sources, loaded beside the tile sums
    const unsigned long long f = tid < m ? found_q[q0 + tid] : 0ull;
    const unsigned long long srcv = tid < m ? src_pos[q0 + tid] : 0ull;
    // prefix of the earlier tiles and the batch total, summed by every warp
    // over all the tile sums (no barrier; <= 32 loads per lane up to 32k tiles)
    unsigned long long pre = 0, all = 0;
    for (uint32_t i = lane; i < ntiles; i += 32) {
        const unsigned long long v = tile_sum[i];
        all += v;
        if (i < t) pre += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pre += __shfl_xor_sync(0xffffffffu, pre, o);
        all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    const unsigned long long prefix = pre;
    FCLSH_TL_MAX(kTlCompLoaded);
    const bool host_cnt = hd.counters != nullptr;
    const bool host_res = host_cnt && all <= hd.cap;
    if (host_res) { // results into the host block
        out_q = hd.q;
        out_id = hd.id;
        out_dist = hd.dist;
    }
    // block exclusive scan of this tile's found counts
    if (tid < m) src_s[tid] = srcv;
    unsigned long long x = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= uint32_t(o)) x += y;
    }
    __syncthreads(); // wsum reuse
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        unsigned long long w = lane < (blockDim.x >> 5) ? wsum[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= uint32_t(o)) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    const unsigned long long excl = x - f + (wid ? wsum[wid - 1] : 0ull);
    const unsigned long long tile_total = wsum[(blockDim.x >> 5) - 1];
    off_s[tid] = excl;
    if (tid == 0) off_s[TQ] = tile_total;
    FCLSH_TL_MAX(kTlCompScanned);
    if (part == 0 && tid < m) res_off[q0 + tid] = prefix + excl;
    // (the query kernels wrote the other counters to the host as each query completed)
    if (host_cnt && tid < m && tid / (TQ / kScanSplit) == part) hd.counters[q0 + tid] = prefix + excl;
    const bool last = q0 + TQ >= nq;
    if (part == 0 && last && tid == 0) {
        res_off[nq] = prefix + tile_total;
        if (host_cnt) hd.counters[nq] = prefix + tile_total;
    }
    __syncthreads();
    // one thread per result of this CTA's share of the tile
    for (unsigned long long idx = uint64_t(part) * blockDim.x + tid; idx < tile_total;
         idx += uint64_t(blockDim.x) * kScanSplit) {
        uint32_t lo = 0, hi = m; // the query j with off_s[j] <= idx < off_s[j+1] (first such: skips empty ones)
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (off_s[mid] <= idx)
                lo = mid;
            else
                hi = mid;
        }
        const unsigned long long k = idx - off_s[lo];
        unsigned long long src = src_s[lo];
        const uint32_t* ti = tmp_id;
        const uint32_t* td = tmp_dist;
        if (src >= tmp_len) {
            src -= tmp_len;
            ti = cta_id;
            td = cta_dist;
        }
        const unsigned long long dst = prefix + idx;
        out_q[dst] = uint32_t(q0 + lo);
        out_id[dst] = uint32_t(ti[src + k] + id_offset);
        out_dist[dst] = td[src + k];
    }
    FCLSH_TL_MAX(kTlCompExit);
    if (!pub || !host_cnt) return;
    // host outputs: publish once every CTA's writes are visible: the
    // barrier orders the CTA's writes before thread 0's system fence
    // (cumulative), which orders them before its count (one fence per CTA:
    // a fence per thread serialises in the memory system, ~0.3 ms per batch)
    __syncthreads();
    if (tid == 0) {
        const unsigned int done = pub_arrive(cnts + 8);
        if (done + 1 == nwork) {
            const unsigned long long seq = *dseq + 1;
            *dseq = seq;
            pub[0] = all;
            pub[1] = reinterpret_cast<volatile unsigned int*>(cnts)[0];
            pub[2] = reinterpret_cast<volatile unsigned int*>(cnts)[1];
            pub_flag(pub + 3, seq);
            FCLSH_TL_MAX(kTlPublish);
        }
    }
}

uint32_t bit_length(uint64_t x) { return x == 0 ? 0 : 64 - __builtin_clzll(x); }

// vector width of the verify's row loads (row_distance): every stored row is
// W words at a cudaMalloc'd base; the query rows' base must be aligned too
int vec_for(uint32_t words, const void* q) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(q);
    if (words % 4 == 0 && a % 32 == 0) return 4;
    if (words % 2 == 0 && a % 16 == 0) return 2;
    return 1;
}

unsigned grid_for(uint64_t work, int device, unsigned threads = 256, unsigned per_sm = 8) {
    const uint64_t want = (work + threads - 1) / threads;
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(sm_count(device)) * per_sm)));
}

template <typename T>
Tables<T> view(const DeviceIndex& ix) {
    Tables<T> tb;
    tb.data = static_cast<const typename T::E*>(ix.entries.p);
    tb.dir = ix.dir.as<uint32_t>();
    tb.n = ix.n;
    tb.cells = ix.cells();
    tb.nbuckets = ix.nbuckets;
    tb.shift = ix.key_shift;
    tb.filter = ix.filter_words ? ix.filter.as<uint32_t>() : nullptr;
    tb.filter_words = ix.filter_words;
    tb.kscale = ix.key_scale;
    return tb;
}

// keys: one part's point-major keys (stride L); builds global tables
// [tg0, tg0 + count) from the part's local tables [t0, t0 + count).
template <typename T>
void build_csr_tables(DeviceIndex& ix, const void* keys, uint32_t L, uint32_t t0, uint32_t tg0, uint32_t count,
                      DevBuf& cnt_buf, DevBuf& cur_buf, DevBuf& big_buf, DevBuf& big_cnt, cudaStream_t s) {
    using K = typename T::K;
    const uint64_t n = ix.n, cells = ix.cells();
    const uint64_t cbytes = uint64_t(count) * (cells + 1) * 4;
    uint32_t* cnt = static_cast<uint32_t*>(cnt_buf.ensure(cbytes));
    uint32_t* cur = static_cast<uint32_t*>(cur_buf.ensure(cbytes));
    uint32_t* dir = ix.dir.as<uint32_t>() + uint64_t(tg0) * (cells + 1);
    auto* entries = static_cast<typename T::E*>(ix.entries.p) + uint64_t(tg0) * n;
    FCLSH_CUDA(cudaMemsetAsync(cnt, 0, cbytes, s));
    const unsigned g = grid_for(n * count, ix.device, 256, 8);
    k_hist<K><<<g, 256, 0, s>>>(static_cast<const K*>(keys), n, L, t0, count, ix.key_shift, ix.key_scale, cells, cnt);
    FCLSH_LAUNCHED();
    k_scan_cells<<<count, 1024, 0, s>>>(cnt, cells, dir, cur);
    FCLSH_LAUNCHED();
    k_scatter<T, K><<<g, 256, 0, s>>>(static_cast<const K*>(keys), n, L, t0, count, ix.key_shift, ix.key_scale, cells, cur, entries);
    FCLSH_LAUNCHED();
    // cells longer than kSmallCell: at most n / (kSmallCell+1) per table
    const uint64_t max_big = uint64_t(count) * (n / (kSmallCell + 1) + 1);
    uint2* big = static_cast<uint2*>(big_buf.ensure(max_big * sizeof(uint2)));
    unsigned int* bc = static_cast<unsigned int*>(big_cnt.ensure(sizeof(unsigned int)));
    FCLSH_CUDA(cudaMemsetAsync(bc, 0, sizeof(unsigned int), s));
    k_sort_cells<T><<<grid_for(uint64_t(count) * cells, ix.device), 256, 0, s>>>(dir, cells, n, count, entries, big, bc);
    FCLSH_LAUNCHED();
    unsigned int nbig = 0;
    FCLSH_CUDA(cudaMemcpyAsync(&nbig, bc, sizeof(nbig), cudaMemcpyDeviceToHost, s));
    FCLSH_CUDA(cudaStreamSynchronize(s));
    if (nbig > 0) {
        const uint32_t cap = uint32_t((96 * 1024) / sizeof(typename T::E));
        const size_t smem = size_t(cap) * sizeof(typename T::E);
        FCLSH_CUDA(cudaFuncSetAttribute(k_sort_big<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k_sort_big<T><<<nbig, 512, smem, s>>>(dir, cells, n, entries, big, cap);
        FCLSH_LAUNCHED();
    }
}

template <typename T>
void build_all(DeviceIndex& ix) {
    using K = typename T::K;
    const uint64_t n = ix.n, L = ix.fs->tables;
    const uint32_t kb = sizeof(K);
    cudaStream_t s = ix.stream;
    DevBuf keys, keys_tm, cnt, cur, big, bigc;
    keys.ensure(L * n * kb);
    if (ix.layout == kLayoutBuckets)
        FCLSH_CUDA(cudaMemsetAsync(ix.entries.p, T::empty_byte(), ix.entries.bytes, s));
    // CSR: tables per chunk bounded by ~1 GiB of cell counters
    const uint64_t per_table = (ix.cells() + 1) * 8;
    const uint32_t chunk = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(L, (1ull << 30) / per_table)));
    for (uint32_t p = 0; p < ix.fs->parts; ++p) {
        // K1, point-major: key of (row i, local table t) at keys[i*L + t]
        hash_rows(*ix.fs, ix.rows.as<uint64_t>(), n, keys.p, kb, L, kLayoutPointMajor, s, p, 1);
        if (ix.layout == kLayoutBuckets) {
            auto* bk = static_cast<typename T::E*>(ix.entries.p) + uint64_t(p) * L * ix.nbuckets * kSlots;
            uint32_t* fl = ix.filter_words ? ix.filter.as<uint32_t>() + uint64_t(p) * L * ix.filter_words : nullptr;
            // keys table-major one slab of tables at a time, then table groups
            // of ~64 MB of buckets (half the L2) inserted from the slab
            const uint64_t tbytes = ix.nbuckets * kSlots * sizeof(typename T::E);
            const uint32_t tg = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(L, (uint64_t(64) << 20) / tbytes)));
            const uint32_t slab = uint32_t(std::min<uint64_t>(L, std::max<uint64_t>(tg, kBuildSlab)));
            K* ktm = static_cast<K*>(keys_tm.ensure(uint64_t(slab) * n * kb));
            for (uint32_t sb = 0; sb < L; sb += slab) {
                const uint32_t sc = uint32_t(std::min<uint64_t>(slab, L - sb));
                k_keys_table_major<K><<<unsigned(std::min<uint64_t>(((sc + 31) / 32) * ((n + 31) / 32),
                                                                     uint64_t(sm_count(ix.device)) * 8)),
                                        256, 0, s>>>(static_cast<const K*>(keys.p), ktm, n, uint32_t(L), sb, sc);
                FCLSH_LAUNCHED();
                for (uint32_t t0 = sb; t0 < sb + sc; t0 += tg) {
                    const uint32_t c = uint32_t(std::min<uint64_t>(tg, sb + sc - t0));
                    k_bucket_insert<T><<<grid_for(n * c, ix.device, 256, 8), 256, 0, s>>>(
                        ktm, sb, n, t0, c, ix.key_shift, ix.nbuckets, bk, fl, ix.filter_words, ix.key_scale);
                    FCLSH_LAUNCHED();
                }
            }
        } else {
            for (uint32_t t = 0; t < L; t += chunk) {
                const uint32_t c = uint32_t(std::min<uint64_t>(chunk, L - t));
                build_csr_tables<T>(ix, keys.p, uint32_t(L), t, uint32_t(p * L + t), c, cnt, cur, big, bigc, s);
            }
        }
    }
    FCLSH_CUDA(cudaStreamSynchronize(s));
}

// The query kernel hashes its own queries (k_query_warp_pf<.., FE>) when the
// keys are narrow (prime < 2^32), the family is a covering family with
// N = 32 x FE columns per part, FE in {1, 2, 4, 8} (per-part radius 4..7),
// and rows fit a warp (d <= 2048): returns FE, else 0 (the separate hash
// kernel runs first). FCLSH_NO_FUSED_HASH=1: never (A/B).
int fused_fe(const DeviceIndex& ix) {
    static const bool off = getenv("FCLSH_NO_FUSED_HASH") != nullptr || getenv("FCLSH_WARP_V1") != nullptr ||
                            getenv("FCLSH_FUSED_SHARED") != nullptr;
    const DeviceFamilySet& fs = *ix.fs;
    if (off || ix.layout != kLayoutBuckets || ix.wide || fs.classic || ix.prime > 0xFFFFFFFFull) return 0;
    // (N = 512, FE = 16 -- cfg2 -- measured slower fused: 0.139 -> 0.186 ms per
    // batch, the 16-deep register transform spills and delays every query's
    // probes; again with the family in shared memory, 4 CTAs/SM: 0.167 ->
    // 0.184 ms per 11k batch; the separate hash kernel runs there)
    if (ix.tables > 600 || ix.row_words > 32 || fs.order < 32 || fs.order > 256) return 0;
    return int(fs.order / 32);
}

FusedHash fused_params(const DeviceIndex& ix, const uint64_t* hash_src) {
    FusedHash f;
    const DeviceFamilySet& fs = *ix.fs;
    if (!fused_fe(ix)) return f;
    f.parts = fs.parts;
    f.N = uint32_t(fs.order);
    f.L = uint32_t(fs.tables);
    f.max_dims = fs.max_part_dims;
    f.col_ptr = fs.col_ptr.as<uint32_t>();
    f.ent_pk = fs.ent_pk.as<uint64_t>();
    f.ent_sk = fs.ent_sk.as<uint64_t>();
    f.ent_pos = fs.ent_pos.as<uint32_t>();
    f.ent_seed = fs.ent_seed.as<uint64_t>();
    f.prime = fs.prime;
    f.hash_src = hash_src;
    // staged in shared memory when small (cfg3: 5.1 KB per CTA; A/B: FCLSH_FAMILY_GLOBAL=1)
    static const bool global_only = getenv("FCLSH_FAMILY_GLOBAL") != nullptr;
    const uint64_t sb = uint64_t(f.parts) * (f.max_dims * 8 + (f.N + 1) * 4);
    f.smem_bytes = !global_only && sb <= 12 * 1024 ? uint32_t((sb + 15) & ~uint64_t(15)) : 0;
    return f;
}

template <typename T, int LAYOUT, int CAP>
void launch_fused(DeviceIndex& ix, typename T::K* qkeys, const uint64_t* d_q, uint64_t nq, uint32_t radius,
                  uint32_t slot_cap, unsigned long long* coll_q, unsigned long long* cand_q,
                  unsigned long long* found_q, unsigned long long* src_pos, uint32_t* tmp_id, uint32_t* tmp_dist,
                  uint32_t* ovf, unsigned int* ovf_cnt, unsigned int* qnext, unsigned long long* tile_sum,
                  const unsigned long long* desc, cudaStream_t s, const uint64_t* hash_src) {
    // default: the id list in registers (no shared memory, all of L1 for the
    // probes in flight); FCLSH_FUSED_SHARED=1 selects the shared-set kernel
    static const bool shared_set = getenv("FCLSH_FUSED_SHARED") != nullptr;
    static const bool v1 = getenv("FCLSH_WARP_V1") != nullptr; // A/B: the unpipelined warp kernel
    if (!shared_set && !v1 && LAYOUT == kLayoutBuckets) {
        const int vec = vec_for(ix.row_words, d_q);
        auto go = [&](auto kern, bool use_smem = false, int sk_fe = 0) {
            FusedHash fh = fused_params(ix, hash_src);
            if (!use_smem) fh.smem_bytes = 0;
            if (sk_fe) { // position-parallel sketch: entries + per-warp row and column accumulators
                fh.sk_warp_bytes = uint32_t((uint64_t(sk_fe) * 32 * 2 * 4 + uint64_t(ix.row_words) * 8 + 15) & ~uint64_t(15));
                fh.smem_bytes = uint32_t((uint64_t(fh.parts) * fh.max_dims * 8 + 15) & ~uint64_t(15)) + 8 * fh.sk_warp_bytes;
            }
            // carveout: none (all of the unified array as L1 for the probes in
            // flight), or just enough shared memory for MINB CTAs' staged family
            static std::atomic<uint64_t> carved{0}; // devices whose carveout is set (per instantiation)
            static std::atomic<int> carve_pct{-1};
            static const int carve_env = getenv("FCLSH_CARVE") ? atoi(getenv("FCLSH_CARVE")) : -1; // A/B (%)
            const int want = carve_env >= 0 ? carve_env
                             : fh.smem_bytes ? int((uint64_t(fh.smem_bytes + 1024) * 6 * 100 + 228 * 1024 - 1) / (228 * 1024))
                                             : 0;
            const uint64_t bit = uint64_t(1) << (ix.device & 63);
            if (!(carved.load(std::memory_order_acquire) & bit) || carve_pct.load() != want) {
                FCLSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, std::min(want, 100)));
                carve_pct.store(want);
                carved.fetch_or(bit, std::memory_order_acq_rel);
            }
            int per_sm = resident_ctas(kern, 256, fh.smem_bytes, ix.device);
            static const int cap = getenv("FCLSH_WARP_CTAS") ? atoi(getenv("FCLSH_WARP_CTAS")) : 0; // A/B
            if (cap > 0) per_sm = std::min(per_sm, cap);
            const uint64_t grid = std::max<uint64_t>(
                1, std::min<uint64_t>((nq + 7) / 8, uint64_t(std::max(per_sm, 1)) * sm_count(ix.device)));
            launch_pdl(kern, unsigned(grid), 256, fh.smem_bytes, s, qkeys, nq, uint32_t(ix.tables), view<T>(ix),
                       ix.rows.as<uint64_t>(), d_q, ix.row_words, radius, slot_cap, coll_q, cand_q, found_q, src_pos,
                       tmp_id, tmp_dist, ovf, ovf_cnt, qnext, tile_sum, desc, vec, fh);
            FCLSH_LAUNCHED();
        };
        // probes per lane in flight per round: 3 for indexes of <= 400
        // tables, else 2 (measured; A/B: FCLSH_WARP_U = 2 | 3 | 4)
        static const int wu_env = getenv("FCLSH_WARP_U") ? atoi(getenv("FCLSH_WARP_U")) : 0;
        const int wu = wu_env ? wu_env : (ix.tables <= 400 ? 3 : 2);
        const int fe = fused_fe(ix);
        const bool fsm = fe > 0 && fused_params(ix, hash_src).smem_bytes > 0;
        // part-major fused hash (keys in registers) with the family in shared
        // memory for one-register parts (cfg1: 34.2 -> 35.7 M q/s); cfg3
        // measured slower part-major (fused kernel 88.3 -> 89.7 us, replayed
        // 1M batch 157.5 -> 145.3 M q/s: profiles/r02/ab_part_major.txt).
        // A/B: FCLSH_FUSED_PM=1 (every FE), FCLSH_FUSED_PF=1 (never)
        static const bool pf_env = getenv("FCLSH_FUSED_PF") != nullptr;
        static const bool pm_env = getenv("FCLSH_FUSED_PM") != nullptr;
        const bool pm = fsm && !pf_env && (fe == 1 || pm_env);
        // the position-parallel sketch (hash_part_sk) for FE = 1 (cfg1: 35.4 ->
        // 36.7 M q/s); for cfg3 (FE = 4) its 1 KB of accumulators per warp
        // take L1 from the probes in flight: kernel 88.4 -> 91.8 us
        // (profiles/r02/ab_sketch.txt). A/B: FCLSH_SKETCH_COLS=1 keeps the
        // per-column lists, FCLSH_SKETCH_ALL=1 uses the sketch for FE = 4 too
        static const bool cols_env = getenv("FCLSH_SKETCH_COLS") != nullptr;
        static const bool sk4_env = getenv("FCLSH_SKETCH_ALL") != nullptr;
        const bool sk = fsm && !cols_env && fused_params(ix, hash_src).ent_sk != nullptr;
        if (fe == 1 && pm && sk)
            go(k_query_warp_pf<T, 3, 4, 1, true, true, true>, true, 1);
        else if (fe == 4 && !pm && wu_env != 3 && sk && sk4_env)
            go(k_query_warp_pf<T, 2, FCLSH_FE4_MINB, 4, true, false, true>, true, 4);
        else if (fe == 1)
            pm ? go(k_query_warp_pf<T, 3, 4, 1, true, true>, true)
               : fsm ? go(k_query_warp_pf<T, 3, 4, 1, true>, true) : go(k_query_warp_pf<T, 3, 4, 1>);
        else if (fe == 2)
            pm ? go(k_query_warp_pf<T, 2, 5, 2, true, true>, true)
               : fsm ? go(k_query_warp_pf<T, 3, 4, 2, true>, true) : go(k_query_warp_pf<T, 3, 4, 2>);
        else if (fe == 4 && wu_env == 3)
            fsm ? go(k_query_warp_pf<T, 3, 4, 4, true>, true) : go(k_query_warp_pf<T, 3, 4, 4>);
        else if (fe == 4) // (cfg3: U = 2 at 5 CTAs/SM measured ~4 % ahead of U = 3 at 4)
            pm ? go(k_query_warp_pf<T, 2, 5, 4, true, true>, true)
               : !fsm ? go(k_query_warp_pf<T, 2, 5, 4>)
                 : ix.row_words <= 16 ? go(k_query_warp_pf<T, 2, FCLSH_FE4_MINB, 4, true, false, false, true>, true)
                                      : go(k_query_warp_pf<T, 2, FCLSH_FE4_MINB, 4, true>, true);
        else if (fe == 8)
            pm ? go(k_query_warp_pf<T, 2, 4, 8, true, true>, true)
               : fsm ? go(k_query_warp_pf<T, 2, 4, 8, true>, true) : go(k_query_warp_pf<T, 2, 4, 8>);
        else if (wu == 4)
            go(k_query_warp_pf<T, 4, 3, 0>);
        else if (wu == 3)
            go(k_query_warp_pf<T, 3, 4, 0>);
        else
            go(k_query_warp_pf<T, 2, 5, 0>);
        return;
    }
    if (!shared_set) {
        auto kern = k_query_warp<T, LAYOUT, kFusedU>;
        static std::atomic<uint64_t> carved{0}; // devices whose carveout is set (per instantiation)
        const uint64_t bit = uint64_t(1) << (ix.device & 63);
        if (!(carved.load(std::memory_order_acquire) & bit)) {
            FCLSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
            carved.fetch_or(bit, std::memory_order_acq_rel);
        }
        const int per_sm = resident_ctas(kern, 256, 0, ix.device);
        const uint64_t grid = std::max<uint64_t>(
            1, std::min<uint64_t>((nq + 7) / 8, uint64_t(std::max(per_sm, 1)) * sm_count(ix.device)));
        launch_pdl(kern, unsigned(grid), 256, 0, s, qkeys, nq, uint32_t(ix.tables), view<T>(ix),
                   ix.rows.as<uint64_t>(), d_q, ix.row_words, radius, slot_cap, coll_q, cand_q, found_q, src_pos,
                   tmp_id, tmp_dist, ovf, ovf_cnt, qnext, tile_sum, desc);
        FCLSH_LAUNCHED();
        return;
    }
    auto kern = k_query_fused<T, LAYOUT, CAP, kFusedU>;
    const size_t smem = (8 + size_t(8) * CAP) * 4; // CAP = set slots per warp
    const int per_sm = resident_ctas(kern, 256, smem, ix.device);
    const uint64_t grid =
        std::max<uint64_t>(1, std::min<uint64_t>((nq + 7) / 8, uint64_t(std::max(per_sm, 1)) * sm_count(ix.device)));
    launch_pdl(kern, unsigned(grid), 256, smem, s, qkeys, nq, uint32_t(ix.tables), view<T>(ix),
               ix.rows.as<uint64_t>(), d_q, ix.row_words, radius, slot_cap, coll_q, cand_q, found_q, src_pos, tmp_id,
               tmp_dist, ovf, ovf_cnt, qnext, tile_sum, desc);
    FCLSH_LAUNCHED();
}

// CTA-kernel shapes (id-set slots: < 3/4 of them distinct candidates; found
// list; threads; CTAs per SM). Big: the warp kernel's hand-over (its heavy
// queries) and CSR indexes (the flattened probe phase wants many threads per
// query). Small: bucket indexes of > 600 tables, every query (cfg4's shards):
// more queries in flight per SM hide the per-query barriers better -- one
// 1.25M-point cfg4 shard 0.377 -> 0.298 ms per 10k batch; queries beyond its
// set or list go on to the general path (profiles/r02/cfg4_dense.md).
struct DenseBig {
    static constexpr int HS = 8192, FCAP = 2048, NT = 512, MINB = 2;
};
struct DenseSmall {
    static constexpr int HS = 2048, FCAP = 1024, NT = 128, MINB = 8;
};

template <typename T, int LAYOUT, typename S>
void launch_dense(DeviceIndex& ix, const typename T::K* qkeys, const uint64_t* d_q, uint32_t radius,
                const uint32_t* ovf, const unsigned int* ovf_cnt, uint64_t direct_n, unsigned long long* coll_q,
                unsigned long long* cand_q, unsigned long long* found_q, unsigned long long* src_pos,
                uint64_t src_base, uint32_t* res_id, uint32_t* res_dist, uint64_t res_cap,
                unsigned long long* res_cursor, uint32_t* ovf2, unsigned int* ovf2_cnt, unsigned int* qnext,
                uint64_t max_grid, unsigned long long* tile_sum, const unsigned long long* desc, uint64_t nq_all,
                uint32_t slot_cap, uint32_t* slot_id, uint32_t* slot_dist, cudaStream_t s) {
    auto kern = k_query_dense<T, LAYOUT, S::HS, S::FCAP, S::NT, S::MINB>;
    const size_t smem = size_t(S::FCAP) * 8 + size_t(S::HS) * 4 + size_t(S::HS) / 4 * 3 * 2 +
                        (LAYOUT == kLayoutCsr ? kFlatSmem : 0);
    const int per_sm = resident_ctas(kern, S::NT, smem, ix.device);
    // persistent grid: the overflow count is only known on the device
    uint64_t grid = uint64_t(std::max(per_sm, 1)) * sm_count(ix.device);
    if (!ovf) grid = std::max<uint64_t>(1, std::min(grid, direct_n));
    else grid = std::max<uint64_t>(1, std::min(grid, max_grid)); // sized by the last batch's hand-over
    launch_pdl(kern, unsigned(grid), S::NT, smem, s, qkeys, uint32_t(ix.tables), view<T>(ix),
               ix.rows.as<uint64_t>(), d_q, ix.row_words, radius, ovf, ovf_cnt, uint32_t(direct_n), coll_q, cand_q,
               found_q, src_pos, src_base, res_id, res_dist, res_cap, res_cursor, ovf2, ovf2_cnt, qnext, tile_sum, desc,
               nq_all, slot_cap, slot_id, slot_dist, vec_for(ix.row_words, d_q));
    FCLSH_LAUNCHED();
}

// Spins until k_compact has published this batch's sequence number in mapped
// host memory (lower latency than a D2H copy + cudaStreamSynchronize). Polls
// the stream now and then so a device fault surfaces instead of hanging.
void wait_published(const unsigned long long* h_pub, unsigned long long seq, cudaStream_t s) {
    const volatile unsigned long long* flag = h_pub + 3;
    for (uint64_t it = 1; *flag != seq; ++it) {
        if ((it & 4095) == 0) {
            const cudaError_t e = cudaStreamQuery(s);
            if (e == cudaSuccess && *flag != seq) throw CudaError("query: batch results were not published");
            if (e != cudaSuccess && e != cudaErrorNotReady) FCLSH_CUDA(e);
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
}

// A batch's host destination (HostDest: counters, query, id, distance
// pointers and the block's capacity; zeros = device outputs only), passed by
// value to the prologue kernel.
struct DescVals {
    unsigned long long v[5];
};

// Batch prologue, one small CTA (first on the batch's stream, or on a side
// branch beside a separate hash kernel): clears
// the batch's counters (overflow counts, result cursor, hand-out counters,
// per-tile result sums) and writes the host destination to device memory for
// the query and compaction kernels. The destination arrives as a kernel
// argument that query_enqueue_impl patches into the replayed graph's node
// (cudaGraphExecKernelNodeSetParams), so one captured graph serves any
// destination without a host-to-device copy node on the critical path
// (a 40-byte memcpy node there cost ~3 us per batch; profiles/r02).
__global__ void k_batch_prologue(unsigned int* __restrict__ cnts, uint32_t words, unsigned long long* __restrict__ d_desc,
                                 DescVals dv) {
    pdl_trigger(); // (the query kernel's CTAs may launch; they wait for this grid to finish)
    pdl_wait();    // (and this one for whatever preceded it on the stream: the previous batch's kernels)
    FCLSH_TL_MIN(kTlProEntry);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) cnts[i] = 0;
    if (threadIdx.x < 5) d_desc[threadIdx.x] = dv.v[threadIdx.x];
    FCLSH_TL_MAX(kTlProExit);
}

// Every buffer a batch of nq queries touches, sized (grow-only) before any
// launch so that a captured graph never needs a reallocation. Called again by
// query_finish_impl: the same sizes return the same pointers.
template <typename T>
struct QueryBufs {
    using K = typename T::K;
    K* qkeys;
    unsigned long long *counters, *res_off, *coll_q, *cand_q, *found_q, *src_pos, *res_cursor, *tile_sum;
    uint32_t *tmp_id, *tmp_dist, *ovf, *ovf2, *cta_id, *cta_dist, *oq, *oi, *od;
    unsigned int* ovf_cnt;
    uint64_t ntiles, cta_cap, out_cap;
    size_t scan_bytes;
    void* scan_tmp;
};
constexpr uint32_t kSlotCap = 32; // results per query in the warp kernel's slots

template <typename T>
QueryBufs<T> query_bufs(DeviceIndex& ix, uint64_t nq, cudaStream_t s) {
    using K = typename T::K;
    QueryBufs<T> b;
    const uint64_t T_ = ix.tables;
    b.qkeys = static_cast<K*>(ix.q_keys.ensure(std::max<uint64_t>(1, nq * T_) * sizeof(K)));
    // per-query outputs in one block [offsets | collisions | candidates | found],
    // nq + 1 words each, so a host caller reads them back with one copy
    b.counters = static_cast<unsigned long long*>(ix.counters.ensure(4 * (nq + 1) * 8));
    b.res_off = b.counters;
    b.coll_q = b.counters + (nq + 1);
    b.cand_q = b.counters + 2 * (nq + 1);
    b.found_q = b.counters + 3 * (nq + 1);
    b.src_pos = static_cast<unsigned long long*>(ix.src_pos.ensure((nq + 1) * 8));
    b.tmp_id = static_cast<uint32_t*>(ix.res_tmp_id.ensure(std::max<uint64_t>(1, nq * kSlotCap) * 4));
    b.tmp_dist = static_cast<uint32_t*>(ix.res_tmp_dist.ensure(std::max<uint64_t>(1, nq * kSlotCap) * 4));
    b.ovf = static_cast<uint32_t*>(ix.overflow.ensure(std::max<uint64_t>(1, nq) * 4));
    b.ovf2 = static_cast<uint32_t*>(ix.overflow2.ensure(std::max<uint64_t>(1, nq) * 4));
    // counters: [0] warp-kernel overflow count, [1] CTA-kernel overflow
    // count, bytes 8..15: the CTA kernel's result cursor, [5]: next
    // query to hand out in the CTA kernel, [8]: k_scan_compact CTAs done;
    // from byte 64 the warp kernel's kQCtr query counters (256 B apart), from
    // byte kCntHeader the results per tile of 1024 queries, added by the
    // query kernels for k_scan_compact. The batch prologue clears all of it.
    b.ntiles = (nq + (uint64_t(1) << kScanTileLog) - 1) >> kScanTileLog;
    b.ovf_cnt = static_cast<unsigned int*>(ix.overflow_cnt.ensure(kCntHeader + std::max<uint64_t>(1, b.ntiles) * 8));
    b.res_cursor = reinterpret_cast<unsigned long long*>(b.ovf_cnt + 2);
    b.tile_sum = reinterpret_cast<unsigned long long*>(b.ovf_cnt + kCntHeader / 4);
    // CTA-kernel result region; queries that do not fit go on to the general path
    b.cta_cap = std::max<uint64_t>(uint64_t(1) << 21, nq * kSlotCap);
    b.cta_id = static_cast<uint32_t*>(ix.res_cta_id.ensure(b.cta_cap * 4));
    b.cta_dist = static_cast<uint32_t*>(ix.res_cta_dist.ensure(b.cta_cap * 4));
    b.out_cap = std::max<uint64_t>(1, nq * kSlotCap + b.cta_cap); // CTA results <= cta_cap
    b.oq = static_cast<uint32_t*>(ix.out_q.ensure(b.out_cap * 4));
    b.oi = static_cast<uint32_t*>(ix.out_id.ensure(b.out_cap * 4));
    b.od = static_cast<uint32_t*>(ix.out_dist.ensure(b.out_cap * 4));
    b.scan_bytes = 0;
    FCLSH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b.scan_bytes, b.found_q, b.res_off, nq + 1, s));
    b.scan_tmp = ix.cub_tmp.ensure(b.scan_bytes);
    return b;
}

// Phase 1 of a batch: enqueue the common path (replayed as a CUDA graph once
// the shape repeats) on the index's stream and return without waiting.
template <typename T, int LAYOUT>
void query_enqueue_impl(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, cudaStream_t s,
                        const HostDest* dest, const uint64_t* hash_src) {
    using K = typename T::K;
    const uint64_t T_ = ix.tables;
    const bool big = T_ > 600;
    const uint32_t slot_cap = kSlotCap;
    const QueryBufs<T> b = query_bufs<T>(ix, nq, s);
    K* const qkeys = b.qkeys;
    for (auto& e : ix.ev)
        if (!e) FCLSH_CUDA(cudaEventCreate(&e));
    // CTAs for the hand-over: most batches hand nothing over, and an idle
    // full grid still costs ~4 us; a batch handing over more than the last
    // one did still completes (queries are handed out dynamically)
    const uint64_t dense_grid = std::max<uint64_t>(32, 2 * ix.last_dense);
    // Many tables (cfg4: 1022): the CTA kernel for every query (a warp per
    // query with a shared id set measured slower there: one 1.25M-point
    // shard 0.44 vs 0.38 ms per 10k batch, the shared-memory atomics and run
    // walks serialise inside a warp; profiles/r02/cfg4_dense.md).
    const bool dense_all = big;
    if (!ix.h_pub) {
        // [0] total, [1] [2] overflow counts, [3] sequence
        FCLSH_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ix.h_pub), 128, cudaHostAllocMapped));
        FCLSH_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ix.d_pub), ix.h_pub, 0));
        std::memset(ix.h_pub, 0, 128);
        FCLSH_CUDA(cudaMemset(ix.pub_seq_dev.ensure(64), 0, 64)); // [0] sequence, [1..5] HostDest
        FCLSH_CUDA(cudaStreamCreateWithFlags(&ix.side, cudaStreamNonBlocking));
        FCLSH_CUDA(cudaEventCreateWithFlags(&ix.ev_fork, cudaEventDisableTiming));
        FCLSH_CUDA(cudaEventCreateWithFlags(&ix.ev_join, cudaEventDisableTiming));
        ix.pub_seq = 0;
    }
    auto* d_seq = ix.pub_seq_dev.as<unsigned long long>();
    // The common path: S1 hash (point-major key[q*T + t]), S2+S3 fused warp
    // per query, the CTA-per-query kernel for what it hands over (count read
    // on the device) or for every query, found scan, compaction + publish.
    bool capturing = false;
    // FCLSH_DEBUG_SYNC=1: synchronize and report after every stage (eager
    // batches only) to find a stage that faults or does not finish
    static const bool debug_sync = getenv("FCLSH_DEBUG_SYNC") != nullptr;
    const bool timing = ix.stage_timing;
    auto rec = [&](int k) { // stage events; inside a capture they must be external record nodes
        // (each costs ~4 us in a replayed graph: none unless stage timing is on)
        if (!timing) return;
        FCLSH_CUDA(capturing ? cudaEventRecordWithFlags(ix.ev[k], s, cudaEventRecordExternal)
                             : cudaEventRecord(ix.ev[k], s));
        if (debug_sync && !capturing) {
            FCLSH_CUDA(cudaStreamSynchronize(s));
            fprintf(stderr, "[fclsh] query nq=%llu stage %d reached\n", (unsigned long long)nq, k);
        }
    };
    const unsigned long long* d_desc = d_seq + 1;
    // the host destination for this batch (written to d_desc by the prologue,
    // read by the query kernels and k_scan_compact at run time, so a replayed
    // graph serves any destination)
    const bool host_cnt = nq && dest && dest->counters;
    DescVals dv{};
    if (host_cnt) {
        dv.v[0] = reinterpret_cast<uintptr_t>(dest->counters);
        dv.v[1] = reinterpret_cast<uintptr_t>(dest->q);
        dv.v[2] = reinterpret_cast<uintptr_t>(dest->id);
        dv.v[3] = reinterpret_cast<uintptr_t>(dest->dist);
        dv.v[4] = dest->cap;
    }
    cudaGraphNode_t prologue_node = nullptr;
    auto enqueue_common = [&] {
        rec(0);
        // hash_src (mapped pinned host rows): hashed from there, copied to d_q on
        // the way; with the hash fused into the query kernel it does both
        const bool fused_hash = !big && fused_fe(ix) > 0;
        // the prologue: with the hash fused, first on the batch's stream (the
        // query kernel follows it by PDL); else on a side branch beside the
        // hash kernel, joined before the query kernel
        const bool on_s = fused_hash;
        cudaStream_t ps = on_s ? s : ix.side;
        if (!on_s) {
            FCLSH_CUDA(cudaEventRecord(ix.ev_fork, s));
            FCLSH_CUDA(cudaStreamWaitEvent(ix.side, ix.ev_fork, 0));
        }
        launch_pdl(k_batch_prologue, 1, 256, 0, ps, b.ovf_cnt, uint32_t((kCntHeader + b.ntiles * 8) / 4),
                   const_cast<unsigned long long*>(d_desc), dv);
        FCLSH_LAUNCHED();
        if (capturing) { // its node, for the per-launch destination patch
            cudaStreamCaptureStatus st;
            const cudaGraphNode_t* deps = nullptr;
            size_t ndeps = 0;
            FCLSH_CUDA(cudaStreamGetCaptureInfo(ps, &st, nullptr, nullptr, &deps, &ndeps));
            if (ndeps != 1) throw CudaError("query: prologue node not found in the capture");
            prologue_node = deps[0];
        }
        if (!on_s) FCLSH_CUDA(cudaEventRecord(ix.ev_join, ix.side));
        if (!fused_hash) {
            hash_rows(*ix.fs, hash_src ? hash_src : d_q, nq, qkeys, sizeof(K), T_, kLayoutPointMajor, s, 0, 0,
                      hash_src ? const_cast<uint64_t*>(d_q) : nullptr);
        }
        rec(1);
        if (!on_s) FCLSH_CUDA(cudaStreamWaitEvent(s, ix.ev_join, 0));
        if (!dense_all)
            launch_fused<T, LAYOUT, kFusedCap>(ix, qkeys, d_q, nq, radius, slot_cap, b.coll_q, b.cand_q, b.found_q,
                                               b.src_pos, b.tmp_id, b.tmp_dist, b.ovf, b.ovf_cnt, b.ovf_cnt + 16,
                                               b.tile_sum, d_desc, s, fused_hash ? hash_src : nullptr);
        rec(2);
        auto dense = [&](auto shape) {
            launch_dense<T, LAYOUT, decltype(shape)>(ix, qkeys, d_q, radius, dense_all ? nullptr : b.ovf, b.ovf_cnt,
                                                     nq, b.coll_q, b.cand_q, b.found_q, b.src_pos, nq * slot_cap,
                                                     b.cta_id, b.cta_dist, b.cta_cap, b.res_cursor, b.ovf2,
                                                     b.ovf_cnt + 1, b.ovf_cnt + 5, dense_grid, b.tile_sum, d_desc, nq,
                                                     slot_cap, b.tmp_id, b.tmp_dist, s);
        };
        if constexpr (LAYOUT == kLayoutBuckets) {
            if (dense_all)
                dense(DenseSmall{});
            else
                dense(DenseBig{});
        } else {
            dense(DenseBig{});
        }
        rec(3);
        rec(4); // (one kernel: scan, offsets, compaction, publish)
        launch_pdl(k_scan_compact, unsigned(b.ntiles * kScanSplit + 1), 1u << kScanTileLog, 0, s, nq,
                   static_cast<const unsigned long long*>(b.found_q), static_cast<const unsigned long long*>(b.tile_sum),
                   b.res_off, static_cast<const unsigned long long*>(b.src_pos),
                   static_cast<const uint32_t*>(b.tmp_id), static_cast<const uint32_t*>(b.tmp_dist), nq * slot_cap,
                   static_cast<const uint32_t*>(b.cta_id), static_cast<const uint32_t*>(b.cta_dist), ix.id_offset,
                   b.oq, b.oi, b.od, ix.d_pub, d_seq, b.ovf_cnt, static_cast<const unsigned long long*>(b.coll_q),
                   static_cast<const unsigned long long*>(b.cand_q), d_desc);
        FCLSH_LAUNCHED();
        rec(5);
    };
    // the host destination for this batch (read by k_scan_compact at run time,
    // so a replayed graph serves any destination)

#ifdef FCLSH_TRACE
    {
        static DevBuf tbuf; // (trace builds: single-threaded tools only)
        void* tp = tbuf.ensure(std::max<uint64_t>(1, nq) * 128);
        FCLSH_CUDA(cudaMemsetAsync(tp, 0, std::max<uint64_t>(1, nq) * 128, s));
        FCLSH_CUDA(cudaMemcpyToSymbolAsync(g_trace, &tp, sizeof(tp), 0, cudaMemcpyHostToDevice, s));
        static const unsigned long long tl0[16] = {~0ull, 0, ~0ull, 0, ~0ull, 0, ~0ull, ~0ull, 0, ~0ull, ~0ull, 0, 0, 0, 0};
        FCLSH_CUDA(cudaMemcpyToSymbolAsync(g_tl, tl0, sizeof(tl0), 0, cudaMemcpyHostToDevice, s));
    }
#endif
    DeviceIndex::Pending& p = ix.pending;
    p.nq = nq;
    p.radius = radius;
    p.d_q = d_q;
    p.host_cnt = host_cnt;
    p.dest_cap = host_cnt ? dest->cap : 0;
    p.dense_all = dense_all;
    if (nq) {
        // A shape seen twice in a row (same rows pointer, batch size, radius,
        // stream and workspace) is captured once into a CUDA graph and
        // relaunched: one host call instead of ~10 launches per batch.
        const std::vector<const void*> key = {d_q, reinterpret_cast<const void*>(nq),
                                              reinterpret_cast<const void*>(uintptr_t(radius)), s, qkeys, b.coll_q,
                                              b.cand_q, b.found_q, b.res_off, b.src_pos, b.tmp_id, b.tmp_dist, b.ovf,
                                              b.ovf2, b.ovf_cnt, b.cta_id, b.cta_dist, b.oq, b.oi, b.od, b.scan_tmp,
                                              ix.d_pub, d_seq, reinterpret_cast<const void*>(uintptr_t(timing)),
                                              reinterpret_cast<const void*>(uintptr_t(dense_grid)), b.tile_sum,
                                              hash_src};
        auto patch_prologue = [&] {
            unsigned int* a0 = b.ovf_cnt;
            uint32_t a1 = uint32_t((kCntHeader + b.ntiles * 8) / 4);
            unsigned long long* a2 = const_cast<unsigned long long*>(d_desc);
            void* args[] = {&a0, &a1, &a2, &dv};
            cudaKernelNodeParams kp = {};
            kp.func = reinterpret_cast<void*>(k_batch_prologue);
            kp.gridDim = dim3(1);
            kp.blockDim = dim3(256);
            kp.sharedMemBytes = 0;
            kp.kernelParams = args;
            kp.extra = nullptr;
            FCLSH_CUDA(cudaGraphExecKernelNodeSetParams(ix.gexec, ix.gprologue, &kp));
        };
        if (ix.gexec && key == ix.gkey) {
            patch_prologue();
            FCLSH_CUDA(cudaGraphLaunch(ix.gexec, s));
            launch_counter() += ix.gkernels;
        } else if (key == ix.gpending) {
            const uint64_t before = launch_counter();
            cudaGraph_t g = nullptr;
            FCLSH_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            capturing = true;
            try {
                enqueue_common();
            } catch (...) {
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            capturing = false;
            FCLSH_CUDA(cudaStreamEndCapture(s, &g));
            ix.gkernels = launch_counter() - before;
            launch_counter() = before;
            if (ix.gexec) {
                cudaGraphExecDestroy(ix.gexec);
                ix.gexec = nullptr;
            }
            if (ix.gsrc) {
                cudaGraphDestroy(ix.gsrc);
                ix.gsrc = nullptr;
            }
            const cudaError_t ie = cudaGraphInstantiate(&ix.gexec, g, 0);
            if (ie != cudaSuccess) cudaGraphDestroy(g);
            FCLSH_CUDA(ie);
            ix.gsrc = g; // kept: gprologue is one of its nodes
            ix.gprologue = prologue_node;
            ix.gkey = key;
            FCLSH_CUDA(cudaGraphLaunch(ix.gexec, s));
            launch_counter() += ix.gkernels;
        } else {
            enqueue_common();
            ix.gpending = key;
        }
        p.seq = ++ix.pub_seq;
    } else {
        FCLSH_CUDA(cudaMemsetAsync(b.res_off, 0, 8, s)); // offsets = [0]
        for (int e = 0; e < 6; ++e) FCLSH_CUDA(cudaEventRecord(ix.ev[e], s));
    }
}

// Phase 2: wait until the batch published its total (mapped host memory),
// run the general path for what both query kernels handed over, and return
// the outputs.
template <typename T, int LAYOUT>
QueryOutput query_finish_impl(DeviceIndex& ix) {
    DeviceIndex::Pending& p = ix.pending;
    const uint64_t nq = p.nq;
    const uint32_t radius = p.radius;
    const uint64_t* d_q = p.d_q;
    cudaStream_t s = ix.stream;
    const uint64_t T_ = ix.tables;
    const uint32_t slot_cap = kSlotCap;
    QueryBufs<T> b = query_bufs<T>(ix, nq, s);
    QueryOutput out;
    out.nq = nq;
    struct {
        unsigned long long total;
        unsigned int cnt[2];
    } hs{0, {0, 0}};
    if (nq) {
        wait_published(ix.h_pub, p.seq, s);
#ifdef FCLSH_TRACE
        if (const char* path = getenv("FCLSH_TRACE_OUT")) {
            unsigned long long* tp = nullptr;
            FCLSH_CUDA(cudaMemcpyFromSymbol(&tp, g_trace, sizeof(tp)));
            std::vector<unsigned long long> h(nq * 16);
            FCLSH_CUDA(cudaMemcpy(h.data(), tp, nq * 128, cudaMemcpyDeviceToHost));
            if (FILE* f = fopen(path, "ab")) {
                const unsigned long long hdr[2] = {nq, 16};
                fwrite(hdr, 8, 2, f);
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
            }
        }
        if (const char* path = getenv("FCLSH_TL_OUT")) {
            unsigned long long tl[16];
            FCLSH_CUDA(cudaMemcpyFromSymbol(tl, g_tl, sizeof(tl)));
            if (FILE* f = fopen(path, "a")) {
                fprintf(f, "nq=%llu", (unsigned long long)nq);
                for (int k = 0; k < kTlSlots; ++k)
                    fprintf(f, " %.2f", tl[k] == ~0ull || tl[k] == 0 ? -1.0 : (double(tl[k]) - double(tl[0])) / 1e3);
                fprintf(f, "\n");
                fclose(f);
            }
        }
#endif
        hs.total = ix.h_pub[0];
        hs.cnt[0] = unsigned(ix.h_pub[1]);
        hs.cnt[1] = unsigned(ix.h_pub[2]);
    }
    const unsigned int ns = hs.cnt[1];
    const uint32_t* ovf = b.ovf2; // what the CTA kernel could not take
    unsigned long long total = hs.total;
    if (ns) {
        // general path for the overflowing queries
        const uint64_t pairs = uint64_t(ns) * T_;
        const Tables<T> tb = view<T>(ix);
        auto* coll_s = static_cast<unsigned long long*>(ix.coll_sel.ensure((ns + 1) * 8));
        auto* coll_off = static_cast<unsigned long long*>(ix.coll_off.ensure((ns + 1) * 8));
        auto* fill = static_cast<unsigned long long*>(ix.fill.ensure((ns + 1) * 8));
        FCLSH_CUDA(cudaMemsetAsync(coll_s, 0, (ns + 1) * 8, s));
        FCLSH_CUDA(cudaMemsetAsync(fill, 0, (ns + 1) * 8, s));
        k_count_sel<T, LAYOUT><<<grid_for(pairs, ix.device), 256, 0, s>>>(b.qkeys, ovf, ns, uint32_t(T_), tb, coll_s);
        FCLSH_LAUNCHED();
        size_t tb_bytes = 0;
        FCLSH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb_bytes, coll_s, coll_off, ns + 1, s));
        FCLSH_CUDA(cub::DeviceScan::ExclusiveSum(ix.cub_tmp2.ensure(tb_bytes), tb_bytes, coll_s, coll_off, ns + 1, s));
        unsigned long long total_coll = 0;
        FCLSH_CUDA(cudaMemcpyAsync(&total_coll, coll_off + ns, 8, cudaMemcpyDeviceToHost, s));
        FCLSH_CUDA(cudaStreamSynchronize(s));
        uint32_t* cand = static_cast<uint32_t*>(ix.cand.ensure(std::max<uint64_t>(1, total_coll) * 4));
        uint32_t* sorted = static_cast<uint32_t*>(ix.cand_sorted.ensure(std::max<uint64_t>(1, total_coll) * 4));
        uint32_t* tmp2_id = static_cast<uint32_t*>(ix.res2_id.ensure(std::max<uint64_t>(1, total_coll) * 4));
        uint32_t* tmp2_dist = static_cast<uint32_t*>(ix.res2_dist.ensure(std::max<uint64_t>(1, total_coll) * 4));
        if (total_coll) {
            k_gather_sel<T, LAYOUT><<<grid_for(pairs, ix.device), 256, 0, s>>>(b.qkeys, ovf, ns, uint32_t(T_), tb,
                                                                                coll_off, fill, cand);
            FCLSH_LAUNCHED();
            size_t sb = 0;
            FCLSH_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, sb, cand, sorted, int64_t(total_coll), int64_t(ns),
                                                          coll_off, coll_off + 1, s));
            FCLSH_CUDA(cub::DeviceSegmentedSort::SortKeys(ix.cub_tmp2.ensure(sb), sb, cand, sorted,
                                                          int64_t(total_coll), int64_t(ns), coll_off, coll_off + 1, s));
        }
        k_verify_sel<<<grid_for(uint64_t(ns) * 32, ix.device), 256, 0, s>>>(
            ns, ovf, coll_off, sorted, ix.rows.as<uint64_t>(), d_q, ix.row_words, radius, nq * slot_cap + b.cta_cap,
            tmp2_id, tmp2_dist, b.coll_q, b.cand_q, b.found_q, b.src_pos);
        FCLSH_LAUNCHED();
        // the overflowing queries' counts are in now: scan and compact again
        FCLSH_CUDA(cudaMemsetAsync(b.found_q + nq, 0, 8, s));
        FCLSH_CUDA(cub::DeviceScan::ExclusiveSum(b.scan_tmp, b.scan_bytes, b.found_q, b.res_off, nq + 1, s));
        FCLSH_CUDA(cudaMemcpyAsync(&hs.total, b.res_off + nq, 8, cudaMemcpyDeviceToHost, s));
        FCLSH_CUDA(cudaStreamSynchronize(s));
        total = hs.total;
        if (total > b.out_cap) {
            b.out_cap = total;
            b.oq = static_cast<uint32_t*>(ix.out_q.ensure(b.out_cap * 4));
            b.oi = static_cast<uint32_t*>(ix.out_id.ensure(b.out_cap * 4));
            b.od = static_cast<uint32_t*>(ix.out_dist.ensure(b.out_cap * 4));
        }
        k_compact<<<grid_for(nq * 32, ix.device), 256, 0, s>>>(
            nq, b.src_pos, b.res_off, b.tmp_id, b.tmp_dist, nq * slot_cap, b.cta_id, b.cta_dist, b.cta_cap, tmp2_id,
            tmp2_dist, ix.id_offset, b.oq, b.oi, b.od, nullptr, ix.pub_seq_dev.as<unsigned long long>(), b.ovf_cnt);
        FCLSH_LAUNCHED();
    }
    FCLSH_CUDA(cudaEventRecord(ix.ev[6], s));
    out.total = total;
    out.d_query = ix.out_q.as<uint32_t>();
    out.d_id = ix.out_id.as<uint32_t>();
    out.d_dist = ix.out_dist.as<uint32_t>();
    out.d_offsets = reinterpret_cast<uint64_t*>(b.res_off);
    out.d_coll = reinterpret_cast<uint64_t*>(b.coll_q);
    out.d_cand = reinterpret_cast<uint64_t*>(b.cand_q);
    out.d_found = reinterpret_cast<uint64_t*>(b.found_q);
    // the general path rewrote counters and results in device memory
    out.host_counters = p.host_cnt && !ns;
    out.host_results = out.host_counters && total <= p.dest_cap;
    ix.last_total = total;
    ix.last_dense = p.dense_all ? nq : hs.cnt[0];
    ix.last_overflow = ns;
    p.active = false;
    return out;
}

} // namespace

namespace {
// Device-wide persisting-L2 limit (cudaLimitPersistingL2CacheSize) raised for
// the key filters of live indexes: the first index on a device records the
// limit it found, the last one to go restores it.
struct L2PersistState {
    int users = 0;
    size_t saved = 0;
};
std::mutex g_l2_mu;
L2PersistState g_l2[64];
} // namespace

bool l2_persist_acquire(int device, uint64_t bytes) {
    if (device < 0 || device >= 64) return false;
    int maxp = 0;
    if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device) != cudaSuccess || maxp <= 0) {
        cudaGetLastError();
        return false;
    }
    std::lock_guard<std::mutex> lk(g_l2_mu);
    L2PersistState& st = g_l2[device];
    size_t cur = 0;
    if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (st.users == 0) st.saved = cur;
    const size_t want = std::min<size_t>(size_t(maxp), size_t(bytes));
    if (cur < want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) cudaGetLastError();
    ++st.users;
    return true;
}

void l2_persist_release(int device) {
    if (device < 0 || device >= 64) return;
    std::lock_guard<std::mutex> lk(g_l2_mu);
    L2PersistState& st = g_l2[device];
    if (st.users <= 0) return;
    if (--st.users == 0) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, st.saved) != cudaSuccess) cudaGetLastError();
        cudaSetDevice(prev);
    }
}

DeviceIndex::~DeviceIndex() {
    if (l2_persist) l2_persist_release(device);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (gsrc) cudaGraphDestroy(gsrc);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (h_pub) cudaFreeHost(h_pub);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
}

std::unique_ptr<DeviceIndex> build_index(const uint64_t* rows, bool rows_on_device, uint64_t n, uint64_t dims,
                                         uint32_t radius, const Plan& plan, uint64_t rng_seed,
                                         const IndexBuildOptions& opt) {
    // index.cpp:51-53, 65-79
    if (n == 0) throw UsageError("index: empty dataset");
    if (dims != plan.dims) throw UsageError("index: dataset width does not match the plan");
    if (radius != plan.radius) throw UsageError("index: radius does not match the plan");
    if (opt.method != kMethodCovering && opt.method != kMethodClassic) throw UsageError("index: unknown method");
    const bool classic = opt.method == kMethodClassic;
    if (classic && plan.kind != PlanKind::identity)
        throw UsageError("index: the classic baseline expects the identity plan");
    const uint64_t classic_tables = opt.tables_override ? opt.tables_override : (uint64_t(1) << (radius + 1)) - 1;
    if ((classic ? classic_tables : plan.table_count()) > opt.table_budget)
        throw ResourceError("index: table count exceeds the budget");
    if (n + opt.id_offset > (uint64_t(1) << 32)) throw UsageError("index: ids must fit 32 bits");
    if (opt.layout < 0 || opt.layout > 2) throw UsageError("index: unknown table layout");

    auto ix = std::make_unique<DeviceIndex>();
    ix->device = opt.device;
    ix->plan = plan;
    ix->radius = radius;
    ix->n = n;
    ix->dims = dims;
    ix->row_words = uint32_t((dims + 63) / 64);
    ix->prime = opt.prime;
    ix->wide = opt.prime > 0xFFFFFFFFull;
    ix->id_offset = opt.id_offset;

    ix->method = opt.method;
    Rng rng(rng_seed);
    std::vector<Family> fams;
    BitSampleFamily bsf;
    if (classic) { // index.cpp:65-76: k from choose_k unless overridden, family stream ("family", 0)
        const uint32_t k = opt.k_override ? opt.k_override : choose_k(dims, radius, classic_tables, opt.delta);
        bsf = build_bit_sample_family(dims, k, classic_tables, rng.stream("family", 0).seed(), opt.prime);
    } else { // families per part from rng.stream("family", p) (index.cpp:83-88)
        for (uint32_t p = 0; p < plan.part_count(); ++p)
            fams.push_back(build_family(plan.part_dims(p), plan.per_part_radius, -1, rng.stream("family", p).seed(),
                                        opt.prime, opt.include_zero_column));
    }

    FCLSH_CUDA(cudaSetDevice(opt.device));
    FCLSH_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
    ix->fs = classic ? make_device_classic_set(bsf, opt.device) : make_device_family_set(plan, std::move(fams), opt.device);
    ix->tables = ix->fs->total_tables();

    const uint32_t kbits = bit_length(opt.prime - 1);
    const uint64_t W = ix->row_words;
    const uint64_t eb = ix->entry_bytes();
    // bucket table: 2^bb buckets of 4 slots, home = key >> (kbits - bb).
    // Preferred: 2^bb >= n (slot load <= 25%): a probe then needs the next
    // bucket (its home bucket full) ~3 % of the time instead of ~18 % at
    // 2^bb >= n/2 (load <= 50%), and each such continuation is a dependent
    // random read (cfg2: fused probe kernel 190 -> 168 us, 8.6 -> 17.2 GB).
    // The sparser table is taken when it fits in half the free memory.
    uint32_t bb = bit_length(std::max<uint64_t>(2, (n + 1) / 2) - 1);
    if (bb < 1) bb = 1;
    // slot load <= 50 %, and no more buckets than keys
    auto bkt_fits = [&](uint32_t bits) { return bits <= std::min<uint32_t>(kbits, 40) && (uint64_t(kSlots) << bits) > n; };
    auto bkt_size = [&](uint32_t bits) { return ix->tables * (uint64_t(1) << bits) * kSlots * eb; };
    // CSR directory: 2^b cells, about two postings per cell
    uint32_t b = opt.directory_bits > 0 ? uint32_t(opt.directory_bits)
                                        : std::max<uint32_t>(1, bit_length(n - 1) > 1 ? bit_length(n - 1) - 1 : 1);
    b = std::min<uint32_t>({b, kbits, 30u});
    const uint64_t csr_bytes = ix->tables * (n * eb + ((uint64_t(1) << b) + 1) * 4);
    int layout = opt.layout;
    {
        size_t free_b = 0, total_b = 0;
        FCLSH_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (opt.mem_budget) free_b = std::min<size_t>(free_b, opt.mem_budget); // (several shards on one GPU)
        // the build's transient buffers: one part's point-major keys + one
        // table-major slab of them
        const uint64_t kbytes = ix->wide ? 8 : 4;
        const uint64_t need_extra = n * W * 8 + ix->fs->tables * n * kbytes +
                                    std::min<uint64_t>(ix->fs->tables, std::max<uint64_t>(kBuildSlab, 64)) * n * kbytes +
                                    (uint64_t(2) << 30);
        // (a 50-75 % tier that fits cfg4's 10M points on one GPU in 137 GB
        // measured slower than CSR there: 2.34 vs 1.14 ms per 10k batch; at
        // that load a probe reads 2.25 buckets on average, p99 23, and the
        // runs are dependent reads; profiles/r02/cfg4_dense.md)
        if (layout != kLayoutCsr && bkt_fits(bb + 1) && bkt_size(bb + 1) + need_extra <= free_b / 2) ++bb; // load <= 25 %
        if (layout == kLayoutAuto)
            layout = (bkt_fits(bb) && bkt_size(bb) + need_extra <= free_b) ? kLayoutBuckets : kLayoutCsr;
    }
    const bool bkt_ok = bkt_fits(bb);
    if (layout == kLayoutBuckets && !bkt_ok)
        throw UsageError("index: bucket layout needs a key field wider than the bucket count");
    ix->layout = layout;
    if (layout == kLayoutBuckets) {
        ix->nbuckets = uint64_t(1) << bb;
        ix->key_shift = 64 - bb;
        ix->dir_bits = 0;
    } else {
        ix->dir_bits = b;
        ix->key_shift = 64 - b;
    }

    // key filter (buckets): FCLSH_FILTER_BPK bits per posting (default 1),
    // at most FCLSH_FILTER_MB (default 80) MiB in all so that it stays in L2;
    // below 3/4 bit per posting it rejects too few probes to pay for its own
    // read. FCLSH_FILTER=0: none.
    ix->filter_words = 0;
    ix->key_scale = ~0ull / opt.prime; // floor((2^64 - 1) / P) = floor(2^64 / P) for odd P
    if (layout == kLayoutBuckets && !(getenv("FCLSH_FILTER") && getenv("FCLSH_FILTER")[0] == '0')) {
        const double bpk = getenv("FCLSH_FILTER_BPK") ? atof(getenv("FCLSH_FILTER_BPK")) : 1.0;
        const double mb = getenv("FCLSH_FILTER_MB") ? atof(getenv("FCLSH_FILTER_MB")) : 80.0;
        const uint64_t cap_words = uint64_t(mb * 1048576.0 / 4.0) / ix->tables;
        const uint64_t want_words = (uint64_t(double(n) * bpk) + 31) / 32;
        const double min_bpk = getenv("FCLSH_FILTER_MIN") ? atof(getenv("FCLSH_FILTER_MIN")) : 0.75;
        const uint64_t words = std::min<uint64_t>({cap_words, want_words, uint64_t(1) << 26});
        if (words > 0 && double(words) * 32 >= double(n) * min_bpk) ix->filter_words = uint32_t(words);
    }
    try {
        ix->rows.ensure(n * W * 8);
        if (ix->filter_words) {
            const uint64_t fbytes = ix->tables * ix->filter_words * 4;
            ix->filter.ensure(fbytes);
            FCLSH_CUDA(cudaMemsetAsync(ix->filter.p, 0, fbytes, ix->stream));
            // room for the filter's evict_last lines in the persisting part of L2
            // (the device-wide limit is restored when the last index holding a
            // filter on this device is destroyed)
            ix->l2_persist = l2_persist_acquire(opt.device, fbytes);
        }
        if (layout == kLayoutBuckets) {
            ix->entries.ensure(bkt_size(bb));
        } else {
            ix->entries.ensure(ix->tables * n * eb);
            ix->dir.ensure(ix->tables * (ix->cells() + 1) * 4);
        }
    } catch (const CudaError& e) {
        throw ResourceError(std::string("index: device memory exhausted (") + e.what() + ")");
    }
    FCLSH_CUDA(cudaMemcpyAsync(ix->rows.p, rows, n * W * 8,
                               rows_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ix->stream));
    cudaEvent_t e0, e1;
    FCLSH_CUDA(cudaEventCreate(&e0));
    FCLSH_CUDA(cudaEventCreate(&e1));
    FCLSH_CUDA(cudaEventRecord(e0, ix->stream));
    if (ix->wide)
        build_all<WideEntry>(*ix);
    else
        build_all<NarrowEntry>(*ix);
    FCLSH_CUDA(cudaEventRecord(e1, ix->stream));
    FCLSH_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ix->build_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ix;
}

namespace {
constexpr int kCHSLog = 14, kCKCAP = 4096; // shared set slots (2^14) and cut-table ids of the budgeted query

__global__ void k_iota(uint32_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = uint32_t(i);
}

template <typename T, int LAYOUT>
void query_c_impl(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, uint64_t budget,
                  unsigned long long* counters, uint32_t* best, cudaStream_t s) {
    using K = typename T::K;
    const uint64_t T_ = ix.tables;
    K* qkeys = static_cast<K*>(ix.q_keys.ensure(std::max<uint64_t>(1, nq * T_) * sizeof(K)));
    auto* ctr = static_cast<unsigned int*>(ix.overflow_cnt.ensure(32)); // [6] hand-out, [7] errors
    hash_rows(*ix.fs, d_q, nq, qkeys, sizeof(K), T_, kLayoutPointMajor, s);
    auto kern = k_query_c<T, LAYOUT>;
    const size_t tbytes = ((T_ + 3) & ~uint64_t(3)) * 4;
    // shared mode: every distinct id of a walk fits the set at load <= 3/4
    if (budget <= (uint64_t(1) << kCHSLog) / 4 * 3 && T_ <= 16384) {
        FCLSH_CUDA(cudaMemsetAsync(ctr + 6, 0, 8, s));
        const size_t smem = tbytes + ((size_t(1) << kCHSLog) + kCKCAP) * 4;
        const int per_sm = resident_ctas(kern, 512, smem, ix.device);
        if (per_sm < 1) throw ResourceError("query_c_r_nn: too many tables for the device kernel");
        const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(nq, uint64_t(per_sm) * sm_count(ix.device)));
        kern<<<unsigned(grid), 512, smem, s>>>(qkeys, nq, uint32_t(T_), view<T>(ix), ix.rows.as<uint64_t>(), d_q,
                                              ix.row_words, radius, budget, counters, best, ctr + 6, ctr + 7,
                                              uint32_t(kCHSLog), uint32_t(kCKCAP), nullptr, ix.id_offset);
        FCLSH_LAUNCHED();
        unsigned int errs = 0;
        FCLSH_CUDA(cudaMemcpyAsync(&errs, ctr + 7, 4, cudaMemcpyDeviceToHost, s));
        FCLSH_CUDA(cudaStreamSynchronize(s));
        if (!errs) return;
        // a cut bucket longer than the shared buffer: the batch again in global mode
    }
    // Global mode (any budget, as the reference's std::optional<uint64_t>,
    // index.hpp:90-93): per-query collision totals bound the distinct ids of
    // a walk (<= min(budget, collisions)) and the cut bucket; every CTA gets
    // a global slice [set (load <= 1/2) | cut ids | inserted slots].
    uint32_t* sel = static_cast<uint32_t*>(ix.overflow.ensure(std::max<uint64_t>(1, nq) * 4));
    auto* coll = static_cast<unsigned long long*>(ix.coll_sel.ensure(std::max<uint64_t>(1, nq) * 8));
    k_iota<<<grid_for(nq, ix.device), 256, 0, s>>>(sel, nq);
    FCLSH_LAUNCHED();
    FCLSH_CUDA(cudaMemsetAsync(coll, 0, nq * 8, s));
    k_count_sel<T, LAYOUT><<<grid_for(nq * T_, ix.device), 256, 0, s>>>(qkeys, sel, nq, uint32_t(T_), view<T>(ix),
                                                                         coll);
    FCLSH_LAUNCHED();
    std::vector<unsigned long long> hc(nq);
    FCLSH_CUDA(cudaMemcpyAsync(hc.data(), coll, nq * 8, cudaMemcpyDeviceToHost, s));
    FCLSH_CUDA(cudaStreamSynchronize(s));
    uint64_t maxc = 1;
    for (auto c : hc) maxc = std::max<uint64_t>(maxc, c);
    const uint64_t maxd = std::min<uint64_t>(maxc, budget); // distinct ids of one walk
    if (maxd >= (uint64_t(1) << 30)) throw ResourceError("query_c_r_nn: walk too long for the device id set");
    uint32_t hs_log = 10;
    while ((uint64_t(1) << hs_log) < 2 * maxd) ++hs_log;
    const uint64_t HS = uint64_t(1) << hs_log;
    uint32_t kcap = 1;
    while (kcap < maxc && kcap < (uint32_t(1) << 31)) kcap <<= 1; // the cut bucket <= all collisions
    const uint64_t per_cta = (tbytes / 4 + HS + kcap + HS / 2) * 4;
    size_t free_b = 0, total_b = 0;
    FCLSH_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t fit = std::max<uint64_t>(1, (free_b / 2) / per_cta);
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>({nq, uint64_t(2) * sm_count(ix.device), fit}));
    DevBuf scratch;
    try {
        scratch.ensure(grid * per_cta);
    } catch (const CudaError& e) {
        throw ResourceError(std::string("query_c_r_nn: device memory exhausted (") + e.what() + ")");
    }
    FCLSH_CUDA(cudaMemsetAsync(ctr + 6, 0, 8, s));
    kern<<<unsigned(grid), 512, 0, s>>>(qkeys, nq, uint32_t(T_), view<T>(ix), ix.rows.as<uint64_t>(), d_q,
                                            ix.row_words, radius, budget, counters, best, ctr + 6, ctr + 7, hs_log,
                                            kcap, scratch.as<uint32_t>(), ix.id_offset);
    FCLSH_LAUNCHED();
    unsigned int errs = 0;
    FCLSH_CUDA(cudaMemcpyAsync(&errs, ctr + 7, 4, cudaMemcpyDeviceToHost, s));
    FCLSH_CUDA(cudaStreamSynchronize(s));
    if (errs) throw CudaError("query_c_r_nn: cut bucket exceeded its bound");
}
} // namespace

void query_c_device(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, int64_t posting_budget,
                    uint64_t* d_counters, uint32_t* d_best, cudaStream_t stream) {
    if (radius > ix.radius) // index.cpp:147-153 (check_query)
        throw UsageError("query radius " + std::to_string(radius) + " exceeds the index radius " +
                         std::to_string(ix.radius));
    const uint64_t budget = posting_budget < 0 ? 3 * ix.tables : uint64_t(posting_budget); // index.cpp:201
    if (nq == 0) return;
    FCLSH_CUDA(cudaSetDevice(ix.device));
    cudaStream_t s = stream ? stream : ix.stream;
    auto* c = reinterpret_cast<unsigned long long*>(d_counters);
    if (ix.wide) {
        if (ix.layout == kLayoutBuckets)
            query_c_impl<WideEntry, kLayoutBuckets>(ix, d_q, nq, radius, budget, c, d_best, s);
        else
            query_c_impl<WideEntry, kLayoutCsr>(ix, d_q, nq, radius, budget, c, d_best, s);
    } else {
        if (ix.layout == kLayoutBuckets)
            query_c_impl<NarrowEntry, kLayoutBuckets>(ix, d_q, nq, radius, budget, c, d_best, s);
        else
            query_c_impl<NarrowEntry, kLayoutCsr>(ix, d_q, nq, radius, budget, c, d_best, s);
    }
}

void query_enqueue(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, cudaStream_t stream,
                   const HostDest* dest, const uint64_t* hash_src) {
    if (radius > ix.radius) // index.cpp:147-153
        throw UsageError("query radius " + std::to_string(radius) + " exceeds the index radius " +
                         std::to_string(ix.radius));
    if (ix.pending.active) throw UsageError("query: the previous batch on this index was not finished");
    FCLSH_CUDA(cudaSetDevice(ix.device));
    // Work runs on the index's stream, ordered after / before the caller's.
    cudaStream_t s = ix.stream;
    const bool join = stream && stream != s;
    if (join) {
        for (auto* e : {&ix.ev_in, &ix.ev_out})
            if (!*e) FCLSH_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        FCLSH_CUDA(cudaEventRecord(ix.ev_in, stream));
        FCLSH_CUDA(cudaStreamWaitEvent(s, ix.ev_in, 0));
    }
    if (ix.wide) {
        if (ix.layout == kLayoutBuckets)
            query_enqueue_impl<WideEntry, kLayoutBuckets>(ix, d_q, nq, radius, s, dest, hash_src);
        else
            query_enqueue_impl<WideEntry, kLayoutCsr>(ix, d_q, nq, radius, s, dest, hash_src);
    } else {
        if (ix.layout == kLayoutBuckets)
            query_enqueue_impl<NarrowEntry, kLayoutBuckets>(ix, d_q, nq, radius, s, dest, hash_src);
        else
            query_enqueue_impl<NarrowEntry, kLayoutCsr>(ix, d_q, nq, radius, s, dest, hash_src);
    }
    ix.pending.active = true;
    ix.pending.caller = join ? stream : nullptr;
}

QueryOutput query_finish(DeviceIndex& ix) {
    if (!ix.pending.active) throw UsageError("query: no batch in flight on this index");
    FCLSH_CUDA(cudaSetDevice(ix.device));
    cudaStream_t caller = ix.pending.caller;
    QueryOutput o;
    try {
        if (ix.wide)
            o = ix.layout == kLayoutBuckets ? query_finish_impl<WideEntry, kLayoutBuckets>(ix)
                                            : query_finish_impl<WideEntry, kLayoutCsr>(ix);
        else
            o = ix.layout == kLayoutBuckets ? query_finish_impl<NarrowEntry, kLayoutBuckets>(ix)
                                            : query_finish_impl<NarrowEntry, kLayoutCsr>(ix);
    } catch (...) {
        ix.pending.active = false;
        throw;
    }
    if (caller) {
        FCLSH_CUDA(cudaEventRecord(ix.ev_out, ix.stream));
        FCLSH_CUDA(cudaStreamWaitEvent(caller, ix.ev_out, 0));
    }
    ix.stages_pending = true;
    ix.stages_timed = ix.stage_timing;
    return o;
}

QueryOutput query_device(DeviceIndex& ix, const uint64_t* d_q, uint64_t nq, uint32_t radius, cudaStream_t stream,
                         const HostDest* dest, const uint64_t* hash_src) {
    query_enqueue(ix, d_q, nq, radius, stream, dest, hash_src);
    return query_finish(ix);
}

void DeviceIndex::collect_stages() {
    if (!stages_pending) return;
    FCLSH_CUDA(cudaEventSynchronize(ev[kStages]));
    batch_ms = -1; // not measured (stage timing off: the events cost ~2 % of a cfg2 batch)
    for (int i = 0; i < kStages; ++i) stage_ms[i] = -1;
    for (int i = 0; i < kStages && stages_timed; ++i) {
        float ms = 0;
        FCLSH_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        stage_ms[i] = ms;
    }
    if (stages_timed) {
        float total = 0;
        FCLSH_CUDA(cudaEventElapsedTime(&total, ev[0], ev[5]));
        batch_ms = total;
        t_hash_ms = stage_ms[0];
        t_probe_ms = stage_ms[1] + stage_ms[2] + stage_ms[5]; // probe + dedup + verify are fused
        t_verify_ms = stage_ms[3] + stage_ms[4];              // result assembly
    } else {
        t_hash_ms = t_probe_ms = t_verify_ms = -1;
    }
    stages_pending = false;
}

} // namespace fclsh_b200
