// K1 -- batched fcLSH covering hash for sm_100a.
//
// Reference semantics (hash_batch_into, covering.cpp:169-182 and
// batch_hash_kernel, hadamard.cpp:66-72): per row, scatter the seeds of set
// bits onto their code columns (sketch t), run an N-point Hadamard transform
// mod P, map x -> (l1 - x)/2 mod P and drop entry 0. Equivalently
//     key[v] = sum_{c : popcount(v & c) odd} t[c]   (mod P),  v = 1..N-1.
//
// Fast path (P = 2^31 - 1, the 32-bit-key field of the BASELINE configs):
// exact integer arithmetic, reduced once at the end. Seeds are split into a
// 16-bit plane and a 15-bit plane; the signed transform F of each plane fits
// int32 (|F| <= sum of the plane <= d' * 2^16 < 2^31 for d' <= 2^15), so the
// butterflies are single 32-bit adds with no modular reduction. Finally
//     O = (F[0] - F[v]) / 2  per plane,   key = (O_lo + 2^16 O_hi) mod P,
// which is the canonical residue the reference stores (bit-exact).
//
// Work decomposition (N = 2^LOGN): G lanes cooperate on one row, each lane
// holding E = N/G elements per plane in registers. Phase 1 runs log2(E)
// butterfly stages in registers, one swizzled shared-memory transpose
// (warp-local, __syncwarp only) regroups the elements, phase 2 runs the
// remaining log2(G) stages in registers. Keys are staged in shared memory
// and written with 16-byte stores so every table row receives full 32-byte
// sectors (table-major layout) -- the pass is a pure stream: rows in, keys
// out, no re-reads. A CTA owns PT = 256/G rows per tile; the grid is
// persistent over tiles.
//
// Generic path (any odd P < 2^63, u64 keys, any N): one CTA per row, mod-P
// butterflies in shared/global memory exactly as the reference sequences
// them. Used for the M61 default field and the small-prime golden tests.

#include "hash.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace fclsh_b200 {

namespace {

constexpr uint32_t kP31 = 0x7FFFFFFFu;
constexpr int kMaxParts = 32;

// lanes per row for a given LOGN
__host__ __device__ constexpr int lanes_for(int logn) {
    return logn <= 5 ? 1 : (logn <= 7 ? 8 : (logn <= 9 ? 16 : 32));
}

struct FastParams {
    const uint64_t* rows;
    uint64_t n;
    uint32_t row_words;
    uint32_t parts;
    uint32_t part_words;   // uint2 per part in fam
    uint32_t lane_entries; // M (general path)
    const uint2* fam;
    uint64_t* rows_copy; // optional: every row also written here (k_hash_f64_pt)
    void* keys;
    uint64_t key_stride;
    uint64_t L;
    int layout;
    int key_bytes;
};

template <int SIZE>
__device__ __forceinline__ void fht_signed(uint32_t* x) {
#pragma unroll
    for (int h = 1; h < SIZE; h <<= 1) {
#pragma unroll
        for (int i = 0; i < SIZE; ++i) {
            if ((i & h) == 0) {
                uint32_t a = x[i], b = x[i + h];
                x[i] = a + b;
                x[i + h] = a - b;
            }
        }
    }
}

// (O_lo + 2^16 * O_hi) mod (2^31-1), canonical. O_lo = (Tlo - Flo)/2 < 2^31,
// O_hi = (Thi - Fhi)/2 < 2^30.
__device__ __forceinline__ uint32_t finish_key(uint32_t Tlo, uint32_t Thi, uint32_t Flo, uint32_t Fhi) {
    uint32_t slo = (Tlo - Flo) >> 1;
    uint32_t shi = (Thi - Fhi) >> 1;
    // 2^16 * shi = (shi >> 15) * 2^31 + (shi & 0x7fff) * 2^16 == (shi >> 15) + ((shi & 0x7fff) << 16)
    uint32_t s = slo + (shi >> 15) + ((shi & 0x7FFFu) << 16); // < 2^32
    s = (s & kP31) + (s >> 31);                               // <= 2^31
    uint32_t s1 = s + 1;
    return (s1 & kP31) + (s1 >> 31) - 1;                      // canonical in [0, P)
}

__device__ __forceinline__ uint32_t row_bit(const uint32_t* row32, uint32_t pos) {
    return (row32[pos >> 5] >> (pos & 31)) & 1u;
}

// staging swizzle for slot s (see the store loop): spreads the PT/4 slot
// groups read by one warp over disjoint bank ranges
template <int PT>
__device__ __forceinline__ uint32_t stage_swz(uint32_t s) {
    constexpr int M = PT / 4;
    constexpr int V = 32 / M;
    return (((s >> 2) & (M - 1)) * V) ^ ((s & 3) << 4);
}

template <int LOGN, bool DIRECT>
__global__ void __launch_bounds__(256) k_hash_m31(const FastParams p) {
    constexpr int N = 1 << LOGN;
    constexpr int G = lanes_for(LOGN);
    constexpr int E = N / G;
    constexpr int PT = 256 / G;
    constexpr int EG = (G > 1) ? E / G : 1;
    static_assert(G == 1 || EG == 1 || EG == 2, "phase-2 layout");

    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* xbuf = reinterpret_cast<uint64_t*>(smem);    // 256 * E u64
    uint64_t* rows_s = xbuf + 256 * E;                      // PT * row_words u64
    uint2* fam_s = reinterpret_cast<uint2*>(rows_s + PT * p.row_words);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int slot = tid / G;
    const int g = tid % G;

    for (uint32_t i = tid; i < p.parts * p.part_words; i += 256) fam_s[i] = p.fam[i];

    const uint64_t ntiles = (p.n + PT - 1) / PT;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t p0 = tile * PT;
        __syncthreads(); // previous tile done with rows_s / xbuf; fam_s staged
        {
            const uint64_t base = p0 * p.row_words;
            const uint64_t lim = p.n * p.row_words;
            for (uint32_t i = tid; i < PT * p.row_words; i += 256)
                rows_s[i] = (base + i < lim) ? __ldg(p.rows + base + i) : 0ull;
        }
        __syncthreads();
        const uint32_t* myrow = reinterpret_cast<const uint32_t*>(rows_s + slot * p.row_words);
        const uint64_t my_point = p0 + slot;

        for (uint32_t part = 0; part < p.parts; ++part) {
            const uint2* fam = fam_s + part * p.part_words;
            uint32_t lo[E], hi[E];

            // ---- sketch: t[c] for this lane's columns c = g*E + j, split into planes
            if constexpr (DIRECT) {
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    const uint2 e = fam[(j / 2) * 2 * G + 2 * g + (j & 1)]; // column pairs, lane-fastest
                    const uint32_t m = 0u - row_bit(myrow, e.x);
                    lo[j] = e.y & m & 0xFFFFu;
                    hi[j] = (e.y >> 16) & m;
                }
            } else {
                // warp-local accumulation buffer sk[col][lane] (conflict-free for any col)
                uint64_t* sk = xbuf + warp * 32 * E;
#pragma unroll
                for (int j = 0; j < E; ++j) sk[j * 32 + lane] = 0ull;
                const uint2* le = fam + g; // entry k of lane g at le[k * G]
                uint32_t cur = le[0].x >> 24;
                uint64_t acc = 0;
                for (uint32_t k = 0; k < p.lane_entries; ++k) {
                    const uint2 e = le[k * G];
                    const uint32_t col = e.x >> 24;
                    if (col != cur) {
                        sk[cur * 32 + lane] = acc;
                        acc = 0;
                        cur = col;
                    }
                    const uint64_t packed = (uint64_t(e.y >> 16) << 32) | (e.y & 0xFFFFu);
                    acc += row_bit(myrow, e.x & 0xFFFFFFu) ? packed : 0ull;
                }
                sk[cur * 32 + lane] = acc;
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    const uint64_t v = sk[j * 32 + lane];
                    lo[j] = uint32_t(v);
                    hi[j] = uint32_t(v >> 32);
                }
                __syncwarp();
            }

            // ---- phase 1: log2(E) stages in registers
            fht_signed<E>(lo);
            fht_signed<E>(hi);

            uint32_t Tlo, Thi;
            if constexpr (G > 1) {
                // ---- swizzled transpose through this row's slot region (warp-local)
                uint64_t* xs = xbuf + slot * N;
#pragma unroll
                for (int j = 0; j < E; j += 2) {
                    const int idx = g * E + (j ^ ((2 * g) & (E - 1)));
                    *reinterpret_cast<uint4*>(xs + idx) = make_uint4(lo[j], hi[j], lo[j + 1], hi[j + 1]);
                }
                __syncwarp();
                // phase-2 layout: register k*G + h holds element c = h*E + g*EG + k
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const int idx = h * E + ((g * EG) ^ ((2 * h) & (E - 1)));
                    if constexpr (EG == 2) {
                        const uint4 v = *reinterpret_cast<const uint4*>(xs + idx);
                        lo[h] = v.x;
                        hi[h] = v.y;
                        lo[G + h] = v.z;
                        hi[G + h] = v.w;
                    } else {
                        const uint2 v = *reinterpret_cast<const uint2*>(xs + idx);
                        lo[h] = v.x;
                        hi[h] = v.y;
                    }
                }
                __syncwarp();
                // ---- phase 2: log2(G) stages in registers
#pragma unroll
                for (int k = 0; k < EG; ++k) {
                    fht_signed<G>(lo + k * G);
                    fht_signed<G>(hi + k * G);
                }
                // totals F[0] sit in lane g == 0 of the row, register 0
                const int src = lane & ~(G - 1);
                Tlo = __shfl_sync(0xffffffffu, lo[0], src);
                Thi = __shfl_sync(0xffffffffu, hi[0], src);
            } else {
                Tlo = lo[0];
                Thi = hi[0];
            }

            // ---- final reduction + output
            if constexpr (G == 1) {
                // thread per row: table-major stores are coalesced across lanes directly
                if (my_point < p.n) {
#pragma unroll
                    for (int v = 1; v < N; ++v) {
                        const uint32_t key = finish_key(Tlo, Thi, lo[v], hi[v]);
                        const uint64_t t = part * p.L + (v - 1);
                        const uint64_t off = p.layout == 0 ? t * p.key_stride + my_point
                                                           : my_point * p.key_stride + t;
                        if (p.key_bytes == 4)
                            static_cast<uint32_t*>(p.keys)[off] = key;
                        else
                            static_cast<uint64_t*>(p.keys)[off] = key;
                    }
                }
            } else {
                // stage keys: slot s occupies u32 [2sN, 2sN + N), element v at v ^ swz(s)
                uint32_t* stg = reinterpret_cast<uint32_t*>(xbuf) + 2 * slot * N;
                const uint32_t sw = stage_swz<PT>(slot);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const int v0 = h * E + g * EG;
                    if constexpr (EG == 2) {
                        const uint32_t k0 = finish_key(Tlo, Thi, lo[h], hi[h]);
                        const uint32_t k1 = finish_key(Tlo, Thi, lo[G + h], hi[G + h]);
                        *reinterpret_cast<uint2*>(stg + (v0 ^ sw)) = make_uint2(k0, k1);
                    } else {
                        stg[v0 ^ sw] = finish_key(Tlo, Thi, lo[h], hi[h]);
                    }
                }
                __syncthreads();
                const uint32_t* stg_all = reinterpret_cast<const uint32_t*>(xbuf);
                if (p.layout == 0) {
                    constexpr int M = PT / 4;
                    for (uint32_t i = tid; i < uint32_t(N) * M; i += 256) {
                        const uint32_t m = i % M;
                        const uint32_t v = i / M;
                        if (v == 0) continue;
                        uint32_t kk[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t s = 4 * m + q;
                            kk[q] = stg_all[2 * s * N + (v ^ stage_swz<PT>(s))];
                        }
                        const uint64_t t = part * p.L + (v - 1);
                        const uint64_t pt = p0 + 4 * m;
                        const uint64_t off = t * p.key_stride + pt;
                        if (p.key_bytes == 4) {
                            uint32_t* kp = static_cast<uint32_t*>(p.keys);
                            if (pt + 4 <= p.n && (off & 3) == 0) {
                                *reinterpret_cast<uint4*>(kp + off) = make_uint4(kk[0], kk[1], kk[2], kk[3]);
                            } else {
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    if (pt + q < p.n) kp[off + q] = kk[q];
                            }
                        } else {
                            uint64_t* kp = static_cast<uint64_t*>(p.keys);
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (pt + q < p.n) kp[off + q] = kk[q];
                        }
                    }
                } else {
                    for (uint32_t i = tid; i < uint32_t(N) * PT; i += 256) {
                        const uint32_t s = i / N;
                        const uint32_t v = i % N;
                        if (v == 0 || p0 + s >= p.n) continue;
                        const uint32_t key = stg_all[2 * s * N + (v ^ stage_swz<PT>(s))];
                        const uint64_t off = (p0 + s) * p.key_stride + part * p.L + (v - 1);
                        if (p.key_bytes == 4)
                            static_cast<uint32_t*>(p.keys)[off] = key;
                        else
                            static_cast<uint64_t*>(p.keys)[off] = key;
                    }
                }
                __syncthreads();
            }
        }
    }
}

// ------------------------------------------------------------- generic path

struct GenericParams {
    const uint64_t* rows;
    uint64_t n;
    uint32_t row_words;
    uint32_t parts;
    uint64_t N;
    uint64_t L;
    uint64_t prime;
    uint64_t max_dims;
    const uint32_t* col_ptr;  // [parts][N+1]
    const uint32_t* ent_pos;  // [parts][max_dims]
    const uint64_t* ent_seed; // [parts][max_dims]
    uint64_t* scratch;        // [gridDim.x][N] when not in shared memory
    int use_smem;
    void* keys;
    uint64_t key_stride;
    int layout;
    int key_bytes;
};

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t p) { // modmath.hpp:12-15
    uint64_t s = a + b;
    return s >= p ? s - p : s;
}
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t p) { // modmath.hpp:17-19
    return a >= b ? a - b : a + p - b;
}

__global__ void __launch_bounds__(256) k_hash_generic(const GenericParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t red[8];
    uint64_t* t = p.use_smem ? reinterpret_cast<uint64_t*>(smem) : p.scratch + blockIdx.x * p.N;
    const uint64_t P = p.prime;
    const int tid = threadIdx.x;
    for (uint64_t pt = blockIdx.x; pt < p.n; pt += gridDim.x) {
        const uint64_t* row = p.rows + pt * p.row_words;
        for (uint32_t part = 0; part < p.parts; ++part) {
            const uint32_t* cp = p.col_ptr + part * (p.N + 1);
            const uint32_t* ep = p.ent_pos + part * p.max_dims;
            const uint64_t* es = p.ent_seed + part * p.max_dims;
            // sketch (covering.cpp:174-179): per column, seeds of set bits in view order
            uint64_t part_l1 = 0;
            for (uint64_t c = tid; c < p.N; c += blockDim.x) {
                uint64_t acc = 0;
                for (uint32_t k = cp[c]; k < cp[c + 1]; ++k) {
                    const uint32_t pos = ep[k];
                    if ((row[pos >> 6] >> (pos & 63)) & 1ull) acc = add_mod(acc, es[k], P);
                }
                t[c] = acc;
                part_l1 = add_mod(part_l1, acc, P);
            }
            // l1 = total mass mod P (exact modular sum, order-free for P < 2^63)
            for (int o = 16; o > 0; o >>= 1) part_l1 = add_mod(part_l1, __shfl_xor_sync(0xffffffffu, part_l1, o), P);
            if ((tid & 31) == 0) red[tid >> 5] = part_l1;
            __syncthreads();
            uint64_t l1 = 0;
            for (int w = 0; w < int(blockDim.x >> 5); ++w) l1 = add_mod(l1, red[w], P);
            // fht_mod_in_place (hadamard.cpp:51-64)
            for (uint64_t half = 1; half < p.N; half <<= 1) {
                for (uint64_t b = tid; b < p.N / 2; b += blockDim.x) {
                    const uint64_t i = (b / half) * 2 * half + (b % half);
                    const uint64_t a = t[i], c = t[i + half];
                    t[i] = add_mod(a, c, P);
                    t[i + half] = sub_mod(a, c, P);
                }
                __syncthreads();
            }
            // x <- half * (l1 - x) mod P (hadamard.cpp:69-71); for canonical y,
            // half*y mod P is y/2 (y even) or (y+P)/2 (y odd).
            for (uint64_t v = 1 + tid; v < p.N; v += blockDim.x) {
                const uint64_t y = sub_mod(l1, t[v], P);
                const uint64_t key = (y & 1) ? (y >> 1) + (P >> 1) + 1 : (y >> 1);
                const uint64_t tt = part * p.L + (v - 1);
                const uint64_t off = p.layout == 0 ? tt * p.key_stride + pt : pt * p.key_stride + tt;
                if (p.key_bytes == 4)
                    static_cast<uint32_t*>(p.keys)[off] = uint32_t(key);
                else
                    static_cast<uint64_t*>(p.keys)[off] = key;
            }
            __syncthreads();
        }
    }
}

// (O_lo + 2^16 * O_hi) mod (2^31-1) from D = 2*O per plane (D even, Dlo <
// 2^32, Dhi < 2^31): s = O_lo + 2^16 O_hi (mod P, lazily) + 1 < 2^32, then
// two Mersenne folds; the +1 makes the second fold land on the canonical
// residue (P -> 0, 2^31 -> 1).
__device__ __forceinline__ uint32_t finish_from_d(uint32_t Dlo, uint32_t Dhi) {
    const uint32_t slo = Dlo >> 1;
    const uint32_t a = Dhi >> 16;                               // (O_hi >> 15) * 2^31 == (O_hi >> 15)
    const uint32_t b = ((Dhi << 15) & 0x7FFF0000u) | 1u;        // (O_hi & 0x7fff) << 16, plus 1
    const uint32_t s1 = slo + a + b;                            // s + 1, s < 2^32 - 1
    const uint32_t y = (s1 & kP31) + (s1 >> 31);                // fold
    return (y & kP31) + (y >> 31) - 1;                          // canonical in [0, P)
}

// Point-major variant (keys[row*stride + part*L + v-1]) for G > 1: every warp
// owns 32/G rows end to end -- row fetch, sketch, both butterfly phases, the
// final reduction and the key stores go straight from registers to HBM (a
// lane's consecutive keys are contiguous across the warp), so there is no
// output staging and no CTA-wide barrier after the family is staged. The
// plane totals T = F[0] come from a lane reduction of the phase-1 block
// totals, which lets the last butterfly stage produce D = T - F directly.
// The transpose rows are padded by one 16-byte unit (E+2 u64) instead of
// XOR-swizzled: conflict-free, and every access is [base + immediate].
template <int LOGN>
__host__ __device__ constexpr int pm_warps() {
    return LOGN == 11 ? 12 : 8; // N = 2048 needs ~200 registers: 12 warps fit the register file
}

template <int LOGN, bool DIRECT>
__global__ void __launch_bounds__(32 * pm_warps<LOGN>(), 1) k_hash_m31_pm(const FastParams p) {
    constexpr int N = 1 << LOGN;
    constexpr int G = lanes_for(LOGN);
    constexpr int E = N / G;
    constexpr int EP = E + 2; // padded transpose row (u64)
    constexpr int EG = E / G;
    constexpr int SPW = 32 / G; // rows per warp
    constexpr int WARPS = pm_warps<LOGN>();
    constexpr int NT = 32 * WARPS;
    static_assert(G > 1 && (EG == 1 || EG == 2), "phase-2 layout");

    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* xbuf = reinterpret_cast<uint64_t*>(smem);    // WARPS x 32*EP u64
    uint64_t* rows_s = xbuf + WARPS * 32 * EP;              // WARPS x SPW x row_words u64
    uint2* fam_s = reinterpret_cast<uint2*>(rows_s + WARPS * SPW * p.row_words);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int slot = lane / G; // row within the warp
    const int g = lane % G;

    for (uint32_t i = tid; i < p.parts * p.part_words; i += NT) fam_s[i] = p.fam[i];
    __syncthreads();

    uint64_t* xw = xbuf + warp * 32 * EP;                   // this warp's transpose region
    uint64_t* rw = rows_s + warp * SPW * p.row_words;       // this warp's rows
    const uint32_t* myrow = reinterpret_cast<const uint32_t*>(rw + slot * p.row_words);
    uint64_t* xs = xw + slot * G * EP;                      // this row's transpose region
    uint64_t* xs_w = xs + g * EP;                           // phase-1 row of this lane
    const uint64_t* xs_r = xs + g * EG;                     // phase-2 column of this lane

    const uint64_t groups = (p.n + SPW - 1) / SPW;
    const uint64_t nwarps = uint64_t(gridDim.x) * WARPS;
    for (uint64_t grp = uint64_t(blockIdx.x) * WARPS + warp; grp < groups; grp += nwarps) {
        const uint64_t p0 = grp * SPW;
        {
            const uint64_t base = p0 * p.row_words;
            const uint64_t lim = p.n * p.row_words;
            for (uint32_t i = lane; i < SPW * p.row_words; i += 32)
                rw[i] = (base + i < lim) ? __ldg(p.rows + base + i) : 0ull;
        }
        __syncwarp();
        const uint64_t my_point = p0 + slot;

        for (uint32_t part = 0; part < p.parts; ++part) {
            const uint2* fam = fam_s + part * p.part_words;
            uint32_t lo[E], hi[E];
            if constexpr (DIRECT) {
                // entries of columns (j, j+1) of lane g are adjacent: one 16-byte load
                const uint4* fam4 = reinterpret_cast<const uint4*>(fam) + g;
#pragma unroll
                for (int j = 0; j < E; j += 2) {
                    const uint4 e = fam4[(j / 2) * G];
                    const uint32_t m0 = 0u - row_bit(myrow, e.x);
                    const uint32_t m1 = 0u - row_bit(myrow, e.z);
                    lo[j] = e.y & m0 & 0xFFFFu;
                    hi[j] = (e.y >> 16) & m0;
                    lo[j + 1] = e.w & m1 & 0xFFFFu;
                    hi[j + 1] = (e.w >> 16) & m1;
                }
            } else {
                uint64_t* sk = xw; // sk[col][lane], conflict-free for any col
#pragma unroll
                for (int j = 0; j < E; ++j) sk[j * 32 + lane] = 0ull;
                const uint2* le = fam + g;
                uint32_t cur = le[0].x >> 24;
                uint64_t acc = 0;
                for (uint32_t k = 0; k < p.lane_entries; ++k) {
                    const uint2 e = le[k * G];
                    const uint32_t col = e.x >> 24;
                    if (col != cur) {
                        sk[cur * 32 + lane] = acc;
                        acc = 0;
                        cur = col;
                    }
                    const uint64_t packed = (uint64_t(e.y >> 16) << 32) | (e.y & 0xFFFFu);
                    acc += row_bit(myrow, e.x & 0xFFFFFFu) ? packed : 0ull;
                }
                sk[cur * 32 + lane] = acc;
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    const uint64_t v = sk[j * 32 + lane];
                    lo[j] = uint32_t(v);
                    hi[j] = uint32_t(v >> 32);
                }
                __syncwarp();
            }

            // phase 1
            fht_signed<E>(lo);
            fht_signed<E>(hi);
            // plane totals: sum of the G block totals (register 0 of each lane)
            uint32_t Tlo = lo[0], Thi = hi[0];
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
                Tlo += __shfl_xor_sync(0xffffffffu, Tlo, o);
                Thi += __shfl_xor_sync(0xffffffffu, Thi, o);
            }
            // transpose (warp-local): element c = hb*E + j lives at xs[hb*EP + j]
#pragma unroll
            for (int j = 0; j < E; j += 2)
                *reinterpret_cast<uint4*>(xs_w + j) = make_uint4(lo[j], hi[j], lo[j + 1], hi[j + 1]);
            __syncwarp();
#pragma unroll
            for (int h = 0; h < G; ++h) {
                if constexpr (EG == 2) {
                    const uint4 v = *reinterpret_cast<const uint4*>(xs_r + h * EP);
                    lo[h] = v.x;
                    hi[h] = v.y;
                    lo[G + h] = v.z;
                    hi[G + h] = v.w;
                } else {
                    const uint2 v = *reinterpret_cast<const uint2*>(xs_r + h * EP);
                    lo[h] = v.x;
                    hi[h] = v.y;
                }
            }
            __syncwarp();
            // phase 2: all but the last stage, then the last stage emits D = T - F
#pragma unroll
            for (int k = 0; k < EG; ++k) {
                uint32_t* xl = lo + k * G;
                uint32_t* xh = hi + k * G;
#pragma unroll
                for (int hs = 1; hs < G / 2; hs <<= 1) {
#pragma unroll
                    for (int i = 0; i < G; ++i) {
                        if ((i & hs) == 0) {
                            uint32_t a = xl[i], b = xl[i + hs];
                            xl[i] = a + b;
                            xl[i + hs] = a - b;
                            a = xh[i];
                            b = xh[i + hs];
                            xh[i] = a + b;
                            xh[i + hs] = a - b;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < G / 2; ++i) {
                    uint32_t a = xl[i], b = xl[i + G / 2];
                    xl[i] = Tlo - a - b;
                    xl[i + G / 2] = Tlo - a + b;
                    a = xh[i];
                    b = xh[i + G / 2];
                    xh[i] = Thi - a - b;
                    xh[i + G / 2] = Thi - a + b;
                }
            }
            // keys straight to HBM: element (k, h) is code v = h*E + g*EG + k
            if (my_point < p.n) {
                if (p.key_bytes == 4) {
                    uint32_t* out = static_cast<uint32_t*>(p.keys) + my_point * p.key_stride + part * p.L +
                                    (g * EG - 1);
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < EG; ++k)
                            if (h * E + g * EG + k != 0) out[h * E + k] = finish_from_d(lo[k * G + h], hi[k * G + h]);
                } else {
                    uint64_t* out = static_cast<uint64_t*>(p.keys) + my_point * p.key_stride + part * p.L +
                                    (g * EG - 1);
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < EG; ++k)
                            if (h * E + g * EG + k != 0) out[h * E + k] = finish_from_d(lo[k * G + h], hi[k * G + h]);
                }
            }
        }
        __syncwarp();
    }
}

// FP64 variant of the point-major kernel for direct families. The sketch t
// and every partial transform are exact doubles (|F| <= d * 2^31 < 2^53 for
// d < 2^22), so one butterfly is a single DADD instead of one 32-bit add on
// each of two planes, and the FP64 pipe runs beside the integer pipes that do
// the sketch and the reduction. The last stage computes (T + 2^52) - F: for
// 0 <= D = T - F < 2^52 that double is exact and its low 52 mantissa bits are
// D, so the final reduction needs no float-to-int conversion.
template <int LOGN>
__global__ void __launch_bounds__(32 * pm_warps<LOGN>(), 1) k_hash_f64_pm(const FastParams p) {
    constexpr int N = 1 << LOGN;
    constexpr int G = lanes_for(LOGN);
    constexpr int E = N / G;
    constexpr int EP = E + 2; // padded transpose row (doubles)
    constexpr int EG = E / G;
    constexpr int SPW = 32 / G; // rows per warp
    constexpr int WARPS = pm_warps<LOGN>();
    constexpr int NT = 32 * WARPS;
    constexpr int NP = N / 2; // column pairs per part
    static_assert(G > 1 && (EG == 1 || EG == 2), "phase-2 layout");
    constexpr double kTwo52 = 4503599627370496.0;
    // added to every final-stage value D (even): moves O = D/2 by P - 0x43300000 (mod P), which
    // cancels the exponent bits 0x43300000 that the high word of 2^52 + D carries (see finish)
    constexpr double kFinishBias = 2.0 * double(kP31 - 0x43300000u);

    extern __shared__ __align__(16) unsigned char smem[];
    double* xbuf = reinterpret_cast<double*>(smem);                            // WARPS x 32*EP
    uint64_t* rows_s = reinterpret_cast<uint64_t*>(xbuf + WARPS * 32 * EP);    // WARPS x SPW x row_words
    double2* seed_s = reinterpret_cast<double2*>(rows_s + WARPS * SPW * p.row_words); // [parts][NP]
    uint2* pos_s = reinterpret_cast<uint2*>(seed_s + p.parts * NP);            // [parts][NP]

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int slot = lane / G; // row within the warp
    const int g = lane % G;

    // the direct table holds {pos, seed} for column pairs, lane-fastest: pair
    // i = (j/2)*G + g of a part is entries 2i, 2i+1 -> positions and seeds apart
    for (uint32_t i = tid; i < p.parts * NP; i += NT) {
        const uint2 e0 = p.fam[2 * i], e1 = p.fam[2 * i + 1];
        pos_s[i] = make_uint2(e0.x, e1.x);
        seed_s[i] = make_double2(double(e0.y), double(e1.y));
    }
    __syncthreads();

    double* xw = xbuf + warp * 32 * EP;                     // this warp's transpose region
    uint64_t* rw = rows_s + warp * SPW * p.row_words;       // this warp's rows
    const uint32_t* myrow = reinterpret_cast<const uint32_t*>(rw + slot * p.row_words);
    double* xs = xw + slot * G * EP;                        // this row's transpose region
    double* xs_w = xs + g * EP;                             // phase-1 row of this lane
    const double* xs_r = xs + g * EG;                       // phase-2 column of this lane

    const uint64_t groups = (p.n + SPW - 1) / SPW;
    const uint64_t nwarps = uint64_t(gridDim.x) * WARPS;
    for (uint64_t grp = uint64_t(blockIdx.x) * WARPS + warp; grp < groups; grp += nwarps) {
        const uint64_t p0 = grp * SPW;
        {
            const uint64_t base = p0 * p.row_words;
            const uint64_t lim = p.n * p.row_words;
            for (uint32_t i = lane; i < SPW * p.row_words; i += 32)
                rw[i] = (base + i < lim) ? __ldg(p.rows + base + i) : 0ull;
        }
        __syncwarp();
        const uint64_t my_point = p0 + slot;

        for (uint32_t part = 0; part < p.parts; ++part) {
            const uint2* ps = pos_s + part * NP + g;
            const double2* sd = seed_s + part * NP + g;
            double x[E];
            // sketch: seed where the row bit is set, +0.0 elsewhere (a 64-bit mask)
#pragma unroll
            for (int j = 0; j < E; j += 2) {
                const uint2 pp = ps[(j / 2) * G];
                const double2 s2 = sd[(j / 2) * G];
                // row bit -> predicate (funnel shift = 1 << (pos mod 32)), then select the seed words
                const bool b0 = (myrow[pp.x >> 5] & __funnelshift_l(0u, 1u, pp.x)) != 0u;
                const bool b1 = (myrow[pp.y >> 5] & __funnelshift_l(0u, 1u, pp.y)) != 0u;
                x[j] = b0 ? s2.x : 0.0;
                x[j + 1] = b1 ? s2.y : 0.0;
            }
            // phase 1
#pragma unroll
            for (int h = 1; h < E; h <<= 1) {
#pragma unroll
                for (int i = 0; i < E; ++i) {
                    if ((i & h) == 0) {
                        const double a = x[i], b = x[i + h];
                        x[i] = a + b;
                        x[i + h] = a - b;
                    }
                }
            }
            // total T: sum of the G block totals (element 0 of each lane)
            double T = x[0];
#pragma unroll
            for (int o = 1; o < G; o <<= 1) T += __shfl_xor_sync(0xffffffffu, T, o);
            const double Tp = T + (kTwo52 + kFinishBias);
            // transpose (warp-local): element c = hb*E + j lives at xs[hb*EP + j]
#pragma unroll
            for (int j = 0; j < E; j += 2) *reinterpret_cast<double2*>(xs_w + j) = make_double2(x[j], x[j + 1]);
            __syncwarp();
#pragma unroll
            for (int h = 0; h < G; ++h) {
                if constexpr (EG == 2) {
                    const double2 v = *reinterpret_cast<const double2*>(xs_r + h * EP);
                    x[h] = v.x;
                    x[G + h] = v.y;
                } else {
                    x[h] = xs_r[h * EP];
                }
            }
            __syncwarp();
            // phase 2: all but the last stage, then the last stage emits 2^52 + D
#pragma unroll
            for (int k = 0; k < EG; ++k) {
                double* xl = x + k * G;
#pragma unroll
                for (int hs = 1; hs < G / 2; hs <<= 1) {
#pragma unroll
                    for (int i = 0; i < G; ++i) {
                        if ((i & hs) == 0) {
                            const double a = xl[i], b = xl[i + hs];
                            xl[i] = a + b;
                            xl[i + hs] = a - b;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < G / 2; ++i) {
                    const double a = xl[i], b = xl[i + G / 2];
                    xl[i] = (Tp - a) - b;
                    xl[i + G / 2] = (Tp - a) + b;
                }
            }
            // keys straight to HBM: element (k, h) is code v = h*E + g*EG + k
            auto finish = [](double v) -> uint32_t {
                // D = bits & (2^52 - 1) = dh * 2^32 + lo (even), O = D / 2 = dh * 2^31 + lo / 2
                // == dh + lo / 2 (mod P)
                // O' = dh + lo/2 < 2P: one conditional subtraction, as an unsigned min
                // the high word is 0x43300000 + dh (dh < 2^20) and kFinishBias has already moved O by
                // -0x43300000 (mod P): no mask; lo/2 + dh + 0x43300000 < 2^31 + 2^20 + 0x43300000 < 2P
                const uint32_t lo = uint32_t(__double2loint(v)), hi = uint32_t(__double2hiint(v));
                const uint32_t o = (lo >> 1) + hi;
                return min(o, o - kP31);
            };
            if (my_point < p.n) {
                if (p.key_bytes == 4) {
                    uint32_t* out = static_cast<uint32_t*>(p.keys) + my_point * p.key_stride + part * p.L +
                                    (g * EG - 1);
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < EG; ++k)
                            if (h * E + g * EG + k != 0) out[h * E + k] = finish(x[k * G + h]);
                } else {
                    uint64_t* out = static_cast<uint64_t*>(p.keys) + my_point * p.key_stride + part * p.L +
                                    (g * EG - 1);
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < EG; ++k)
                            if (h * E + g * EG + k != 0) out[h * E + k] = finish(x[k * G + h]);
                }
            }
        }
        __syncwarp();
    }
}

// FP64 point-major kernel with a column-pair table. The sketch and the first
// butterfly stage of a column pair (j, j+1) depend only on the two row bits,
// so the shared table holds the four outcomes {(0,0), (s0,s0), (s1,-s1),
// (s0+s1, s0-s1)} per pair, and one 16-byte load replaces two selects per
// column and the first stage. Layout [part][outcome][pair] (16 B entries):
// lanes read consecutive pairs, so a quarter-warp's loads hit distinct banks
// whatever outcome each lane selects. The outcome is bits S, S+1 of the byte
// offset (S = log2(16 * N/2)); the pair's positions are stored with their low
// five bits pre-rotated so that rotating the row word moves the bit straight
// to bit S (S+1).
// The transpose runs in E/G rounds of G columns through a (G+2)-double padded
// buffer, half the size of a one-round transpose: after round k lane g holds
// column k*G + g of every lane's block, so the keys of one store are G
// consecutive codes.
// d = LUT(a, b, c) bitwise; 0xE2 = b ? a : c, 0xEA = (a & b) | c
template <uint32_t LUT, uint32_t B>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "n"(B), "r"(c), "n"(LUT));
    return d;
}

// 8-byte global -> shared async copy; src_bytes 0 zero-fills the destination
__device__ __forceinline__ void cp_async8(void* dst, const void* src, uint32_t src_bytes) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_one() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int LOGN>
__host__ __device__ constexpr int pt_warps() {
    return LOGN == 11 ? 12 : 8;
}

// P16: both positions of a pair in one 32-bit word (16 bits each: row-word
// byte offset << 5 | rotation; rows up to 2 KB), halving the position loads
template <int LOGN, bool P16>
__global__ void __launch_bounds__(32 * pt_warps<LOGN>(), 1) k_hash_f64_pt(const FastParams p) {
    constexpr int N = 1 << LOGN;
    constexpr int G = lanes_for(LOGN);
    constexpr int E = N / G;
    constexpr int GP = G + 2; // padded transpose row (doubles)
    constexpr int EG = E / G;
    constexpr int SPW = 32 / G; // rows per warp
    constexpr int WARPS = pt_warps<LOGN>();
    constexpr int NT = 32 * WARPS;
    constexpr int NP = N / 2; // column pairs per part
    static_assert(G > 1 && EG >= 1 && E % 2 == 0, "layout");
    constexpr double kTwo52 = 4503599627370496.0;
    // added to every final-stage value D (even): moves O = D/2 by P - 0x43300000 (mod P), which
    // cancels the exponent bits 0x43300000 that the high word of 2^52 + D carries (see finish)
    constexpr double kFinishBias = 2.0 * double(kP31 - 0x43300000u);

    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int S = LOGN + 3; // outcome bit of the table byte offset
    double2* tab_s = reinterpret_cast<double2*>(smem);                         // [parts][4][NP]
    double* xbuf = reinterpret_cast<double*>(tab_s + size_t(p.parts) * NP * 4); // WARPS x 32*GP
    uint2* pk_s = reinterpret_cast<uint2*>(xbuf + WARPS * 32 * GP);             // [parts][NP]
    uint64_t* rows_s = reinterpret_cast<uint64_t*>(pk_s + p.parts * NP);        // WARPS x 2 x SPW x row_words

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int slot = lane / G; // row within the warp
    const int g = lane % G;
    pdl_trigger(); // the query kernel may be scheduled behind this grid (it waits for its completion)

    // pair i = (j/2)*G + g of a part is entries 2i, 2i+1 of the direct table
    for (uint32_t i = tid; i < p.parts * NP; i += NT) {
        const uint2 e0 = p.fam[2 * i], e1 = p.fam[2 * i + 1];
        const double s0 = double(e0.y), s1 = double(e1.y);
        double2* t = tab_s + size_t(i / NP) * 4 * NP + (i % NP);
        t[0] = make_double2(0.0, 0.0);
        t[NP] = make_double2(s0, s0);
        t[2 * NP] = make_double2(s1, -s1);
        t[3 * NP] = make_double2(s0 + s1, s0 - s1);
        // (byte offset of the row word) << 5 | rotation: bit (pos mod 32) -> bit S (S+1)
        if constexpr (P16)
            reinterpret_cast<uint32_t*>(pk_s)[i] = ((((e0.x >> 5) << 7) | ((e0.x - S) & 31u)) & 0xFFFFu) |
                                                   ((((e1.x >> 5) << 7) | ((e1.x - S - 1) & 31u)) << 16);
        else
            pk_s[i] = make_uint2(((e0.x & ~31u) << 2) | ((e0.x - S) & 31u),
                                 ((e1.x & ~31u) << 2) | ((e1.x - S - 1) & 31u));
    }
    __syncthreads();

    double* xw = xbuf + warp * 32 * GP; // this warp's transpose region
    const uint32_t wrow = SPW * p.row_words;
    uint64_t* rw = rows_s + warp * 2 * wrow; // this warp's rows, double-buffered
    double* xs = xw + slot * G * GP;         // this row's transpose region
    double* xs_w = xs + g * GP;              // round write: row g
    const double* xs_r = xs + g;             // round read: column g

    const uint64_t groups = (p.n + SPW - 1) / SPW;
    const uint64_t nwarps = uint64_t(gridDim.x) * WARPS;
    // the next group's rows stream into the other buffer (cp.async) while
    // this group computes: the row loads' latency is off the critical path
    auto fetch = [&](uint64_t gr, uint64_t* dst) {
        const uint64_t base = gr * wrow, lim = p.n * p.row_words;
        for (uint32_t i = lane; i < wrow; i += 32) {
            const bool ok = gr < groups && base + i < lim;
            cp_async8(dst + i, ok ? p.rows + base + i : p.rows, ok ? 8u : 0u);
        }
        cp_async_commit();
    };
    uint64_t grp = uint64_t(blockIdx.x) * WARPS + warp;
    fetch(grp, rw);
    for (uint32_t it = 0; grp < groups; grp += nwarps, ++it) {
        fetch(grp + nwarps, rw + ((it + 1) & 1) * wrow);
        cp_async_wait_one();
        __syncwarp();
        if (p.rows_copy) { // this group's rows, staged, also to the device copy
            const uint64_t base = grp * wrow, lim = p.n * p.row_words;
            for (uint32_t i = lane; i < wrow && base + i < lim; i += 32) p.rows_copy[base + i] = rw[(it & 1) * wrow + i];
        }
        const uint32_t* myrow = reinterpret_cast<const uint32_t*>(rw + (it & 1) * wrow + slot * p.row_words);
        const uint64_t p0 = grp * SPW;
        const uint64_t my_point = p0 + slot;

        for (uint32_t part = 0; part < p.parts; ++part) {
            const uint2* pk = pk_s + part * NP + g;
            const uint32_t tb_off = part * NP * 64u + g * 16u; // this lane's first pair, outcome 0
            const char* rowb = reinterpret_cast<const char*>(myrow);
            const char* tabb = reinterpret_cast<const char*>(tab_s);
            double x[E];
            // sketch + first stage: one table entry per column pair
#pragma unroll
            for (int j = 0; j < E; j += 2) {
                uint32_t r0, r1;
                if constexpr (P16) {
                    const uint32_t v = reinterpret_cast<const uint32_t*>(pk_s)[part * NP + g + (j / 2) * G];
                    const uint32_t w0 = *reinterpret_cast<const uint32_t*>(rowb + ((v << 16) >> 21));
                    const uint32_t w1 = *reinterpret_cast<const uint32_t*>(rowb + (v >> 21));
                    r0 = __funnelshift_r(w0, w0, v);
                    r1 = __funnelshift_r(w1, w1, v >> 16);
                } else {
                    const uint2 pp = pk[(j / 2) * G];
                    const uint32_t w0 = *reinterpret_cast<const uint32_t*>(rowb + (pp.x >> 5));
                    const uint32_t w1 = *reinterpret_cast<const uint32_t*>(rowb + (pp.y >> 5));
                    r0 = __funnelshift_r(w0, w0, pp.x);
                    r1 = __funnelshift_r(w1, w1, pp.y);
                }
                const uint32_t t = lop3<0xE2, 1u << S>(r0, r1);      // bit S from r0, S+1 from r1
                const uint32_t off = lop3<0xEA, 3u << S>(t, tb_off); // + outcome (b0 + 2 b1) * NP * 16
                const double2 v = *reinterpret_cast<const double2*>(tabb + off + (j / 2) * G * 16);
                x[j] = v.x;
                x[j + 1] = v.y;
            }
            // phase 1, remaining stages
#pragma unroll
            for (int h = 2; h < E; h <<= 1) {
#pragma unroll
                for (int i = 0; i < E; ++i) {
                    if ((i & h) == 0) {
                        const double a = x[i], b = x[i + h];
                        x[i] = a + b;
                        x[i + h] = a - b;
                    }
                }
            }
            // total T: sum of the G block totals (element 0 of each lane)
            double T = x[0];
#pragma unroll
            for (int o = 1; o < G; o <<= 1) T += __shfl_xor_sync(0xffffffffu, T, o);
            const double Tp = T + (kTwo52 + kFinishBias);
            // transpose, G columns per round: x[k*G + h] <- element h*E + k*G + g
#pragma unroll
            for (int k = 0; k < EG; ++k) {
#pragma unroll
                for (int j = 0; j < G; j += 2)
                    *reinterpret_cast<double2*>(xs_w + j) = make_double2(x[k * G + j], x[k * G + j + 1]);
                __syncwarp();
#pragma unroll
                for (int h = 0; h < G; ++h) x[k * G + h] = xs_r[h * GP];
                __syncwarp();
            }
            // phase 2: all but the last stage, then the last stage emits 2^52 + D
#pragma unroll
            for (int k = 0; k < EG; ++k) {
                double* xl = x + k * G;
#pragma unroll
                for (int hs = 1; hs < G / 2; hs <<= 1) {
#pragma unroll
                    for (int i = 0; i < G; ++i) {
                        if ((i & hs) == 0) {
                            const double a = xl[i], b = xl[i + hs];
                            xl[i] = a + b;
                            xl[i + hs] = a - b;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < G / 2; ++i) {
                    const double a = xl[i], b = xl[i + G / 2];
                    xl[i] = (Tp - a) - b;
                    xl[i + G / 2] = (Tp - a) + b;
                }
            }
            auto finish = [](double v) -> uint32_t {
                // the high word is 0x43300000 + dh (dh < 2^20) and kFinishBias has already moved O by
                // -0x43300000 (mod P): no mask; lo/2 + dh + 0x43300000 < 2^31 + 2^20 + 0x43300000 < 2P
                const uint32_t lo = uint32_t(__double2loint(v)), hi = uint32_t(__double2hiint(v));
                const uint32_t o = (lo >> 1) + hi;
                return min(o, o - kP31);
            };
            // element (k, h) is code v = h*E + k*G + g: G consecutive keys per store
            if (my_point < p.n) {
                if (p.key_bytes == 4) {
                    uint32_t* out = static_cast<uint32_t*>(p.keys) + my_point * p.key_stride + part * p.L + g - 1;
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < EG; ++k)
                            if (h * E + k * G + g != 0) out[h * E + k * G] = finish(x[k * G + h]);
                } else {
                    uint64_t* out = static_cast<uint64_t*>(p.keys) + my_point * p.key_stride + part * p.L + g - 1;
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < EG; ++k)
                            if (h * E + k * G + g != 0) out[h * E + k * G] = finish(x[k * G + h]);
                }
            }
        }
        __syncwarp();
    }
    cp_async_wait_all();
}

template <int LOGN, bool DIRECT>
size_t fast_smem_bytes(const DeviceFamilySet& fs) {
    constexpr int G = lanes_for(LOGN);
    constexpr int E = (1 << LOGN) / G;
    constexpr int PT = 256 / G;
    return size_t(256) * E * 8 + size_t(PT) * fs.row_words * 8 + size_t(fs.parts) * fs.part_words * 8;
}

template <int LOGN, bool DIRECT>
void launch_fast(DeviceFamilySet& fs, const FastParams& prm_in, cudaStream_t stream) {
    constexpr int G = lanes_for(LOGN);
    FastParams prm = prm_in;
    // kernels other than k_hash_f64_pt do not copy the rows: copy first, hash the copy
    auto copy_first = [&]() {
        if (!prm.rows_copy) return;
        FCLSH_CUDA(cudaMemcpyAsync(prm.rows_copy, prm.rows, prm.n * prm.row_words * 8, cudaMemcpyDefault, stream));
        prm.rows = prm.rows_copy;
        prm.rows_copy = nullptr;
    };
    constexpr int PT = 256 / G;
    const size_t smem = fast_smem_bytes<LOGN, DIRECT>(fs);
    if constexpr (G > 1) {
        constexpr int WARPS = pm_warps<LOGN>();
        constexpr int E = (1 << LOGN) / G;
        const size_t smem_pm = size_t(WARPS) * 32 * (E + 2) * 8 + size_t(WARPS) * (32 / G) * fs.row_words * 8 +
                               size_t(fs.parts) * fs.part_words * 8;
        // FP64 butterflies for direct families (FCLSH_HASH_INT=1 keeps the two int32 planes)
        static const bool use_int = getenv("FCLSH_HASH_INT") != nullptr;
        static const bool use_pm = getenv("FCLSH_HASH_F64_PM") != nullptr;
        constexpr int PW = pt_warps<LOGN>();
        const size_t smem_pt = size_t(fs.parts) * (1 << LOGN) / 2 * 72 + size_t(PW) * 32 * (G + 2) * 8 +
                               size_t(PW) * 2 * (32 / G) * fs.row_words * 8;
        if (DIRECT && !use_int && !use_pm && prm.layout == kLayoutPointMajor && smem_pt <= 227 * 1024) {
            static const bool pk32 = getenv("FCLSH_HASH_PK32") != nullptr; // A/B: 32-bit positions
            auto kern = (!pk32 && fs.row_words * 8 <= 2048) ? k_hash_f64_pt<LOGN, true> : k_hash_f64_pt<LOGN, false>;
            const int per_sm = resident_ctas(kern, 32 * PW, smem_pt, fs.device);
            if (per_sm < 1) throw ResourceError("hash: kernel does not fit on an SM (shared memory)");
            const uint64_t groups = (prm.n + (32 / G) - 1) / (32 / G);
            const uint64_t grid = std::min<uint64_t>((groups + PW - 1) / PW, uint64_t(per_sm) * sm_count(fs.device));
            kern<<<unsigned(std::max<uint64_t>(grid, 1)), 32 * PW, smem_pt, stream>>>(prm);
            FCLSH_LAUNCHED();
            return;
        }
        copy_first();
        const size_t smem_f64 = size_t(WARPS) * 32 * (E + 2) * 8 + size_t(WARPS) * (32 / G) * fs.row_words * 8 +
                                size_t(fs.parts) * (1 << LOGN) / 2 * 24;
        if (DIRECT && !use_int && prm.layout == kLayoutPointMajor && smem_f64 <= 227 * 1024) {
            auto kern = k_hash_f64_pm<LOGN>;
            const int per_sm = resident_ctas(kern, 32 * WARPS, smem_f64, fs.device);
            if (per_sm < 1) throw ResourceError("hash: kernel does not fit on an SM (shared memory)");
            const uint64_t groups = (prm.n + (32 / G) - 1) / (32 / G);
            const uint64_t grid = std::min<uint64_t>((groups + WARPS - 1) / WARPS, uint64_t(per_sm) * sm_count(fs.device));
            kern<<<unsigned(std::max<uint64_t>(grid, 1)), 32 * WARPS, smem_f64, stream>>>(prm);
            FCLSH_LAUNCHED();
            return;
        }
        // (a family table too large for the 12-warp layout falls back to the staged kernel)
        if (prm.layout == kLayoutPointMajor && smem_pm <= 227 * 1024) {
            auto kern = k_hash_m31_pm<LOGN, DIRECT>;
            const int per_sm = resident_ctas(kern, 32 * WARPS, smem_pm, fs.device);
            if (per_sm < 1) throw ResourceError("hash: kernel does not fit on an SM (shared memory)");
            const uint64_t groups = (prm.n + (32 / G) - 1) / (32 / G);
            const uint64_t grid = std::min<uint64_t>((groups + WARPS - 1) / WARPS, uint64_t(per_sm) * sm_count(fs.device));
            kern<<<unsigned(std::max<uint64_t>(grid, 1)), 32 * WARPS, smem_pm, stream>>>(prm);
            FCLSH_LAUNCHED();
            return;
        }
    }
    copy_first();
    auto kern = k_hash_m31<LOGN, DIRECT>;
    const int per_sm = resident_ctas(kern, 256, smem, fs.device);
    if (per_sm < 1) throw ResourceError("hash: kernel does not fit on an SM (shared memory)");
    const uint64_t tiles = (prm.n + PT - 1) / PT;
    const uint64_t grid = std::min<uint64_t>(tiles, uint64_t(per_sm) * sm_count(fs.device));
    kern<<<unsigned(std::max<uint64_t>(grid, 1)), 256, smem, stream>>>(prm);
    FCLSH_LAUNCHED();
}

template <bool DIRECT>
void dispatch_fast(DeviceFamilySet& fs, const FastParams& prm, cudaStream_t s) {
    switch (fs.logn) {
    case 2: launch_fast<2, DIRECT>(fs, prm, s); break;
    case 3: launch_fast<3, DIRECT>(fs, prm, s); break;
    case 4: launch_fast<4, DIRECT>(fs, prm, s); break;
    case 5: launch_fast<5, DIRECT>(fs, prm, s); break;
    case 6: launch_fast<6, DIRECT>(fs, prm, s); break;
    case 7: launch_fast<7, DIRECT>(fs, prm, s); break;
    case 8: launch_fast<8, DIRECT>(fs, prm, s); break;
    case 9: launch_fast<9, DIRECT>(fs, prm, s); break;
    case 10: launch_fast<10, DIRECT>(fs, prm, s); break;
    case 11: launch_fast<11, DIRECT>(fs, prm, s); break;
    default: throw UsageError("hash: no fast kernel for this code order");
    }
}

} // namespace

std::unique_ptr<DeviceFamilySet> make_device_family_set(const Plan& plan, std::vector<Family> families,
                                                        int device) {
    auto fs = std::make_unique<DeviceFamilySet>();
    fs->device = device;
    fs->parts = plan.part_count();
    if (families.size() != fs->parts) throw UsageError("hash: one family per plan part required");
    if (fs->parts > kMaxParts) throw ResourceError("hash: too many plan parts");
    fs->radius = families[0].radius;
    fs->logn = fs->radius + 1;
    fs->order = uint64_t(1) << fs->logn;
    fs->tables = fs->order - 1;
    fs->prime = families[0].prime;
    fs->dims = plan.dims;
    fs->row_words = uint32_t((plan.dims + 63) / 64);
    for (uint32_t p = 0; p < fs->parts; ++p) {
        const Family& f = families[p];
        if (f.radius != fs->radius || f.prime != fs->prime)
            throw UsageError("hash: plan parts must share radius and prime");
        if (f.dims != plan.part_dims(p)) throw UsageError("hash: family width does not match the plan part");
        fs->max_part_dims = std::max<uint64_t>(fs->max_part_dims, f.dims);
    }
    const uint64_t N = fs->order;
    FCLSH_CUDA(cudaSetDevice(device));

    // ---------------- generic CSR (always built; the fast path may be unavailable)
    {
        std::vector<uint32_t> cp(size_t(fs->parts) * (N + 1), 0);
        std::vector<uint32_t> epos(size_t(fs->parts) * fs->max_part_dims, 0);
        std::vector<uint64_t> eseed(size_t(fs->parts) * fs->max_part_dims, 0);
        for (uint32_t p = 0; p < fs->parts; ++p) {
            const Family& f = families[p];
            uint32_t* c = cp.data() + size_t(p) * (N + 1);
            for (uint64_t j = 0; j < f.dims; ++j) c[f.mapping[j] + 1]++;
            for (uint64_t k = 0; k < N; ++k) c[k + 1] += c[k];
            std::vector<uint32_t> fill(c, c + N);
            for (uint64_t j = 0; j < f.dims; ++j) { // ascending view position per column
                const uint32_t at = fill[f.mapping[j]]++;
                epos[size_t(p) * fs->max_part_dims + at] = uint32_t(plan.source_bit(p, j));
                eseed[size_t(p) * fs->max_part_dims + at] = f.seeds[j];
            }
        }
        FCLSH_CUDA(cudaMemcpy(fs->col_ptr.ensure(cp.size() * 4), cp.data(), cp.size() * 4, cudaMemcpyHostToDevice));
        FCLSH_CUDA(cudaMemcpy(fs->ent_pos.ensure(epos.size() * 4), epos.data(), epos.size() * 4, cudaMemcpyHostToDevice));
        FCLSH_CUDA(cudaMemcpy(fs->ent_seed.ensure(eseed.size() * 8), eseed.data(), eseed.size() * 8, cudaMemcpyHostToDevice));
        if (fs->prime <= 0xFFFFFFFFull) { // one 8-byte load per entry (seed < P < 2^32)
            std::vector<uint64_t> pk(eseed.size());
            for (size_t k = 0; k < pk.size(); ++k) pk[k] = (eseed[k] << 32) | epos[k];
            FCLSH_CUDA(cudaMemcpy(fs->ent_pk.ensure(pk.size() * 8), pk.data(), pk.size() * 8, cudaMemcpyHostToDevice));
            if (N <= (uint64_t(1) << 16) && plan.dims <= (uint64_t(1) << 16)) {
                // the fused query hash's position-parallel sketch: one entry per
                // view position (missing positions of a short part: seed 0)
                std::vector<uint64_t> sk(size_t(fs->parts) * fs->max_part_dims, 0);
                for (uint32_t p = 0; p < fs->parts; ++p) {
                    const Family& f = families[p];
                    for (uint64_t j = 0; j < f.dims; ++j)
                        sk[size_t(p) * fs->max_part_dims + j] =
                            (f.seeds[j] << 32) | (uint64_t(f.mapping[j]) << 16) | uint64_t(plan.source_bit(p, j));
                }
                FCLSH_CUDA(cudaMemcpy(fs->ent_sk.ensure(sk.size() * 8), sk.data(), sk.size() * 8, cudaMemcpyHostToDevice));
            }
        }
    }

    // ---------------- fast path tables
    fs->fast = fs->prime == kMersenne31 && fs->logn >= 2 && fs->logn <= 11 &&
               fs->max_part_dims <= (uint64_t(1) << 15) && plan.dims < (uint64_t(1) << 24);
    if (fs->fast) {
        // Positions on column 0 never reach a key (they cancel in l1 - FHT[v]); drop them.
        bool direct = true;
        for (const Family& f : families) {
            std::vector<uint32_t> cnt(N, 0);
            for (uint64_t j = 0; j < f.dims; ++j)
                if (f.mapping[j] != 0 && ++cnt[f.mapping[j]] > 1) direct = false;
        }
        fs->direct = direct;
        const int G = lanes_for(int(fs->logn));
        const uint64_t E = N / G;
        std::vector<uint2> blob;
        if (direct) {
            fs->part_words = uint32_t(N);
            blob.assign(size_t(fs->parts) * N, make_uint2(0, 0));
            for (uint32_t p = 0; p < fs->parts; ++p) {
                const Family& f = families[p];
                for (uint64_t j = 0; j < f.dims; ++j)
                    if (f.mapping[j] != 0)
                        // column c = g*E + j -> pair (j/2) of lane g, lanes fastest (16-byte loads)
                        blob[size_t(p) * N + ((f.mapping[j] % E) / 2) * 2 * G + 2 * (f.mapping[j] / E) +
                             (f.mapping[j] % E) % 2] =
                            make_uint2(uint32_t(plan.source_bit(p, j)), uint32_t(f.seeds[j]));
            }
        } else {
            // per lane g: entries of columns [gE, gE+E), sorted by column, padded to M
            std::vector<std::vector<std::vector<uint2>>> lists(fs->parts, std::vector<std::vector<uint2>>(G));
            uint32_t M = 1;
            for (uint32_t p = 0; p < fs->parts; ++p) {
                const Family& f = families[p];
                std::vector<std::vector<uint64_t>> bycol(N);
                for (uint64_t j = 0; j < f.dims; ++j)
                    if (f.mapping[j] != 0) bycol[f.mapping[j]].push_back(j);
                for (int g = 0; g < G; ++g) {
                    auto& L = lists[p][g];
                    for (uint64_t c = g * E; c < (g + 1) * E; ++c)
                        for (uint64_t j : bycol[c])
                            L.push_back(make_uint2(uint32_t(plan.source_bit(p, j)) | (uint32_t(c - g * E) << 24),
                                                   uint32_t(f.seeds[j])));
                    M = std::max<uint32_t>(M, uint32_t(L.size()));
                }
            }
            fs->lane_entries = M;
            fs->part_words = uint32_t(G) * M;
            blob.assign(size_t(fs->parts) * fs->part_words, make_uint2(uint32_t(E - 1) << 24, 0));
            for (uint32_t p = 0; p < fs->parts; ++p)
                for (int g = 0; g < G; ++g)
                    for (size_t k = 0; k < lists[p][g].size(); ++k) // lane-fastest: conflict-free
                        blob[size_t(p) * fs->part_words + k * G + g] = lists[p][g][k];
        }
        // shared-memory budget check (227 KB per CTA)
        const uint64_t smem = uint64_t(256) * E * 8 + uint64_t(256 / G) * fs->row_words * 8 +
                              uint64_t(fs->parts) * fs->part_words * 8;
        if (smem > 227 * 1024) {
            fs->fast = false;
        } else {
            FCLSH_CUDA(cudaMemcpy(fs->fam.ensure(blob.size() * 8), blob.data(), blob.size() * 8,
                                  cudaMemcpyHostToDevice));
        }
    }
    fs->families = std::move(families);
    return fs;
}

namespace {
// hash_tables_into (classic.cpp:48-63) for n rows: thread per (row, table),
// consecutive threads on consecutive tables of a row (point-major keys
// coalesce); key = sum of the seeds at the set sampled positions mod prime,
// reduced term by term (every partial sum < prime < 2^63: the same residue
// as the reference's 128-bit sum % prime).
__global__ void __launch_bounds__(256) k_hash_classic(const uint64_t* __restrict__ rows, uint64_t n, uint32_t words,
                                                      uint64_t tables, uint32_t k, const uint32_t* __restrict__ pos,
                                                      const uint64_t* __restrict__ seeds, uint64_t prime,
                                                      void* __restrict__ keys, uint64_t key_stride, int layout,
                                                      int key_bytes) {
    const uint64_t total = n * tables;
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < total;
         x += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = x / tables, t = x % tables;
        const uint64_t* r = rows + i * words;
        const uint32_t* p = pos + t * k;
        const uint64_t* sd = seeds + t * k;
        uint64_t acc = 0;
        for (uint32_t j = 0; j < k; ++j) {
            const uint32_t b = __ldg(p + j);
            FCLSH_DCHECK((b >> 6) < words);
            const uint64_t bit = (__ldg(r + (b >> 6)) >> (b & 63)) & 1;
            acc += __ldg(sd + j) & (0ull - bit);
            acc = acc >= prime ? acc - prime : acc;
        }
        const uint64_t dst = layout == kLayoutPointMajor ? i * key_stride + t : t * key_stride + i;
        if (key_bytes == 4)
            static_cast<uint32_t*>(keys)[dst] = uint32_t(acc);
        else
            static_cast<uint64_t*>(keys)[dst] = acc;
    }
}
} // namespace

std::unique_ptr<DeviceFamilySet> make_device_classic_set(const BitSampleFamily& f, int device) {
    if (f.prime >= (uint64_t(1) << 63)) throw UsageError("hash: primes >= 2^63 are not supported");
    auto fs = std::make_unique<DeviceFamilySet>();
    fs->device = device;
    fs->parts = 1;
    fs->classic = true;
    fs->cls_k = f.k;
    fs->tables = f.tables;
    fs->prime = f.prime;
    fs->dims = f.dims;
    fs->row_words = uint32_t((f.dims + 63) / 64);
    fs->max_part_dims = f.dims;
    FCLSH_CUDA(cudaSetDevice(device));
    fs->cls_pos.ensure(f.positions.size() * 4);
    fs->cls_seed.ensure(f.seeds.size() * 8);
    FCLSH_CUDA(cudaMemcpy(fs->cls_pos.p, f.positions.data(), f.positions.size() * 4, cudaMemcpyHostToDevice));
    FCLSH_CUDA(cudaMemcpy(fs->cls_seed.p, f.seeds.data(), f.seeds.size() * 8, cudaMemcpyHostToDevice));
    fs->classic_family = f;
    return fs;
}

std::unique_ptr<DeviceFamilySet> make_device_family_set(const Family& f, int device) {
    Plan plan;
    plan.kind = PlanKind::identity;
    plan.dims = f.dims;
    plan.radius = f.radius;
    plan.t = 1;
    plan.per_part_radius = f.radius;
    return make_device_family_set(plan, std::vector<Family>{f}, device);
}

void hash_rows(DeviceFamilySet& fs, const uint64_t* d_rows, uint64_t n, void* d_keys,
               uint32_t key_bytes, uint64_t key_stride, int layout, cudaStream_t stream,
               uint32_t part_begin, uint32_t part_count, uint64_t* rows_copy) {
    if (part_count == 0) part_count = fs.parts - part_begin;
    if (part_begin + part_count > fs.parts) throw UsageError("hash: part range out of bounds");
    if (key_bytes != 4 && key_bytes != 8) throw UsageError("hash: key_bytes must be 4 or 8");
    if (key_bytes == 4 && fs.prime > 0xFFFFFFFFull)
        throw UsageError("hash: 4-byte keys need a prime below 2^32");
    if (layout != 0 && layout != 1) throw UsageError("hash: unknown key layout");
    if (layout == 0 && key_stride < n) throw UsageError("hash: key_stride below the row count");
    if (layout == 1 && key_stride < uint64_t(part_count) * fs.tables)
        throw UsageError("hash: key_stride below the table count");
    if (n == 0) return;
    FCLSH_CUDA(cudaSetDevice(fs.device));
    if (fs.classic) {
        if (rows_copy) {
            FCLSH_CUDA(cudaMemcpyAsync(rows_copy, d_rows, n * fs.row_words * 8, cudaMemcpyDefault, stream));
            d_rows = rows_copy;
        }
        const uint64_t work = n * fs.tables;
        const unsigned grid = unsigned(std::max<uint64_t>(
            1, std::min<uint64_t>((work + 255) / 256, uint64_t(sm_count(fs.device)) * 8)));
        k_hash_classic<<<grid, 256, 0, stream>>>(d_rows, n, fs.row_words, fs.tables, fs.cls_k,
                                                fs.cls_pos.as<uint32_t>(), fs.cls_seed.as<uint64_t>(), fs.prime,
                                                d_keys, key_stride, layout, int(key_bytes));
        FCLSH_LAUNCHED();
        return;
    }
    if (rows_copy && !fs.fast) {
        // only k_hash_f64_pt copies as it goes: copy first, hash the copy
        FCLSH_CUDA(cudaMemcpyAsync(rows_copy, d_rows, n * fs.row_words * 8, cudaMemcpyDefault, stream));
        d_rows = rows_copy;
        rows_copy = nullptr;
    }
    if (fs.fast) {
        FastParams prm{};
        prm.rows = d_rows;
        prm.rows_copy = rows_copy;
        prm.n = n;
        prm.row_words = fs.row_words;
        prm.parts = part_count;
        prm.part_words = fs.part_words;
        prm.lane_entries = fs.lane_entries;
        prm.fam = fs.fam.as<uint2>() + size_t(part_begin) * fs.part_words;
        prm.keys = d_keys;
        prm.key_stride = key_stride;
        prm.L = fs.tables;
        prm.layout = layout;
        prm.key_bytes = int(key_bytes);
        if (fs.direct)
            dispatch_fast<true>(fs, prm, stream);
        else
            dispatch_fast<false>(fs, prm, stream);
        return;
    }
    GenericParams prm{};
    prm.rows = d_rows;
    prm.n = n;
    prm.row_words = fs.row_words;
    prm.parts = part_count;
    prm.N = fs.order;
    prm.L = fs.tables;
    prm.prime = fs.prime;
    prm.max_dims = fs.max_part_dims;
    prm.col_ptr = fs.col_ptr.as<uint32_t>() + size_t(part_begin) * (fs.order + 1);
    prm.ent_pos = fs.ent_pos.as<uint32_t>() + size_t(part_begin) * fs.max_part_dims;
    prm.ent_seed = fs.ent_seed.as<uint64_t>() + size_t(part_begin) * fs.max_part_dims;
    prm.keys = d_keys;
    prm.key_stride = key_stride;
    prm.layout = layout;
    prm.key_bytes = int(key_bytes);
    const size_t tbytes = size_t(fs.order) * 8;
    const uint64_t grid = std::min<uint64_t>(n, uint64_t(sm_count(fs.device)) * 8);
    size_t smem = 0;
    if (tbytes <= 96 * 1024) {
        prm.use_smem = 1;
        smem = tbytes;
        FCLSH_CUDA(cudaFuncSetAttribute(k_hash_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    } else {
        prm.use_smem = 0;
        prm.scratch = static_cast<uint64_t*>(fs.scratch.ensure(grid * tbytes));
    }
    k_hash_generic<<<unsigned(grid), 256, smem, stream>>>(prm);
    FCLSH_LAUNCHED();
}

} // namespace fclsh_b200
