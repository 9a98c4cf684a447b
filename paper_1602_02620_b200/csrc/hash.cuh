// K1: batched fcLSH covering-hash evaluation (reference: hash_batch_into,
// covering.cpp:169-182 -> batch_hash_kernel, hadamard.cpp:51-72).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "common.cuh"
#include "host.hpp"

namespace fclsh_b200 {

constexpr int kLayoutTableMajor = 0; // key[(part*L + v-1)*stride + row]
constexpr int kLayoutPointMajor = 1; // key[row*stride + part*L + v-1]

// One covering family per view ("part") of a preprocessing plan, with the
// plan's bit gather (partition permutation / replicate wrap) folded into the
// family's position table: view position j of part p reads source bit
// plan.source_bit(p, j) of the stored row. Device-resident, immutable.
struct DeviceFamilySet {
    int device = 0;
    uint32_t parts = 0;
    uint32_t radius = 0;   // per-part radius r'
    uint32_t logn = 0;     // r' + 1
    uint64_t order = 0;    // N = 2^(r'+1)
    uint64_t tables = 0;   // L = N - 1 per part
    uint64_t prime = 0;
    uint64_t dims = 0;     // source row width in bits
    uint32_t row_words = 0;
    std::vector<Family> families; // host copies, one per part

    // Fast path (prime == 2^31-1): per part, either a direct column table
    // ({pos, seed}[N], every column has <= 1 position) or per-lane lists
    // ({pos | col_local << 24, seed}[G][M], sorted by column).
    bool fast = false;
    bool direct = false;
    uint32_t lane_entries = 0; // M
    uint32_t part_words = 0;   // uint2 per part in `fam`
    DevBuf fam;

    // Generic path (any odd prime < 2^63): CSR over columns, per part.
    DevBuf col_ptr;  // uint32 [parts][N+1]
    DevBuf ent_pos;  // uint32 [parts][max_dims]
    DevBuf ent_seed; // uint64 [parts][max_dims]
    DevBuf ent_pk;   // uint64 [parts][max_dims]: seed << 32 | source bit, primes < 2^32 (the fused query hash)
    DevBuf ent_sk;   // uint64 [parts][max_dims], view order: seed << 32 | column << 16 | source bit (fused hash, N <= 2^16, d <= 2^16)
    uint64_t max_part_dims = 0;
    DevBuf scratch;  // generic path workspace

    // Classic bit sampling (Method::classic, classic.hpp): one part of
    // `tables` tables, k sampled positions each; hash_rows runs
    // k_hash_classic (hash_tables_into, classic.cpp:48-63).
    bool classic = false;
    uint32_t cls_k = 0;
    DevBuf cls_pos;  // uint32 [tables][k]
    DevBuf cls_seed; // uint64 [tables][k]
    BitSampleFamily classic_family; // host copy

    uint64_t total_tables() const { return uint64_t(parts) * tables; }
};

// Builds the device family set for `plan` with the given per-part families
// (families[p].dims == plan.part_dims(p)).
std::unique_ptr<DeviceFamilySet> make_device_family_set(const Plan& plan,
                                                        std::vector<Family> families, int device);
// The classic bit-sampling family over rows of f.dims bits (identity plan).
std::unique_ptr<DeviceFamilySet> make_device_classic_set(const BitSampleFamily& f, int device);
// A single family over rows of exactly f.dims bits (identity plan).
std::unique_ptr<DeviceFamilySet> make_device_family_set(const Family& f, int device);

// Hash n rows (d_rows: n x row_words) for every part; keys in `layout`
// (0 table-major: key[(p*L + v-1)*stride + i]; 1 point-major:
// key[i*stride + p*L + v-1]). key_bytes 4 requires prime < 2^32.
// Only parts [part_begin, part_begin + part_count) are hashed (part_count 0
// = all); table indices in the output are relative to part_begin.
void hash_rows(DeviceFamilySet& fs, const uint64_t* d_rows, uint64_t n, void* d_keys,
               uint32_t key_bytes, uint64_t key_stride, int layout, cudaStream_t stream,
               uint32_t part_begin = 0, uint32_t part_count = 0, uint64_t* rows_copy = nullptr);
// rows_copy (optional): the rows are also written there (n * row_words
// words); the point-major FP64 kernel does it as it stages each row, so a
// query batch can be hashed straight from mapped pinned host memory while
// its device copy (for the verify) is made on the way.

} // namespace fclsh_b200
