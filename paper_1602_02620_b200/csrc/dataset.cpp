// Dataset containers (reference: dataset.hpp:20-31, dataset.cpp:29-111), read
// straight into the engine's row layout.
//
// FCL1: "FCL1", n and d as little-endian u64, then n rows of ceil(d/8) bytes,
// bit j of a row in byte j/8 at offset j%8, padding bits zero. On a
// little-endian host those bytes ARE the row's u64 words (bit j in word j/64
// at offset j%64), so a row is a byte copy into a W*8-byte slot; for
// d % 64 == 0 the whole file body is the [n][W] row array and is read with
// one fread into the destination (pinned host memory for an upload).
// Text: one '0'/'1' line per vector, '\r' stripped, empty lines skipped.
// Validation and messages follow the reference, in its order: per row,
// truncation then dirty padding; then trailing bytes.

#include "dataset.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace fclsh_b200 {

namespace {

struct File {
    FILE* f = nullptr;
    explicit File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

uint64_t le_u64(const unsigned char* b) {
    uint64_t x = 0;
    for (int i = 0; i < 8; ++i) x |= uint64_t(b[i]) << (8 * i);
    return x;
}

bool has_magic(FILE* f) {
    unsigned char m[4] = {0, 0, 0, 0};
    const size_t got = std::fread(m, 1, 4, f);
    return got == 4 && m[0] == 'F' && m[1] == 'C' && m[2] == 'L' && m[3] == '1';
}

// Text rows: parse all lines (the width of the first defines d).
void parse_text(FILE* f, uint64_t& dims, std::vector<uint64_t>& rows, uint64_t& n) {
    std::string line;
    dims = 0;
    n = 0;
    auto flush_line = [&]() {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) return;
        const uint64_t w = line.size();
        // the characters first (BitVector::from_string, bitvec.cpp:21-31), then the width
        std::vector<uint64_t> v((w + 63) / 64, 0);
        for (uint64_t i = 0; i < w; ++i) {
            const char c = line[i];
            if (c == '1')
                v[i / 64] |= uint64_t(1) << (i % 64);
            else if (c != '0')
                throw DataError("bit string: unexpected character '" + std::string(1, c) + "'");
        }
        if (n == 0) {
            dims = w;
        } else if (w != dims) {
            throw DataError("dataset: line " + std::to_string(n) + " has width " + std::to_string(w) +
                            ", expected " + std::to_string(dims));
        }
        rows.insert(rows.end(), v.begin(), v.end());
        ++n;
    };
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) {
        for (size_t i = 0; i < got; ++i) {
            if (buf[i] == '\n') {
                flush_line();
                line.clear();
            } else {
                line.push_back(buf[i]);
            }
        }
    }
    flush_line();
    if (n == 0) throw DataError("dataset: no vectors in text input");
}

// FCL1 body after the magic: header, then rows into out ([n][W] words; out
// may be null to validate only). Returns (n, d).
void read_fcl1(FILE* f, uint64_t& n, uint64_t& dims, uint64_t* out, bool header_only) {
    unsigned char h[16];
    if (std::fread(h, 1, 8, f) != 8) throw DataError("dataset: truncated header");
    n = le_u64(h);
    if (std::fread(h + 8, 1, 8, f) != 8) throw DataError("dataset: truncated header");
    dims = le_u64(h + 8);
    if (dims == 0) throw DataError("dataset: zero width");
    if (header_only) return;
    const uint64_t rb = (dims + 7) / 8, W = (dims + 63) / 64;
    const unsigned pad_bits = unsigned(dims % 8);
    if (rb == W * 8 && out) { // d % 64 == 0: the body is the row array
        const uint64_t got = std::fread(out, 1, n * rb, f);
        if (got != n * rb) throw DataError("dataset: truncated at row " + std::to_string(got / rb));
    } else {
        std::vector<unsigned char> chunk;
        const uint64_t per = std::max<uint64_t>(1, (uint64_t(8) << 20) / rb); // rows per 8 MB read
        for (uint64_t i0 = 0; i0 < n; i0 += per) {
            const uint64_t m = std::min(per, n - i0);
            chunk.resize(m * rb);
            const uint64_t got = std::fread(chunk.data(), 1, m * rb, f);
            const uint64_t full = got / rb;
            for (uint64_t k = 0; k < full; ++k) {
                const unsigned char* src = chunk.data() + k * rb;
                if (pad_bits && (src[rb - 1] >> pad_bits) != 0)
                    throw DataError("dataset: nonzero padding bits in row " + std::to_string(i0 + k));
                if (out) {
                    uint64_t* dst = out + (i0 + k) * W;
                    dst[W - 1] = 0;
                    std::memcpy(dst, src, rb);
                }
            }
            if (full < m) throw DataError("dataset: truncated at row " + std::to_string(i0 + full));
        }
    }
    if (std::fgetc(f) != EOF) throw DataError("dataset: trailing bytes after last row");
}

} // namespace

HostDataset load_dataset(const std::string& path) {
    HostDataset ds;
    {
        File f(path, "rb");
        if (!f.f) throw UsageError("dataset: cannot open '" + path + "'");
        if (has_magic(f.f)) {
            read_fcl1(f.f, ds.n, ds.dims, nullptr, true);
            ds.format = kDatasetFcl1;
        } else {
            ds.format = kDatasetText;
        }
    }
    if (ds.format == kDatasetText) {
        File f(path, "rb");
        std::vector<uint64_t> rows;
        parse_text(f.f, ds.dims, rows, ds.n);
        ds.alloc(ds.n * ds.words());
        std::memcpy(ds.rows, rows.data(), rows.size() * 8);
        return ds;
    }
    File f(path, "rb");
    has_magic(f.f);
    uint64_t n = 0, d = 0;
    // a file whose size disagrees with its header fails: run the validating
    // pass (no allocation from a bad header) to raise the reference's error
    const uint64_t rb = (ds.dims + 7) / 8;
    std::fseek(f.f, 0, SEEK_END);
    const long long size = std::ftell(f.f);
    const bool consistent = ds.n <= (uint64_t(1) << 62) / std::max<uint64_t>(1, rb) &&
                            uint64_t(size) == 20 + ds.n * rb;
    std::fseek(f.f, 4, SEEK_SET);
    if (!consistent) {
        read_fcl1(f.f, n, d, nullptr, false);
        throw DataError("dataset: size does not match the header"); // not reached: the pass above throws
    }
    ds.alloc(std::max<uint64_t>(1, ds.n * ds.words()));
    read_fcl1(f.f, n, d, ds.rows, false);
    return ds;
}

void HostDataset::alloc(uint64_t words_needed) {
    release();
    // pinned when a CUDA device is usable (full-speed uploads), else plain host memory
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<uint64_t>(8, words_needed * 8), cudaHostAllocDefault) == cudaSuccess) {
        pinned = true;
    } else {
        cudaGetLastError();
        p = std::calloc(std::max<uint64_t>(1, words_needed), 8);
        if (!p) throw ResourceError("dataset: host memory exhausted");
        pinned = false;
    }
    rows = static_cast<uint64_t*>(p);
}

void HostDataset::release() {
    if (!rows) return;
    if (pinned)
        cudaFreeHost(rows);
    else
        std::free(rows);
    rows = nullptr;
}

void save_dataset(const std::string& path, const uint64_t* rows, uint64_t n, uint64_t dims, int format) {
    if (format != kDatasetFcl1 && format != kDatasetText) throw UsageError("dataset: unknown container format");
    File f(path, format == kDatasetText ? "w" : "wb");
    if (!f.f) throw UsageError("dataset: cannot open '" + path + "' for writing");
    const uint64_t W = (dims + 63) / 64, rb = (dims + 7) / 8;
    bool ok = true;
    if (format == kDatasetFcl1) {
        unsigned char h[20] = {'F', 'C', 'L', '1'};
        for (int i = 0; i < 8; ++i) {
            h[4 + i] = static_cast<unsigned char>((n >> (8 * i)) & 0xff);
            h[12 + i] = static_cast<unsigned char>((dims >> (8 * i)) & 0xff);
        }
        ok = std::fwrite(h, 1, 20, f.f) == 20;
        std::vector<unsigned char> row(rb);
        for (uint64_t i = 0; ok && i < n; ++i) {
            std::memcpy(row.data(), rows + i * W, rb);
            if (dims % 8) row[rb - 1] &= static_cast<unsigned char>((1u << (dims % 8)) - 1); // zero padding
            ok = std::fwrite(row.data(), 1, rb, f.f) == rb;
        }
    } else {
        std::string line(dims + 1, '\n');
        for (uint64_t i = 0; ok && i < n; ++i) {
            const uint64_t* r = rows + i * W;
            for (uint64_t j = 0; j < dims; ++j) line[j] = ((r[j / 64] >> (j % 64)) & 1) ? '1' : '0';
            ok = std::fwrite(line.data(), 1, line.size(), f.f) == line.size();
        }
    }
    if (!ok || std::fflush(f.f) != 0) throw DataError("dataset: write to '" + path + "' failed");
}

} // namespace fclsh_b200
