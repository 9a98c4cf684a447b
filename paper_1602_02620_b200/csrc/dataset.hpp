// Dataset containers (dataset.hpp:20-31): FCL1 and text, read into the
// engine's row layout ([n][ceil(d/64)] u64 words, BitVector's word layout).
#pragma once

#include <cstdint>
#include <string>

#include "host.hpp"

namespace fclsh_b200 {

constexpr int kDatasetFcl1 = 1;
constexpr int kDatasetText = 2;

struct HostDataset {
    uint64_t n = 0, dims = 0;
    int format = 0;
    uint64_t* rows = nullptr; // [n][words()], pinned when a CUDA device is usable
    bool pinned = false;
    HostDataset() = default;
    HostDataset(const HostDataset&) = delete;
    HostDataset& operator=(const HostDataset&) = delete;
    HostDataset(HostDataset&& o) noexcept { *this = std::move(o); }
    HostDataset& operator=(HostDataset&& o) noexcept {
        if (this != &o) {
            release();
            n = o.n;
            dims = o.dims;
            format = o.format;
            rows = o.rows;
            pinned = o.pinned;
            o.rows = nullptr;
        }
        return *this;
    }
    ~HostDataset() { release(); }
    uint64_t words() const { return (dims + 63) / 64; }
    void alloc(uint64_t words_needed);
    void release();
};

// load_dataset (dataset.cpp:101-111): sniffs the FCL1 magic, else text.
HostDataset load_dataset(const std::string& path);
// save_dataset / save_dataset_text (dataset.cpp:82-98).
void save_dataset(const std::string& path, const uint64_t* rows, uint64_t n, uint64_t dims, int format);

} // namespace fclsh_b200
