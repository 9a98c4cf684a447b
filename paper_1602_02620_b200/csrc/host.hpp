// Host-side model of the fcLSH objects: errors, Rng, covering families and
// preprocessing plans. Restates the reference's semantics (cited per
// function) so that families, permutations and seeds are bit-identical to
// the reference's for the same seed; the device code consumes these.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace fclsh_b200 {

// errors.hpp:8-29 (codes = CLI exit codes); CudaError has no reference
// counterpart.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct UsageError : Error {
    explicit UsageError(const std::string& m) : Error(2, m) {}
};
struct DataError : Error {
    explicit DataError(const std::string& m) : Error(3, m) {}
};
struct ResourceError : Error {
    explicit ResourceError(const std::string& m) : Error(4, m) {}
};
struct CudaError : Error {
    explicit CudaError(const std::string& m) : Error(5, m) {}
};

inline constexpr uint64_t kMersenne61 = (uint64_t(1) << 61) - 1; // modmath.hpp:10
inline constexpr uint64_t kMersenne31 = (uint64_t(1) << 31) - 1;
inline constexpr uint32_t kMaxCoveringRadius = 20;                // covering.hpp:53
inline constexpr uint64_t kDefaultTableBudget = uint64_t(1) << 21; // transform.hpp:52

uint64_t splitmix64(uint64_t x); // rng.cpp:9-14

// rng.hpp:18-51 restated: seed fans out into labelled sub-streams; draws come
// from std::mt19937_64 (standard-specified, so identical everywhere).
class Rng {
public:
    explicit Rng(uint64_t seed) : seed_(seed), eng_(splitmix64(seed)) {}
    Rng stream(std::string_view label) const;
    Rng stream(std::string_view label, uint64_t index) const;
    uint64_t seed() const { return seed_; }
    uint64_t next_u64() { return eng_(); }
    uint64_t below(uint64_t bound); // rng.cpp:41-50
    template <typename T>
    void shuffle(std::vector<T>& v) { // rng.hpp:38-44
        for (size_t i = v.size(); i > 1; --i) {
            size_t j = static_cast<size_t>(below(i));
            std::swap(v[i - 1], v[j]);
        }
    }

private:
    uint64_t seed_;
    std::mt19937_64 eng_;
};

enum class Kind : int32_t { general = 0, specific = 1 };

// CoveringFamily (covering.hpp:34-43)
struct Family {
    uint64_t dims = 0;
    uint32_t radius = 0;
    uint64_t prime = kMersenne61;
    Kind kind = Kind::general;
    std::vector<uint32_t> mapping;
    std::vector<uint64_t> seeds;
    uint64_t order() const { return uint64_t(1) << (radius + 1); }
    uint64_t tables() const { return order() - 1; }
};

// build_covering_family (covering.cpp:40-80); kind < 0 derives it.
Family build_family(uint64_t dims, uint32_t radius, int kind, uint64_t rng_seed, uint64_t prime,
                    bool include_zero_column);
// make_covering_family (covering.cpp:84-111)
Family make_family(uint64_t dims, uint32_t radius, Kind kind, std::vector<uint32_t> mapping,
                   std::vector<uint64_t> seeds, uint64_t prime);

// BitSampleFamily (classic.hpp:15-27): the classic bit-sampling baseline.
// Table t's key is the sum, mod prime, of the seeds of its k sampled
// positions (with replacement) that are set in the row.
struct BitSampleFamily {
    uint64_t dims = 0;
    uint32_t k = 0;
    uint64_t tables = 0;
    uint64_t prime = kMersenne61;
    std::vector<uint32_t> positions; // tables * k
    std::vector<uint64_t> seeds;     // tables * k, each < prime
};
constexpr uint32_t kMaxSamplesPerDim = 4; // classic.hpp:30
// choose_k (classic.cpp:10-23)
uint32_t choose_k(uint64_t dims, uint32_t radius, uint64_t tables, double delta);
// build_bit_sample_family (classic.cpp:25-46)
BitSampleFamily build_bit_sample_family(uint64_t dims, uint32_t k, uint64_t tables, uint64_t rng_seed,
                                        uint64_t prime);

enum class PlanKind : int32_t { identity = 0, replicate = 1, partition = 2 };

// PreprocessPlan (transform.hpp:26-44)
struct Plan {
    PlanKind kind = PlanKind::identity;
    uint64_t dims = 0;
    uint32_t radius = 0;
    uint32_t t = 1;
    uint32_t per_part_radius = 0;
    std::vector<uint32_t> permutation;
    std::vector<std::pair<uint64_t, uint64_t>> parts;
    uint32_t part_count() const { return kind == PlanKind::partition ? t : 1; }
    uint64_t part_dims(uint32_t p) const {
        if (kind == PlanKind::partition) return parts[p].second - parts[p].first;
        return kind == PlanKind::replicate ? dims * t : dims;
    }
    // Source bit of view p's position j (transform.cpp:115-135).
    uint64_t source_bit(uint32_t p, uint64_t j) const {
        if (kind == PlanKind::partition) return permutation[parts[p].first + j];
        if (kind == PlanKind::replicate) return j % dims;
        return j;
    }
    uint64_t table_count() const { // plan_table_count (transform.cpp:155-158)
        return uint64_t(part_count()) * ((uint64_t(1) << (per_part_radius + 1)) - 1);
    }
};

struct PlanOverride {
    PlanKind kind;
    uint32_t t;
};

// make_plan (transform.cpp:32-113)
Plan make_plan(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t rng_seed,
               const PlanOverride* force, uint64_t table_budget);

} // namespace fclsh_b200
