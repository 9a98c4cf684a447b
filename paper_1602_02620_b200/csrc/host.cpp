#include "host.hpp"

#include <cmath>
#include <numeric>

namespace fclsh_b200 {

uint64_t splitmix64(uint64_t x) { // rng.cpp:9-14
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

namespace {

uint64_t fnv1a(std::string_view s) { // rng.cpp:18-25
    uint64_t h = 0xcbf29ce484222325ull;
    for (char c : s) {
        h ^= static_cast<uint8_t>(c);
        h *= 0x100000001b3ull;
    }
    return h;
}

void check_basic(uint64_t dims, uint32_t radius, uint64_t prime) { // covering.cpp:14-22
    if (dims == 0) throw UsageError("covering family: dims must be positive");
    if (radius == 0) throw UsageError("covering family: radius must be >= 1");
    if (radius > kMaxCoveringRadius)
        throw ResourceError("covering family: radius " + std::to_string(radius) +
                            " exceeds the table budget (max " + std::to_string(kMaxCoveringRadius) + ")");
    if (prime < 3 || prime % 2 == 0) throw UsageError("covering family: prime must be odd and > 2");
    // The reference's add_mod is exact only while a + b < 2^64
    // (modmath.hpp:12-15); the device field code keeps that domain.
    if (prime >= (uint64_t(1) << 63))
        throw UsageError("covering family: prime must be below 2^63");
}

void check_kind_fits(uint64_t dims, uint32_t radius, Kind kind) { // covering.cpp:24-32
    uint64_t order = uint64_t(1) << (radius + 1);
    if (kind == Kind::specific && dims > order)
        throw UsageError("covering family: specific construction needs dims <= " +
                         std::to_string(order) + ", got " + std::to_string(dims));
    if (kind == Kind::general && dims <= order)
        throw UsageError("covering family: general construction needs dims > " +
                         std::to_string(order) + ", got " + std::to_string(dims));
}

uint64_t tables_for_radius(uint32_t r) { return (uint64_t(1) << (r + 1)) - 1; }

} // namespace

Rng Rng::stream(std::string_view label) const { // rng.cpp:31-33
    return Rng(splitmix64(seed_ ^ fnv1a(label)));
}

Rng Rng::stream(std::string_view label, uint64_t index) const { // rng.cpp:35-37
    return Rng(splitmix64(seed_ ^ fnv1a(label) ^ splitmix64(index + 1)));
}

uint64_t Rng::below(uint64_t bound) { // rng.cpp:41-50
    if (bound == 0) throw UsageError("rng: zero bound");
    uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
        x = next_u64();
    } while (x >= limit);
    return x % bound;
}

Family build_family(uint64_t dims, uint32_t radius, int kind_in, uint64_t rng_seed, uint64_t prime,
                    bool include_zero_column) {
    check_basic(dims, radius, prime);
    uint64_t order = uint64_t(1) << (radius + 1);
    Kind kind = kind_in < 0 ? (dims > order ? Kind::general : Kind::specific) // covering.cpp:74-80
                            : static_cast<Kind>(kind_in);
    check_kind_fits(dims, radius, kind);
    Rng rng(rng_seed);
    Family f;
    f.dims = dims;
    f.radius = radius;
    f.prime = prime;
    f.kind = kind;
    f.mapping.resize(dims);
    f.seeds.resize(dims);
    if (kind == Kind::general) { // covering.cpp:53-59
        Rng map_rng = rng.stream("mapping");
        for (uint64_t i = 0; i < dims; ++i)
            f.mapping[i] = include_zero_column ? static_cast<uint32_t>(map_rng.below(order))
                                               : static_cast<uint32_t>(1 + map_rng.below(order - 1));
    } else { // covering.cpp:60-66
        Rng perm_rng = rng.stream("permutation");
        std::vector<uint32_t> columns(order);
        std::iota(columns.begin(), columns.end(), 0u);
        perm_rng.shuffle(columns);
        for (uint64_t i = 0; i < dims; ++i) f.mapping[i] = columns[i];
    }
    Rng seed_rng = rng.stream("seeds"); // covering.cpp:68-69
    for (uint64_t i = 0; i < dims; ++i) f.seeds[i] = seed_rng.below(prime);
    return f;
}

Family make_family(uint64_t dims, uint32_t radius, Kind kind, std::vector<uint32_t> mapping,
                   std::vector<uint64_t> seeds, uint64_t prime) { // covering.cpp:84-111
    check_basic(dims, radius, prime);
    if (mapping.size() != dims || seeds.size() != dims)
        throw UsageError("covering family: mapping/seeds must have one entry per dimension");
    Family f;
    f.dims = dims;
    f.radius = radius;
    f.prime = prime;
    f.kind = kind;
    f.mapping = std::move(mapping);
    f.seeds = std::move(seeds);
    uint64_t order = f.order();
    std::vector<bool> seen(order, false);
    for (uint32_t m : f.mapping) {
        if (m >= order) throw UsageError("covering family: mapping entry out of range");
        if (kind == Kind::specific) {
            if (seen[m]) throw UsageError("covering family: specific mapping must be injective");
            seen[m] = true;
        }
    }
    for (uint64_t b : f.seeds)
        if (b >= f.prime) throw UsageError("covering family: seed out of field range");
    return f;
}

Plan make_plan(uint64_t dims, uint32_t radius, double c, uint64_t n, uint64_t rng_seed,
               const PlanOverride* force, uint64_t table_budget) { // transform.cpp:32-113
    if (dims == 0) throw UsageError("plan: dims must be positive");
    if (radius == 0) throw UsageError("plan: radius must be >= 1");
    if (radius >= dims) throw UsageError("plan: radius must be below dims");
    if (c < 1.0) throw UsageError("plan: approximation factor must be >= 1");
    if (n < 2) throw UsageError("plan: need at least two data points");

    PlanKind kind;
    uint32_t t;
    double logn = std::log2(static_cast<double>(n));
    double cr = c * static_cast<double>(radius);
    if (force) {
        if (force->t == 0) throw UsageError("plan: override factor must be >= 1");
        if (force->kind == PlanKind::identity && force->t != 1)
            throw UsageError("plan: identity override must have t = 1");
        kind = force->kind;
        t = force->t;
    } else if (cr < logn - 1e-9) {
        kind = PlanKind::replicate;
        t = static_cast<uint32_t>(std::floor(logn / cr + 1e-9));
    } else if (cr > logn + 1e-9) {
        kind = PlanKind::partition;
        t = static_cast<uint32_t>(std::ceil(cr / logn - 1e-9));
    } else {
        kind = PlanKind::identity;
        t = 1;
    }
    if (t <= 1) kind = PlanKind::identity;

    Plan plan;
    plan.dims = dims;
    plan.radius = radius;
    if (kind == PlanKind::identity) {
        if (radius > kMaxCoveringRadius || tables_for_radius(radius) > table_budget)
            throw ResourceError("plan: radius " + std::to_string(radius) +
                                " needs more tables than the budget allows");
        plan.kind = PlanKind::identity;
        plan.t = 1;
        plan.per_part_radius = radius;
        return plan;
    }
    if (kind == PlanKind::replicate) {
        while (t > 1 && (uint64_t(t) * radius > kMaxCoveringRadius ||
                         tables_for_radius(t * radius) > table_budget))
            --t;
        if (t == 1) {
            plan.kind = PlanKind::identity;
            plan.t = 1;
            plan.per_part_radius = radius;
            return plan;
        }
        plan.kind = PlanKind::replicate;
        plan.t = t;
        plan.per_part_radius = t * radius;
        return plan;
    }
    if (t > radius)
        throw UsageError("plan: cannot cut radius " + std::to_string(radius) + " into " +
                         std::to_string(t) + " parts");
    if (t > dims) throw UsageError("plan: more parts than dimensions");
    uint32_t part_radius = radius / t;
    if (part_radius > kMaxCoveringRadius || uint64_t(t) * tables_for_radius(part_radius) > table_budget)
        throw ResourceError("plan: partition table count exceeds the budget");
    plan.kind = PlanKind::partition;
    plan.t = t;
    plan.per_part_radius = part_radius;
    plan.permutation.resize(dims);
    std::iota(plan.permutation.begin(), plan.permutation.end(), 0u);
    Rng perm_rng = Rng(rng_seed).stream("plan-permutation");
    perm_rng.shuffle(plan.permutation);
    uint64_t base = dims / t, rem = dims % t, begin = 0;
    for (uint32_t p = 0; p < t; ++p) {
        uint64_t width = base + (p >= t - rem ? 1 : 0);
        plan.parts.emplace_back(begin, begin + width);
        begin += width;
    }
    return plan;
}

uint32_t choose_k(uint64_t dims, uint32_t radius, uint64_t tables, double delta) {
    if (dims == 0) throw UsageError("choose_k: dims must be positive");
    if (radius == 0 || radius >= dims) throw UsageError("choose_k: radius must be in [1, dims)");
    if (tables == 0) throw UsageError("choose_k: need at least one table");
    if (!(delta > 0.0 && delta < 1.0)) throw UsageError("choose_k: delta must be in (0, 1)");
    // k = ceil(log(1 - delta^(1/L)) / log(1 - r/d)), clamped into [1, 4d]
    const double per_table = 1.0 - std::exp(std::log(delta) / static_cast<double>(tables));
    const double raw = std::log(per_table) / std::log1p(-static_cast<double>(radius) / static_cast<double>(dims));
    const double k = std::ceil(raw);
    const double cap = static_cast<double>(kMaxSamplesPerDim) * static_cast<double>(dims);
    if (!(k >= 1.0)) return 1;
    if (k > cap) return static_cast<uint32_t>(cap);
    return static_cast<uint32_t>(k);
}

BitSampleFamily build_bit_sample_family(uint64_t dims, uint32_t k, uint64_t tables, uint64_t rng_seed,
                                        uint64_t prime) {
    if (dims == 0) throw UsageError("bit sample family: dims must be positive");
    if (k == 0) throw UsageError("bit sample family: k must be >= 1");
    if (tables == 0) throw UsageError("bit sample family: need at least one table");
    if (prime < 3 || prime % 2 == 0) throw UsageError("bit sample family: prime must be odd and > 2");
    BitSampleFamily f;
    f.dims = dims;
    f.k = k;
    f.tables = tables;
    f.prime = prime;
    f.positions.resize(tables * uint64_t(k));
    f.seeds.resize(tables * uint64_t(k));
    const Rng rng(rng_seed);
    Rng pos_rng = rng.stream("positions");
    Rng seed_rng = rng.stream("seeds");
    for (uint64_t j = 0; j < f.positions.size(); ++j) { // positions and seeds from their own streams
        f.positions[j] = static_cast<uint32_t>(pos_rng.below(dims));
        f.seeds[j] = seed_rng.below(prime);
    }
    return f;
}

} // namespace fclsh_b200
