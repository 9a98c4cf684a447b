// Seeded synthetic inputs for the BASELINE configs.
//
// Counter-based: word k of a stream with key K is splitmix64(K + k*gamma),
// i.e. the k-th output of the standard SplitMix64 sequence seeded with K
// (splitmix64 as in rng.cpp:9-14). Any thread count gives identical bytes.
// Stream keys derive from the root seed through the reference's own labelled
// sub-streams (Rng(seed).stream(label), rng.cpp:31-33).

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <thread>
#include <vector>

#include "host.hpp"

namespace fclsh_b200 {

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

inline uint64_t word_at(uint64_t key, uint64_t k) { return splitmix64(key + k * kGamma); }

// floor(r * bound / 2^64): uniform on [0, bound) up to a bias below bound/2^64
inline uint64_t scale(uint64_t r, uint64_t bound) {
    return uint64_t((unsigned __int128)r * bound >> 64);
}

template <typename F>
void parallel_rows(uint64_t n, int threads, F&& f) {
    int T = std::max(1, threads);
    if (T == 1 || n < 1024) {
        f(0, n);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
        uint64_t b = n * t / T, e = n * (t + 1) / T;
        pool.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& th : pool) th.join();
}

} // namespace

// rows [row0, row0 + n) of the stream (any slice of one global dataset)
void gen_bernoulli(uint64_t seed, uint64_t row0, uint64_t n, uint64_t dims, uint64_t* rows, int threads) {
    const uint64_t key = Rng(seed).stream("data").seed();
    const uint64_t W = (dims + 63) / 64;
    const uint64_t tail = dims % 64 ? (uint64_t(1) << (dims % 64)) - 1 : ~0ull;
    parallel_rows(n, threads, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) {
            const uint64_t g = row0 + i;
            for (uint64_t w = 0; w < W; ++w) rows[i * W + w] = word_at(key, g * W + w);
            rows[i * W + W - 1] &= tail;
        }
    });
}

void gen_clustered(uint64_t seed, uint64_t centres, uint64_t row0, uint64_t n, uint64_t dims, double flip_p,
                   uint64_t* rows, int threads) {
    const uint64_t W = (dims + 63) / 64;
    std::vector<uint64_t> cen(centres * W);
    gen_bernoulli(Rng(seed).stream("centres").seed(), 0, centres, dims, cen.data(), threads);
    const uint64_t kc = Rng(seed).stream("assign").seed();
    const uint64_t kf = Rng(seed).stream("flips").seed();
    const double scaled = flip_p * 18446744073709551616.0; // 2^64
    const uint64_t thresh = flip_p >= 1.0 ? ~0ull : uint64_t(scaled);
    parallel_rows(n, threads, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) {
            const uint64_t g = row0 + i;
            const uint64_t c = scale(word_at(kc, g), centres);
            for (uint64_t w = 0; w < W; ++w) {
                uint64_t flips = 0;
                const uint64_t bits = std::min<uint64_t>(64, dims - w * 64);
                for (uint64_t k = 0; k < bits; ++k)
                    if (word_at(kf, g * dims + w * 64 + k) < thresh) flips |= uint64_t(1) << k;
                rows[i * W + w] = cen[c * W + w] ^ flips;
            }
        }
    });
}

void gen_planted(uint64_t seed, const uint64_t* data, uint64_t n, uint64_t dims, uint64_t nq, uint32_t kmax,
                 uint64_t* qrows, uint32_t* src_out) {
    const uint64_t W = (dims + 63) / 64;
    const uint64_t kq = Rng(seed).stream("queries").seed();
    const uint64_t kp = Rng(seed).stream("positions").seed();
    std::vector<uint32_t> pos(dims);
    for (uint64_t j = 0; j < nq; ++j) {
        const uint64_t src = scale(word_at(kq, 2 * j), n);
        const uint64_t k = scale(word_at(kq, 2 * j + 1), uint64_t(kmax) + 1);
        std::copy(data + src * W, data + src * W + W, qrows + j * W);
        std::iota(pos.begin(), pos.end(), 0u);
        // k distinct positions: prefix of a Fisher-Yates shuffle
        for (uint64_t s = 0; s < k && s < dims; ++s) {
            const uint64_t r = s + scale(word_at(kp, j * dims + s), dims - s);
            std::swap(pos[s], pos[r]);
            qrows[j * W + pos[s] / 64] ^= uint64_t(1) << (pos[s] % 64);
        }
        if (src_out) src_out[j] = uint32_t(src);
    }
}

} // namespace fclsh_b200
