// Reference-style C++ caller of the B200 engine through include/fclsh_gpu.hpp.
// Mirrors the reference CLI `build` seed chain (tools/fclsh.cpp:248-263):
// plan seed = Rng(seed).stream("run",0).stream("plan"), index seed = ...("index").
// Usage: cpp_drop_in [--host-only | --dump PATH]  (PATH: the index's and a
// 4-shard cluster's results, for tests/test_cpp_adapter.py to check)
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fclsh_gpu.hpp"

int main(int argc, char** argv) {
    namespace G = fclsh::gpu;
    const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
    const char* dump = argc > 2 && std::strcmp(argv[1], "--dump") == 0 ? argv[2] : nullptr;
    const uint64_t seed = 42, n = 20000, d = 128;
    const uint32_t r = 4;
    const uint64_t run = fclsh_rng_stream_index(seed, "run", 0);
    const uint64_t plan_seed = fclsh_rng_stream(run, "plan"), index_seed = fclsh_rng_stream(run, "index");
    try {
        auto fam = G::build_covering_family(d, r, fclsh_rng_stream_index(index_seed, "family", 0), G::kMersenne31);
        auto m = fam.mapping();
        auto s = fam.seeds();
        std::printf("family tables=%llu mapping0=%u seed0=%llu\n", (unsigned long long)fam.table_count(), m[0],
                    (unsigned long long)s[0]);
        fclsh_plan_override ov{FCLSH_PLAN_IDENTITY, 1};
        auto plan = G::make_plan(d, r, 1.0, n, plan_seed, &ov);
        std::printf("plan tables=%llu\n", (unsigned long long)plan.info().table_count);
        try {
            G::make_plan(d, 0, 1.0, n, plan_seed);
        } catch (const G::UsageError& e) {
            std::printf("usage error ok: %s\n", e.what());
        }
        if (host_only) return 0;
        std::vector<uint64_t> rows(n * (d / 64));
        fclsh_gen_bernoulli(seed, 0, n, d, rows.data(), 4);
        // 200 queries: data rows 0, 100, 200, ... with their bits 0..(k-1) flipped, k = i % 6
        const uint64_t nq = 200, W = d / 64;
        std::vector<uint64_t> q(nq * W);
        for (uint64_t i = 0; i < nq; ++i) {
            for (uint64_t w = 0; w < W; ++w) q[i * W + w] = rows[(i * 100) * W + w];
            for (uint64_t b = 0; b < i % 6; ++b) q[i * W + b / 64] ^= uint64_t(1) << (b % 64);
        }
        auto ix = G::build_index(rows.data(), n, d, r, plan, index_seed, G::kMersenne31);
        auto res = ix.query_r_nn(q.data(), nq, r);
        auto cix = G::build_classic_index(rows.data(), n, d, r, plan, index_seed, G::kMersenne31);
        auto clres = cix.query_r_nn(q.data(), nq, r);
        std::printf("classic tables=%llu found0=%llu\n", (unsigned long long)cix.table_count(),
                    (unsigned long long)clres.found[0]);
        G::Cluster cl({0}, 4);
        cl.build(rows.data(), n, d, r, plan, index_seed, G::kMersenne31);
        auto cres = cl.query_r_nn(q.data(), nq, r);
        std::printf("index tables=%llu found0=%llu first_id=%u total=%zu cluster_total=%zu\n",
                    (unsigned long long)ix.table_count(), (unsigned long long)res.found[0],
                    res.id.empty() ? 0u : res.id[0], res.id.size(), cres.id.size());
        if (dump) {
            FILE* f = std::fopen(dump, "w");
            if (!f) return 3;
            for (const G::RnnBatch* b : {&res, &cres}) {
                std::fprintf(f, "%zu\n", b->id.size());
                for (uint64_t i = 0; i < nq; ++i)
                    std::fprintf(f, "%llu %llu %llu %llu\n", (unsigned long long)b->offsets[i + 1],
                                 (unsigned long long)b->collisions[i], (unsigned long long)b->candidates[i],
                                 (unsigned long long)b->found[i]);
                for (size_t k = 0; k < b->id.size(); ++k) std::fprintf(f, "%u %u\n", b->id[k], b->distance[k]);
            }
            std::fclose(f);
        }
        return (res.found[0] >= 1 && res.id[0] == 0) ? 0 : 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
