// TEST INFRASTRUCTURE ONLY. Prints the reference's write_metrics
// (bench.cpp:160-170) for metric rows read from a file, so the engine's CSV
// writer can be compared byte for byte. A separate executable: iostreams of
// the statically linked libstdc++ cannot share a process with Python's.
//
//   ref_write_metrics <rows.bin> <method>
//   rows.bin: u64 count, then count x 12 little-endian doubles
//             {query_id, radius, collisions, candidates, found, true_near,
//              precision, recall, time_s1_us, time_s2_us, time_s3_us, unused}
#include "fclsh/bench.hpp"

#include <cstdint>
#include <cstdio>
#include <iostream>
#include <vector>

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: %s rows.bin method\n", argv[0]);
        return 2;
    }
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    uint64_t n = 0;
    if (std::fread(&n, 8, 1, f) != 1) return 2;
    std::vector<double> v(n * 12);
    if (std::fread(v.data(), 8, v.size(), f) != v.size()) return 2;
    std::fclose(f);
    std::vector<fclsh::MetricsRow> rows(n);
    for (uint64_t i = 0; i < n; ++i) {
        const double* d = v.data() + 12 * i;
        fclsh::MetricsRow& r = rows[i];
        r.query_id = static_cast<uint32_t>(d[0]);
        r.method = argv[2];
        r.radius = static_cast<uint32_t>(d[1]);
        r.collisions = d[2];
        r.candidates = d[3];
        r.found = d[4];
        r.true_near = d[5];
        r.precision = d[6];
        r.recall = d[7];
        r.time_s1_us = d[8];
        r.time_s2_us = d[9];
        r.time_s3_us = d[10];
    }
    fclsh::write_metrics(rows, std::cout);
    return 0;
}
