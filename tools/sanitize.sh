#!/bin/bash
# compute-sanitizer over a representative slice of the -m gpu suite (SURVEY
# §5): memcheck (out-of-bounds / misaligned / leaked device memory),
# racecheck (shared-memory hazards: k_query_dense's id set and found list,
# k_query_c, k_scan_compact's tile scan, the CSR sorts), synccheck (barrier
# misuse) and initcheck (uninitialised device reads). Logs to gpurun_out/.
# Usage (GPU box): bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLICE=(
  "tests/test_index_gpu.py::test_small_indexes_match_oracle"
  "tests/test_index_gpu.py::test_clustered_data_long_cells"
  "tests/test_index_gpu.py::test_three_query_paths"
  "tests/test_index_gpu.py::test_many_tables_cta_per_query"
  "tests/test_index_gpu.py::test_edge_queries"
  "tests/test_index_gpu.py::test_query_c_r_nn_matches_the_reference"
  "tests/test_cluster_gpu.py::test_cluster_equals_single_index"
  "tests/test_scan_gpu.py"
  "tests/test_hash_gpu.py::test_fast_path_random_families"
  "tests/test_hash_gpu.py::test_generic_path_random_families"
  "tests/test_classic.py::test_hash_tables_equals_reference"
)
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 3000 compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
    python -m pytest -x -q -p no:cacheprovider "${SLICE[@]}" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3 >> gpurun_out/sanitize_summary.txt
done
