#!/bin/bash
# Device-side bounds checks over the GPU suite (compute-sanitizer is closed on
# this pool): the library rebuilt with -DFCLSH_DEBUG_BOUNDS (FCLSH_DCHECK in
# the bucket insert, the query kernels' slot / hand-over / home-bucket
# accesses, the fused hash's row-word reads, the CTA kernel's result region,
# the budgeted query's id set, the classic hash, the cluster merge), then
# every -m gpu test but the multi-minute full-size ones against it
# (FCLSH_LIB). A failed check traps, so the batch fails with a CUDA error.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DBG=paper_1602_02620_b200/lib/libfclsh_b200_dbg.so
make -C paper_1602_02620_b200 -j8 EXTRA=-DFCLSH_DEBUG_BOUNDS BUILD=build_dbg OUT=lib/libfclsh_b200_dbg.so
FCLSH_LIB=$PWD/$DBG timeout 3000 python -m pytest tests -q -m gpu -k "not every_key and not full_size" \
  > gpurun_out/bounds_check.log 2>&1
echo "bounds-checked GPU suite rc=$?" | tee gpurun_out/bounds_check_summary.txt
grep -E "passed|failed|FCLSH_DCHECK" gpurun_out/bounds_check.log | tail -5 | tee -a gpurun_out/bounds_check_summary.txt
