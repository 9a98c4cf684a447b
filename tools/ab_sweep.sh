#!/bin/bash
# A/B sweep of the warp kernel occupancy / U on cfg3 (headline) and cfg2
run() { name=$1; shift; env "$@" python bench.py --steps 10 --warmup 3 --no-cpu --no-hash --configs 2 --replay 1 > gpurun_out/sw_$name.log 2>&1; }
run base
run c1 FCLSH_WARP_CTAS=1
run c2 FCLSH_WARP_CTAS=2
run c3 FCLSH_WARP_CTAS=3
run u2 FCLSH_WARP_U=2
run u2c3 FCLSH_WARP_U=2 FCLSH_WARP_CTAS=3
run u2c4 FCLSH_WARP_U=2 FCLSH_WARP_CTAS=4
echo done
