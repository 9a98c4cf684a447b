# final evidence of a session: GPU suite, smoke, both bench arms, then (after those exited) the ncu launch list and one full capture of the headline kernel
mkdir -p gpurun_out
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6d_gpu_suite.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s6d_gpu_suite.log)
(timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s6d_smoke.log 2>&1)
(timeout 400 python bench.py --impl reference > gpurun_out/s6d_bench_ref.json 2> gpurun_out/s6d_bench_ref.err)
(timeout 600 python bench.py > gpurun_out/s6d_bench.json 2> gpurun_out/s6d_bench.err)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s6d.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-hash --configs 2 --replay 1 > gpurun_out/s6d_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_query_warp_pf -s 1 -c 1 -o gpurun_out/qwarp_cfg3_s6d python tools/prof_workload.py cfg3 > gpurun_out/s6d_ncu_cfg3.log 2>&1
tail -3 gpurun_out/s6d_gpu_suite.log; tail -1 gpurun_out/s6d_smoke.log
