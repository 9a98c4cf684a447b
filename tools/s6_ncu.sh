mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-hash --configs 2 --replay 1 > gpurun_out/s6_trun.json 2> gpurun_out/s6_trun.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s6.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-hash --configs 2 --replay 1 > gpurun_out/s6_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_query_warp_pf -s 1 -c 1 -o gpurun_out/qwarp_cfg3_s6 python tools/prof_workload.py cfg3 > gpurun_out/s6_ncu_cfg3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_hash_f64_pt -s 1 -c 1 -o gpurun_out/hash_cfg5_s6 python tools/prof_workload.py hash > gpurun_out/s6_ncu_hash.log 2>&1
echo done
