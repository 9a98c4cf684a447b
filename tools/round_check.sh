mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/full.json 2> gpurun_out/full.err
timeout 400 python bench.py --impl reference > gpurun_out/ref2.json 2> gpurun_out/ref2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-hash --configs 2 --replay 1 > gpurun_out/trun.json 2> gpurun_out/trun.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-hash --configs 2 --replay 1 > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_query_warp_pf -s 1 -c 1 -o gpurun_out/qwarp_cfg3_s4 python tools/prof_workload.py cfg3 > gpurun_out/ncu_cfg3b.log 2>&1
echo done
