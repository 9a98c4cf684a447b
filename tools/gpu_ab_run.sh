# GPU A/B helper (edited per experiment): parity tests on the default build, then tools/ab_lib.sh over the listed builds
timeout 900 python -m pytest tests/test_index_gpu.py tests/test_classic.py tests/test_cluster_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/ab_tests.log
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q -k "cfg3 or cfg1 or cfg2" 2>&1 | tail -2 >> gpurun_out/ab_tests.log
CONFIGS=1,2 REPLAY=100 bash tools/ab_lib.sh libfclsh_b200.so libfclsh_b200_base.so > gpurun_out/ab_run.txt 2>&1
CONFIGS=1,2 REPLAY=1 bash tools/ab_lib.sh libfclsh_b200.so libfclsh_b200_base.so >> gpurun_out/ab_run.txt 2>&1
cat gpurun_out/ab_tests.log gpurun_out/ab_run.txt
