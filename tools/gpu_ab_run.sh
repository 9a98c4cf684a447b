timeout 900 python -m pytest tests/test_index_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/idx_tests.log
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q -k "cfg4" 2>&1 | tail -3 >> gpurun_out/idx_tests.log
CONFIGS=4 bash tools/ab_lib.sh libfclsh_b200.so libfclsh_b200_old.so > gpurun_out/ab_seg.txt 2>&1
cat gpurun_out/idx_tests.log gpurun_out/ab_seg.txt
