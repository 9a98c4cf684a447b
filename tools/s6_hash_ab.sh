# A/B of the cfg5 hash kernel: the default library vs lib/libfclsh_b200_base.so (FCLSH_LIB), parity first
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_hash_gpu.py tests/test_configs_gpu.py -x -q -k "hash or cfg5 or key" 2>&1 | tail -2 > gpurun_out/s6_hash_tests.log
L=$PWD/paper_1602_02620_b200/lib
for rep in 1 2 3; do for lib in libfclsh_b200.so libfclsh_b200_base.so; do
  echo "== $lib"; FCLSH_LIB=$L/$lib timeout 300 python bench.py --no-cpu --no-configs --replay 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); h=d['hash']; print(f'{h[\"ms_per_step\"]:.3f} ms  {h[\"value\"]/1e9:.1f} Gkeys/s  frac {h[\"roofline\"][\"frac\"]:.4f}  cfg3 {d[\"value\"]/1e6:.2f}')
"; done; done > gpurun_out/s6_hash_ab.txt 2>&1
cat gpurun_out/s6_hash_tests.log gpurun_out/s6_hash_ab.txt
