mkdir -p gpurun_out
B="python bench.py --no-cpu --no-hash --configs 2 --replay 1"
L=$PWD/paper_1602_02620_b200/lib
for i in 1 2; do for lib in libfclsh_b200.so libfclsh_b200_pubsc.so; do echo "== $lib"; FCLSH_LIB=$L/$lib timeout 300 $B 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['configs']['cfg2']; print('cfg3', round(d['value']/1e6,2), round(d['e2e']['value']/1e6,2), round(d['stages_ms_shard0']['fused']*1e3,1), round(d['stages_ms_shard0']['compact']*1e3,1), 'cfg2', round(c['value']/1e6,2), round(c['e2e']['value']/1e6,2))
    else: print(l.strip()[:200])
"; done; done
