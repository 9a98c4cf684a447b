# A/B of library builds on the quick bench: bash tools/ab_lib.sh libA.so libB.so ...
B="python bench.py --no-cpu --no-hash --configs ${CONFIGS:-1,2} --replay ${REPLAY:-1}"
L=$PWD/paper_1602_02620_b200/lib
for rep in 1 2; do for lib in "$@"; do echo "== $lib"; FCLSH_LIB=$L/$lib timeout 300 $B 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); o=' '.join(f'{k} {v[\"value\"]/1e6:.2f}/{v[\"e2e\"][\"value\"]/1e6:.2f}' for k,v in d['configs'].items())
        r=(d.get('replay') or {}).get('queries_per_s',0)/1e6
        print(f'cfg3 {d[\"value\"]/1e6:.2f}/{d[\"e2e\"][\"value\"]/1e6:.2f} fused {d[\"stages_ms_shard0\"][\"fused\"]*1e3:.1f}us', o, f'replay {r:.1f}')
    else: print(l.strip()[:200])
"; done; done
