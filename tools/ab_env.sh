# A/B of env knobs on the quick bench: bash tools/ab_env.sh "X=1" "FCLSH_FUSED_PF=1" ...
B="python bench.py --no-cpu --no-hash --configs ${CONFIGS:-1,2} --replay ${REPLAY:-1}"
for rep in 1 2; do for e in "$@"; do echo "== $e"; env $e timeout 300 $B 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); o=' '.join(f'{k} {v[\"value\"]/1e6:.2f}/{v[\"e2e\"][\"value\"]/1e6:.2f}' for k,v in d['configs'].items())
        r=(d.get('replay') or {}).get('queries_per_s',0)/1e6
        print(f'cfg3 {d[\"value\"]/1e6:.2f}/{d[\"e2e\"][\"value\"]/1e6:.2f} fused {d[\"stages_ms_shard0\"][\"fused\"]*1e3:.1f}us', o, f'replay {r:.1f}')
    else: print(l.strip()[:200])
"; done; done
