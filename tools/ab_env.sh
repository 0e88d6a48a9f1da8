#!/bin/bash
# A/B the attention kernel by environment: ab_env.sh "ENV=a" "ENV=b" ...  (in-tree build)
cd "$(dirname "$0")/.."
for envs in "$@"; do
  for c in ${CFGS:-c3 c2}; do
    env $envs timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()[:300]); continue
    print('$envs $c', 'value %.1f TFLOPS'%d['value'], 'attn %.4f ms'%d['phases_ms']['attention'], 'clk', d['clocks'].get('sm_mhz'))
"
  done
done
