#!/bin/bash
# programmatic dependent launch A/B: DMA_PDL=1 (default) vs 0 on c1 / c2 / c3 (+ --graph on c1)
cd "$(dirname "$0")/.."
for cfg in c1 c2 c3; do
  for pdl in 1 0; do
    for extra in "" "--graph"; do
      [ "$cfg" != c1 ] && [ -n "$extra" ] && continue
      DMA_PDL=$pdl timeout 200 python bench.py --config $cfg --no-cpu-baseline --steps 20 $extra 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); e=d.get('e2e') or {}
    print('$cfg pdl=$pdl $extra', 'ms %.4f'%d['ms_per_step'], 'TF %.1f'%d['value'], 'e2e_ms', e.get('ms_per_step'), d.get('phases_ms'))"
    done
  done
done
