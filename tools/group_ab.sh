#!/bin/bash
# A/B of the head-major group size (DMA_GROUP_MB=0: one head pair per group, the round-2 order)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c4 c3 c5; do
  for g in 0 48 96; do
    DMA_GROUP_MB=$g timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/grp_${c}_$g.json 2>&1
    python -c "
import json
d=json.load(open('gpurun_out/grp_${c}_$g.json')); print('$c', 'group_mb=$g', round(d['ms_per_step'],4), round(d['value'],1), d['phases_ms']['two_phase_attention'], d['roofline'].get('traffic'))"
  done
done
