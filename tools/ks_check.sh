#!/bin/bash
# KV-split check on the box: split-sensitive GPU tests, smoke, c1 / c2 / c3 bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fused.py tests/test_gpu_fuzz.py tests/test_gpu_api.py -m gpu -q -x 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c1 c2 c3; do timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/ks_$c.json 2>&1; done
timeout 300 python bench.py --config c1 --steps 20 --no-cpu-baseline --no-e2e --graph > gpurun_out/ks_c1g.json 2>&1
DMA_KV_SPLIT=0 timeout 300 python bench.py --config c1 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/ks_c1_off.json 2>&1
for f in gpurun_out/ks_*.json; do python -c "
import json,sys
try:
  d=json.load(open('$f')); print('$f', d['ms_per_step'], d['value'], d.get('phases_ms'))
except Exception as e: print('$f', open('$f').read()[-600:])
"; done
