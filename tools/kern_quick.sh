#!/bin/bash
# Fast A/B of the phase-2 kernels: parity subset + c3/c2 device-time bench per kernel.
# usage: KERNELS="pp ws" PYTEST_K="vs_oracle" tools/kern_quick.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for kern in ${KERNELS:-ws}; do
  echo "=== kernel $kern"
  DMA_ATTN_KERNEL=$kern timeout 300 python -m pytest tests/test_gpu_attention.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -4
  for c in ${CONFIGS:-c3 c2}; do
    DMA_ATTN_KERNEL=$kern timeout 200 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()[:300]); continue
    print('$kern $c', 'value %.1f TFLOPS'%d['value'], 'phases', {k: round(v,4) for k,v in d['phases_ms'].items()}, 'frac %.3f'%d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'))
"
  done
done
