#!/bin/bash
# A/B of the split-KV kernel (default) against the round-1 ping-pong kernel: parity tests + device-time bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15
for c in ${CONFIGS:-c3 c2}; do
  for k in sk pp; do
    DMA_ATTN_KERNEL=$k timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('$c $k', 'value %.1f TFLOPS'%d['value'], 'phases', {k: round(v,4) for k,v in d['phases_ms'].items()}, 'frac %.3f'%d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'))
"
  done
done
