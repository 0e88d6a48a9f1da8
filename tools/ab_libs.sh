#!/bin/bash
# A/B device-time bench of several builds of libdma (DMA_LIB_PATH), interleaved: LIBS="a.so b.so" CONFIGS="c3 c2"
cd "$(dirname "$0")/.."
for r in 1 2; do
for c in ${CONFIGS:-c3}; do
  for L in ${LIBS}; do
    DMA_LIB_PATH=$L timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('$c $L', 'value %.1f'%d['value'], {k: round(v,4) for k,v in d['phases_ms'].items()}, 'clk', d['clocks'].get('sm_mhz'))
"
  done
done
done
