#!/bin/bash
# Fast GPU iteration: attention parity tests, c3/c2 bench (device time only), optional phase profile.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -4
for c in c3 c2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('$c', 'value %.1f TFLOPS'%d['value'], 'phases', {k: round(v,4) for k,v in d['phases_ms'].items()}, 'frac %.3f'%d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'))
"
done
if [ -f build_prof/libdma_prof.so ]; then
  DMA_LIB_PATH=build_prof/libdma_prof.so timeout 120 python tools/prof_phases.py c3
fi
