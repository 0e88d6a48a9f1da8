#!/bin/bash
# split-KV kernel: trace of CTA 0 (c3) + device-time bench (c3, c2), optional parity tests (TESTS=1)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -5; fi
if [ -f build_trace/libdma.so ]; then DMA_LIB_PATH=build_trace/libdma.so timeout 300 python tools/trace_sk.py c3 2>&1 | head -${TRACE_LINES:-45}; fi
for c in ${CONFIGS:-c3 c2}; do
  for k in ${KERNELS:-sk}; do
    DMA_ATTN_KERNEL=$k timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('$c $k', 'value %.1f TFLOPS'%d['value'], 'phases', {k: round(v,4) for k,v in d['phases_ms'].items()}, 'frac %.3f'%d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'))
"
  done
done
