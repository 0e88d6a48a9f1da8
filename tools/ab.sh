#!/bin/bash
# A/B the attention kernel of several builds: ab.sh dir1 dir2 ... (each holding libdma.so); "." = in-tree build
cd "$(dirname "$0")/.."
for d in "$@"; do
  lib=$d/libdma.so; [ "$d" = "." ] && lib=paper_2604_03950_b200/libdma.so
  for c in ${CFGS:-c3 c2}; do
    DMA_LIB_PATH=$lib timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('$d $c', 'value %.1f TFLOPS'%d['value'], 'attn %.4f ms'%d['phases_ms']['attention'], 'quant %.4f'%d['phases_ms']['quantize'], 'clk', d['clocks'].get('sm_mhz'))
"
  done
done
