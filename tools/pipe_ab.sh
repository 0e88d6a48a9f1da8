#!/bin/bash
# attention-kernel time at c3 for library variants x kernels (pipe experiments)
cd "$(dirname "$0")/.."
for lib in ${LIBS:-paper_2604_03950_b200/libdma.so}; do
  for kern in ${KERNELS:-pp ws}; do
    DMA_LIB_PATH=$lib DMA_ATTN_KERNEL=$kern timeout 120 python bench.py --config ${CFG:-c3} --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib $kern', 'attention %.3f ms'%d['phases_ms']['two_phase_attention'])"
  done
done
