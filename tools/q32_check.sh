#!/bin/bash
# phase-1 (bf16 quantizer) parity + timing A/B: LIBS="a.so b.so" tools/q32_check.sh
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_quant.py -q -x 2>&1 | tail -2
[ -n "$FULL" ] && timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fused.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
for lib in ${LIBS:-paper_2604_03950_b200/libdma.so}; do
  for cfg in c3 c2; do
  DMA_LIB_PATH=$lib timeout 120 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib $cfg', round(d['value'],1), 'quant %.4f attn %.4f'%(d['phases_ms']['two_phase_quantize'],d['phases_ms']['two_phase_attention']), 'qfrac %.3f'%d['quant_phase']['frac'])"
  done
done
[ -n "$NCU" ] && ncu --kernel-name regex:quant32 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/$NCU python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > /dev/null 2>&1
true
