#!/bin/bash
# ncu --set full of one attention launch (DMA_ATTN_KERNEL selects the kernel) at ${CFG:-c3} -> gpurun_out/attn_${TAG:-sk}.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dma_attn -s 3 -c 1 \
  -o gpurun_out/attn_${TAG:-sk} -f python bench.py --config ${CFG:-c3} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_${TAG:-sk}.log 2>&1
tail -2 gpurun_out/ncu_${TAG:-sk}.log
