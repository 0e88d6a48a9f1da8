#!/bin/bash
# One GPU session: smoke, bench (c3 + c2), launch list, full ncu capture of the attention kernel.
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
cat gpurun_out/bench_c3.json
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; cat gpurun_out/bench_c2.json
timeout 300 python bench.py --config c3 --pv bf16 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_bf16.json 2>&1; cat gpurun_out/bench_c3_bf16.json
if [ -z "${NO_NCU}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dma_attn -s 3 -c 1 -o gpurun_out/attn_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant16 -s 6 -c 1 -o gpurun_out/quant_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_quant.log 2>&1; tail -3 gpurun_out/ncu_quant.log
fi
