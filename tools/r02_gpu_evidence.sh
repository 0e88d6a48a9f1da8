#!/bin/bash
# Round-2 evidence run: quant16 full ncu capture, launch list of the c3 bench, compute-sanitizer
# racecheck / synccheck / memcheck of the attention, quantize and decode kernels at small shapes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant16 -s 2 -c 1 -o gpurun_out/r02_quant -f \
  python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_quant.log 2>&1
tail -1 gpurun_out/r02_ncu_quant.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv \
  python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r02_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r02_sanitizer_$tool.log
done
