#!/bin/bash
# Round-2 final evidence: full GPU suite (parity rows logged), smoke, bench lines for every config,
# the c4 ablation sweep, launch list + full ncu capture of the attention and quantize kernels,
# compute-sanitizer racecheck / synccheck / memcheck of the small cases.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/parity_*.jsonl
DMA_PARITY_LOG=1 timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
for c in c1 c2 c4; do timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/r02_bench_$c.json 2>&1; done
timeout 300 python bench.py --config c1 --steps 20 --no-cpu-baseline --graph > gpurun_out/r02_bench_c1_graph.json 2>&1
timeout 600 python bench.py --config c5 --steps 3 --no-cpu-baseline > gpurun_out/r02_bench_c5.json 2>&1
timeout 400 python bench.py --pv bf16 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_c3_bf16.json 2>&1
timeout 600 python tools/ablation_c4.py --steps 10 --heads 2 --tag r02 > gpurun_out/r02_c4_sweep.log 2>&1; tail -2 gpurun_out/r02_c4_sweep.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dma_attn_pp -s 3 -c 1 -o gpurun_out/r02_attn_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_attn.log 2>&1; tail -1 gpurun_out/r02_ncu_attn.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant32 -s 2 -c 1 -o gpurun_out/r02_quant32_final -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_quant.log 2>&1; tail -1 gpurun_out/r02_ncu_quant.log
timeout 300 python tools/ks_sweep.py > gpurun_out/r02_kvsplit_sweep.txt 2>&1; tail -4 gpurun_out/r02_kvsplit_sweep.txt
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r02_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/r02_sanitizer_$tool.log
done
for f in gpurun_out/r02_bench_*.json; do echo "$f: $(head -c 300 $f)"; done
