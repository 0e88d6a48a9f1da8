#!/bin/bash
# Quick HEAD check on the box: GPU suite, smoke, bench lines c3 / c1 / c2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/chk_c3.json 2> gpurun_out/chk_c3.err
for c in c1 c2 c4; do timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/chk_$c.json 2>&1; done
for f in gpurun_out/chk_*.json; do echo "$f: $(head -c 400 $f)"; done
