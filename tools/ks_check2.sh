#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fused.py tests/test_gpu_fuzz.py tests/test_gpu_api.py -m gpu -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c1 c3; do timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/ks_$c.json 2>&1; done
DMA_KV_SPLIT=0 timeout 300 python bench.py --config c1 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/ks_c1_off.json 2>&1
for f in gpurun_out/ks_c1.json gpurun_out/ks_c1_off.json gpurun_out/ks_c3.json; do python -c "
import json
d=json.load(open('$f')); print('$f', d['ms_per_step'], d['value'], d.get('phases_ms'))"; done
for m in -1 0; do DMA_KV_SPLIT=$m ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_ks$m.csv python bench.py --config c1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; done
python - <<'PY'
import csv,collections
for f in ['gpurun_out/c1_ks-1.csv','gpurun_out/c1_ks0.csv']:
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
    d=collections.defaultdict(list)
    for r in rows[1:]: d[r[ki][:50]].append(float(r[vi].replace(',','')))
    print(f, {k:(len(v), round(sorted(v)[len(v)//2]/1000,2)) for k,v in d.items()})
PY
