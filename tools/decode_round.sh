#!/bin/bash
# GPU session for the decode kernel: parity tests, six bench shapes -> gpurun_out/r01_decode.jsonl, one ncu --set full capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/r01_decode.jsonl
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3
for a in "" "--batch 1 --heads 32 --kv-heads 32" "--batch 32 --ctx 8192" "--batch 8 --nq 2" "--batch 8 --nq 4" "--batch 64 --heads 64 --kv-heads 8 --ctx 4096"; do
timeout 300 python tools/bench_decode.py $a 2>&1 | tail -1 | tee -a gpurun_out/r01_decode.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['batch'],d['heads'],d['kv_heads'],d['ctx'],d['n_q'],round(d['value'],4),'ms',round(d['achieved_GBps']),'GB/s')"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dma_decode_kernel -s 5 -c 1 -o gpurun_out/decode_r01c -f python tools/bench_decode.py --steps 2 > gpurun_out/ncu_decode.log 2>&1
tail -1 gpurun_out/ncu_decode.log
