cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3
for a in "" "--batch 1 --heads 32 --kv-heads 32" "--batch 32 --ctx 8192" "--batch 8 --nq 4"; do
timeout 300 python tools/bench_decode.py $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['batch'],d['heads'],d['kv_heads'],d['ctx'],d['n_q'],round(d['value'],4),'ms',round(d['achieved_GBps']),'GB/s')"
done
