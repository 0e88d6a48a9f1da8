for lib in ${FLIBS:-paper_2604_03950_b200/libdma.so}; do for c in c3 c2; do DMA_LIB_PATH=$lib timeout 300 python bench.py --config $c --fused --no-cpu-baseline --no-e2e --steps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(\"$lib $c fused\", round(d[\"value\"],1), round(d[\"phases_ms\"][\"forward\"],4))"; done; done
