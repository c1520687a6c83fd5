for v in 12 16 17 9; do python tools/scale_check.py --no-oracle --repeats 5 --variant $v --layout chunk_sorted rmat22 grid4096 2>&1 | grep "{"; done > gpurun_out/cg.jsonl
cat gpurun_out/cg.jsonl | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], r['layout'], 'v', r['variant'], round(r['device_s']*1e3,3), r['sweeps'], r['sweep_ms'][:6], r['verify'])
"
