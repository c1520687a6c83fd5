for sm in 1 3; do python tools/scale_check.py --no-oracle --repeats 3 --store-mode $sm grid4096 rmat22 forest 2>&1 | grep "{"; done > gpurun_out/smode.jsonl
cat gpurun_out/smode.jsonl | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], r['layout'], 'sm', r['store_mode'], round(r['device_s']*1e3,3), r['sweeps'], r['sweep_ms'][:6], r['verify'])
"
