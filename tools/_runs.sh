for fs in 0 1; do python tools/scale_check.py --no-oracle --repeats 2 --host-loop 1 --first-scatter $fs forest rmat28 grid4096 rmat22 2>&1 | grep "{"; done > gpurun_out/fs.jsonl
cat gpurun_out/fs.jsonl | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], r['layout'], 'fs', r['first_scatter'], round(r['device_s']*1e3,3), r['sweeps'], r['sweep_ms'][:8], r['verify'])
"
