for sc in 0 1 2; do python tools/scale_check.py --no-oracle --repeats 2 --shortcut $sc forest 2>&1 | grep "{"; done > gpurun_out/fsc.jsonl
python tools/scale_check.py --no-oracle --repeats 1 --host-loop 1 forest 2>&1 | grep "{" >> gpurun_out/fsc.jsonl
cat gpurun_out/fsc.jsonl | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], r['layout'], 'sc', r['shortcut'], 'hl', r['host_loop'], round(r['device_s']*1e3,3), r['sweeps'], r['sweep_ms'][:8], r['verify'])
"
