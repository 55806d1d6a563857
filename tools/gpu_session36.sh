timeout 1500 python tools/calibration_pass.py > gpurun_out/calpass36.jsonl 2> gpurun_out/calpass36.err; tail -3 gpurun_out/calpass36.err; python -c "
import json
for l in open('gpurun_out/calpass36.jsonl'):
    d=json.loads(l); d.pop('per_layer',None); print(json.dumps(d)[:1500])
"
