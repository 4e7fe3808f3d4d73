mkdir -p gpurun_out
timeout 600 python tools/trace_cp.py C3 C5 C3d C4 > gpurun_out/trace.jsonl 2> gpurun_out/trace.err
python - <<'PY'
import json
for l in open("gpurun_out/trace.jsonl"):
    d = json.loads(l); d.pop("in_flight_per_40th", None); print(json.dumps(d))
PY
tail -3 gpurun_out/trace.err
