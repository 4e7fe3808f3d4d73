mkdir -p gpurun_out
timeout 1200 python tools/ab.py $AB_CFGS $AB_LIBS > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
python - <<'PY'
import json
for l in open("gpurun_out/ab.jsonl"):
    d = json.loads(l)
    print(d["cfg"], d["lib"], round(d["ms"], 3), "proc", d["proc"], "ingest", round(d["ms_ingest"], 3), "cell", round(d["ms_cell"], 3), "egress", round(d["ms_egress"], 3), "csum", d["csum"])
PY
tail -3 gpurun_out/ab.err
