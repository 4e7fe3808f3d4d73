set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout 900 python tools/ab.py C3,C5,C4,C3d,C2,P2 $AB_LIBS > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
python - <<'PY'
import json
for l in open("gpurun_out/ab.jsonl"):
    d = json.loads(l)
    print(d["cfg"], d["lib"], round(d["ms"], 3), "proc", d["proc"], "ingest", round(d["ms_ingest"], 3), "cell", round(d["ms_cell"], 3), "egress", round(d["ms_egress"], 3), "csum", d["csum"])
PY
