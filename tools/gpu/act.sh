mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
timeout 900 python tools/ab.py C5,C3,C3d,C4 build_ab/lib_u2.so build_ab/lib_actcpp.so build_ab/lib_actptx.so build_ab/lib_actnoclob.so build_ab/lib_ing2.so build_ab/lib_l2k.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
python - <<'PY'
import json
for l in open("gpurun_out/ab.jsonl"):
    d = json.loads(l)
    print(d["cfg"], d["lib"], round(d["ms"], 3), "proc", d["proc"], "ingest", round(d["ms_ingest"], 3), "cell", round(d["ms_cell"], 3), "egress", round(d["ms_egress"], 3))
PY
