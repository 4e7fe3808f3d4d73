mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=12 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
rm -f gpurun_out/ab.jsonl
timeout 600 python tools/ab.py C3,C4,C5,C3d,C2 build_ab/lib_head.so build_ab/lib_wt.so build_ab/lib_head.so build_ab/lib_wt.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
python - <<'PY'
import json
for l in open("gpurun_out/ab.jsonl"):
    d = json.loads(l)
    print(d["cfg"], d["lib"], round(d["ms"], 3), "proc", d["proc"], "ingest", round(d["ms_ingest"], 3), "cell", round(d["ms_cell"], 3), "egress", round(d["ms_egress"], 3))
PY
