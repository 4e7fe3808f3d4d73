mkdir -p gpurun_out
rm -f gpurun_out/ing.jsonl
timeout 600 python tools/ab.py C3,C5,C3d build_ab/lib_u2.so build_ab/lib_u4.so build_ab/lib_u2.so build_ab/lib_u4.so > gpurun_out/ing.jsonl 2> gpurun_out/ing.err
python - <<'PY'
import json
for l in open("gpurun_out/ing.jsonl"):
    d = json.loads(l)
    print(d["cfg"], d["lib"], round(d["ms"], 3), "ingest", round(d["ms_ingest"], 3), "loop", round(d["ms_loop"], 3), "egress", round(d["ms_egress"], 3), "cell", round(d["ms_cell"], 3))
PY
(free -g; nproc) > gpurun_out/golden_box.txt
timeout 2400 python tools/make_c5_golden.py --out gpurun_out/c5_oracle_samples > gpurun_out/golden.log 2>&1
tail -5 gpurun_out/golden.log
ls -la gpurun_out/c5_oracle_samples*
