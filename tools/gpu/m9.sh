mkdir -p gpurun_out
rm -f gpurun_out/m9.jsonl
for o in "5=8" "5=9,0=0.003" "5=9,0=0.01" "5=9,0=0.03" "5=9,0=0.1"; do
  echo "{\"opts\": \"$o\"}" >> gpurun_out/m9.jsonl
  AB_OPTS=$o timeout 600 python tools/ab.py C3,C3d,C5,C4,PMAZE,P2,C2d build_ab/lib_m9.so >> gpurun_out/m9.jsonl 2>> gpurun_out/m9.err
done
python - <<'PY'
import json
for l in open("gpurun_out/m9.jsonl"):
    d = json.loads(l)
    print(d.get("opts") or f'{d["cfg"]:6s} {d["ms"]:8.2f} ms  proc {d["proc"]}')
PY
