mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 3000 bash tools/bench_all.sh > gpurun_out/bench_all.log 2>&1
for f in gpurun_out/bench_*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1])); print(sys.argv[1].split('/')[-1], round(d.get('ms_per_step',0),3), (d.get('roofline') or {}).get('frac'))
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
