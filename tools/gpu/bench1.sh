mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_C3.json').read().strip().splitlines()[-1])
print('C3', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'cpu', d['cpu_baseline'], 'e2e', round(d['e2e']['ms_per_step'],2))
f=d['c3_fp64']; print('C3d', round(f['ms_per_step'],3), 'frac', round(f['roofline']['frac'],4))
print('work', d['work'])"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
timeout 900 python tools/cellkey_study.py > gpurun_out/cellkey.jsonl 2> gpurun_out/cellkey.err; echo "cellkey rc=$?"; cat gpurun_out/cellkey.jsonl
