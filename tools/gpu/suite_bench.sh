mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; tail -c 300 gpurun_out/bench_C3.json
for c in C1 C2 C2d C4 C5; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c',round(d['ms_per_step'],3),'frac',round(d['roofline']['frac'],4),'e2e',round(d['e2e']['ms_per_step'],2))"; done
