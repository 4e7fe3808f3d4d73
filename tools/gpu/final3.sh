mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; grep "Elapsed" gpurun_out/bench_default.err; python -c "
import json;d=json.load(open('gpurun_out/bench_default.json'));print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['c3_fp64']['ms_per_step'], d['gpu_launches'], d['clocks'])"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_reference.json'));print(d['config'])"
