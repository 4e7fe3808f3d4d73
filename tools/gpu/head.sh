set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_head.json 2> gpurun_out/bench_head.err; tail -c 600 gpurun_out/bench_head.json
timeout 600 python tools/ab.py C3,C5,C4,C3d paper_1306_4743_b200/libeik.so > gpurun_out/ab_head.jsonl 2> gpurun_out/ab_head.err; cat gpurun_out/ab_head.jsonl
