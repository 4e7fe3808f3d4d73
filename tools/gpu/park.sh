set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout 300 python tools/stress_async.py 3 > gpurun_out/stress.log 2>&1; tail -2 gpurun_out/stress.log
timeout 600 python tools/ab.py C3,C4,C5,C3d build_ab/lib_nopark.so build_ab/lib_park.so build_ab/lib_nopark.so build_ab/lib_park.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
cat gpurun_out/ab.jsonl
timeout 600 python tools/trace_cp.py C3 C4 C5 C3d > gpurun_out/trace.jsonl 2> gpurun_out/trace.err
cat gpurun_out/trace.jsonl | cut -c1-600
