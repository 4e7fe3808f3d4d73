set -x
mkdir -p gpurun_out
rm -f gpurun_out/ws.jsonl
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 900 python tools/ab.py C3,C4,C5,C3d,C2 build_ab/lib_r6.so build_ab/lib_ws.so build_ab/lib_r6.so build_ab/lib_ws.so >> gpurun_out/ws.jsonl 2>> gpurun_out/ws.err
cat gpurun_out/ws.jsonl
timeout 300 python tools/diag.py C3:mode=0:defer=8:msw=0 C5:mode=0:defer=8:msw=0 > gpurun_out/diag.jsonl 2>&1; cat gpurun_out/diag.jsonl
