set -x
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
for o in "11=0" "11=1" "11=0" "11=1"; do AB_OPTS=$o timeout 600 python tools/ab.py C3,C4,C5,C3d build_ab/lib_b2.so >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err; done
cat gpurun_out/ab.jsonl
timeout 300 python tools/diag.py C3:mode=0:defer=6:msw=0 C5:mode=0:defer=6:msw=0 C3d:mode=0:defer=6:msw=0 > gpurun_out/diag.jsonl 2>&1; cat gpurun_out/diag.jsonl
