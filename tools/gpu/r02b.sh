set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 1200 bash tools/ncu_all.sh C3 r02b_C3 > gpurun_out/ncu_C3.log 2>&1
timeout 1200 bash tools/ncu_all.sh C5 r02b_C5 > gpurun_out/ncu_C5.log 2>&1
timeout 1200 bash tools/ncu_all.sh C3d r02b_C3d > gpurun_out/ncu_C3d.log 2>&1
for c in C3:mode=0:defer=8:msw=0 C3d:mode=0:defer=8:msw=0 C4:mode=0:defer=8:msw=0 C5:mode=0:defer=8:msw=0; do
  timeout 300 python tools/diag.py $c >> gpurun_out/diag_r02b.jsonl 2>> gpurun_out/diag.err
done
ls -la gpurun_out | tail -30
