set -x
mkdir -p gpurun_out
timeout 600 python tools/trace_cp.py C3 C4 C5 C3d > gpurun_out/trace.jsonl 2> gpurun_out/trace.err
cat gpurun_out/trace.jsonl
tail -5 gpurun_out/trace.err
