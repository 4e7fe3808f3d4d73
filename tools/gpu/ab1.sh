set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout 600 python tools/ab.py C3,C4,C5,C3d build_ab/lib_old.so build_ab/lib_new.so build_ab/lib_old.so build_ab/lib_new.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
cat gpurun_out/ab.jsonl
