set -x
mkdir -p gpurun_out
rm -f gpurun_out/auto.jsonl
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout 300 python tools/stress_async.py 3 > gpurun_out/stress.log 2>&1; tail -1 gpurun_out/stress.log
timeout 900 python tools/ab.py C3,C4,C5,C3d,PMAZE,C1,C2,C2d,P1,P2,P3,PCB11 build_ab/lib_r4.so build_ab/lib_r3.so build_ab/lib_r6.so >> gpurun_out/auto.jsonl 2>> gpurun_out/auto.err
for o in "5=6" "5=2"; do echo "{\"opts\": \"$o\"}" >> gpurun_out/auto.jsonl; AB_OPTS=$o timeout 600 python tools/ab.py C1,C2,C2d,P1,P2,P3,PCB11 build_ab/lib_r4.so >> gpurun_out/auto.jsonl 2>> gpurun_out/auto.err; done
cat gpurun_out/auto.jsonl
