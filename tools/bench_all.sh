# Every bench line of BASELINE.md section 4 (GPU box): pHCM on C1-C5 and the paper's suite,
# the sweeping comparison methods on C3 and the paper's examples, and the reference arm.
# (The C3 line times the full CPU oracle once, ~150 s; the other lines skip the CPU leg.)
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config C3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
for c in C1 C2 C2d C3d C4 C5 P1 P2 P3 PCB11 PMAZE; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for c in C3 C1 C4 P1 P2 P3 PCB11; do
  for m in dlsm dfsm; do
    timeout 900 python bench.py --config $c --method $m --no-cpu --steps 3 > gpurun_out/bench_${c}_$m.json 2> gpurun_out/bench_${c}_$m.err
  done
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
tail -c 400 gpurun_out/bench_C3.json
