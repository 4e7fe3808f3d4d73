set -x
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc; lscpu | head -20) > gpurun_out/box.txt 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/b_C3.json 2> gpurun_out/b_C3.err
for c in C3:mode=0:defer=6:msw=0 C3d:mode=0:defer=6:msw=0 C4:mode=0:defer=6:msw=0 C5:mode=0:defer=6:msw=0 PMAZE:mode=0:defer=6:msw=0; do
  timeout 300 python tools/diag.py $c >> gpurun_out/diag.jsonl 2>> gpurun_out/diag.err
done
timeout 900 bash tools/ncu_all.sh C4 r02a_C4 > gpurun_out/ncu_C4.log 2>&1
timeout 900 bash tools/ncu_all.sh C5 r02a_C5 > gpurun_out/ncu_C5.log 2>&1
