# ncu evidence for one config (GPU box): launch list of the bench command, DRAM bytes of the
# cell kernel (default scheduler: the persistent k_async, one launch per solve), one --set full
# capture of the measured solve's k_async launch (the second; the first is the warm-up).
# Every command runs once without ncu first (exit 0) before it is profiled.
# usage: bash tools/ncu_all.sh C3 [tag]  -> gpurun_out/ncu_<cfg>_*.{csv,ncu-rep,json}
set -x
C=${1:-C3}; T=${2:-$C}; SKIP=1
mkdir -p gpurun_out
python tools/profile_run.py $C > gpurun_out/ncu_${T}_stats.json || exit 1
python bench.py --config $C --steps 2 --warmup 1 --no-cpu --e2e-steps 0 > gpurun_out/ncu_${T}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ncu_${T}_launches.csv python bench.py --config $C --steps 2 --warmup 1 --no-cpu --e2e-steps 0 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_async --csv --log-file gpurun_out/ncu_${T}_kmet.csv python tools/profile_run.py $C > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_async --launch-skip $SKIP --launch-count 1 \
    -o gpurun_out/ncu_${T}_full -f python tools/profile_run.py $C > gpurun_out/ncu_${T}_full.log 2>&1
ls -la gpurun_out/
