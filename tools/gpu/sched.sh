set -x
mkdir -p gpurun_out
rm -f gpurun_out/sched.jsonl
for o in "5=6" "5=7" "5=2" "5=3,0=0.01" "5=3,0=0.03" "5=3,0=0.1" "5=3,0=0.3" "5=6"; do
  echo "{\"opts\": \"$o\"}" >> gpurun_out/sched.jsonl
  AB_OPTS=$o timeout 600 python tools/ab.py C3,C4,C5,C3d,PMAZE build_ab/lib_cur.so >> gpurun_out/sched.jsonl 2>> gpurun_out/sched.err
done
cat gpurun_out/sched.jsonl
