mkdir -p gpurun_out
rm -f gpurun_out/trace.jsonl
TRACE_TAG=_g timeout 600 python tools/trace_cp.py C3 C3d >> gpurun_out/trace.jsonl 2>> gpurun_out/trace.err
TRACE_TAG=_k timeout 600 python tools/trace_cp.py C3 C3d --opt=5=7 >> gpurun_out/trace.jsonl 2>> gpurun_out/trace.err
TRACE_TAG=_kp EIK_LIB=build_ab/lib_park.so timeout 600 python tools/trace_cp.py C3 C3d --opt=5=7 >> gpurun_out/trace.jsonl 2>> gpurun_out/trace.err
python - <<'PY'
import json
for l in open("gpurun_out/trace.jsonl"):
    d = json.loads(l); occ = d.pop("in_flight_per_40th", None)
    print(d["cfg"], d["tag"], "ms", round(d["ms_total"], 2), "proc", d["processings"], "path", d["path_len"], "first", round(d["path_first_frac"], 2),
          "wait", round(d["path_wait_mean_us"], 1), "work", round(d["path_work_mean_us"], 1), "tail", round(d["path_tail_mean_us"], 1),
          "allwork", round(d["all_work_mean_us"], 1), "sweeps", round(d["path_sweeps_mean"], 2))
    print("   occ", occ)
PY
tail -3 gpurun_out/trace.err
