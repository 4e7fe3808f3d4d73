mkdir -p gpurun_out; rm -f gpurun_out/diag_r02c.jsonl
for c in C3:mode=0:defer=8:msw=0 C3d:mode=0:defer=8:msw=0 C4:mode=0:defer=8:msw=0 C5:mode=0:defer=8:msw=0 C1:mode=0:defer=8:msw=0; do
  timeout 300 python tools/diag.py $c >> gpurun_out/diag_r02c.jsonl 2>> gpurun_out/diag.err
done
timeout 600 python tools/trace_cp.py C3 C4 > gpurun_out/trace_r02c.jsonl 2> gpurun_out/trace.err
cat gpurun_out/diag_r02c.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print({k:(round(v,1) if isinstance(v,float) else v) for k,v in d.items() if k in ('cfg','ms_total','ms_cell','proc','cyc_per_proc','steps_per_proc','sweeps_per_proc','stage','mask','stepcyc','wb','tile','cyc_per_step','defers','list_it')})"
cat gpurun_out/trace_r02c.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print({k:(round(v,1) if isinstance(v,float) else v) for k,v in d.items() if k!='in_flight_per_40th'}); print([round(x) for x in d['in_flight_per_40th']])"
