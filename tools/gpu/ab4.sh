mkdir -p gpurun_out
run() { AB_OPTS="$1" timeout 1200 python tools/ab.py $AB_CFGS $2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$3', d['cfg'], round(d['ms'],3), 'proc', d['proc'], 'cell', round(d['ms_cell'],3))"; }
run "" build_ab/lib_cur.so cur
run "" build_ab/lib_g2.so g2-mode8to2
run "" build_ab/lib_g2n9.so g2-mode8to9
run "5=9" build_ab/lib_g2.so g2-mode9
