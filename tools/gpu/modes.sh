mkdir -p gpurun_out
for m in 8 2 7; do
  echo "== defer mode $m"
  AB_OPTS="5=$m" timeout 900 python tools/ab.py $AB_CFGS paper_1306_4743_b200/libeik.so 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], round(d['ms'],3), 'proc', d['proc'], 'cell', round(d['ms_cell'],3))"
done
