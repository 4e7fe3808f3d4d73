import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_1306_4743_b200 as eik
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg, prec, r = bench.WORKLOADS[name]
n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
s = eik.Solver(loop_mode=2)
s.solve(F, m, q, cell_size=r, n=n); s.solve(F, m, q, cell_size=r, n=n)
a = np.zeros(2092, dtype=np.uint64)
eik.lib.eik_get_debug(s._ctx, a.ctypes.data, len(a))
st = s.stats()
tr = a[42:].reshape(-1, 2)[:st["rounds"]]
print(json.dumps({"cfg": name, "rounds": st["rounds"], "ms_total": st["ms_total"], "sum_span_ms": float(tr[:, 1].sum()) / 1e6,
                  "trace": [[int(c), round(int(t) / 1e3, 1)] for c, t in tr]}))
