import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_1306_4743_b200 as eik
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg, prec, r = bench.WORKLOADS[name]
n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
s = eik.Solver(loop_mode=2)
s.solve(F, m, q, cell_size=r, n=n); s.solve(F, m, q, cell_size=r, n=n)
a = np.zeros(2092 + 2048 + 12, dtype=np.uint64)
eik.lib.eik_get_debug(s._ctx, a.ctypes.data, len(a))
st = s.stats()
tr = a[42:42 + 2048].reshape(-1, 2)[:st["rounds"]]
t2 = a[44 + 2048:44 + 4096].reshape(-1, 2)[:st["rounds"]]
ghz = 1.92
slots = 148 * (4 if r == 16 and prec == "f32" else 2 if r == 16 else 8)
util = [float(x[0]) * 1024 / max(float(t[1]) * ghz * slots, 1) for x, t in zip(t2, tr)]
ls = a[44 + 4096:44 + 4096 + 12].reshape(2, 6).astype(float)
print(json.dumps({"lstat": [{"count": x[0], "cyc": x[1] / max(x[0], 1), "sweeps": x[2] / max(x[0], 1), "list_it": x[3] / max(x[0], 1),
                             "steps": x[4] / max(x[0], 1), "cont": x[5] / max(x[0], 1)} for x in ls]}))
print(json.dumps({"cfg": name, "rounds": st["rounds"], "ms_total": st["ms_total"], "sum_span_ms": float(tr[:, 1].sum()) / 1e6,
                  "util_mean": float(np.sum(t2[:, 0].astype(float)) * 1024 / (float(tr[:, 1].sum()) * ghz * slots)),
                  "trace": [[int(c), round(int(t) / 1e3, 1), round(u, 2), round(int(x[1]) / ghz / 1e3, 1)] for (c, t), u, x in zip(tr, util, t2)]}))
