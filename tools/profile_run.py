"""Profiling driver: one warm-up solve + one measured solve of a config with the library's
default scheduler (async: one persistent k_async launch per solve), or with the host-driven
round loop (argv[2] = "rounds": every cell-sweep launch a plain kernel launch); prints the
stats JSON."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1306_4743_b200 as eik
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg, prec, r = bench.WORKLOADS[name]
n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
s = eik.Solver(loop_mode=1) if len(sys.argv) > 2 and sys.argv[2] == "rounds" else eik.Solver()
s.solve(F, m, q, cell_size=r, n=n)
s.solve(F, m, q, cell_size=r, n=n)
st = s.stats()
print(json.dumps({"config": name, "stats": st}))
