"""Profiling driver: one warm-up solve + one host-loop (mode 1) solve of a config, so that
every cell-sweep launch is a plain kernel launch ncu can see; prints the stats JSON."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1306_4743_b200 as eik
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg, prec, r = bench.WORKLOADS[name]
n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
s = eik.Solver(loop_mode=1)
s.solve(F, m, q, cell_size=r, n=n)
s.solve(F, m, q, cell_size=r, n=n)
st = s.stats()
print(json.dumps({"config": name, "stats": st}))
