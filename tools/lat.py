"""Uncontended cell-processing latency: a one-cell grid (n = r - 1), corner exit."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1306_4743_b200 as eik
for r in (16, 8):
    for dt in (torch.float32, torch.float64):
        n = r - 1
        M = (n + 1) ** 3
        F = torch.ones(M, dtype=dt, device="cuda")
        m = torch.zeros(M, dtype=torch.uint8, device="cuda"); m[0] = 1
        q = torch.zeros(M, dtype=dt, device="cuda")
        s = eik.Solver(loop_mode=1)
        for _ in range(3):
            s.solve(F, m, q, cell_size=r, n=n)
        st, d = s.stats(), s.debug()
        p = max(d["processings"], 1)
        print(json.dumps({"r": r, "dt": str(dt), "proc": p, "sweeps": st["cell_sweeps"], "steps": d["plane_steps"],
                          "cyc": d["cycles_sum"] / p, "stage": d["cyc_stage"] / p, "mask": d["cyc_mask"] / p,
                          "steps_cyc": d["cyc_steps"] / p, "per_step": d["cyc_steps"] / max(d["plane_steps"], 1),
                          "upd": st["point_updates"], "ms": st["ms_total"]}))
        s.close()
