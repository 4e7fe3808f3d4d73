"""Cell-value heuristic study: Eq. (3) (default) vs the legacy
Eq. (4) on the paper's permeable shell maze (fp64, r = 8) with narrow priority bins (1e-6: nearly
the serial heap order the paper measured: HCM8 20.4 vs 8366 sweeps per
cell at M = 64^3), and on Ex.3.  The bin width orders work only in the round scheduler
(loop mode 2: each round takes the queued cells with keys in [kmin, kmin + Delta]); the async
default ignores it, so every run here is loop mode 2.  Prints one JSON line per run (GPU box)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1306_4743_b200 as eik
import workloads as W

for name, w, deltas in (("PMAZE64", W.paper_shell_maze(64), (1e-6, 0.05, float("inf"))),
                        ("PMAZE128", W.paper_shell_maze(128), (0.05, float("inf"))),
                        ("P3_128", W.paper_example(3, 128), (1e-6, 0.05, float("inf")))):
    F, m, q = (torch.from_numpy(a.reshape(-1)).cuda() for a in w.as_dtype("float64"))
    for delta in deltas:
        for key in (0, 1):
            s = eik.Solver(bin_width=delta, loop_mode=2)
            s.set_option(eik.EIK_OPT_MAX_SWEEPS, 0)   # no sweep cap: a processing converges its cell (HCM)
            s.set_option(eik.EIK_OPT_CELL_KEY, key)
            s.set_option(eik.EIK_OPT_MAX_ROUNDS, 3_000_000)
            s.set_option(eik.EIK_OPT_TIMEOUT_S, 100)
            rec = {"workload": name, "bin_width": delta, "loop_mode": 2, "cell_key": "Eq.4" if key else "Eq.3"}
            try:
                s.solve(F, m, q, h=w.h, cell_size=8, n=w.n)
                st = s.stats()
                rec.update(ms=st["ms_total"], rounds=st["rounds"],
                           processings_per_cell=st["cell_processings"] / st["J"],
                           sweeps_per_cell=st["cell_sweeps"] / st["J"],
                           updates_per_point=st["point_updates"] / st["M"])
            except eik.EikError as e:
                rec["error"] = str(e)[:120]
            print(json.dumps(rec), flush=True)
            s.close()
