"""Small solves in every mode/precision/cell size, for compute-sanitizer (one tool per run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, workloads as W
import paper_1306_4743_b200 as eik
w = W.random_instance(20, 7, p_wall=0.15, n_exits=3, q_max=0.2)
U_orc = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals)
bad = 0
for mode in (2, 1, 0):
    s = eik.Solver(loop_mode=mode)
    for r in (4, 8, 16):
        for dt in (np.float64, np.float32):
            F, m, q = w.as_dtype(dt)
            U = s.solve(torch.from_numpy(F).cuda(), torch.from_numpy(m).cuda(), torch.from_numpy(q).cuda(),
                        cell_size=r, n=w.n).cpu().numpy().astype(np.float64)
            fin = np.isfinite(U_orc)
            ok = np.array_equal(np.isfinite(U), fin) and np.abs(U[fin] - U_orc[fin]).max() < (1e-10 if dt == np.float64 else 1e-5)
            bad += not ok
    s.close()
print("sanitize_run done, mismatches:", bad)
