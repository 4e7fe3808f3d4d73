"""kappa early-termination study on the GPU box: the paper's
Ex. 1-3 at M = 320^3 (fp64, r = 8) with kappa in {0, 1e-8}, for pHCM
(eik_solve) and the sweeping methods (eik_solve_sweep dlsm/dfsm): solve ms (mean of 3 after a
warm-up), updates per point, sweeps, and the max / mean deviation from the kappa = 0 result of
the same method.  Not a parity claim (no error bound)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1306_4743_b200 as eik

out = []
cfgs = sys.argv[1:] or ["P1", "P2", "P3"]
for name in cfgs:
    cfg, prec, r = bench.WORKLOADS[name]
    n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
    h = bench.grid_h(cfg, n)
    s = eik.Solver()
    for method in ("hcm", "dlsm", "dfsm"):
        ref = None
        for kap in (0.0, 1e-8):
            s.set_option(eik.EIK_OPT_KAPPA, kap)
            U = torch.empty_like(F)
            run = (lambda: s.solve(F, m, q, h=h, cell_size=r, n=n, out=U)) if method == "hcm" else \
                  (lambda: s.solve_sweep(F, m, q, h=h, cell_size=r, n=n, out=U, method=method))
            run()
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); run(); e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            st = s.stats()
            fin = torch.isfinite(U)
            if ref is None:
                ref = U.clone()
                dmax = dmean = 0.0
            else:
                d = (U[fin] - ref[fin]).abs()
                dmax, dmean = float(d.max()), float(d.mean())
            rec = {"cfg": name, "method": method, "kappa": kap, "ms": float(np.mean(ts)),
                   "updates_per_point": st["point_updates"] / st["M"],
                   "processings_per_cell": st["cell_processings"] / st["J"],
                   "grid_sweeps": st["grid_sweeps"], "max_dev_from_kappa0": dmax,
                   "mean_dev_from_kappa0": dmean, "min_diff_sign_ok": bool((U[fin] >= ref[fin] - 1e-12).all())}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    s.set_option(eik.EIK_OPT_KAPPA, 0.0)
    s.close()
    del F, m, q
    torch.cuda.empty_cache()
