"""Async readiness-order study (EIK_OPT_ASYNC_DEFER): solve ms (mean of 3
after a warm-up) and processings per cell for each mode on the bench configs.  GPU box."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1306_4743_b200 as eik

for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3", "C5", "C4", "C2", "P2", "P3", "PCB11", "PMAZE"]):
    cfg, prec, r = bench.WORKLOADS[name]
    n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
    h = bench.grid_h(cfg, n)
    for mode, defer in ((2, None), (0, 1), (0, 2), (0, 5), (0, 6), (0, 7)):
        s = eik.Solver(loop_mode=mode)
        if defer is not None:
            s.set_option(eik.EIK_OPT_ASYNC_DEFER, defer)
        U = torch.empty_like(F)
        s.solve(F, m, q, h=h, cell_size=r, n=n, out=U)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); s.solve(F, m, q, h=h, cell_size=r, n=n, out=U); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        st = s.stats()
        print(json.dumps({"cfg": name, "scheduler": "rounds (fused, bin +inf)" if mode == 2 else f"async defer {defer}",
                          "ms": sum(ts) / 3, "processings_per_cell": st["cell_processings"] / st["J"],
                          "updates_per_point": st["point_updates"] / st["M"]}), flush=True)
        s.close()
    del F, m, q
    torch.cuda.empty_cache()
