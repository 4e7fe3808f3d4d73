"""Diagnostics: run one config and print eik stats + per-processing counters (GPU box)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1306_4743_b200 as eik  # noqa: E402

cfgs = sys.argv[1:] or ["C3"]
for name in cfgs:
    bw, mode, defer, msw = None, 2, 1, 4
    if ":" in name:
        parts = name.split(":")
        name = parts[0]
        for kv in parts[1:]:
            k, v = kv.split("=")
            if k == "bw": bw = float(v)
            if k == "bwr": bw = -float(v)   # multiple of r*h, resolved below
            if k == "mode": mode = int(v)
            if k == "defer": defer = int(v)
            if k == "msw": msw = int(v)
    cfg, prec, r = bench.WORKLOADS[name]
    n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
    if bw is not None and bw < 0:
        bw = -bw * r * bench.grid_h(cfg, n)
    s = eik.Solver(bin_width=bw, loop_mode=mode)
    if bw is not None and mode == 0:
        s.set_option(eik.EIK_OPT_BIN_WIDTH, bw)
    s.set_option(eik.EIK_OPT_ASYNC_DEFER, defer)
    s.set_option(eik.EIK_OPT_MAX_SWEEPS, msw)
    U = s.solve(F, m, q, cell_size=r, n=n)
    U = s.solve(F, m, q, cell_size=r, n=n)
    st, dbg = s.stats(), s.debug()
    p = max(dbg["processings"], 1)
    out = {"cfg": name, "bw": bw, "mode": mode, "defer": defer, "msw": msw, "defers": dbg["defers"], "ms_total": st["ms_total"], "ms_loop": st["ms_loop"],
           "ms_cell": st["ms_cell_device"], "rounds": st["rounds"], "proc": st["cell_processings"],
           "cyc_per_proc": dbg["cycles_sum"] / p, "cyc_max": dbg["cycles_max"],
           "steps_per_proc": dbg["plane_steps"] / p, "sweeps_per_proc": st["cell_sweeps"] / p,
           "upd_per_proc": st["point_updates"] / p, "hist": dbg["sweep_hist"][:16],
           "stage": dbg["cyc_stage"] / p, "mask": dbg["cyc_mask"] / p, "stepcyc": dbg["cyc_steps"] / p,
           "wb": dbg["cyc_writeback"] / p, "tile": dbg["cyc_tile"] / p, "halo": dbg["cyc_halo"] / p, "list_it": dbg["list_iters"] / p, "cyc_per_step": dbg["cyc_steps"] / max(dbg["plane_steps"], 1)}
    print(json.dumps(out))
    s.close()
