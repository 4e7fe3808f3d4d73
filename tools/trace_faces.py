"""Per-processing statistics from the async trace (EIK_OPT_TRACE): processings, sweeps and work
time by the number of inflow faces and by first visit / re-processing.
usage (GPU box): python tools/trace_faces.py C3 [C4 ...]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1306_4743_b200 as eik  # noqa: E402

for name in sys.argv[1:] or ["C3"]:
    cfg, prec, r = bench.WORKLOADS[name]
    n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
    s = eik.Solver()
    s.set_option(eik.EIK_OPT_TRACE, 8_000_000)
    for _ in range(2):
        s.solve(F, m, q, cell_size=r, n=n, h=bench.grid_h(cfg, n))
    tr = s.trace().astype(np.int64)
    s.close()
    cell, tag, tpop, tsw, tend, nsw, fl, wr = tr.T
    order = np.argsort(tpop, kind="stable")
    seen = set()
    first = np.zeros(len(tr), bool)
    for k in order:
        c = int(cell[k])
        if c not in seen:
            seen.add(c)
            first[k] = True
    nf = np.array([bin(int(x) & 63).count("1") for x in fl])
    init = (fl & 64) != 0
    work = (tsw - tpop) / 1e3
    out = {"cfg": name, "processings": int(len(tr)), "by": []}
    for label, sel in (("first", first), ("again", ~first)):
        for k in range(0, 7):
            mk = sel & (nf == k)
            if mk.sum() == 0:
                continue
            out["by"].append({"visit": label, "inflow_faces": k, "n": int(mk.sum()), "init": int((mk & init).sum()),
                              "sweeps_mean": float(nsw[mk].mean()), "work_us_mean": float(work[mk].mean()),
                              "writes_mean": float(wr[mk].mean()),
                              "sweeps_hist": np.bincount(np.minimum(nsw[mk], 8), minlength=9).tolist()})
    print(json.dumps(out), flush=True)
    del F, m, q
    torch.cuda.empty_cache()
