"""Critical-path analysis of one async solve from its processing trace (EIK_OPT_TRACE).
usage (GPU box): python tools/trace_cp.py C3 [C4 ...] [--opt k=v,...]
For every processing: its last tagger (the processing whose tag queued it), pop / swept / end
times.  The critical path follows last taggers back from the last processing to finish; per
link: wait = child's pop - tagger's sweep end (fence + tags + ring + deferrals + pop), work =
child's sweep end - pop (staging, sweeps, write-back), tail = end - sweep end (fence, tags,
release).  Also: concurrency (processings in flight) over time."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1306_4743_b200 as eik  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
opts = {}
for a in sys.argv[1:]:
    if a.startswith("--opt="):
        for kv in a[6:].split(","):
            k, v = kv.split("=")
            opts[int(k)] = float(v)
for name in args or ["C3"]:
    cfg, prec, r = bench.WORKLOADS[name]
    n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
    s = eik.Solver()
    for k, v in opts.items():
        s.set_option(k, v)
    s.set_option(eik.EIK_OPT_TRACE, 8_000_000)
    U = s.solve(F, m, q, cell_size=r, n=n, h=bench.grid_h(cfg, n))
    U = s.solve(F, m, q, cell_size=r, n=n, h=bench.grid_h(cfg, n))
    st = s.stats()
    tr = s.trace().astype(np.int64)
    s.close()
    cell, tag, tpop, tsw, tend, nsw, fl, wr = tr.T
    N = len(tr)
    NONE = 0xFFFFFFFF
    # critical path
    i = int(np.argmax(tend))
    path = []
    while i != NONE and i < N and len(path) < N:
        path.append(i)
        i = int(tag[i])
    path = path[::-1]
    p = np.array(path)
    par = tag[p[1:]]
    wait = tpop[p[1:]] - tsw[par]
    work = tsw[p] - tpop[p]
    tail = tend[p] - tsw[p]
    # first processing of each cell?
    first_seen = {}
    is_first = np.zeros(N, bool)
    for k in np.argsort(tpop, kind="stable"):
        c = int(cell[k])
        if c not in first_seen:
            first_seen[c] = k
            is_first[k] = True
    # concurrency over time
    T = int(tend.max())
    bins = np.linspace(0, T, 41)
    ev = np.zeros(len(bins) - 1)
    for a, b in zip(tpop, tend):
        ia, ib = np.searchsorted(bins, [a, b])
        ev[max(ia - 1, 0):ib] += 1
    occ = []
    for k in range(len(bins) - 1):
        lo, hi = bins[k], bins[k + 1]
        ov = np.clip(np.minimum(tend, hi) - np.maximum(tpop, lo), 0, None).sum() / (hi - lo)
        occ.append(round(float(ov), 1))
    out = {"cfg": name, "tag": os.environ.get("TRACE_TAG", ""), "opts": opts, "ms_total": st["ms_total"], "ms_cell": st["ms_cell_device"], "processings": N,
           "T_last_end_us": T / 1e3, "path_len": len(path),
           "path_first_frac": float(is_first[p].mean()),
           "path_wait_us": float(wait.sum()) / 1e3, "path_work_us": float(work.sum()) / 1e3,
           "path_tail_us": float(tail.sum()) / 1e3,
           "path_wait_mean_us": float(wait.mean()) / 1e3 if len(wait) else 0,
           "path_work_mean_us": float(work.mean()) / 1e3, "path_tail_mean_us": float(tail.mean()) / 1e3,
           "all_work_mean_us": float((tsw - tpop).mean()) / 1e3, "all_tail_mean_us": float((tend - tsw).mean()) / 1e3,
           "path_start_us": float(tpop[p[0]]) / 1e3,
           "path_sweeps_mean": float(nsw[p].mean()), "all_sweeps_mean": float(nsw.mean()),
           "in_flight_per_40th": occ,
           "writes_pct_10_50_90": [float(x) for x in np.percentile(wr, [10, 50, 90])],
           "procs_writes_lt64": float((wr < 64).mean()), "procs_writes_lt512": float((wr < 512).mean()),
           "ctatime_share_writes_lt64": float(((tend - tpop) * (wr < 64)).sum() / (tend - tpop).sum()),
           "ctatime_share_writes_lt512": float(((tend - tpop) * (wr < 512)).sum() / (tend - tpop).sum()),
           "reproc_writes_median": float(np.median(wr[~is_first])) if (~is_first).any() else 0.0}
    print(json.dumps(out), flush=True)
    np.save(f"gpurun_out/trace_{name}{os.environ.get('TRACE_TAG', '')}.npy", tr)
    del F, m, q, U
    torch.cuda.empty_cache()
