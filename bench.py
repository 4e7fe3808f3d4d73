#!/usr/bin/env python
"""Benchmark of the B200 cell-sweep Eikonal solver (pHCM hot path, arXiv 1306.4743).

Metric (BASELINE.json): "Eikonal solve ms & gridpoints/s at 513^3; HBM GB/s as fraction of peak".
Workload (default): C3 = n=512 (513^3 points), 8^3 checkerboard F in {1, 10}, corner exit,
fp32, cell size 16 -- configs[2], the 513^3 configuration the metric is quoted on.
A "step" is one full eik_solve (ingest -> device scheduler loop -> egress) over the resident
inputs; value = gridpoints/s = M / (step time), summed over ranks (independent replicas).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C4|...] [--impl reference]

N > 1: one process per GPU (launched by torchrun; `--gpus N` without torchrun re-executes
itself under torch.distributed.run); the path does not shard ("replicas only"):
each rank solves its own copy, no data-path collective; barrier + max over ranks.
--impl reference: the CPU fp64 FMM oracle (the only "reference" this tier has) on the host
cores, each step a bounded sample of the same workload: the oracle on a corner sub-box of the
very same input (same F, h and exits inside it), rank 0 only.
cpu_baseline (our arm, rank 0, N = 1): the oracle once on the full fp64 input of the workload
(~75 s for C3), or on a 257^3 sub-box for inputs above 1.5e8 points.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Eikonal solve ms & gridpoints/s at 513^3; HBM GB/s as fraction of peak"
UNIT = "gridpoints/s"
WORKLOADS = {
    # name: (config, precision, cell size)
    "C1": ("C1", "f64", 8), "C2": ("C2", "f32", 16), "C2d": ("C2", "f64", 8),
    "C3": ("C3", "f32", 16), "C3d": ("C3", "f64", 16), "C4": ("C4", "f32", 16),
    "C5": ("C5", "f32", 16),
    # the paper's own suite, M = 320^3 / 352^3 as in P:837-906, fp64, r = 8
    "P1": ("P1", "f64", 8), "P2": ("P2", "f64", 8), "P3": ("P3", "f64", 8),
    "PCB11": ("PCB11", "f64", 8), "PMAZE": ("PMAZE", "f64", 8),
}
DESC = {
    "C1": "n=128 (129^3), F=1, centre exit",
    "C2": "n=256 (257^3), F=1+0.5 sin(8pi x)sin(8pi y)sin(8pi z), centre exit",
    "C3": "n=512 (513^3), 8^3 checkerboard F in {1,10}, exit (0,0,0)",
    "C4": "n=512 (513^3), 8 F=0 walls with 4 random holes each, exit face z=0",
    "C5": "n=1024 (1025^3), 32 Gaussian bumps, 64 random exits",
    "P1": "paper Ex.1, M=320^3, F=1, 8-point centre exit (P:760)",
    "P2": "paper Ex.2, M=320^3, F=1+.5 sin(20pi x)sin(20pi y)sin(20pi z) (P:762)",
    "P3": "paper Ex.3, M=320^3, F=1+.99 sin(2pi x)sin(2pi y)sin(2pi z) (P:764)",
    "PCB11": "paper checkerboard K=11, M=352^3, F in {1,2} (P:1596)",
    "PMAZE": "paper shell maze, M=320^3 on [-1,1]^3, F=.001 barriers (P:1627)",
}
PAPER_N = {"P1": 320, "P2": 320, "P3": 320, "PCB11": 352, "PMAZE": 320}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        # wait for the first sample (nvidia-smi starts in ~0.1-1 s) so that the sampler is live
        # when the timed region starts; a region of a few ms still gets the sample at its start
        self.pre = ""
        if self.p is not None:
            import select
            r, _, _ = select.select([self.p.stdout], [], [], 5.0)
            if r:
                self.pre = self.p.stdout.readline()
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.15)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = []
        for line in (self.pre + (self.out or "")).strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) == 6 and f[0].replace(".", "").isdigit():
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def make_inputs(cfg, prec, device, n=None):
    """Seeded synthetic inputs of the config (workloads/), resident on `device`."""
    import torch
    import workloads as W
    dt = torch.float32 if prec == "f32" else torch.float64
    if cfg == "C5":
        n = n or 1024
        a, c, sig, ex = W.c5_params(n)
        F = W.c5_field_torch(n, a, c, sig, device=device, dtype=torch.float64).to(dt).reshape(-1)
        m = torch.zeros((n + 1) ** 3, dtype=torch.uint8, device=device)
        idx = torch.tensor([i + (n + 1) * (j + (n + 1) * k) for (i, j, k) in ex], device=device)
        m[idx] = 1
        q = torch.zeros((n + 1) ** 3, dtype=dt, device=device)
        return n, F.contiguous(), m, q
    w = paper_workload(cfg, n) if cfg in PAPER_N else W.make(cfg, n)
    Fh, mh, qh = w.as_dtype(np.float32 if prec == "f32" else np.float64)
    return (w.n, torch.from_numpy(Fh.reshape(-1)).to(device), torch.from_numpy(mh.reshape(-1)).to(device),
            torch.from_numpy(qh.reshape(-1)).to(device))


def paper_workload(cfg, N=None):
    import workloads as W
    N = N or PAPER_N[cfg]
    if cfg in ("P1", "P2", "P3"):
        return W.paper_example(int(cfg[1]), N)
    if cfg == "PCB11":
        return W.paper_checkerboard(11, N)
    return W.paper_shell_maze(N)


def grid_h(cfg, n):
    """grid spacing of a config (the shell maze lives on [-1, 1]^3)"""
    return 2.0 / n if cfg == "PMAZE" else 1.0 / n


def job_time(t_local: float, pg=None, device=None) -> float:
    """Whole-job time of one step: the MAX over ranks of each rank's device time (replicas
    only: no data-path collective, the reduction is timing plumbing)."""
    if pg is None:
        return float(t_local)
    import torch
    tt = torch.tensor([float(t_local)], dtype=torch.float64, device=device)
    pg.all_reduce(tt, op=pg.ReduceOp.MAX)
    return float(tt.item())


def job_value(points_per_rank: int, world: int, t_seconds: float) -> float:
    """gridpoints/s of the whole job: every rank solves its own copy (weak scaling)."""
    return points_per_rank * world / t_seconds


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), ws


def full_workload(cfg):
    """the workload at its BASELINE / paper size (fp64 F, as the oracle always takes it)"""
    import workloads as W
    return paper_workload(cfg) if cfg in PAPER_N else W.make(cfg)


def sub_box(w, ns):
    """Corner-anchored sub-box [i0, i0 + ns]^3 of workload w around its first exit: the same
    F, h and the exits that fall inside (a bounded sample of the SAME input; the sub-box
    faces act as the domain boundary)."""
    import workloads as W
    n = w.n
    ns = min(ns, n)
    k, j, i = [int(v[0]) for v in np.nonzero(w.exit_mask)]
    lo = [min(max(c - ns // 2, 0), n - ns) for c in (k, j, i)]
    sl = tuple(slice(a, a + ns + 1) for a in lo)
    meta = dict(w.meta, h=w.h, box_lo_kji=lo)
    return W.Workload(w.name, ns, np.ascontiguousarray(w.F[sl]), np.ascontiguousarray(w.exit_mask[sl]),
                      np.ascontiguousarray(w.exit_vals[sl]), meta), lo


def time_oracle(w):
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals, h=w.h)
    return time.perf_counter() - t0


def run_reference(args):
    rank, _, ws = dist_env()
    if rank != 0:
        return 0
    cfg, prec, r = WORKLOADS[args.config]
    wf = full_workload(cfg)
    w, lo = sub_box(wf, args.ref_n)
    del wf
    times = []
    for s in range(args.warmup + args.steps):
        dt = time_oracle(w)
        if s >= args.warmup:
            times.append(dt)
    t = float(np.mean(times))
    val = w.M / t
    sample = (f"serial fp64 FMM oracle (1 host core of {os.cpu_count()}) per step on the "
              f"{w.n + 1}^3 sub-box at (k, j, i) = {tuple(lo)} of the {cfg} input ({w.M} of its "
              f"{(WN[cfg] + 1) ** 3} points; same F, h = {w.h:g} and the exits inside)")
    cb = config_block(cfg, prec, r)
    # the workload is the arm's (same name and size: the driver matches the two lines on it); what
    # actually ran per step is stated next to it, and keys that only describe the GPU path go
    cb.update({"precision": "f64", "solve": "oracle FMM (serial, fp64) on a bounded sample of this input",
               "sample_n": w.n, "sample_points": w.M, "sample": sample})
    cb.pop("l2", None)
    cb.pop("cell_size", None)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cb,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


WN = {"C1": 128, "C2": 256, "C3": 512, "C4": 512, "C5": 1024, **{k: v - 1 for k, v in PAPER_N.items()}}


def cpu_baseline(cfg):
    """the oracle as it stands, once, on the full fp64 input (or a 257^3 sub-box above 1.5e8
    points: C5's full run takes ~15 min)"""
    w = full_workload(cfg)
    full = w.M <= 150_000_000
    if not full:
        w, lo = sub_box(w, 256)
    secs = time_oracle(w)
    what = (f"the full {cfg} input ({w.M} points)" if full else
            f"the {w.n + 1}^3 sub-box at (k, j, i) = {tuple(lo)} of the {cfg} input ({w.M} points)")
    return {"value": w.M / secs, "unit": UNIT, "cores": 1, "kind": "oracle", "seconds": round(secs, 2),
            "sample": f"serial fp64 FMM oracle once on {what}, {secs:.1f} s, 1 of {os.cpu_count()} host cores"}


def config_block(cfg, prec, r, n=None):
    n = n or {"C1": 128, "C2": 256, "C3": 512, "C4": 512, "C5": 1024}.get(cfg) or PAPER_N[cfg] - 1
    return {"workload": f"{cfg}: {DESC[cfg]}", "n": n, "points": (n + 1) ** 3, "cell_size": r,
            "precision": prec, "solve": "eik_solve: ingest + device scheduler loop + egress",
            "l2": "inputs (F + exit_mask + exit_vals) and tiles are > 4x the 126 MB L2; no flush"
            if n >= 256 else "L2-resident (small config)"}


def sweep_method(args):
    return getattr(args, "method", "hcm") != "hcm"


def free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def self_launch(n, argv):
    """`--gpus N` (N > 1) outside torchrun: re-execute this script under torch.distributed.run,
    one process per GPU (replicas only); rank 0's JSON line passes through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def measure(eik, solver, cfg, prec, r, dev, args, sweep=False, async_mode=True, barrier=None,
            pg=None, steps=None, warmup=None):
    """Device-timed steps of one workload: W untimed warm-up solves, then K solves between CUDA
    events on the launching stream (barrier + synchronize on both sides), max over ranks.
    Returns the timing, roofline and work blocks."""
    import torch
    steps = steps or args.steps
    warmup = args.warmup if warmup is None else warmup
    n, F, m, q = make_inputs(cfg, prec, dev, args.n)
    M = (n + 1) ** 3
    U = torch.empty_like(F)
    stream = torch.cuda.current_stream(dev)

    def run_once():
        if sweep:
            solver.solve_sweep(F, m, q, h=grid_h(cfg, n), cell_size=r, n=n, out=U, method=args.method)
        else:
            solver.solve(F, m, q, h=grid_h(cfg, n), cell_size=r, n=n, out=U)

    for _ in range(warmup):
        run_once()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    barrier()
    with Clocks(dev.index) as clk:
        ev0.record(stream)
        for _ in range(steps):
            run_once()
            stats.append(solver.stats())
        ev1.record(stream)
        barrier()
    t_ms = job_time(ev0.elapsed_time(ev1) / steps, pg, dev)

    # roofline of the dominant kernel (cell sweep): algorithmic bytes / its device time
    cell_ms = float(np.mean([s["ms_cell_device"] for s in stats]))            # %globaltimer span
    ev_ms = float(np.mean([s["ms_cell_events"] for s in stats]))              # CUDA events (async)
    if async_mode and ev_ms > 0:
        cell_ms = ev_ms
    alg_bytes = float(np.mean([s["bytes_cell_alg"] for s in stats]))
    launches = float(np.mean([s["cell_launches"] for s in stats]))
    peak, peak_src = peaks()
    achieved = alg_bytes / (cell_ms * 1e-3) / 1e9 if cell_ms > 0 else None
    st2 = {"ms_cell_events": 0.0, "cell_launches": 1}
    if async_mode:
        st2 = {"ms_cell_events": ev_ms, "cell_launches": 1}
    elif not sweep:
        # CUDA events around every round's cell-kernel launch in the host-driven loop
        s2 = eik.Solver(device=dev.index, loop_mode=1, bin_width=args.bin_width)
        s2.set_option(eik.EIK_OPT_TIME_CELL_EVENTS, 1)
        s2.solve(F, m, q, h=grid_h(cfg, n), cell_size=r, n=n, out=torch.empty_like(F))
        st2 = s2.stats()
        s2.close()
    tag = f"{args.config if (cfg, prec, r) == WORKLOADS[args.config] else cfg + ('d' if prec == 'f64' else '')}"
    traffic, tsrc = None, None
    for rr in ("r02", "r01"):
        tp = os.path.join(ROOT, "profiles", f"{rr}_ncu_{tag}.json")
        if os.path.exists(tp) and not sweep:
            # ncu DRAM bytes of the cell kernel per processing x processings per launch
            d = json.load(open(tp))["kcell_traffic"]
            traffic = d["dram_bytes_per_processing"] * (stats[-1]["cell_processings"] / max(launches, 1))
            tsrc = f"profiles/{rr}_ncu_{tag}.json (ncu --set full, per processing x this run's processings)"
            break
    st = stats[-1]
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic, "traffic_source": tsrc,
            "kernel": f"{'k_dsweep' if sweep else 'k_async' if async_mode else 'k_cell'}<{'float' if prec == 'f32' else 'double'},{r}>",
            "alg_bytes_per_launch": alg_bytes / max(launches, 1),
            "ms_per_launch_device": float(np.mean([s["ms_cell_device"] for s in stats])) / max(launches, 1),
            "ms_per_launch_events": (st2["ms_cell_events"] / max(st2["cell_launches"], 1)),
            "cell_share_of_step": cell_ms / t_ms, "peak_source": peak_src,
            "alg_bytes_def": "per processing (2 r^3 + 6 r^2) s read + changed points * s written",
            "kernel_timer": ("CUDA events around the persistent k_async launch on its stream, every timed solve"
                             if async_mode and ev_ms > 0 else "%globaltimer span of the cell-kernel launches")}
    work = {"rounds": st["rounds"], "grid_sweeps": st["grid_sweeps"], "cell_processings": st["cell_processings"],
            "processings_per_cell": st["cell_processings"] / st["J"],
            "sweeps_per_cell": st["cell_sweeps"] / st["J"],
            "updates_per_point": st["point_updates"] / st["M"],
            "writes_per_point": st["point_writes"] / st["M"],
            "max_worklist": st["max_worklist"], "J": st["J"],
            "grid_pass_equivalents": st["real_points_processed"] / st["M"],
            "bytes_min_GBps": st["bytes_min"] / (t_ms * 1e-3) / 1e9,
            "ms_ingest": st["ms_ingest"], "ms_loop": st["ms_loop"], "ms_egress": st["ms_egress"],
            "ms_total_lib": st["ms_total"]}
    rounds = float(np.mean([s["rounds"] for s in stats]))
    launches_per_step = (5 if async_mode else
                         4 + (launches + rounds if sweep else rounds * (1 if args.bin_width is None else 3)))
    return dict(n=n, M=M, F=F, m=m, q=q, t_ms=t_ms, roof=roof, work=work, clk=clk.summary(),
                launches_per_step=launches_per_step)


def plumbing_test(args):
    """CPU-only check of the multi-rank plumbing (tests/test_dist_cpu.py): gloo, a fixed fake
    step time per rank, the max over ranks and the whole-job value; never a bench number."""
    import torch.distributed as dist
    rank, _, ws = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    t = 0.010 * (rank + 1)
    tj = job_time(t, dist if ws > 1 else None, "cpu")
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": job_value(1000, ws, tj), "unit": UNIT,
                          "n_gpus": ws, "ms_per_step": tj * 1e3, "data": "plumbing-test"}), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="override n (reduced size; not a bench line)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-n", type=int, default=128,
                    help="--impl reference: side (intervals) of the sub-box of the input timed per step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 sub-line of the C3 bench")
    ap.add_argument("--bin-width", type=float, default=None,
                    help="priority bin width (round modes; implies --loop-mode 2)")
    ap.add_argument("--loop-mode", type=int, default=None,
                    help="scheduler (EIK_OPT_LOOP_MODE): 0 async [library default], 1 host rounds, 2 graph rounds")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--method", default="hcm", choices=["hcm", "dfsm", "dlsm"],
                    help="hcm: the product path (eik_solve); dfsm / dlsm: the paper's comparison "
                         "sweeping methods on the GPU (eik_solve_sweep, SURVEY 8(f) F2)")
    ap.add_argument("--plumbing-test", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus, sys.argv[1:])
    if args.plumbing_test:
        return plumbing_test(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1306_4743_b200 as eik

    rank, local, ws = dist_env()
    if ws > 1 and args.gpus not in (1, ws):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {ws}")
    if local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: local rank {local} but {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()

    cfg, prec, r = WORKLOADS[args.config]
    loop_mode = args.loop_mode if args.loop_mode is not None else (2 if args.bin_width is not None else None)
    solver = eik.Solver(device=local, bin_width=args.bin_width, loop_mode=loop_mode)
    sweep = args.method != "hcm"
    async_mode = loop_mode in (None, 0) and not sweep
    if async_mode:
        # CUDA events around the persistent cell-kernel launch, recorded by the library on the
        # launching stream inside every timed solve (the roofline's denominator)
        solver.set_option(eik.EIK_OPT_TIME_CELL_EVENTS, 1)
    res = measure(eik, solver, cfg, prec, r, dev, args, sweep=sweep, async_mode=async_mode,
                  barrier=barrier, pg=pg)
    n, M, F, m, q, t_ms = res["n"], res["M"], res["F"], res["m"], res["q"], res["t_ms"]
    value = job_value(M, ws, t_ms * 1e-3)

    # e2e: the same solve through the C ABI with pinned HOST buffers, copies inside the timing
    e2e = None
    if args.e2e_steps > 0 and not sweep:
        Fh = F.cpu().pin_memory()
        mh = m.cpu().pin_memory()
        qh = q.cpu().pin_memory()
        Uh = torch.empty_like(Fh).pin_memory()
        solver.solve_host(Fh, mh, qh, h=grid_h(cfg, n), cell_size=r, n=n, out=Uh)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            solver.solve_host(Fh, mh, qh, h=grid_h(cfg, n), cell_size=r, n=n, out=Uh)
        t_e = job_time((time.perf_counter() - t0) / args.e2e_steps, pg, dev)
        st_h = solver.stats()   # bytes the C call moved (F and mask copied; exit_vals read in
        # place at the exits: page-locked host memory, mapped)
        e2e = {"value": job_value(M, ws, t_e), "unit": UNIT, "ms_per_step": t_e * 1e3,
               "h2d_bytes_per_step": int(st_h["h2d_bytes"]),
               "d2h_bytes_per_step": int(st_h["d2h_bytes"]),
               "timer": "host wall clock around the blocking C-ABI call (pinned buffers)",
               "transfers": "F and exit_mask copied H2D; exit_vals read in place at the exit points "
                            "(mapped pinned memory); U copied D2H"}
        del Fh, mh, qh, Uh
    del F, m, q
    res.pop("F"), res.pop("m"), res.pop("q")

    # the paper's default precision on the headline config, device-timed the same way
    fp64 = None
    if args.config == "C3" and not args.no_fp64 and not sweep and args.n is None:
        r64 = measure(eik, solver, "C3", "f64", 16, dev, args, sweep=False, async_mode=async_mode,
                      barrier=barrier, pg=pg)
        fp64 = {"workload": "C3d: " + DESC["C3"] + ", fp64, cell size 16", "dtype": "f64",
                "ms_per_step": r64["t_ms"], "value": job_value(r64["M"], ws, r64["t_ms"] * 1e-3),
                "unit": UNIT, "roofline": r64["roof"], "work": r64["work"], "clocks": r64["clk"],
                "gpu_launches": int(args.steps * r64["launches_per_step"])}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu and args.n is None:
        cpu = cpu_baseline(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "config": dict(config_block(cfg, prec, r, n), **({"solve": f"eik_solve_sweep ({args.method}): "
                           "ingest + whole-grid sweep loop (CUDA graph) + egress"} if sweep else {}),
                           **({"bin_width": args.bin_width} if args.bin_width is not None else {})),
            "roofline": res["roof"], "cpu_baseline": cpu, "e2e": e2e,
            # per solve: init, ingest, (worklist build), egress + the loop's launches: fused
            # rounds = one k_cell each (k_select + k_cell + k_round_end otherwise); sweeping =
            # one k_dsweep per cell diagonal + k_sweep_end per sweep
            # async: init, ingest, seed, the persistent k_async, egress
            "gpu_launches": int(args.steps * res["launches_per_step"]),
            "clocks": res["clk"],
            "method": args.method,
            "work": res["work"],
        }
        if fp64 is not None:
            line["c3_fp64"] = fp64
        print(json.dumps(line), flush=True)
    solver.close()
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
