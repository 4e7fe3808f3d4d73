"""A/B timing of experimental builds (GPU box).  usage:
    python tools/ab.py C3,C5 lib_a.so lib_b.so ...   [env AB_OPTS="6=2"  option=value list]
Each library runs in its own process (EIK_LIB); prints mean ms of 5 solves after 2 warm-ups
(CUDA events on the solve stream) and the work counters."""
import json, os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import bench
    import paper_1306_4743_b200 as eik
    for name in sys.argv[2].split(","):
        cfg, prec, r = bench.WORKLOADS[name]
        n, F, m, q = bench.make_inputs(cfg, prec, torch.device("cuda", 0))
        s = eik.Solver()
        for kv in filter(None, os.environ.get("AB_OPTS", "").split(",")):
            k, v = kv.split("=")
            s.set_option(int(k), float(v))
        U = torch.empty_like(F)
        for _ in range(2):
            s.solve(F, m, q, cell_size=r, n=n, out=U)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); s.solve(F, m, q, cell_size=r, n=n, out=U); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        st = s.stats()
        print(json.dumps({"cfg": name, "lib": os.path.basename(eik.LIB_PATH), "ms": sum(ts) / len(ts),
                          "ms_min": min(ts), "proc": st["cell_processings"], "rounds": st["rounds"],
                          "upd_pt": st["point_updates"] / st["M"],
                          "ms_ingest": st["ms_ingest"], "ms_loop": st["ms_loop"], "ms_egress": st["ms_egress"],
                          "ms_cell": st["ms_cell_device"],
                          "csum": float(U[torch.isfinite(U)].double().sum())}), flush=True)
        s.close()
        del F, m, q, U
        torch.cuda.empty_cache()
    sys.exit(0)

cfgs = sys.argv[1]
for lib in sys.argv[2:]:
    env = dict(os.environ, EIK_LIB=os.path.abspath(lib))
    subprocess.run([sys.executable, os.path.abspath(__file__), "--child", cfgs], env=env)
