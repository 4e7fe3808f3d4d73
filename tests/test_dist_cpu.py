"""Multi-process plumbing of bench.py on CPU (gloo, world_size 2): the replicas-only path
 reduces each rank's step time with MAX and reports the whole-job throughput."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = [0.010, 0.025][rank]                      # rank 1 is the slow one
    tj = bench.job_time(t, dist, "cpu")
    out[rank] = (tj, bench.job_value(1000, world, tj))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_max_time_and_weak_value():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        tj, val = out[r]
        assert tj == pytest.approx(0.025)
        assert val == pytest.approx(1000 * 2 / 0.025)


def test_single_rank_passthrough():
    import bench
    assert bench.job_time(0.5) == 0.5
    assert bench.job_value(10, 1, 0.5) == 20.0


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` without torchrun re-executes itself under torch.distributed.run
    (one process per GPU, replicas only); here through the CPU plumbing mode (gloo): rank 0
    prints one line with n_gpus = 2, the max-over-ranks step time and the whole-job value."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--plumbing-test"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2
    assert lines[0]["ms_per_step"] == pytest.approx(20.0)          # rank 1's 20 ms (max)
    assert lines[0]["value"] == pytest.approx(1000 * 2 / 0.020)
