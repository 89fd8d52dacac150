"""Multi-process host logic on CPU (gloo, world size 2): the replicas-only bench
 -- max-over-ranks timing, identical seeded inputs on every
replica, and `bench.py --impl reference` under torchrun printing exactly one line
from rank 0."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from bench import max_over_ranks
    from workloads import configs as W

    v = max_over_ranks(10.0 + rank, dist)
    c = W.config4(12, 10, 8)
    h = [float(np.sum(x * np.arange(1, len(x) + 1))) for x in c["u"]] + [float(np.sum(c["op"]["kappa"]))]
    hs = [None] * world
    dist.all_gather_object(hs, h)
    out[rank] = (v, hs)
    dist.destroy_process_group()


def test_gloo_world2_max_and_identical_replicas():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 11.0
    assert res[0][1][0] == res[0][1][1]  # every replica draws the same seeded input


def test_reference_arm_under_torchrun_world2():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1", "--gpus", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "ms/call" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
