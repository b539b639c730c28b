"""Host logic of bench.py (no GPU): replica aggregation over ranks with gloo,
and the reference arm's JSON contract."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    ms, dof = bench.combine_ranks(10.0 + rank, 100.0 * (rank + 1), world, device="cpu")
    q.put((rank, ms, dof))
    dist.destroy_process_group()


def test_combine_ranks_gloo_world2():
    import multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, ms, dof in res:
        assert ms == 11.0 and dof == 300.0     # max time, summed work


def test_reference_arm_json(tmp_path):
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                                   "--config", "c0_2d_const", "--steps", "5"], timeout=600).decode()
    line = json.loads(out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
