"""World-size-2 gloo tests of the host-side multi-process plumbing (CPU)."""
from __future__ import annotations

import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(WORLD_SIZE=str(world), RANK=str(rank), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2312_02493_b200 import dist

    env = dist.init_from_env("gloo")
    assert (env.world, env.rank) == (world, rank)
    payload = bytes(range(128)) if rank == 0 else None
    got = env.broadcast_bytes(payload)
    m = env.max_over_ranks(float(rank) + 0.5)
    g = env.gather_arrays(np.full(3, rank, np.float32))
    env.barrier()
    q.put((rank, got == bytes(range(128)), m,
           None if g is None else [a.tolist() for a in g]))
    env.close()


def test_gloo_world2_plumbing():
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert all(ok for _, ok, _, _ in out)
    assert all(m == 1.5 for _, _, m, _ in out)
    assert out[0][3] == [[0.0] * 3, [1.0] * 3] and out[1][3] is None


def test_single_process_env(monkeypatch):
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    from paper_2312_02493_b200 import dist

    env = dist.init_from_env()
    assert env.world == 1 and env.pg is None
    assert env.max_over_ranks(3.0) == 3.0
    assert env.broadcast_bytes(b"x") == b"x"
