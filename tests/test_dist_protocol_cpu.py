"""The multi-rank exchange protocol of AR-Top-k / AG-Top-k, run as real
processes over gloo (CPU), checked bit-exact against the single-process
oracle (`oracle.F32.artopk_step` / `ag_step`, which restate
inc/artopk.hpp:62-111 and :128-161).

Each rank holds only its own worker's gradient and residual, exactly as one
GPU does under `bench.py --gpus N`, and follows the order the peer-memory
path uses on the device:

- STAR: selected rank = step % N (inc/artopk.hpp:27-30, `fc.select_star`);
- VAR: every rank publishes its fp64 squared norm of its Top-k values, all
  ranks take the argmax, strict `>`, ties to the lowest rank
  (inc/artopk.hpp:35-48);
- the selected rank's index list is broadcast (collectives.hpp:58);
- every rank gathers g_e at those indices and zeros them in its residual
  (artopk.hpp:92-102);
- the allreduce sums contributions in ascending rank order, then /N
  (collectives.hpp:82-87) — the order the device's rank-ordered sums keep;
- AG: allgather of (idx, val) lists, scatter-add in rank order, /N.

The oracle is the checker here only; the product path is the CUDA one.
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]

G, C, STEPS, SEED = 4099, 0.02, 4, 77


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grad(f32, rank, step, same):
    return f32.synth(G, SEED, 0 if same else rank, step)


def _worker(rank, world, port, mode, same, c, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(WORLD_SIZE=str(world), RANK=str(rank), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2312_02493_b200 import flexcomm as fc

    dist.init_process_group("gloo", rank=rank, world_size=world)
    f32 = oracle.F32()
    res = np.zeros(G, np.float32)
    out = []
    for step in range(STEPS):
        ge = _grad(f32, rank, step, same) + res
        idx, val = f32.topk_exact(ge, c)
        k = idx.size
        if mode == "ag":
            idxs = [torch.empty(k, dtype=torch.int64) for _ in range(world)]
            vals = [torch.empty(k, dtype=torch.float32) for _ in range(world)]
            dist.all_gather(idxs, torch.from_numpy(idx.astype(np.int64)))
            dist.all_gather(vals, torch.from_numpy(val))
            agg = np.zeros(G, np.float32)
            for r in range(world):
                agg[idxs[r].numpy()] += vals[r].numpy()
            agg /= np.float32(world)
            res = ge.copy()
            res[idx] -= val
            out.append((agg, res.copy(), -1))
            continue
        if mode == "star":
            sel = fc.select_star(step, world)
        else:
            score = torch.tensor([f32.squared_norm(val)], dtype=torch.float64)
            scores = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(scores, score)
            s = [float(t.item()) for t in scores]
            sel = 0
            for r in range(1, world):
                if s[r] > s[sel]:
                    sel = r
        bidx = torch.from_numpy(idx.astype(np.int64)) if rank == sel else torch.empty(k, dtype=torch.int64)
        dist.broadcast(bidx, src=sel)
        b = bidx.numpy()
        contrib = torch.from_numpy(ge[b].copy())
        parts = [torch.empty(k, dtype=torch.float32) for _ in range(world)]
        dist.all_gather(parts, contrib)
        red = parts[0].numpy().copy()
        for r in range(1, world):
            red += parts[r].numpy()
        red /= np.float32(world)
        agg = np.zeros(G, np.float32)
        agg[b] = red
        res = ge.copy()
        res[b] = 0.0
        out.append((agg, res.copy(), sel))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, out))


def _run(world, mode, same=False, c=C):
    port = _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, same, c, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world,mode,same,c", [
    (2, "star", False, C), (3, "star", False, C),
    (2, "var", False, C), (3, "var", False, C),
    (3, "var", True, C),  # equal scores on every rank -> rank 0 (strict >)
    (2, "ag", False, C), (3, "ag", False, C),
    (2, "star", False, 1.0), (2, "ag", False, 1.0),  # k = G: every index sent
    (3, "var", False, 1e-4),  # k = 1
])
def test_gloo_protocol_matches_oracle(f32, world, mode, same, c):
    got = _run(world, mode, same, c)
    res = np.zeros((world, G), np.float32)
    for step in range(STEPS):
        g_o = np.stack([_grad(f32, r, step, same) for r in range(world)])
        if mode == "ag":
            agg = f32.ag_step(g_o, res, c)
            sel = -1
        else:
            agg, sel, _, _ = f32.artopk_step(g_o, res, c, 0 if mode == "star" else 1, step)
        if same and mode == "var":
            assert sel == 0
        for r in range(world):
            a, rr, s = got[r][step]
            assert s == sel, (step, r)
            np.testing.assert_array_equal(a, agg)
            np.testing.assert_array_equal(rr, res[r])
