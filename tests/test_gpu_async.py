"""Async host copies (FC_HOST_ASYNC): uploads of step s+1 overlap downloads of
step s; the results must be exactly those of the synchronous path."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pipeline", [False, True])
@pytest.mark.parametrize("kind", ["star", "ag", "dense"])
def test_async_pipeline_matches_oracle(fc, f32, kind, pipeline):
    import torch

    from paper_2312_02493_b200 import _abi

    g, steps, c = 200_003, 5, 0.01
    uid = fc.get_unique_id()
    hosts = [torch.from_numpy(f32.synth(g, 31, 0, s)).pin_memory() for s in range(steps)]
    outs = [torch.empty(g, dtype=torch.float32).pin_memory() for _ in range(steps)]
    flags = _abi.FC_FLAG_ASYNC | (_abi.FC_FLAG_PIPELINE if pipeline else 0)
    with fc.Cluster.nccl(1, 0, uid, g, device=0, max_cr=0.1, flags=flags) as cl:
        for s in range(steps):
            cl.set_grad(0, hosts[s], async_=True)
            if kind == "ag":
                cl.ag_step(c, stats=False)
            elif kind == "dense":
                cl.dense_step(fc.RING, fc.AVG, stats=False)
            else:
                cl.artopk_step(c, fc.STAR, fc.RING, s, fc.AVG, stats=False)
            cl.aggregate(outs[s], async_=True)
        cl.sync()
        res_gpu = cl.residual(0)
    res = np.zeros((1, g), np.float32)
    for s in range(steps):
        g_o = hosts[s].numpy()[None, :]
        if kind == "dense":
            ref = f32.dense(g_o, 1)
        elif kind == "ag":
            ref = f32.ag_step(g_o, res, c)
        else:
            ref = f32.artopk_step(g_o, res, c, 0, s, 1)[0]
        assert np.array_equal(outs[s].numpy().view(np.uint32), ref.view(np.uint32)), f"step {s}"
    assert np.array_equal(res_gpu.view(np.uint32), res[0].view(np.uint32))


def test_async_then_sync_copies_interleave(fc, f32):
    import torch

    g = 50_000
    host = torch.from_numpy(f32.synth(g, 3, 0, 0)).pin_memory()
    with fc.Cluster(1, g) as cl:
        cl.set_grad(0, host, async_=True)
        cl.dense_step(op=fc.SUM)  # waits for the upload
        out = torch.empty(g, dtype=torch.float32).pin_memory()
        cl.aggregate(out, async_=True)
        cl.set_grad(0, np.zeros(g, np.float32))  # sync upload after async traffic
        cl.sync()
        assert np.array_equal(out.numpy(), host.numpy())
