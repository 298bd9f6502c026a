"""Peer-only contexts (FC_FLAG_PEER_ONLY: no NCCL, exchange-buffer handles
allgathered over gloo) -- which lets several ranks share one GPU, so the
8-rank protocol (kMaxPeers = 8: mailboxes, parity rows, the two-stage list
broadcast from 5 ranks on) runs on a 4-GPU lease: correctness only.

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tests/mp_peer_only.py [G]

Ranks r and r + ngpu share GPU r % ngpu.  Every rank runs STAR / VAR (Ring
and Tree) and AG steps; rank 0 regenerates all ranks' gradients (counter-
based generator) and checks selection, aggregates and residuals bit-exact
against the fp32 oracle.  Exit 0 on success.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402


def main() -> int:
    env = dist.init_from_env("gloo")
    import torch

    ngpu = torch.cuda.device_count()
    dev = env.rank % ngpu
    torch.cuda.set_device(dev)
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 50_021

    def allgather(b: bytes):
        out = [None] * env.world
        env.pg.all_gather_object(out, b)
        return out

    f32 = oracle.F32() if env.rank == 0 else None
    plan = [("star", fc.RING, 0.01), ("var", fc.RING, 0.02), ("ag", fc.RING, 0.01), ("star", fc.TREE, 0.05),
            ("var", fc.TREE, 0.01), ("star", fc.RING, 0.002)]
    failures = []
    with fc.Cluster.peer_only(env.world, env.rank, G, allgather, device=dev, max_cr=0.05) as cl:
        cl.set_peer_timeout(600.0)  # ranks sharing a GPU are time-sliced
        res = np.zeros((env.world, G), np.float32) if env.rank == 0 else None
        for s, (kind, algo, c) in enumerate(plan):
            cl.fill_synthetic(0, 4321, env.rank, s)
            sel = -1
            if kind == "ag":
                cl.ag_step(c)
            else:
                sel = cl.artopk_step(c, fc.STAR if kind == "star" else fc.VAR, algo, s, fc.AVG).selected_rank
            aggs = env.gather_arrays(cl.aggregate())
            resid = env.gather_arrays(cl.residual(0))
            sels = env.gather_arrays(np.array([sel]))
            if env.rank != 0:
                continue
            g_o = np.stack([f32.synth(G, 4321, r, s) for r in range(env.world)])
            if kind == "ag":
                ref, rsel = f32.ag_step(g_o, res, c), -1
            else:
                ref, rsel, _, _ = f32.artopk_step(g_o, res, c, 0 if kind == "star" else 1, s, 1)
            for r in range(env.world):
                if int(sels[r][0]) != rsel:
                    failures.append(f"step {s} {kind}: rank {r} selected {int(sels[r][0])} != {rsel}")
                if not np.array_equal(aggs[r].view(np.uint32), ref.view(np.uint32)):
                    failures.append(f"step {s} {kind}: aggregate of rank {r} not bit-exact")
                if not np.array_equal(resid[r].view(np.uint32), res[r].view(np.uint32)):
                    failures.append(f"step {s} {kind}: residual of rank {r} differs")
        # NCCL-only operations fail loudly in a peer-only context
        try:
            cl.dense_step(fc.RING, fc.AVG)
            failures.append("dense step did not fail in a peer-only context")
        except fc.InvalidArgument:
            pass
        env.barrier()
    if env.rank == 0:
        print(f"[mp_peer_only] world={env.world} gpus={ngpu} G={G} failures={len(failures)}", flush=True)
        for f in failures[:20]:
            print("  ", f, flush=True)
        print("MP_PEER_ONLY PASS" if not failures else "MP_PEER_ONLY FAIL", flush=True)
    env.close()
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
