"""Multi-GPU parity of the NCCL path (one process per GPU).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tests/mp_check.py

Every rank runs a trajectory of STAR/VAR AR-Top-k (Ring and Tree) and
AG-Top-k steps on its own synthetic gradient; rank 0 regenerates all ranks'
gradients (the generator is counter-based) and checks against the fp32
oracle:
  * selected rank, residuals and the AG aggregate: bit-exact;
  * AR aggregates: NCCL's ring/tree summation order differs from the
    reference's rank-ascending order, so |gpu - oracle| <= 1e-5 * mean_r |c_r|
    (the north star's 1e-5 relative bar, cancellation-safe).
Exit code 0 on success.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402


def main() -> int:
    env = dist.init_from_env("gloo")
    import torch

    torch.cuda.set_device(env.local_rank)
    uid = dist.share_nccl_uid(env)
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_003
    f32 = oracle.F32() if env.rank == 0 else None
    plan = [("star", fc.RING, 0.01), ("star", fc.TREE, 0.05), ("var", fc.RING, 0.01),
            ("var", fc.TREE, 0.002), ("ag", fc.RING, 0.01), ("ag", fc.RING, 0.1),
            ("star", fc.RING, 0.001), ("dense", fc.TREE, 1.0),
            # AG with the layerwise / threshold compressors (threshold sizes
            # differ per rank: padded allgather)
            ("ag-lw", fc.RING, 0.05), ("ag-thr", fc.RING, 0.01), ("ag-thr", fc.RING, 0.1)]
    layers = [(0, 3), (3, 1000), (1005, G // 2 - 1005), (G // 2, G - G // 2)]
    failures = []
    with fc.Cluster.nccl(env.world, env.rank, uid, G, device=env.local_rank, max_cr=0.2) as cl:
        cl.set_layer_map(layers)
        p2p = cl.peer_exchange
        if env.rank == 0:
            print(f"[mp_check] peer exchange: {p2p}", flush=True)
        res = np.zeros((env.world, G), np.float32) if env.rank == 0 else None
        for s, (kind, algo, c) in enumerate(plan):
            cl.fill_synthetic(0, 1234, env.rank, s)
            sel = -1
            if kind == "ag":
                cl.ag_step(c)
            elif kind == "ag-lw":
                cl.ag_step(c, fc.LAYERWISE)
            elif kind == "ag-thr":
                cl.ag_step(c, fc.THRESHOLD)
            elif kind == "dense":
                cl.dense_step(algo, fc.AVG)
            else:
                st = cl.artopk_step(c, fc.STAR if kind == "star" else fc.VAR, algo, s, fc.AVG)
                sel = st.selected_rank
            agg = cl.aggregate()
            mine = cl.residual(0)
            aggs = env.gather_arrays(agg)
            resid = env.gather_arrays(mine)
            sels = env.gather_arrays(np.array([sel]))
            if env.rank != 0:
                continue
            g_o = np.stack([f32.synth(G, 1234, r, s) for r in range(env.world)])
            if kind == "ag":
                ref = f32.ag_step(g_o, res, c)
                exact = True
            elif kind in ("ag-lw", "ag-thr"):
                ref, _ = f32.ag_step_kind(g_o, res, c, 1 if kind == "ag-lw" else 2,
                                          layers if kind == "ag-lw" else None, 25)
                exact = True
            elif kind == "dense":
                ref = f32.dense(g_o, 1)
                exact = False
            else:
                ge = g_o + res  # the error-fed gradients (for the tolerance scale)
                ref, rsel, _, _ = f32.artopk_step(g_o, res, c, 0 if kind == "star" else 1, s, 1)
                if any(int(x[0]) != rsel for x in sels):
                    failures.append(f"step {s} {kind}: selected {[int(x[0]) for x in sels]} != {rsel}")
                exact = False
            for r in range(env.world):
                if kind != "dense" and not np.array_equal(resid[r].view(np.uint32), res[r].view(np.uint32)):
                    failures.append(f"step {s} {kind}: residual of rank {r} differs")
                if exact:
                    if not np.array_equal(aggs[r].view(np.uint32), ref.view(np.uint32)):
                        failures.append(f"step {s} {kind}: aggregate on rank {r} not bit-exact")
                else:
                    base = g_o if kind == "dense" else ge
                    scale = np.abs(base).sum(axis=0) / env.world
                    if (kind != "dense"):
                        scale = np.where(ref != 0, scale, 0)
                    if kind in ("star", "var") and p2p and not np.array_equal(aggs[r].view(np.uint32),
                                                                       ref.view(np.uint32)):
                        # rank-ordered sums over peer memory: bit-exact
                        failures.append(f"step {s} {kind}: peer-exchange aggregate on rank {r} not bit-exact")
                    err = np.abs(aggs[r].astype(np.float64) - ref)
                    if not np.all(err <= 1e-5 * scale + 1e-30):
                        failures.append(f"step {s} {kind}: aggregate on rank {r} off by {err.max():.3g}")
                    if kind != "dense" and not np.array_equal(aggs[r] != 0, ref != 0):
                        # support = the broadcast index set (zeros elsewhere)
                        nz = np.nonzero((aggs[r] != 0) != (ref != 0))[0]
                        if np.any(np.abs(ref[nz]) > 0):
                            failures.append(f"step {s} {kind}: aggregate support differs")
            print(f"[mp_check] step {s} {kind} algo={algo} c={c} ok={not failures}", flush=True)

        # MOO controller over the NCCL path: every rank must take the same
        # decisions (gains and measured compression times are rank-identical)
        from paper_2312_02493_b200 import moo

        sched = moo.NetworkSchedule([moo.Segment(0, fc.NetParams(5e-6, 4.5e12)),
                                     moo.Segment(1, fc.NetParams(5e-6, 4.5e10))])
        tr = moo.SyncTrainer(cl, moo.SyncConfig(epochs=2, steps_per_epoch=3, adaptive=True,
                                                seed=77), sched)
        ctl = moo.Controller(moo.ControllerConfig(probe_iters=2))
        tr.run(ctl.hook())
        summary = np.array([x for cnd in ctl.candidates
                            for x in (cnd.c, cnd.gain_avg, cnd.t_comp_avg, cnd.t_sync_modeled)]
                           + [x for e in ctl.events
                              for x in (e.step, e.chosen_c, int(e.collective), e.front_size)]
                           + [m.gain for m in tr.metrics] + [m.cr_used for m in tr.metrics])
        allsum = env.gather_arrays(summary)
        if env.rank == 0:
            if any(not np.array_equal(a, allsum[0]) for a in allsum):
                failures.append("MOO: ranks took different decisions")
            if len([e for e in ctl.events if e.trigger == "network"]) != 1:
                failures.append(f"MOO: expected one network event, got {ctl.events}")
            print(f"[mp_check] moo events={[(e.step, e.trigger, e.chosen_c) for e in ctl.events]} "
                  f"ok={not failures}", flush=True)
    if env.rank == 0:
        print("MP_CHECK", "PASS" if not failures else "FAIL", env.world, flush=True)
        for f in failures[:20]:
            print("  ", f)
    env.close()
    return 0 if not failures else 1


if __name__ == "__main__":
    sys.exit(main())
