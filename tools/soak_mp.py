"""Long-run soak of the multi-GPU exchange (peer memory or NCCL): STEPS
back-to-back steps cycling STAR / VAR (Ring), STAR / VAR (Tree) and AG, and
CR 0.01 / 0.003 / 0.05 (the aggregate updated in place, then rewritten
whole, then in place again), with the residual carried, one
rank per GPU.  Rank 0 follows the same trajectory with the fp32 oracle (the
checker) and compares every rank's aggregate and residual bit-exact every
CHECK steps and at the last step — exercises the mailbox epochs and parity
rows of the peer exchange over many reuses, not just the first few.

torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/soak_mp.py [G] [STEPS] [CHECK]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 200_003
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
    check = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    env = dist.init_from_env("gloo")
    uid = dist.share_nccl_uid(env)
    f32 = oracle.F32() if env.rank == 0 else None
    res = np.zeros((env.world, G), np.float32) if env.rank == 0 else None
    kinds = ("star", "var", "ag", "star-tree", "var-tree")
    crs = (0.01, 0.003, 0.05)
    failures, checks = [], 0
    t0 = time.time()
    with fc.Cluster.nccl(env.world, env.rank, uid, G, device=env.local_rank, max_cr=0.05) as cl:
        p2p = cl.peer_exchange
        for s in range(steps):
            kind = kinds[s % len(kinds)]
            c = crs[(s // len(kinds)) % len(crs)]
            cl.fill_synthetic(0, 99, env.rank, s)
            sel = -1
            if kind == "ag":
                cl.ag_step(c)
            else:
                sel = cl.artopk_step(c, fc.STAR if kind.startswith("star") else fc.VAR,
                                     fc.TREE if kind.endswith("tree") else fc.RING, s, fc.AVG).selected_rank
            last = s == steps - 1
            do_check = last or (s + 1) % check == 0 or s < 2 * len(kinds)
            if do_check:
                aggs = env.gather_arrays(cl.aggregate())
                resid = env.gather_arrays(cl.residual(0))
                sels = env.gather_arrays(np.array([sel]))
            if env.rank != 0:
                continue
            g_o = np.stack([f32.synth(G, 99, r, s) for r in range(env.world)])
            if kind == "ag":
                ref, rsel = f32.ag_step(g_o, res, c), -1
            else:
                ref, rsel, _, _ = f32.artopk_step(g_o, res, c, 0 if kind.startswith("star") else 1, s, 1)
            if not do_check:
                continue
            checks += 1
            for r in range(env.world):
                if int(sels[r][0]) != rsel:
                    failures.append(f"step {s} {kind}: rank {r} selected {int(sels[r][0])} != {rsel}")
                if not np.array_equal(resid[r].view(np.uint32), res[r].view(np.uint32)):
                    failures.append(f"step {s} {kind}: residual of rank {r} differs")
                exact = kind == "ag" or p2p
                if exact and not np.array_equal(aggs[r].view(np.uint32), ref.view(np.uint32)):
                    failures.append(f"step {s} {kind}: aggregate on rank {r} not bit-exact")
                # NCCL sums in its own order: 1e-5 relative, cancellation-safe
                # (a sum that cancels to ~0 keeps the summands' rounding)
                tol = 1e-5 * np.abs(ref) + 1e-6 * float(np.abs(ref).max(initial=0.0)) + 1e-30
                bad = np.abs(aggs[r].astype(np.float64) - ref) > tol
                if not exact and bad.any():
                    j = int(np.argmax(bad))
                    failures.append(f"step {s} {kind} c={c}: aggregate on rank {r} off: {int(bad.sum())} elements, "
                                    f"first at {j} (got {aggs[r][j]:.9g}, want {ref[j]:.9g}), "
                                    f"nonzero got/want {int((aggs[r] != 0).sum())}/{int((ref != 0).sum())}")
    if env.rank == 0:
        print(f"[soak_mp] world={env.world} G={G} steps={steps} peer={p2p} checks={checks} "
              f"failures={len(failures)} wall={time.time() - t0:.1f}s", flush=True)
        for f in failures[:20]:
            print("  ", f, flush=True)
        print("SOAK PASS" if not failures else "SOAK FAIL", flush=True)
    env.close()
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
