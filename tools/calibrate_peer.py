"""NVLink calibration of the cost model on the exchange the library runs.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/calibrate_peer.py [out_dir]

The reference's selector (select_collective, inc/costmodel.hpp:153-167)
picks AG, ART-Ring or ART-Tree from one NetParams(alpha, bandwidth); the
reference validates that choice against measured collective times
(inc/sweep.hpp:63-108, tests/test_acceptance.cpp:45-60).  This tool measures
the three exchanges as the product runs them -- over NVLink peer memory,
with the product's own kernels -- on this box's GPUs, max over ranks:

  step grid       whole steps (fc_artopk_step Ring / Tree, fc_ag_step) at
                  BASELINE configs 1-3 (G, CR) and seven more (G, CR) points
                  (Mc = 4 G c = 47 KB .. 55 MB), plus the same steps of a
                  one-worker context on the same GPU (no exchange): the
                  measured sync time of a collective is its step minus the
                  one-worker step of the same kind -- what choosing that
                  collective costs the step (the fit's input)
  exchange grid   fc_diag_exchange_ms(AG / ART-Ring / ART-Tree) for k
                  (index, value) pairs, k = 1e3 .. 1.38e7 (Mc = 4k bytes):
                  the communication alone, from the selections being
                  published to the decode's inputs being in place (reported
                  beside the fit: it leaves out the N-list decode of AG)

Writes fixtures/peer_exchange_n{N}.csv and fixtures/peer_steps_n{N}.csv;
tools/fit_peer.py fits NetParams to them (no GPU needed).
"""
from __future__ import annotations

import csv
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

KS = [1_000, 4_000, 25_600, 117_000, 400_000, 1_380_000, 4_000_000, 13_800_000]
# BASELINE configs 1-3, plus more (G, CR) points spanning Mc = 4 G c bytes
# from 47 KB to 55 MB for the fit
CONFIGS = [("C1", 11_700_000, 0.01), ("C2", 25_600_000, 0.001), ("C3", 138_000_000, 0.01),
           ("G11.7M-c0.001", 11_700_000, 0.001), ("G11.7M-c0.1", 11_700_000, 0.1),
           ("G25.6M-c0.01", 25_600_000, 0.01), ("G138M-c0.001", 138_000_000, 0.001),
           ("G138M-c0.003", 138_000_000, 0.003), ("G138M-c0.03", 138_000_000, 0.03),
           ("G138M-c0.1", 138_000_000, 0.1)]
KINDS = ["ag", "art_ring", "art_tree"]


def time_steps(cl, kind, cr, steps, warmup, env=None):
    """Mean device ms per step (CUDA events on the library stream)."""
    import torch

    def one(s):
        if kind == "ag":
            cl.ag_step(cr, stats=False)
        else:
            cl.artopk_step(cr, fc.STAR, fc.TREE if kind == "art_tree" else fc.RING, s, fc.AVG, stats=False)

    stream = torch.cuda.ExternalStream(cl.stream_ptr())
    for s in range(warmup):
        one(s)
    cl.sync()
    if env:
        env.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(steps):
        one(warmup + s)
    e1.record(stream)
    cl.sync()
    return e0.elapsed_time(e1) / steps


def main() -> int:
    env = dist.init_from_env("gloo")
    import torch

    torch.cuda.set_device(env.local_rank)
    n = env.world
    if n < 2:
        print("calibration needs >= 2 GPUs", file=sys.stderr)
        return 2
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "fixtures"
    flags = _abi.FC_FLAG_ASYNC

    # ---- exchange grid ------------------------------------------------------
    ex_rows = []
    uid = dist.share_nccl_uid(env)
    with fc.Cluster.nccl(n, env.rank, uid, 138_000_000, device=env.local_rank, max_cr=0.1, flags=flags) as cl:
        cl.fill_synthetic(0, 42, env.rank, 0)
        cl.artopk_step(0.01, fc.STAR, fc.RING, 0, fc.AVG, stats=False)  # g_e in place
        cl.sync()
        p2p = cl.peer_exchange
        for k in KS:
            row = {"n": n, "k": k, "mc_bytes": 4 * k}
            for which, nm in enumerate(KINDS):
                ms = C.c_double()
                iters = 20 if k >= 1_000_000 else 100
                env.barrier()
                check(lib.fc_diag_exchange_ms(cl._ctx, which, k, iters, C.byref(ms)))
                row[nm + "_us"] = env.max_over_ranks(ms.value) * 1e3
            ex_rows.append(row)
            if env.rank == 0:
                print(json.dumps(row), flush=True)

    # ---- step grid ------------------------------------------------------------
    st_rows = []
    for name, G, cr in CONFIGS:
        uid = dist.share_nccl_uid(env)
        row = {"n": n, "config": name, "grad_len": G, "cr": cr, "k": fc.k_of(cr, G)}
        with fc.Cluster.nccl(n, env.rank, uid, G, device=env.local_rank, max_cr=cr, flags=flags) as cl:
            cl.fill_synthetic(0, 42, env.rank, 0)
            for kind in KINDS:  # best of 3 runs of 30 steps (max over ranks each)
                ts = []
                for _ in range(3):
                    env.barrier()
                    ts.append(env.max_over_ranks(time_steps(cl, kind, cr, 30, 5, env)) * 1e3)
                row[kind + "_step_us"] = min(ts)
        # the same steps without an exchange: one worker on this GPU
        with fc.Cluster(1, G, device=env.local_rank, max_cr=cr, flags=flags) as one:
            one.fill_synthetic(0, 42, env.rank, 0)
            for kind, key in (("art_ring", "art_one_worker_us"), ("ag", "ag_one_worker_us")):
                ts = []
                for _ in range(3):
                    env.barrier()
                    ts.append(env.max_over_ranks(time_steps(one, kind, cr, 30, 5)) * 1e3)
                row[key] = min(ts)
        st_rows.append(row)
        if env.rank == 0:
            print(json.dumps(row), flush=True)

    if env.rank == 0:
        out.mkdir(parents=True, exist_ok=True)
        for fname, rows in ((f"peer_exchange_n{n}.csv", ex_rows), (f"peer_steps_n{n}.csv", st_rows)):
            with open(out / fname, "w", newline="") as f:
                wr = csv.DictWriter(f, fieldnames=list(rows[0]))
                wr.writeheader()
                for r in rows:
                    wr.writerow({k: (f"{v:.3f}" if isinstance(v, float) and k != "cr" else v)
                                 for k, v in r.items()})
        print(json.dumps({"n": n, "peer_exchange": p2p, "out": str(out)}), flush=True)
    env.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
