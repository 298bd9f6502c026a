"""NVLink bytes per step of each exchange, from the GPUs' own NVLink data
counters (NVML field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX,
KiB, summed over the links) read around S steps -- no profiler replay, so
the peer waits run as in production.  One process per GPU:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_bytes.py [out.json]

Per rank and kind: TX / RX bytes per step against the algorithmic bytes the
bench reports (STAR ring / tree: list pull + contribution push + reduced
list; AG: (N-1) packs; dense: NCCL ring allreduce).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2312_02493_b200 import _abi, dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

G, CR, S = 138_000_000, 0.01, 50


def counters(h, pynvml):
    tx = rx = 0
    for link in range(18):
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                     (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
        except pynvml.NVMLError:
            continue
        if v[0].nvmlReturn == 0:
            tx += v[0].value.ullVal
        if v[1].nvmlReturn == 0:
            rx += v[1].value.ullVal
    return tx * 1024, rx * 1024


def main() -> int:
    env = dist.init_from_env("gloo")
    import pynvml
    import torch

    torch.cuda.set_device(env.local_rank)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(env.local_rank)
    n = env.world
    k = fc.k_of(CR, G)
    uid = dist.share_nccl_uid(env)
    out = {}
    with fc.Cluster.nccl(n, env.rank, uid, G, device=env.local_rank, max_cr=0.01, flags=_abi.FC_FLAG_ASYNC) as cl:
        cl.fill_synthetic(0, 42, env.rank, 0)
        kinds = {
            "star_ring": lambda s: cl.artopk_step(CR, fc.STAR, fc.RING, s, fc.AVG, stats=False),
            "star_tree": lambda s: cl.artopk_step(CR, fc.STAR, fc.TREE, s, fc.AVG, stats=False),
            "ag": lambda s: cl.ag_step(CR, stats=False),
            "dense": lambda s: cl.dense_step(fc.RING, fc.AVG, stats=False),
        }
        alg = {  # bytes one rank sends per step (the bench's bus bytes / N for the peer exchanges)
            "star_ring": 4.0 * k * (n - 1) / n + 2.0 * (n - 1) / n * 4.0 * k,
            "star_tree": 4.0 * k * (n - 1) / n + 2.0 * (n - 1) / n * 4.0 * k,
            "ag": (n - 1) * 8.0 * k,
            "dense": 2.0 * (n - 1) / n * 4.0 * G,
        }
        for name, step in kinds.items():
            for s in range(5):
                step(s)
            cl.sync()
            env.barrier()
            t0, r0 = counters(h, pynvml)
            for s in range(S):
                step(5 + s)
            cl.sync()
            env.barrier()
            t1, r1 = counters(h, pynvml)
            out[name] = {"tx_bytes_per_step": (t1 - t0) / S, "rx_bytes_per_step": (r1 - r0) / S,
                         "alg_bytes_per_rank_step": alg[name]}
        out["peer_exchange"] = cl.peer_exchange
    allr = [None] * n
    import torch.distributed as tdist

    tdist.all_gather_object(allr, out)
    if env.rank == 0:
        rec = {"n": n, "grad_len": G, "cr": CR, "k": k, "steps": S,
               "source": "NVML NVLink data counters (TX/RX KiB over the links) around S steps, per rank",
               "ranks": allr}
        print(json.dumps(rec, indent=1))
        if len(sys.argv) > 1:
            Path(sys.argv[1]).write_text(json.dumps(rec, indent=1))
    env.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
