"""BASELINE config 4: the CR sweep with the AG / ART-Ring / ART-Tree switching
heuristic (crossover_cr / select_collective, inc/costmodel.hpp:
153-203), on this box's GPUs.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/c4_sweep.py [out.jsonl]

For every CR of the sweep on the GPT-2-medium-sized 355M gradient per GPU:
the three collectives' whole steps (ms, max over ranks; STAR AR-Top-k Ring
/ Tree and AG-Top-k) and the collective the unchanged selector picks with
the NVLink-calibrated NetParams (paper_2312_02493_b200/nvlink.py), with the
regret of that choice (its measured step over the fastest).  One JSON line
per CR (rank 0).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2312_02493_b200 import _abi, dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200 import nvlink  # noqa: E402

G = 355_000_000
CRS = [1e-4, 3e-4, 1e-3, 3e-3, 1e-2, 3e-2, 1e-1]
NAMES = {0: "ag", 1: "art_ring", 2: "art_tree"}


def main() -> int:
    env = dist.init_from_env("gloo")
    import torch

    torch.cuda.set_device(env.local_rank)
    n = env.world
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else None
    net = nvlink.net_params(n)
    uid = dist.share_nccl_uid(env)
    rows = []
    with fc.Cluster.nccl(n, env.rank, uid, G, device=env.local_rank, max_cr=0.1, flags=_abi.FC_FLAG_ASYNC) as cl:
        cl.fill_synthetic(0, 42, env.rank, 0)
        stream = torch.cuda.ExternalStream(cl.stream_ptr())
        for cr in CRS:
            row = {"n": n, "grad_len": G, "cr": cr, "k": fc.k_of(cr, G)}
            for kind in NAMES.values():
                def one(s):
                    if kind == "ag":
                        cl.ag_step(cr, stats=False)
                    else:
                        cl.artopk_step(cr, fc.STAR, fc.TREE if kind == "art_tree" else fc.RING, s, fc.AVG,
                                       stats=False)
                for s in range(3):
                    one(s)
                cl.sync()
                env.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for s in range(10):
                    one(3 + s)
                e1.record(stream)
                cl.sync()
                row[kind + "_ms"] = round(env.max_over_ranks(e0.elapsed_time(e1) / 10), 4)
            ch = fc.select_collective(net, fc.MessageSpec(4.0 * G, cr, n))
            pick = NAMES[int(ch.collective)]
            best = min(NAMES.values(), key=lambda kk: row[kk + "_ms"])
            row.update({"selected": pick, "fastest": best,
                        "regret": round(row[pick + "_ms"] / row[best + "_ms"] - 1.0, 3),
                        "net": {"alpha_s": net.alpha, "bandwidth_bps": net.bandwidth}})
            rows.append(row)
            if env.rank == 0:
                print(json.dumps(row), flush=True)
    if env.rank == 0 and out:
        out.write_text("".join(json.dumps(r) + "\n" for r in rows))
    env.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
