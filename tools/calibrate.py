"""NVLink calibration of the reference's alpha-beta cost model.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/calibrate.py [out_dir]

Measures, on this box's GPUs through the library's own NCCL communicators
(fc_diag_collective_ms, CUDA events, max over ranks), the three compressed
exchanges the reference's selector chooses between, over payload sizes
Mc = 4 KB ... 142 MB:
    AG-compressed   allgather of 2·Mc bytes per rank      (cost_ag_compressed)
    ART-Ring        broadcast(Mc) + ring allreduce(Mc)     (cost_art_ring, Eq. 4a)
    ART-Tree        broadcast(Mc) + tree allreduce(Mc)     (cost_art_tree, Eq. 4b)
plus the primitives.  Fits ONE NetParams(alpha, bandwidth) — the reference's
API has a single one (inc/costmodel.hpp:12-27) — by least squares on log
time, then checks select_collective (unchanged, inc/costmodel.hpp:153) with
the fitted NetParams against the measured-fastest exchange at every point,
in the spirit of the reference's Acceptance C2 (tests/test_acceptance.cpp:47-60).
Writes fixtures/nvlink_grid_n{N}.csv and fixtures/nvlink_fit_n{N}.json.
"""
from __future__ import annotations

import ctypes as C
import csv
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

SIZES = [4 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 55_200_000,
         142_000_000]
NAMES = {0: "broadcast", 1: "ring_ar", 2: "tree_ar", 3: "allgather", 4: "art_ring",
         5: "art_tree", 6: "ag_compressed"}


def model(alpha, beta, n, mc):
    lg = math.log2(n)
    nm1 = n - 1
    return {"ag_compressed": alpha * lg + 2.0 * mc * beta * nm1,
            "art_ring": alpha * (2 * nm1 + lg) + mc * beta * (2 * nm1 / n + lg),
            "art_tree": 3 * alpha * lg + 3 * mc * beta * lg}


def fit(rows, n):
    """Least squares on log time over the three exchanges; grid + refine."""
    best = None
    for la in np.linspace(-7, -3, 81):         # alpha 0.1 us .. 1 ms
        for lb in np.linspace(-13, -9, 81):    # beta  (1/bytes-per-second)
            a, b = 10 ** la, 10 ** lb
            err = 0.0
            for r in rows:
                m = model(a, b, n, r["mc"])
                for key in ("ag_compressed", "art_ring", "art_tree"):
                    err += (math.log(m[key]) - math.log(r[key])) ** 2
            if best is None or err < best[0]:
                best = (err, a, b)
    return best[1], best[2]


def main() -> int:
    env = dist.init_from_env("gloo")
    import torch

    torch.cuda.set_device(env.local_rank)
    n = env.world
    if n < 2:
        print("calibration needs >= 2 GPUs", file=sys.stderr)
        return 2
    uid = dist.share_nccl_uid(env)
    G = 355_000_000
    rows = []
    with fc.Cluster.nccl(n, env.rank, uid, G, device=env.local_rank, max_cr=0.1) as cl:
        for mc in SIZES:
            row = {"n": n, "mc": mc}
            for which, nm in NAMES.items():
                ms = C.c_double()
                iters = 20 if mc >= (16 << 20) else 100
                check(lib.fc_diag_collective_ms(cl._ctx, which, mc, iters, C.byref(ms)))
                row[nm] = env.max_over_ranks(ms.value) * 1e-3  # seconds, max over ranks
            rows.append(row)
            if env.rank == 0:
                print(json.dumps({k: (round(v * 1e6, 2) if k not in ("n", "mc") else v)
                                  for k, v in row.items()}), flush=True)
    if env.rank == 0:
        out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "fixtures"
        out.mkdir(parents=True, exist_ok=True)
        with open(out / f"nvlink_grid_n{n}.csv", "w", newline="") as f:
            wr = csv.writer(f)
            wr.writerow(["n", "payload_bytes"] + [f"{v}_us" for v in NAMES.values()])
            for r in rows:
                wr.writerow([n, r["mc"]] + [f"{r[v] * 1e6:.3f}" for v in NAMES.values()])
        alpha, beta = fit(rows, n)
        net = fc.NetParams(alpha, 8.0 / beta)
        checks = []
        for r in rows:
            m = model(alpha, beta, n, r["mc"])
            meas = {k: r[k] for k in ("ag_compressed", "art_ring", "art_tree")}
            order = sorted(meas, key=meas.get)
            margin = meas[order[1]] / meas[order[0]] - 1.0
            # select_collective with M, c such that M*c = payload (c = 0.01)
            ch = fc.select_collective(net, fc.MessageSpec(r["mc"] / 0.01, 0.01, n))
            pred = {0: "ag_compressed", 1: "art_ring", 2: "art_tree"}[int(ch.collective)]
            checks.append({"payload_bytes": r["mc"], "measured_fastest": order[0],
                           "margin": round(margin, 3), "predicted": pred,
                           "agree": pred == order[0],
                           "rel_err": {k: round(abs(m[k] - meas[k]) / meas[k], 3) for k in meas}})
        decisive = [c for c in checks if c["margin"] > 0.15]
        res = {"n": n, "alpha_s": alpha, "bandwidth_bps": 8.0 / beta,
               "bandwidth_GBps": 1.0 / beta / 1e9,
               "argmin_agreement_all": sum(c["agree"] for c in checks) / len(checks),
               "argmin_agreement_margin_gt_15pct": (sum(c["agree"] for c in decisive) / len(decisive)
                                                    if decisive else None),
               "max_rel_err": max(max(c["rel_err"].values()) for c in checks),
               "points": checks}
        (out / f"nvlink_fit_n{n}.json").write_text(json.dumps(res, indent=1))
        print(json.dumps({k: v for k, v in res.items() if k != "points"}), flush=True)
    env.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
