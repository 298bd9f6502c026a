"""MOO-driven sync run (BASELINE config 5).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/moo_run.py [options]
    python tools/moo_run.py --workers 2 ...      # 1 GPU, loopback workers

Runs the adaptive-CR Controller (inc/moo.hpp semantics, default
ControllerConfig: ladder {0.1, 0.0333, 0.0111, 0.0037, 0.001}, 10 probe
iterations) over `--steps` synchronous STAR/VAR steps of a `--grad-len`
fp32 gradient per worker, with the NVLink-calibrated NetParams
(fixtures/nvlink_fit_n{N}.json) and, optionally, a network change halfway.
Candidate compression times are measured on the device.  Prints one JSON
object (rank 0) with the candidates, events, per-category seconds and the
per-step device time; `--out` also writes it to a file.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200 import moo, nvlink  # noqa: E402


def main() -> int:
    p = argparse.ArgumentParser()
    p.add_argument("--grad-len", type=int, default=1_000_000_000)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--steps-per-epoch", type=int, default=10)
    p.add_argument("--mode", choices=["star", "var"], default="star")
    p.add_argument("--probe-iters", type=int, default=10)
    p.add_argument("--workers", type=int, default=2, help="loopback workers when not under torchrun")
    p.add_argument("--net-change", type=float, default=0.0,
                   help="bandwidth factor applied at the middle epoch (0: constant network)")
    p.add_argument("--out", default=None)
    a = p.parse_args()

    env = dist.init_from_env("gloo")
    import torch

    torch.cuda.set_device(env.local_rank)
    if env.world > 1:
        uid = dist.share_nccl_uid(env)
        cl = fc.Cluster.nccl(env.world, env.rank, uid, a.grad_len, device=env.local_rank,
                             max_cr=0.1)
    else:
        cl = fc.Cluster(a.workers, a.grad_len, device=env.local_rank, max_cr=0.1)
    n = cl.world
    net0 = nvlink.net_params(n)
    segs = [moo.Segment(0, net0)]
    epochs = max(1, a.steps // a.steps_per_epoch)
    if a.net_change > 0 and epochs >= 2:
        segs.append(moo.Segment(epochs // 2, fc.NetParams(net0.alpha, net0.bandwidth * a.net_change)))
    cfg = moo.SyncConfig(epochs=epochs, steps_per_epoch=a.steps_per_epoch, adaptive=True,
                         mode=moo.SyncMode.VAR if a.mode == "var" else moo.SyncMode.STAR)
    tr = moo.SyncTrainer(cl, cfg, moo.NetworkSchedule(segs))
    ctl = moo.Controller(moo.ControllerConfig(probe_iters=a.probe_iters))
    env.barrier()
    t0 = time.time()
    tr.run(ctl.hook())
    cl.sync()
    env.barrier()
    wall = env.max_over_ranks(time.time() - t0)
    steps = tr.metrics
    out = {
        "workload": f"C5 MOO-driven {a.mode.upper()} over {len(steps)} steps, "
                    f"{a.grad_len / 1e6:g}M fp32 per worker, N={n}",
        "n": n, "grad_len": a.grad_len, "net": {"alpha_s": net0.alpha, "bandwidth_bps": net0.bandwidth,
                                                "source": "fixtures/nvlink_fit (calibrated)"},
        "net_change": a.net_change,
        "candidates": [vars(c) for c in ctl.candidates],
        "events": [{"step": e.step, "trigger": e.trigger, "chosen_c": e.chosen_c,
                    "collective": e.collective.name, "front_size": e.front_size} for e in ctl.events],
        "chosen_c_final": tr.current_c(),
        "collective_final": tr.current_collective().name,
        "clock_s": {c.name.lower(): tr.clock.of(c) for c in moo.Category},
        "steps": len(steps),
        "mean_step_ms": 1e3 * sum(m.t_step for m in steps) / max(1, len(steps)),
        "mean_comp_ms": 1e3 * sum(m.t_comp_decomp for m in steps) / max(1, len(steps)),
        "mean_sync_ms": 1e3 * sum(m.t_sync for m in steps) / max(1, len(steps)),
        "mean_gain": sum(m.gain for m in steps) / max(1, len(steps)),
        "wall_s_incl_exploration": wall,
    }
    if env.rank == 0:
        s = json.dumps(out)
        print(s, flush=True)
        if a.out:
            Path(a.out).parent.mkdir(parents=True, exist_ok=True)
            Path(a.out).write_text(json.dumps(out, indent=1))
    cl.close()
    env.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
