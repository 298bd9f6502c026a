"""Event-timed vs wall-timed per-step time on the same loop."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

G = 138_000_000
for flags, nm in [(_abi.FC_FLAG_ASYNC, "timing"), (_abi.FC_FLAG_ASYNC | _abi.FC_FLAG_NO_TIMING, "no-timing")]:
    uid = fc.get_unique_id()
    with fc.Cluster.nccl(1, 0, uid, G, device=0, max_cr=0.1, flags=flags) as cl:
        stream = torch.cuda.ExternalStream(cl.stream_ptr(), device=0)
        cl.fill_synthetic(0, 42, 0, 0)
        for s in range(5):
            cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=False)
        for n in (20, 50, 200):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cl.sync()
            t0 = time.perf_counter()
            e0.record(stream)
            for s in range(n):
                cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=False)
            e1.record(stream)
            t1 = time.perf_counter()
            cl.sync()
            t2 = time.perf_counter()
            print(f"{nm} n={n}: events {e0.elapsed_time(e1)/n*1e3:.1f} us/step, wall {(t2-t0)/n*1e6:.1f} us/step, enqueue {(t1-t0)/n*1e6:.1f}")
