"""Does a long back-to-back soak change the per-step time?"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

G = 138_000_000
uid = fc.get_unique_id()
with fc.Cluster.nccl(1, 0, uid, G, device=0, max_cr=0.1, flags=_abi.FC_FLAG_ASYNC) as cl:
    stream = torch.cuda.ExternalStream(cl.stream_ptr(), device=0)
    cl.fill_synthetic(0, 42, 0, 0)

    def timed(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cl.sync()
        e0.record(stream)
        for s in range(n):
            cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=False)
        e1.record(stream)
        cl.sync()
        return e0.elapsed_time(e1) / n * 1e3

    print("fresh 20:", round(timed(20), 1))
    for soak_s in (0.5, 1.5, 3.0):
        t = time.time()
        n = 0
        while time.time() - t < soak_s:
            for _ in range(20):
                cl.artopk_step(0.01, fc.STAR, fc.RING, n, stats=False)
                n += 1
            cl.sync()
        print(f"after {soak_s}s soak ({n} steps): 20 steps", round(timed(20), 1), "us/step")
        time.sleep(1.0)
        print("  after 1s idle:", round(timed(20), 1))
    print("ef timing", cl.ef_kernel_timing(reset=True))
