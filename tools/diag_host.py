"""Host enqueue time per step vs device time per step (NCCL path, world 1)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 138_000_000
for flags, name in [(_abi.FC_FLAG_ASYNC, "async+timing"), (_abi.FC_FLAG_ASYNC | _abi.FC_FLAG_NO_TIMING, "async no-timing")]:
    uid = fc.get_unique_id()
    with fc.Cluster.nccl(1, 0, uid, G, device=0, max_cr=0.1, flags=flags) as cl:
        cl.fill_synthetic(0, 42, 0, 0)
        for s in range(5):
            cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=False)
        cl.sync()
        n = 50
        t0 = time.perf_counter()
        for s in range(n):
            cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=False)
        t1 = time.perf_counter()
        cl.sync()
        t2 = time.perf_counter()
        print(f"{name}: host enqueue {(t1-t0)/n*1e6:.1f} us/step, wall incl. drain {(t2-t0)/n*1e6:.1f} us/step")
