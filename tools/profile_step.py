"""A short run of the bench workload for profilers (ncu): config 3's per-GPU
worker (138M fp32, CR 0.01, STAR, world-1 NCCL context), `warmup` steps then
`steps` steps, nothing else.  Usage: python tools/profile_step.py [warmup] [steps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
G = 138_000_000
with fc.Cluster.nccl(1, 0, fc.get_unique_id(), G, max_cr=0.1, flags=_abi.FC_FLAG_ASYNC) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    for s in range(warm + steps):
        cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=False)
    cl.sync()
print("ok")
