"""Steps of every peer-exchange kind at BASELINE config 3 (138M fp32, CR
0.01), one rank per GPU -- the workload for the NVLink counter capture
(tools/nvlink_profile.sh runs rank 0 under ncu, the other ranks plain)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

env = dist.init_from_env("gloo")
import torch  # noqa: E402

torch.cuda.set_device(env.local_rank)
uid = dist.share_nccl_uid(env)
G = int(os.environ.get("NVL_G", "138000000"))
with fc.Cluster.nccl(env.world, env.rank, uid, G, device=env.local_rank, max_cr=0.01) as cl:
    cl.set_peer_timeout(900.0)  # rank 0 runs under ncu (kernel replays)
    cl.fill_synthetic(0, 42, env.rank, 0)
    for s in range(2 * env.world):
        cl.artopk_step(0.01, fc.STAR, fc.RING, s)
    for s in range(2 * env.world):
        cl.artopk_step(0.01, fc.STAR, fc.TREE, s)
    for s in range(2):
        cl.ag_step(0.01)
    cl.sync()
    print(f"rank {env.rank}: peer={cl.peer_exchange} done", flush=True)
env.close()
