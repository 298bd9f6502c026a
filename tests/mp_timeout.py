"""A peer that never arrives: the waiting rank's exchange kernel gives up
after the peer timeout, skips its remaining reads, and the step call (or
fc_sync) reports FC_ERR_RUNTIME -- never a hang, never a silent result.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_timeout.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2312_02493_b200 import dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402


def main() -> int:
    env = dist.init_from_env("gloo")
    import torch

    torch.cuda.set_device(env.local_rank)
    uid = dist.share_nccl_uid(env)
    ok = True
    with fc.Cluster.nccl(env.world, env.rank, uid, 100_003, device=env.local_rank, max_cr=0.05) as cl:
        if not cl.peer_exchange:
            print("MP_TIMEOUT SKIP (no peer exchange)", flush=True)
            env.close()
            return 0
        cl.set_peer_timeout(2.0)
        cl.fill_synthetic(0, 1, env.rank, 0)
        cl.artopk_step(0.01, fc.STAR, fc.RING, 0)  # both ranks: fine
        env.barrier()
        if env.rank == 0:
            # step 1 selects rank 1, which does not take part: rank 0 waits
            t0 = time.time()
            try:
                cl.artopk_step(0.01, fc.STAR, fc.RING, 1)
                cl.sync()
                ok = False
                print("rank 0: no error reported", flush=True)
            except fc.RuntimeFailure as e:
                ok = "timed out" in str(e)
                print(f"rank 0: {e} after {time.time() - t0:.1f} s", flush=True)
            # the report is returned once, then cleared
            try:
                cl.sync()
            except fc.RuntimeFailure:
                ok = False
        env.barrier()
    if env.rank == 0:
        print("MP_TIMEOUT PASS" if ok else "MP_TIMEOUT FAIL", flush=True)
    env.close()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
