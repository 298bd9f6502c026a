"""Per-rank device timeline of one multi-GPU AR-Top-k step over the peer
exchange (%globaltimer marks; the GPUs of one node share the clock closely
enough for a microsecond view).  Run under torchrun:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P \\
        tools/diag_mp_timeline.py [star|var] [ring|tree] [G] [cr]
"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import _abi, dist  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

mode = fc.VAR if "var" in sys.argv[1:] else fc.STAR
algo = fc.TREE if "tree" in sys.argv[1:] else fc.RING
nums = [a for a in sys.argv[1:] if a[0].isdigit()]
G = int(nums[0]) if nums else 138_000_000
cr = float(nums[1]) if len(nums) > 1 else 0.01
env = dist.init_from_env("gloo")
import torch  # noqa: E402

torch.cuda.set_device(env.local_rank)
uid = dist.share_nccl_uid(env)
nb = torch.cuda.get_device_properties(env.local_rank).multi_processor_count
with fc.Cluster.nccl(env.world, env.rank, uid, G, device=env.local_rank, max_cr=0.1,
                     flags=_abi.FC_FLAG_ASYNC) as cl:
    cl.set_ef_timing_period(1 << 30)
    cl.fill_synthetic(0, 42, env.rank, 0)
    for s in range(8):
        cl.artopk_step(cr, mode, algo, s, stats=False)
    cl.sync()
    torch.distributed.barrier()
    st = torch.cuda.ExternalStream(cl.stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for s in range(20):
        cl.artopk_step(cr, mode, algo, 8 + s, stats=False)
    e1.record(st)
    cl.sync()
    period = e0.elapsed_time(e1) / 20 * 1e3
    rows = []
    for s in range(4):  # one step at a time (synchronised): marks of that step
        torch.distributed.barrier()
        stt = cl.artopk_step(cr, mode, algo, 28 + s, stats=False)
        cl.sync()
        ng = 2 * 148 * 8
        tb = (C.c_uint64 * (2 * nb + 8 + ng))()
        check(lib.fc_diag_ef_blocks(cl._ctx, 0, tb, 2 * nb + 8 + ng))
        ts = (C.c_uint64 * 24)()
        check(lib.fc_diag_select_phases(cl._ctx, 0, ts))
        ef0 = min(tb[2 * b] for b in range(nb))
        ef1 = max(tb[2 * b + 1] for b in range(nb))
        d = list(tb[2 * nb: 2 * nb + 8])
        rel = lambda t: (t - ef0) / 1e3 if t >= ef0 else float("nan")
        gb = [(tb[2 * nb + 8 + 2 * b], tb[2 * nb + 8 + 2 * b + 1]) for b in range(ng // 2)]
        gb = [(a, e) for a, e in gb if a >= ef0 and e >= a]
        gstat = ""
        if gb:
            st_ = sorted(a for a, _ in gb)
            en_ = sorted(e for _, e in gb)
            gstat = (f" | gather blocks {len(gb)}: start {rel(st_[0]):.1f}/{rel(st_[-1]):.1f} "
                     f"end {rel(en_[0]):.1f}/{rel(en_[len(en_) // 2]):.1f}/{rel(en_[-1]):.1f}")
            if os.environ.get("DUMP_BLOCKS"):
                gstat += "\n  block durations (us, block order): " + " ".join(
                    f"{(e - a) / 1e3:.0f}" for a, e in gb)
        rows.append(
            f"rank {env.rank} step {28 + s}: EF 0..{rel(ef1):.1f} | select {rel(ts[0]):.1f}..{rel(ts[7]):.1f} | "
            f"gather wait {rel(d[2]):.1f} start {rel(d[3]):.1f} published {rel(d[4]):.1f} | "
            f"reduce/pregather-end {rel(d[6]):.1f}..{rel(d[7]):.1f} | decode wait/pregather-start {rel(d[5]):.1f} start {rel(d[0]):.1f} "
            f"end {rel(d[1]):.1f}{gstat}")
    out = [None] * env.world
    torch.distributed.all_gather_object(out, (period, rows))
    if env.rank == 0:
        for r, (p, rr) in enumerate(out):
            print(f"rank {r}: period {p:.1f} us/step")
        for i in range(4):
            for r in range(env.world):
                print(out[r][1][i])
