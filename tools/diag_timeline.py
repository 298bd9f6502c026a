"""Device timeline of one step (138M, STAR, N=1 loopback), %globaltimer marks:
EF blocks (start, end), select phases, decode (start, end) -> the gaps
between kernels.  Usage: python tools/diag_timeline.py [async]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

G = 138_000_000
flags = (_abi.FC_FLAG_ASYNC if "async" in sys.argv[1:] else 0) | (
    _abi.FC_FLAG_NO_TIMING if "notiming" in sys.argv[1:] else 0)
nb = 148
period = next((int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("period=")), 4)
stats = "stats" in sys.argv[1:]


def marks(cl):
    tb = (C.c_uint64 * (2 * nb + 2))()
    check(lib.fc_diag_ef_blocks(cl._ctx, 0, tb, 2 * nb + 2))
    ts = (C.c_uint64 * 16)()
    check(lib.fc_diag_select_phases(cl._ctx, 0, ts))
    ef0 = min(tb[2 * b] for b in range(nb))
    ef1 = max(tb[2 * b + 1] for b in range(nb))
    return ef0, ef1, ts[0], ts[7], tb[2 * nb], tb[2 * nb + 1]


with fc.Cluster(1, G, max_cr=0.1, flags=flags) as cl:
    cl.set_ef_timing_period(period)
    cl.fill_synthetic(0, 42, 0, 0)
    import torch
    for s in range(6):
        cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=stats)
    cl.sync()
    st = torch.cuda.ExternalStream(cl.stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for s in range(20):
        cl.artopk_step(0.01, fc.STAR, fc.RING, 6 + s, stats=stats)
    e1.record(st)
    cl.sync()
    print(f"period {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/step (EF timing period {period}, stats={stats})")
    ef0, ef1, sel0, sel1, dec0, dec1 = marks(cl)
    r = lambda t: (t - ef0) / 1e3
    print(f"EF     {r(ef0):8.1f} .. {r(ef1):8.1f} us  ({(ef1 - ef0) / 1e3:.1f})")
    print(f"select {r(sel0):8.1f} .. {r(sel1):8.1f} us  ({(sel1 - sel0) / 1e3:.1f})  gap after EF {(sel0 - ef1) / 1e3:.1f}")
    print(f"decode {r(dec0):8.1f} .. {r(dec1):8.1f} us  ({(dec1 - dec0) / 1e3:.1f})  gap after select {(dec0 - sel1) / 1e3:.1f}")
    gaps = []
    for s in range(8):  # one synchronised step at a time: the gap of each
        cl.artopk_step(0.01, fc.STAR, fc.RING, 26 + s, stats=stats)
        cl.sync()
        ef0, ef1, sel0, sel1, dec0, dec1 = marks(cl)
        gaps.append(f"{(sel0 - ef1) / 1e3:.1f}/{(dec0 - sel1) / 1e3:.1f}")
    print("per-step gaps EF->select / select->decode (us):", " ".join(gaps))
