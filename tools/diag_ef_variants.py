"""EF kernel time in different call patterns (same process, 138M): async
steps (fc_ef_kernel_timing), synchronous steps, fc_diag_kernel_ms variants."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

G = 138_000_000
for flags, name in ((_abi.FC_FLAG_ASYNC, "async steps"), (0, "sync steps")):
    with fc.Cluster(1, G, max_cr=0.1, flags=flags) as cl:
        cl.fill_synthetic(0, 42, 0, 0)
        for s in range(5):
            cl.artopk_step(0.01, fc.STAR, fc.RING, s, stats=False)
        cl.sync()
        cl.ef_kernel_timing(reset=True)
        for s in range(20):
            cl.artopk_step(0.01, fc.STAR, fc.RING, 5 + s, stats=False)
        cl.sync()
        ms, n = cl.ef_kernel_timing()
        print(f"{name}: EF {ms * 1e3:.1f} us over {n}", flush=True)
        out = []
        for w in (6, 5, 4, 6):
            m = C.c_double()
            check(lib.fc_diag_kernel_ms(cl._ctx, w, 10, C.byref(m)))
            out.append((w, round(m.value * 1e3, 1)))
        print("  diag variants", out, flush=True)
