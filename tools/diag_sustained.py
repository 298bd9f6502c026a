"""HBM streaming under sustained load: mean triad time over short vs long runs."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

G = 138_000_000
with fc.Cluster(1, G, max_cr=0.1) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    for iters in (10, 200, 2000, 10):
        ms = C.c_double()
        check(lib.fc_diag_kernel_ms(cl._ctx, 2, iters, C.byref(ms)))
        print(f"triad x{iters}: {ms.value*1e3:.1f} us = {12*G/ms.value/1e6:.0f} GB/s")
