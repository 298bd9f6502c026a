"""Roofline calibration on a B200: times the EF pass variants against a plain
streaming triad (b += a) and a write-only fill over the same buffers, with
CUDA events (fc_diag_kernel_ms).  Usage: python tools/diag_kernels.py [G]"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 138_000_000
names = {0: "triad 3blk/SM", 1: "triad 4blk/SM", 2: "triad 8blk/SM", 3: "zero-fill 8blk/SM",
         4: "EF", 5: "EF+emit", 6: "EF+emit+owed zeros"}
bytes_ = {w: (4 * G if w == 3 else 12 * G) for w in names}
out = {}
with fc.Cluster(1, G, max_cr=0.1) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    cl.artopk_step(0.01, fc.STAR, fc.RING, 0)  # leaves a zero map for variant 6
    for w, nm in names.items():
        ms = C.c_double()
        check(lib.fc_diag_kernel_ms(cl._ctx, w, 10, C.byref(ms)))
        out[nm] = {"ms": round(ms.value, 4), "GB/s": round(bytes_[w] / ms.value / 1e6, 1)}
print(json.dumps({"G": G, "kernels": out}))
