"""Per-segment phases of the layerwise compressor's segmented launches
(VGG-16 map at 138M, CR 0.01, N=1): for each large layer, its blocks and
the EF-emission / select marks of its block 0 (fc_diag_seg_phases)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import check, lib  # noqa: E402

import bench  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 138_000_000
cr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
with fc.Cluster(1, G, max_cr=0.1) as cl:
    cl.set_layer_map(bench.vgg16_layers(G))
    cl.fill_synthetic(0, 42, 0, 0)
    for s in range(4):
        cl.ag_step(cr, fc.LAYERWISE)
    cl.sync()
    out = (C.c_uint64 * (26 * 64))()
    n = C.c_int()
    check(lib.fc_diag_seg_phases(cl._ctx, 0, out, 64, C.byref(n)))
    rows = [list(out[26 * q: 26 * q + 26]) for q in range(n.value)]
    t0 = min(r[2 + 8] for r in rows)  # earliest EF start
    for r in rows:
        ln, nb = r[0], r[1]
        sel, ef = r[2:10], r[10:14]
        rel = lambda t: (t - t0) / 1e3 if t >= t0 else float("nan")
        print(f"len {ln:>10} blocks {nb:>3} | EF start {rel(ef[0]):7.1f} barrier {rel(ef[1]):7.1f} bound {rel(ef[2]):7.1f} "
              f"end(b0) {rel(ef[3]):7.1f} | select start {rel(sel[0]):7.1f} window {rel(sel[1]):7.1f} "
              f"look-back {rel(sel[4]):7.1f} emitted {rel(sel[5]):7.1f} b0-done {rel(sel[6]):7.1f}")
