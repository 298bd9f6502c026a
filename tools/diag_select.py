"""Phase timing of the select kernel and the EF kernel (block 0, %globaltimer),
plus the EF blocks' start/end spread."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402
from paper_2312_02493_b200._abi import FC_FLAG_DENSE_DECODE, check, lib  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 138_000_000
cr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
flags = FC_FLAG_DENSE_DECODE if "dense" in sys.argv[3:] else 0
names = ["load+window+bar", "windowbin", "inbin+bar", "T+lookback", "emit", "write+bounds", "final"]
with fc.Cluster(1, G, max_cr=max(cr, 0.1), flags=flags) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    for s in range(4):
        st = cl.artopk_step(cr, fc.STAR, fc.RING, s)
        t = (C.c_uint64 * 24)()
        check(lib.fc_diag_select_phases(cl._ctx, 0, t))
        ws = cl.worker_stats(0)
        print(f"step {s}: total {st.ms_total * 1e3:.0f}us ef {st.ms_ef * 1e3:.0f}us select {st.ms_select * 1e3:.0f}us "
              f"exch {st.ms_exchange * 1e3:.0f}us decode {st.ms_decode * 1e3:.0f}us cand {ws.candidates} "
              + " ".join(f"{n}={(t[i + 1] - t[i]) / 1e3:.1f}us" for i, n in enumerate(names))
              + f" | EF: preamble={(t[10] - t[8]) / 1e3:.1f}us sample+hist1={(t[12] - t[8]) / 1e3:.1f}us flush={(t[13] - t[12]) / 1e3:.1f}us "
              f"barrier={(t[9] - t[13]) / 1e3:.1f}us bound={(t[10] - t[9]) / 1e3:.1f}us "
              f"stream={(t[11] - t[10]) / 1e3:.1f}us EF-end->select-start={(t[0] - t[11]) / 1e3:.1f}us"
              + (f" | sx: setup={(t[22] - t[0]) / 1e3:.1f} idxtma={(t[23] - t[22]) / 1e3:.1f} "
                 f"p1pass={(t[16] - t[23]) / 1e3:.1f} flush={(t[17] - t[16]) / 1e3:.1f} "
                 f"bar1={(t[1] - t[17]) / 1e3:.1f} p2pass={(t[18] - t[2]) / 1e3:.1f} flush+bar2={(t[3] - t[18]) / 1e3:.1f} "
                 f"idxwait={(t[19] - t[4]) / 1e3:.1f} emit={(t[5] - t[19]) / 1e3:.1f} write={(t[20] - t[5]) / 1e3:.1f} "
                 f"bounds={(t[21] - t[20]) / 1e3:.1f} bsum={(t[6] - t[21]) / 1e3:.1f}" if t[16] else ""))

# EF block imbalance of the last step: per-block start/end spread
nb = 148
t = (C.c_uint64 * (2 * nb))()
with fc.Cluster(1, G, max_cr=max(cr, 0.1), flags=flags) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    for s in range(4):
        cl.artopk_step(cr, fc.STAR, fc.RING, s)
    check(lib.fc_diag_ef_blocks(cl._ctx, 0, t, 2 * nb))
st = [t[2 * b] for b in range(nb)]
en = [t[2 * b + 1] for b in range(nb)]
t0 = min(st)
dur = sorted((e - s) / 1e3 for s, e in zip(st, en))
print(f"EF blocks: start spread {(max(st) - t0) / 1e3:.1f}us, end min/median/max "
      f"{(min(en) - t0) / 1e3:.1f}/{(sorted(en)[nb // 2] - t0) / 1e3:.1f}/{(max(en) - t0) / 1e3:.1f}us, "
      f"duration min/median/max {dur[0]:.1f}/{dur[nb // 2]:.1f}/{dur[-1]:.1f}us")

# select blocks: P1 / P2 pass end per block (k_select_x writes them at
# g_part[2048 + 2b], returned after the EF marks and 8 exchange marks)
with fc.Cluster(1, G, max_cr=max(cr, 0.1), flags=flags) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    for s in range(4):
        cl.artopk_step(cr, fc.STAR, fc.RING, s)
    n = 2 * nb + 8 + 2048 + 2 * nb
    t = (C.c_uint64 * n)()
    check(lib.fc_diag_ef_blocks(cl._ctx, 0, t, n))
    base = 2 * nb + 8 + 2048
    p1 = [t[base + 2 * b] for b in range(nb)]
    p2 = [t[base + 2 * b + 1] for b in range(nb)]
    t0 = min(p1)
    order = sorted(range(nb), key=lambda b: p1[b])
    print("select P1 end per block (us from the first): "
          + " ".join(f"{b}:{(p1[b] - t0) / 1e3:.1f}" for b in order[-12:]) + f" | median {(p1[order[nb // 2]] - t0) / 1e3:.1f}")
    t0 = min(p2)
    order = sorted(range(nb), key=lambda b: p2[b])
    print("select P2 end per block (us from the first): "
          + " ".join(f"{b}:{(p2[b] - t0) / 1e3:.1f}" for b in order[-12:]) + f" | median {(p2[order[nb // 2]] - t0) / 1e3:.1f}")
