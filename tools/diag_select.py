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
        t = (C.c_uint64 * 16)()
        check(lib.fc_diag_select_phases(cl._ctx, 0, t))
        ws = cl.worker_stats(0)
        print(f"step {s}: total {st.ms_total * 1e3:.0f}us ef {st.ms_ef * 1e3:.0f}us select {st.ms_select * 1e3:.0f}us "
              f"exch {st.ms_exchange * 1e3:.0f}us decode {st.ms_decode * 1e3:.0f}us cand {ws.candidates} "
              + " ".join(f"{n}={(t[i + 1] - t[i]) / 1e3:.1f}us" for i, n in enumerate(names))
              + f" | EF: sample={(t[12] - t[8]) / 1e3:.1f}us flush={(t[13] - t[12]) / 1e3:.1f}us "
              f"barrier={(t[9] - t[13]) / 1e3:.1f}us bound={(t[10] - t[9]) / 1e3:.1f}us "
              f"stream={(t[11] - t[10]) / 1e3:.1f}us EF-end->select-start={(t[0] - t[11]) / 1e3:.1f}us"
              + (f" | emit: base={(t[14] - t[5]) / 1e3:.1f}us assemble={(t[15] - t[14]) / 1e3:.1f}us "
                 f"write={(t[6] - t[15]) / 1e3:.1f}us" if t[15] > t[14] else ""))

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
