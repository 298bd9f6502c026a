"""Per-phase device time (CUDA events on the library stream) of single steps
for the BASELINE configurations, one GPU (loopback workers).
Usage: python tools/diag_step.py [dense]   (dense: FC_FLAG_DENSE_DECODE)"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

FLAGS = _abi.FC_FLAG_DENSE_DECODE if "dense" in sys.argv[1:] else 0

CONFIGS = [
    ("C1 STAR 11.7M CR.01 N=2", 11_700_000, 2, "star", 0.01),
    ("C2 VAR 25.6M CR.001 N=4", 25_600_000, 4, "var", 0.001),
    ("C3 STAR 138M CR.01 N=1", 138_000_000, 1, "star", 0.01),
    ("C3 AG 138M CR.01 N=1", 138_000_000, 1, "ag", 0.01),
    ("C4 STAR 355M CR.001 N=1", 355_000_000, 1, "star", 0.001),
    ("C4 STAR 355M CR.1 N=1", 355_000_000, 1, "star", 0.1),
]
out = []
for name, G, n, mode, cr in CONFIGS:
    with fc.Cluster(n, G, max_cr=max(cr, 0.1), flags=FLAGS) as cl:
        for r in range(n):
            cl.fill_synthetic(r, 42, r, 0)
        rows = []
        for s in range(6):
            if mode == "ag":
                st = cl.ag_step(cr)
            else:
                st = cl.artopk_step(cr, fc.STAR if mode == "star" else fc.VAR, fc.RING, s)
            rows.append(st)
        st = rows[-1]
        ws = cl.worker_stats(0)
        out.append({"config": name, "total_us": round(st.ms_total * 1e3, 1),
                    "ef_us": round(st.ms_ef * 1e3, 1), "select_us": round(st.ms_select * 1e3, 1),
                    "exchange_us": round(st.ms_exchange * 1e3, 1),
                    "decode_us": round(st.ms_decode * 1e3, 1),
                    "lower_bound_us": round(16 * G / 6535.7e3 * (1 if n == 1 else 1), 1),
                    "candidates": ws.candidates, "k": st.k, "fallback": st.fallback,
                    "launches": st.launches})
        print(json.dumps(out[-1]), flush=True)
