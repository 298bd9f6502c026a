"""Per-phase times of the NCCL (one process per GPU) path at world size 1."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 138_000_000
cr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
uid = fc.get_unique_id()
with fc.Cluster.nccl(1, 0, uid, G, device=0, max_cr=max(cr, 0.1)) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    for s in range(8):
        st = cl.artopk_step(cr, fc.STAR, fc.RING, s)
        print(f"step {s}: total {st.ms_total*1e3:.1f} ef {st.ms_ef*1e3:.1f} select {st.ms_select*1e3:.1f} "
              f"exchange {st.ms_exchange*1e3:.1f} decode {st.ms_decode*1e3:.1f} launches {st.launches}")
