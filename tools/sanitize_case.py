"""Small driver for compute-sanitizer (tools/sanitize.sh): every kernel of
the path at small sizes on one GPU (loopback workers), checked against the
oracle so that a sanitizer run is also a parity run.  Exit 0 on parity."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2312_02493_b200 import _abi  # noqa: E402
from paper_2312_02493_b200 import flexcomm as fc  # noqa: E402

f32 = oracle.F32()
bad = 0


def same(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


for flags in (0, _abi.FC_FLAG_NO_COOPERATIVE):
    n, g = 2, 70_001
    with fc.Cluster(n, g, flags=flags) as cl:
        res = np.zeros((n, g), np.float32)
        for s, (kind, c) in enumerate([("star", 0.01), ("var", 0.05), ("ag", 0.01), ("star", 0.3), ("var", 0.002)]):
            g_o = np.stack([f32.synth(g, 5, r, s, s % 3) for r in range(n)])
            for r in range(n):
                cl.fill_synthetic(r, 5, r, s, s % 3)
            if kind == "ag":
                cl.ag_step(c)
                agg = f32.ag_step(g_o, res, c)
            else:
                cl.artopk_step(c, fc.STAR if kind == "star" else fc.VAR, fc.RING, s, fc.AVG)
                agg, _, _, _ = f32.artopk_step(g_o, res, c, 0 if kind == "star" else 1, s, 1)
            bad += not same(cl.aggregate(), agg)
        for r in range(n):
            bad += not same(cl.residual(r), res[r])
    # threshold / layerwise compressors and the forced fallback
    v = f32.synth(50_000, 3, 0, 0)
    with fc.Cluster(1, v.size, flags=flags) as cl:
        cl.set_grad(0, v)
        idx, _ = cl.topk_exact(0, 0.02)
        bad += not np.array_equal(idx, f32.topk_exact(v, 0.02)[0])
        cl.set_layer_map([(0, 10_000), (10_000, 40_000)])
        cl.ag_step(0.05, fc.LAYERWISE)
        cl.ag_step(0.05, fc.THRESHOLD)
    import os

    os.environ["FC_FORCE_FALLBACK"] = "1"
    with fc.Cluster(1, v.size, flags=flags) as cl:
        cl.set_grad(0, v)
        idx, _ = cl.topk_exact(0, 0.01)
        bad += not np.array_equal(idx, f32.topk_exact(v, 0.01)[0])
    del os.environ["FC_FORCE_FALLBACK"]
print("SANITIZE CASE", "PASS" if not bad else f"FAIL ({bad})")
sys.exit(1 if bad else 0)
