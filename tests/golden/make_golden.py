"""Generate tests/golden/golden.json from the UNMODIFIED reference.

Run in the dev container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py

Contents
  hand:      the reference tests' hand-executed vectors, transcribed with
             their file:line (tests/test_artopk.cpp, tests/test_compress.cpp,
             SPEC.md gain example).
  topk:      reference topk_exact (fp64, inc/compress.hpp:57) on fp32 values
             from the shared synthetic generator (include/fc_synth.h),
             widened to double: index sets are identical for fp32 and fp64.
  artopk:    reference artopk_step trajectories (inc/artopk.hpp:62) on
             dyadic inputs (multiples of 1/8, |x| <= 8) so every fp64 sum is
             exact in fp32 too: the fp32 GPU path must reproduce them bit
             for bit (aggregates compared after rounding to fp32).
  ag:        reference ag_step trajectories, same inputs.
  costmodel: reference select_collective / crossover_cr / candidate_ladder.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).with_name("golden.json")


def hand_vectors():
    return {
        # tests/test_artopk.cpp:28-53 (Artopk.HandExecutedTwoWorkerStep)
        "artopk_two_worker": {
            "source": "tests/test_artopk.cpp:28-53",
            "g_o": [[2.0, 0.0, 1.0], [3.0, 4.0, 2.0]],
            "c": 1.0 / 3.0,
            "steps": [
                {"step": 0, "selected": 0, "aggregate": [2.5, 0.0, 0.0],
                 "residuals": [[0.0, 0.0, 1.0], [0.0, 4.0, 2.0]]},
                {"step": 1, "selected": 1, "aggregate": [0.0, 4.0, 0.0],
                 "residuals": [[2.0, 0.0, 2.0], [3.0, 0.0, 4.0]]},
            ],
        },
        # tests/test_artopk.cpp:187-202 (AgStep.AveragesContributionsByWorkerCount);
        # 0.1 / 0.2 are restated as their fp32 values.
        "ag_two_worker": {
            "source": "tests/test_artopk.cpp:187-202",
            "g_o": [[4.0, 0.1, 0.0], [0.2, 6.0, 0.0]],
            "c": 1.0 / 3.0,
            "aggregate": [2.0, 3.0, 0.0],
            "residuals": [[0.0, 0.1, 0.0], [0.2, 0.0, 0.0]],
        },
        # tests/test_compress.cpp:66-71 (TopkExact.TieBreaksToLowerIndex)
        "topk_ties": {"source": "tests/test_compress.cpp:66-71",
                      "values": [1.0, -1.0, 1.0, -2.0, 1.0], "c": 0.6, "indices": [0, 1, 3]},
        # tests/test_compress.cpp:38-48 (KOf.ExactValues)
        "k_of": {"source": "tests/test_compress.cpp:38-48",
                 "cases": [[1.0, 17, 17], [0.5, 10, 5], [0.1, 10, 1], [0.01, 10, 1],
                           [0.3, 10, 3], [0.31, 10, 4]],
                 "invalid_c": [0.0, 1.5], "invalid_g": [0]},
        # SPEC.md compression_gain example: g_e=[3,-7,1,0,5], g_c={1:-7,4:5} -> 74/84
        "gain": {"source": "SPEC.md (compression_gain examples)",
                 "g_e": [3.0, -7.0, 1.0, 0.0, 5.0], "c": 0.4, "indices": [1, 4],
                 "gain": 74.0 / 84.0},
        # tests/test_collectives.cpp:43-54 (Allreduce.SumAndAverage)
        "allreduce": {"source": "tests/test_collectives.cpp:43-54",
                      "per_worker": [[1.0, 2.0], [3.0, 6.0]], "sum": [4.0, 8.0],
                      "avg": [2.0, 4.0]},
    }


def topk_cases(ref, f32):
    cases = []
    rng = np.random.default_rng(20231202)
    for t in range(40):
        g = int(rng.integers(1, 20000))
        c = float(rng.choice([1e-3, 3e-3, 1e-2, 0.05, 0.1, 0.25, 0.5, 1.0, rng.uniform(1e-3, 1)]))
        dist = int(t % 3)
        v = f32.synth(g, 42 + t, t % 4, t, dist)
        idx, _ = ref.topk_exact(v.astype(np.float64), c)
        cases.append({"g": g, "c": c, "seed": 42 + t, "rank": t % 4, "step": t, "dist": dist,
                      "k": int(idx.size), "indices": idx.astype(int).tolist()})
    # k_of quirk at the C5 rung: 1e9 x 0.0333 -> 33,300,001
    quirk = {"c": 0.0333, "g": 1_000_000_000, "k": ref.k_of(0.0333, 1_000_000_000)}
    return cases, quirk


def dyadic(rng, shape):
    return (rng.integers(-64, 65, size=shape) / 8.0).astype(np.float64)


def artopk_cases(ref):
    out = []
    rng = np.random.default_rng(62)
    for t in range(60):
        n = int(rng.integers(1, 5))
        g = int(rng.integers(1, 48))
        mode = int(t % 2)
        algo = int((t // 2) % 2)
        op = 1 if t % 5 else 0
        steps = []
        res = np.zeros((n, g))
        grads = []
        for s in range(4):
            c = float(rng.uniform(0.05, 1.0))
            g_o = dyadic(rng, (n, g))
            grads.append(g_o.tolist())
            agg, sel, charge = ref.artopk_step(g_o, res, c, mode, algo, s, op)
            steps.append({"c": c, "step": s, "selected": sel, "aggregate": agg.tolist(),
                          "residuals": res.tolist(), "sync_charge": charge})
        out.append({"n": n, "g": g, "mode": mode, "algo": algo, "op": op, "g_o": grads,
                    "steps": steps})
    return out


def ag_cases(ref):
    out = []
    rng = np.random.default_rng(128)
    for t in range(40):
        n = int(rng.integers(1, 5))
        g = int(rng.integers(1, 48))
        res = np.zeros((n, g))
        steps, grads = [], []
        for s in range(4):
            c = float(rng.uniform(0.05, 1.0))
            g_o = dyadic(rng, (n, g))
            grads.append(g_o.tolist())
            agg, charge = ref.ag_step(g_o, res, c)
            steps.append({"c": c, "aggregate": agg.tolist(), "residuals": res.tolist(),
                          "sync_charge": charge})
        out.append({"n": n, "g": g, "g_o": grads, "steps": steps})
    return out


def costmodel_cases(ref):
    rng = np.random.default_rng(2024)
    sel = []
    for _ in range(400):
        alpha = float(rng.uniform(1e-6, 0.2))
        bw = float(10 ** rng.uniform(8, 13))
        m = float(10 ** rng.uniform(4, 10))
        c = float(10 ** rng.uniform(-4, 0))
        n = int(rng.integers(2, 513))
        ch, costs = ref.select_collective(alpha, bw, m, c, n)
        sel.append({"alpha": alpha, "bw": bw, "m": m, "c": c, "n": n, "choice": ch,
                    "costs": costs.tolist()})
    cross = []
    for _ in range(100):
        alpha = float(rng.uniform(1e-6, 0.05))
        bw = float(10 ** rng.uniform(8, 13))
        m = float(10 ** rng.uniform(6, 10))
        n = int(rng.integers(2, 65))
        for pair in range(3):
            cross.append({"alpha": alpha, "bw": bw, "m": m, "n": n, "pair": pair,
                          "c": ref.crossover_cr(alpha, bw, m, n, pair)})
    ladder = ref.candidate_ladder()
    return {"select": sel, "crossover": cross, "ladder_default": ladder}


def moo_cases(ref):
    """MOO controller decision functions (inc/moo.hpp:44-146, netsched.hpp:50-58)."""
    rng = np.random.default_rng(77)
    ladders = []
    for _ in range(120):
        c_high = float(10 ** rng.uniform(-3, 0))
        c_low = float(c_high * 10 ** -rng.uniform(0, 3))
        factor = float(rng.choice([1.5, 2.0, 3.0, 3.3, 10.0]) if rng.random() < 0.5
                       else rng.uniform(1.01, 12))
        ladders.append({"c_low": c_low, "c_high": c_high, "factor": factor,
                        "ladder": ref.candidate_ladder(c_low, c_high, factor)})
    r3 = []
    for v in list(10 ** rng.uniform(-9, 9, 200)) + [0.0333333, 0.0111111, 0.0037037, 123456.0,
                                                      0.0, 0.00125, 0.0445, 2.5e-3]:
        v = float(v) * (-1.0 if rng.random() < 0.2 else 1.0)
        r3.append([v, ref.round_3sig(v)])
    knee = []
    for _ in range(300):
        m = int(rng.integers(1, 9))
        rows = []
        for i in range(m):
            if rows and rng.random() < 0.2:  # exact duplicates / ties
                rows.append(list(rows[int(rng.integers(0, len(rows)))]))
                rows[-1][0] = float(rng.choice([0.1, 0.0333, 0.0111, 0.0037, 0.001]))
                continue
            rows.append([float(rng.choice([0.1, 0.0333, 0.0111, 0.0037, 0.001])),
                         float(rng.uniform(0.05, 1.0)), float(10 ** rng.uniform(-5, -1)),
                         float(10 ** rng.uniform(-5, 0))])
        alpha = float(rng.uniform(1e-6, 0.01))
        bw = float(10 ** rng.uniform(9, 13))
        mb = float(10 ** rng.uniform(5, 10))
        n = int(rng.integers(2, 65))
        mask, chosen, coll = ref.choose_cr(np.array(rows), alpha, bw, mb, n)
        knee.append({"rows": rows, "alpha": alpha, "bw": bw, "m": mb, "n": n,
                     "mask": [int(x) for x in mask], "chosen": chosen, "collective": coll})
    trig = []
    for _ in range(200):
        cnt = int(rng.integers(0, 12))
        samples = [float(x) for x in rng.uniform(0.2, 1.0, cnt)]
        window = int(rng.integers(1, 10))
        gref = float(rng.choice([-1.0, 0.0, float(rng.uniform(0.2, 1.0))]))
        thr = float(rng.choice([0.0, 0.05, 0.1, 0.25]))
        trig.append({"gain_ref": gref, "samples": samples, "window": window, "threshold": thr,
                     "fire": ref.trigger_gain(gref, samples, window, thr)})
    net = []
    for _ in range(200):
        a0 = float(rng.uniform(0, 0.01))
        b0 = float(10 ** rng.uniform(8, 12))
        a1 = a0 * float(rng.choice([1.0, 1.0 + rng.uniform(-0.2, 0.2)]))
        b1 = b0 * float(rng.choice([1.0, 1.0 + rng.uniform(-0.2, 0.2)]))
        rel = float(rng.choice([0.0, 0.05, 0.1]))
        net.append({"a0": a0, "b0": b0, "a1": a1, "b1": b1, "rel": rel,
                    "changed": ref.network_changed(a0, b0, a1, b1, rel)})
    return {"ladder": ladders, "round_3sig": r3, "knee": knee, "trigger": trig, "network": net}


def main():
    oracle.build()
    ref, f32 = oracle.Ref(), oracle.F32()
    topk, quirk = topk_cases(ref, f32)
    data = {
        "generator": "tests/golden/make_golden.py (reference: /root/reference/proj/include)",
        "hand": hand_vectors(),
        "topk": topk,
        "k_of_quirk": quirk,
        "artopk": artopk_cases(ref),
        "ag": ag_cases(ref),
        "costmodel": costmodel_cases(ref),
        "moo": moo_cases(ref),
    }
    OUT.write_text(json.dumps(data, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
