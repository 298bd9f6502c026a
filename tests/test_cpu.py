"""CPU-only tests (no GPU): the oracle pinned against the reference and its
golden vectors, the host cost model vs the reference, and the C-ABI library
(loads, exports every declared symbol, fails loudly without a GPU)."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


# ------------------------------------------------------------------ C-ABI --

def test_library_exports_every_declared_symbol():
    from paper_2312_02493_b200 import _abi

    header = (ROOT / "include" / "flexcomm_b200.h").read_text()
    declared = sorted(set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(fc_\w+)\(", header, re.M)))
    assert len(declared) >= 30
    missing = [n for n in declared if not hasattr(_abi.lib, n)]
    assert not missing, missing
    assert sorted(_abi.EXPORTS) == declared
    assert _abi.lib.fc_abi_version() == 1


def test_no_gpu_fails_loudly():
    import torch

    from paper_2312_02493_b200 import flexcomm as fc

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(fc.NoDevice):
        fc.Cluster(1, 1000)


def test_k_of_known_answers(golden, fc):
    h = golden["hand"]["k_of"]
    for c, g, k in h["cases"]:
        assert fc.k_of(c, g) == k
    for c in h["invalid_c"]:
        with pytest.raises(fc.InvalidArgument):
            fc.k_of(c, 10)
    with pytest.raises(fc.InvalidArgument):
        fc.k_of(0.5, 0)
    q = golden["k_of_quirk"]
    assert fc.k_of(q["c"], q["g"]) == q["k"] == 33_300_001


def test_select_star_round_robin(fc):
    # tests/test_artopk.cpp:106-113
    counts = [0] * 4
    for step in range(100):
        counts[fc.select_star(step, 4)] += 1
    assert counts == [25] * 4
    with pytest.raises(fc.InvalidArgument):
        fc.select_star(0, 0)


# ---------------------------------------------------------------- oracle --

def test_oracle_hand_vectors(golden, f32):
    h = golden["hand"]
    a = h["artopk_two_worker"]
    g_o = np.array(a["g_o"], np.float32)
    res = np.zeros_like(g_o)
    for st in a["steps"]:
        agg, sel, _, _ = f32.artopk_step(g_o, res, a["c"], 0, st["step"], 1)
        assert sel == st["selected"]
        np.testing.assert_array_equal(agg, np.float32(st["aggregate"]))
        np.testing.assert_array_equal(res, np.float32(st["residuals"]))
    b = h["ag_two_worker"]
    g_o = np.array(b["g_o"], np.float32)
    res = np.zeros_like(g_o)
    agg = f32.ag_step(g_o, res, b["c"])
    np.testing.assert_array_equal(agg, np.float32(b["aggregate"]))
    np.testing.assert_array_equal(res, np.array(b["residuals"], np.float32))
    t = h["topk_ties"]
    assert f32.topk_exact(np.float32(t["values"]), t["c"])[0].tolist() == t["indices"]
    gn = h["gain"]
    idx, val = f32.topk_exact(np.float32(gn["g_e"]), gn["c"])
    assert idx.tolist() == gn["indices"]
    assert abs(f32.squared_norm(val) / f32.squared_norm(np.float32(gn["g_e"])) - gn["gain"]) < 1e-15
    ar = h["allreduce"]
    per = np.array(ar["per_worker"], np.float32)
    np.testing.assert_array_equal(f32.dense(per, 0), np.float32(ar["sum"]))
    np.testing.assert_array_equal(f32.dense(per, 1), np.float32(ar["avg"]))


def test_oracle_vs_reference_topk_golden(golden, f32):
    for case in golden["topk"]:
        v = f32.synth(case["g"], case["seed"], case["rank"], case["step"], case["dist"])
        idx, _ = f32.topk_exact(v, case["c"])
        assert idx.tolist() == case["indices"]


def test_oracle_vs_reference_artopk_golden(golden, f32):
    for case in golden["artopk"]:
        res = np.zeros((case["n"], case["g"]), np.float32)
        for s, st in enumerate(case["steps"]):
            g_o = np.array(case["g_o"][s], np.float32)
            agg, sel, _, _ = f32.artopk_step(g_o, res, st["c"], case["mode"], st["step"], case["op"])
            assert sel == st["selected"]
            np.testing.assert_array_equal(agg, np.array(st["aggregate"], np.float32))
            np.testing.assert_array_equal(res, np.array(st["residuals"], np.float32))


def test_oracle_vs_reference_ag_golden(golden, f32):
    for case in golden["ag"]:
        res = np.zeros((case["n"], case["g"]), np.float32)
        for s, st in enumerate(case["steps"]):
            agg = f32.ag_step(np.array(case["g_o"][s], np.float32), res, st["c"])
            np.testing.assert_array_equal(agg, np.array(st["aggregate"], np.float32))
            np.testing.assert_array_equal(res, np.array(st["residuals"], np.float32))


def test_oracle_vs_live_reference_random(ref, f32):
    """Acceptance C4/C5 style fuzz (tests/test_acceptance.cpp:97-118, 142-171)
    against the live reference build: step-0 index sets and selections, and
    per-step parity with the residual folded into g_o (so both precisions
    see identical g_e)."""
    rng = np.random.default_rng(4096)
    for t in range(300):
        g = int(rng.integers(1, 3000))
        c = float(rng.uniform(0.0005, 1.0))
        v = rng.standard_normal(g).astype(np.float32)
        if t % 4 == 0:
            v = np.round(v * 8) / 8  # tie-heavy
        assert np.array_equal(f32.topk_exact(v, c)[0].astype(np.uint64),
                              ref.topk_exact(v.astype(np.float64), c)[0])
    for t in range(150):
        n = int(rng.integers(1, 5))
        g = int(rng.integers(1, 64))
        mode = t % 2
        res32 = np.zeros((n, g), np.float32)
        for s in range(3):
            c = float(rng.uniform(0.05, 1.0))
            g_o = rng.standard_normal((n, g)).astype(np.float32)
            ge = g_o + res32  # the fp32 error-fed gradient
            res64 = np.zeros((n, g))
            a64, s64, _ = ref.artopk_step(ge.astype(np.float64), res64, c, mode, 0, s, 1)
            a32, s32, _, _ = f32.artopk_step(g_o, res32, c, mode, s, 1)
            assert s32 == s64
            np.testing.assert_array_equal(res32.astype(np.float64), res64)
            # fp32 vs fp64 rank-ascending sums: the north star's 1e-5 relative
            # bar, scaled by the contributions' magnitude (cancellation-safe)
            scale = np.abs(ge).sum(axis=0) / n
            assert np.all(np.abs(a32 - a64) <= 1e-5 * scale + 1e-30)


def test_synth_generator_deterministic(f32):
    a = f32.synth(10_000, 42, 0, 0)
    b = f32.synth(10_000, 42, 0, 0)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, f32.synth(10_000, 42, 1, 0))
    assert abs(float(a.mean())) < 0.05 and abs(float(a.std()) - 1.0) < 0.05
    t = f32.synth(10_000, 42, 0, 0, 1)
    assert np.all(np.round(t * 256) == t * 256)  # tie-stress grid


# ------------------------------------------------------------ cost model --

def test_costmodel_matches_reference_golden(golden, fc):
    cm = golden["costmodel"]
    for row in cm["select"]:
        ch = fc.select_collective(fc.NetParams(row["alpha"], row["bw"]),
                                  fc.MessageSpec(row["m"], row["c"], row["n"]))
        assert int(ch.collective) == row["choice"]
        assert [ch.costs[k] for k in fc.COST_FIELDS] == row["costs"]  # bit-exact
    for row in cm["crossover"]:
        got = fc.crossover_cr(fc.NetParams(row["alpha"], row["bw"]), row["m"], row["n"], row["pair"])
        assert got == row["c"]


def test_costmodel_matches_live_reference(ref, fc):
    """Acceptance C3 (tests/test_acceptance.cpp:63-94) + bit-exact argmin."""
    rng = np.random.default_rng(2024)
    non_tie = 0
    for _ in range(30_000):
        net = fc.NetParams(float(rng.uniform(1e-5, 0.2)), float(rng.uniform(1e8, 1e11)))
        msg = fc.MessageSpec(float(10 ** rng.uniform(4, 10)), float(10 ** rng.uniform(-4, 0)),
                             int(rng.integers(2, 513)))
        ch = fc.select_collective(net, msg)
        rch, rcosts = ref.select_collective(net.alpha, net.bandwidth, msg.m_bytes, msg.c, msg.n)
        assert int(ch.collective) == rch
        ring, tree, ag = ch.costs["art_ring"], ch.costs["art_tree"], ch.costs["ag_compressed"]

        def near(a, b):
            return abs(a - b) <= 1e-9 * max(abs(a), abs(b))

        if not near(ring, tree):
            assert fc.prefer(net, msg, 0) == (ring < tree)
            non_tie += 1
        if not near(ring, ag):
            assert fc.prefer(net, msg, 1) == (ring < ag)
            non_tie += 1
        if not near(tree, ag):
            assert fc.prefer(net, msg, 2) == (tree < ag)
            non_tie += 1
    assert non_tie >= 10_000


def test_costmodel_errors(fc):
    with pytest.raises(fc.InvalidArgument):
        fc.select_collective(fc.NetParams(0.001, 1e9), fc.MessageSpec(100.0, 0.1, 1))
    with pytest.raises(fc.InvalidArgument):
        fc.NetParams(-1.0, 1e9)
    with pytest.raises(fc.InvalidArgument):
        fc.MessageSpec(2.0, 0.1, 2)
    with pytest.raises(fc.InvalidArgument):
        fc.crossover_cr(fc.NetParams(0.001, 1e9), 1e6, 1, 0)


# ---- layerwise / threshold compressors ----------------------------

def _random_layers(rng, g):
    cuts = sorted(set(int(x) for x in rng.integers(1, g, int(rng.integers(0, 6))))) if g > 2 else []
    b = [0] + cuts + [g]
    return [(a, e - a) for a, e in zip(b, b[1:]) if e > a]


def test_oracle_compressors_vs_live_reference(ref, f32):
    """topk_layerwise / topk_threshold (inc/compress.hpp:67-112): the fp32
    restatement selects exactly what the reference selects."""
    rng = np.random.default_rng(21)
    for _ in range(400):
        g = int(rng.integers(1, 600))
        c = float(rng.uniform(0.005, 1.0))
        kind = int(rng.integers(1, 3))
        dist = rng.integers(0, 3)
        v = rng.standard_normal(g).astype(np.float32)
        if dist == 1:
            v = np.round(v * 4) / 4  # ties
        elif dist == 2:
            v = v * np.float32(10.0) ** rng.integers(-3, 3, g).astype(np.float32)
        layers = _random_layers(rng, g) if kind == 1 else None
        rounds = int(rng.integers(1, 40))
        i1, v1 = f32.topk_kind(v, c, kind, layers, rounds)
        i2, v2 = ref.topk_kind(v.astype(np.float64), c, kind, layers, rounds)
        np.testing.assert_array_equal(i1.astype(np.uint64), i2)
        np.testing.assert_array_equal(v1.astype(np.float64), v2)


def test_oracle_ag_step_kinds_vs_live_reference(ref, f32):
    """ag_step with Layerwise / Threshold (inc/artopk.hpp:128-161) on dyadic
    inputs (sums exact in fp32 and fp64): aggregates and residuals equal."""
    rng = np.random.default_rng(22)
    for _ in range(60):
        n = int(rng.choice([1, 2, 4]))  # /N exact in both precisions
        g = int(rng.integers(4, 300))
        kind = int(rng.integers(1, 3))
        layers = _random_layers(rng, g) if kind == 1 else None
        rounds = int(rng.integers(1, 30))
        res32 = np.zeros((n, g), np.float32)
        res64 = np.zeros((n, g), np.float64)
        for s in range(3):
            c = float(rng.choice([0.05, 0.1, 0.25, 0.5]))
            g_o = (rng.integers(-64, 65, (n, g)) / 16.0).astype(np.float32)
            a32, _ = f32.ag_step_kind(g_o, res32, c, kind, layers, rounds)
            a64 = ref.ag_step_kind(g_o.astype(np.float64), res64, c, kind, layers, rounds)
            np.testing.assert_array_equal(a32.astype(np.float64), a64)
            np.testing.assert_array_equal(res32.astype(np.float64), res64)


def test_oracle_compressor_reference_cases(f32):
    # tests/test_compress.cpp:73-78
    v = np.array([5.0, 0.1, 0.2, 0.3, 0.01, 9.0, 0.02, 0.03], np.float32)
    idx, val = f32.topk_kind(v, 0.25, 1, [(0, 4), (4, 4)])
    assert list(idx) == [0, 5] and list(val) == [5.0, 9.0]
    # tests/test_compress.cpp:80-91: distinct magnitudes -> threshold == exact
    rng = np.random.default_rng(11)
    for _ in range(50):
        g = int(rng.integers(2, 400))
        v = rng.standard_normal(g).astype(np.float32)
        c = float(rng.uniform(0.01, 1.0))
        np.testing.assert_array_equal(f32.topk_kind(v, c, 2)[0], f32.topk_exact(v, c)[0])
    # tests/test_compress.cpp:93-98
    v = rng.standard_normal(97).astype(np.float32)
    assert f32.topk_kind(v, 1.0, 2)[0].size == 97
