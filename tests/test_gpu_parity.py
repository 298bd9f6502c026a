"""GPU parity: the CUDA path through the C-ABI vs the oracle and the
reference's own golden vectors.

Bar (SURVEY §8c / BASELINE north star):
  * Top-k index sets, selected worker: bit-exact.
  * Loopback aggregates and residuals: bit-exact vs the fp32 restatement
    (same rank-ascending summation order as the reference, collectives.hpp:82).
  * Against the fp64 reference on dyadic inputs: bit-exact after rounding to
    fp32 (the sums are exact in both precisions).
  * Gain inputs (fp64 norms): relative 1e-9 (summation order differs).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bitwise(a, b, what=""):
    a, b = bits(a), bits(b)
    if not np.array_equal(a, b):
        bad = np.nonzero(a != b)[0]
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[:5]}: "
                             f"{a[bad[:5]].view(np.float32)} vs {b[bad[:5]].view(np.float32)}")


# ----------------------------------------------------------------- generator --

@pytest.mark.parametrize("dist", [0, 1, 2])
def test_synthetic_generator_bit_identical(fc, f32, dist):
    g = 300_007
    with fc.Cluster(1, g) as cl:
        cl.fill_synthetic(0, 42, 3, 7, dist)
        cl.dense_step(op=fc.SUM)
        assert_bitwise(cl.aggregate(), f32.synth(g, 42, 3, 7, dist), "synth")


# ---------------------------------------------------------------------- top-k --

TOPK_CASES = [(g, c, d) for g in (1, 2, 3, 7, 16, 100, 8191, 8192, 8193, 65_537, 1_000_003)
              for c in (1e-3, 0.01, 0.1, 0.37, 1.0) for d in (0, 1, 2)]


@pytest.mark.parametrize("g,c,dist", TOPK_CASES)
def test_topk_exact_matches_oracle(fc, f32, g, c, dist):
    v = f32.synth(g, 7 + g, 1, 2, dist)
    with fc.Cluster(1, g) as cl:
        cl.set_grad(0, v)
        idx, val = cl.topk_exact(0, c)
    ridx, rval = f32.topk_exact(v, c)
    np.testing.assert_array_equal(idx, ridx)
    assert_bitwise(val, rval, "values")


def test_topk_forced_fallback(fc, f32, monkeypatch):
    monkeypatch.setenv("FC_FORCE_FALLBACK", "1")
    for g, c, dist in [(50_000, 0.01, 0), (123_457, 0.1, 1), (10, 0.3, 0)]:
        v = f32.synth(g, 11, 0, 0, dist)
        with fc.Cluster(1, g) as cl:
            cl.set_grad(0, v)
            idx, _ = cl.topk_exact(0, c)
            assert cl.worker_stats(0).fallback == 1
        np.testing.assert_array_equal(idx, f32.topk_exact(v, c)[0])


def test_topk_adversarial_ties(fc, f32):
    # every magnitude equal: the whole selection is the tie-break
    g = 100_000
    v = np.where(np.arange(g) % 3 == 0, 1.0, -1.0).astype(np.float32)
    with fc.Cluster(1, g) as cl:
        cl.set_grad(0, v)
        for c in (1e-4, 0.01, 0.5):
            idx, _ = cl.topk_exact(0, c)
            np.testing.assert_array_equal(idx, np.arange(idx.size, dtype=np.uint32))
    # zeros and negative zeros share one magnitude
    v = np.zeros(5000, np.float32)
    v[::2] = -0.0
    v[4000] = 3.0
    with fc.Cluster(1, v.size) as cl:
        cl.set_grad(0, v)
        idx, _ = cl.topk_exact(0, 0.01)
    np.testing.assert_array_equal(idx, f32.topk_exact(v, 0.01)[0])


# ------------------------------------------------------------ full protocol --

def trajectory(fc, f32, n, g, steps, mode, op, crs, dist, seed, algo=0, flags=0, max_cr=1.0):
    with fc.Cluster(n, g, max_cr=max_cr, flags=flags) as cl:
        res = np.zeros((n, g), np.float32)
        for s in range(steps):
            c = crs[s % len(crs)]
            g_o = np.stack([f32.synth(g, seed, r, s, dist) for r in range(n)])
            for r in range(n):
                cl.fill_synthetic(r, seed, r, s, dist)
            st = cl.artopk_step(c, mode, algo, s, op)
            agg, sel, _, norms = f32.artopk_step(g_o, res, c, mode, s, op)
            assert st.selected_rank == sel, (s, st.selected_rank, sel, norms)
            assert_bitwise(cl.aggregate(), agg, f"aggregate step {s}")
            for r in range(n):
                assert_bitwise(cl.residual(r), res[r], f"residual r{r} step {s}")
                ws = cl.worker_stats(r)
                ge = g_o[r].astype(np.float64)  # only used for magnitude checks
                assert ws.ge_norm2 > 0 or not ge.any()
            if mode == fc.VAR:
                for r in range(n):
                    np.testing.assert_allclose(cl.worker_stats(r).topk_norm2, norms[r], rtol=1e-9)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("mode", [0, 1])
def test_artopk_trajectory_bit_exact(fc, f32, n, mode):
    trajectory(fc, f32, n, 40_000 + 17 * n, 5, mode, 1, [0.01, 0.1, 0.003], n % 3, 100 + n)


def test_artopk_dense_decode_flag(fc, f32):
    """FC_FLAG_DENSE_DECODE: the tile decode at every k (no in-place support
    update), bit-exact like the default path."""
    from paper_2312_02493_b200 import _abi

    for n, mode in ((1, 0), (3, 0), (2, 1)):
        trajectory(fc, f32, n, 70_001, 6, mode, 1, [0.01, 0.001, 0.2, 0.003], 0, 31 + n,
                   flags=_abi.FC_FLAG_DENSE_DECODE)


def test_aggregate_in_place_update(fc, f32):
    """The aggregate kept by whole-sector in-place updates (k <= G/80): the
    previous support's sectors zeroed, the new one's rewritten -- bit-exact
    with a full decode while k moves across the dense/in-place boundary,
    with lists whose entries share sectors and owed-zero words (dense
    clusters) and a gradient length that ends mid-sector."""
    from paper_2312_02493_b200 import _abi

    g = 262_147  # ends 3 floats into a sector
    for flags, expect in ((0, True), (_abi.FC_FLAG_DENSE_DECODE, False)):
        with fc.Cluster(1, g, flags=flags) as cl:
            res = np.zeros((1, g), np.float32)
            for s, c in enumerate([0.01, 0.005, 0.5, 0.001, 0.012, 0.003]):
                g_o = f32.synth(g, 77, 0, s, s % 2)[None]
                if s == 3:  # a dense run of large magnitudes: whole sectors / words selected
                    g_o[0, 1000:1400] = 50.0 + np.arange(400, dtype=np.float32)
                cl.set_grad(0, g_o[0])
                cl.artopk_step(c, fc.STAR, 0, s, fc.AVG)
                agg, _, _, _ = f32.artopk_step(g_o, res, c, fc.STAR, s, fc.AVG)
                assert_bitwise(cl.aggregate(), agg, f"aggregate step {s} cr {c}")
                assert_bitwise(cl.residual(0), res[0], f"residual step {s}")
                k = fc.k_of(c, g)
                assert cl.aggregate_in_place == (expect and k * 80 <= g), (s, c)


def test_non_cooperative_launch_path(fc, f32):
    """FC_FLAG_NO_COOPERATIVE: the grid-barrier kernels as plain launches
    (occupancy-checked), bit-exact like the default cooperative launches."""
    from paper_2312_02493_b200 import _abi

    for n, mode in ((1, 0), (2, 1)):
        trajectory(fc, f32, n, 90_001, 3, mode, 1, [0.01, 0.1], 0, 3 + n,
                   flags=_abi.FC_FLAG_NO_COOPERATIVE)


@pytest.mark.parametrize("op", [0, 1])
@pytest.mark.parametrize("algo", [0, 1])
def test_artopk_ops_algos(fc, f32, op, algo):
    trajectory(fc, f32, 3, 9_999, 3, 0, op, [0.05], 0, 5, algo)


def test_artopk_tiny_sizes(fc, f32):
    for g in (1, 2, 3, 5, 16):
        for n in (1, 2, 4):
            trajectory(fc, f32, n, g, 3, (g + n) % 2, 1, [0.3, 1.0, 0.05], 0, g * 10 + n)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_ag_trajectory_bit_exact(fc, f32, n):
    g = 30_011
    with fc.Cluster(n, g) as cl:
        res = np.zeros((n, g), np.float32)
        for s, c in enumerate([0.01, 0.1, 0.001, 0.5]):
            g_o = np.stack([f32.synth(g, 9, r, s, s % 3) for r in range(n)])
            for r in range(n):
                cl.fill_synthetic(r, 9, r, s, s % 3)
            cl.ag_step(c)
            agg = f32.ag_step(g_o, res, c)
            assert_bitwise(cl.aggregate(), agg, f"ag aggregate step {s}")
            for r in range(n):
                assert_bitwise(cl.residual(r), res[r], f"ag residual r{r}")


@pytest.mark.parametrize("op", [0, 1])
def test_dense_step(fc, f32, op):
    n, g = 3, 12_345
    with fc.Cluster(n, g) as cl:
        g_o = np.stack([f32.synth(g, 1, r, 0) for r in range(n)])
        cl.set_grads(list(g_o))
        cl.dense_step(op=op)
        assert_bitwise(cl.aggregate(), f32.dense(g_o, op), "dense")


# ------------------------------------------------------- reference goldens --

def test_golden_hand_vectors(fc, golden):
    h = golden["hand"]
    a = h["artopk_two_worker"]
    g_o = np.array(a["g_o"], np.float32)
    with fc.Cluster(2, 3) as cl:
        cl.set_grads(list(g_o))
        for st in a["steps"]:
            s = cl.artopk_step(a["c"], fc.STAR, fc.RING, st["step"], fc.AVG)
            assert s.selected_rank == st["selected"]
            np.testing.assert_array_equal(cl.aggregate(), np.float32(st["aggregate"]))
            for r in range(2):
                np.testing.assert_array_equal(cl.residual(r), np.float32(st["residuals"][r]))
    b = h["ag_two_worker"]
    with fc.Cluster(2, 3) as cl:
        cl.set_grads(list(np.array(b["g_o"], np.float32)))
        cl.ag_step(b["c"])
        np.testing.assert_array_equal(cl.aggregate(), np.float32(b["aggregate"]))
        for r in range(2):
            np.testing.assert_array_equal(cl.residual(r), np.array(b["residuals"][r], np.float32))
    t = h["topk_ties"]
    with fc.Cluster(1, len(t["values"])) as cl:
        cl.set_grad(0, np.float32(t["values"]))
        idx, _ = cl.topk_exact(0, t["c"])
        assert idx.tolist() == t["indices"]
    gn = h["gain"]
    with fc.Cluster(1, len(gn["g_e"])) as cl:
        cl.set_grad(0, np.float32(gn["g_e"]))
        cl.ag_step(gn["c"])
        ws = cl.worker_stats(0)
        assert cl.topk(0)[0].tolist() == gn["indices"]
        assert abs(ws.topk_norm2 / ws.ge_norm2 - gn["gain"]) < 1e-12


def test_golden_reference_topk(fc, f32, golden):
    for case in golden["topk"]:
        v = f32.synth(case["g"], case["seed"], case["rank"], case["step"], case["dist"])
        with fc.Cluster(1, case["g"]) as cl:
            cl.set_grad(0, v)
            idx, _ = cl.topk_exact(0, case["c"])
        assert idx.tolist() == case["indices"], case["g"]


def test_golden_reference_artopk(fc, golden):
    for case in golden["artopk"]:
        n, g = case["n"], case["g"]
        with fc.Cluster(n, g) as cl:
            for s, st in enumerate(case["steps"]):
                cl.set_grads(list(np.array(case["g_o"][s], np.float32)))
                out = cl.artopk_step(st["c"], case["mode"], case["algo"], st["step"], case["op"])
                assert out.selected_rank == st["selected"]
                np.testing.assert_array_equal(cl.aggregate(), np.array(st["aggregate"], np.float32))
                for r in range(n):
                    np.testing.assert_array_equal(cl.residual(r),
                                                  np.array(st["residuals"][r], np.float32))


def test_golden_reference_ag(fc, golden):
    for case in golden["ag"]:
        n, g = case["n"], case["g"]
        with fc.Cluster(n, g) as cl:
            for s, st in enumerate(case["steps"]):
                cl.set_grads(list(np.array(case["g_o"][s], np.float32)))
                cl.ag_step(st["c"])
                np.testing.assert_array_equal(cl.aggregate(), np.array(st["aggregate"], np.float32))
                for r in range(n):
                    np.testing.assert_array_equal(cl.residual(r),
                                                  np.array(st["residuals"][r], np.float32))


# ------------------------------------------------------------------- errors --

def test_errors_map_to_reference_exceptions(fc):
    with fc.Cluster(2, 100, max_cr=0.5) as cl:
        with pytest.raises(fc.InvalidArgument):
            cl.artopk_step(0.0)
        with pytest.raises(fc.InvalidArgument):
            cl.artopk_step(1.5)
        with pytest.raises(fc.InvalidArgument):
            cl.artopk_step(0.9)  # above max_cr
        with pytest.raises(fc.InvalidArgument):
            cl.artopk_step(0.1, step=-1)  # select_star -> bad source rank
        with pytest.raises(fc.OutOfRange):
            cl.residual(2)
        with pytest.raises(fc.InvalidArgument):
            cl.set_grads([np.zeros(100, np.float32)])
    with pytest.raises(fc.InvalidArgument):
        fc.Cluster(1, 0)
    with pytest.raises(fc.InvalidArgument):
        fc.Cluster(0, 10)


# -------------------------------------------------------------- gain / state --

def test_gain_inputs(fc, f32):
    n, g, c = 2, 50_000, 0.01
    with fc.Cluster(n, g) as cl:
        g_o = np.stack([f32.synth(g, 3, r, 0) for r in range(n)])
        cl.set_grads(list(g_o))
        st = cl.artopk_step(c, fc.STAR, fc.RING, 0)
        idx = f32.topk_exact(g_o[st.selected_rank], c)[0]
        for r in range(n):
            ge = g_o[r].astype(np.float64)
            ws = cl.worker_stats(r)
            np.testing.assert_allclose(ws.ge_norm2, (ge * ge).sum(), rtol=1e-9)
            np.testing.assert_allclose(ws.kept_norm2, (ge[idx] ** 2).sum(), rtol=1e-9)


def test_snapshot_restore_replays(fc, f32):
    n, g = 2, 20_000
    with fc.Cluster(n, g) as cl:
        for r in range(n):
            cl.fill_synthetic(r, 1, r, 0)
        cl.artopk_step(0.01, fc.STAR, fc.RING, 0)
        cl.snapshot()
        outs = []
        for s in range(1, 3):
            cl.artopk_step(0.01, fc.STAR, fc.RING, s)
            outs.append(cl.aggregate().copy())
        cl.restore()
        for s in range(1, 3):
            cl.artopk_step(0.01, fc.STAR, fc.RING, s)
            assert_bitwise(cl.aggregate(), outs[s - 1], "replay")


# --------------------------------------------------------- BASELINE sizes --

def test_c1_full_size_bit_exact(fc, f32):
    """BASELINE config 1: STAR, 11.7M fp32, CR 0.01, 2 workers, seed 42."""
    trajectory(fc, f32, 2, 11_700_000, 2, fc.STAR, fc.AVG, [0.01], 0, 42)


@pytest.mark.slow
@pytest.mark.parametrize("c", [0.01, 0.001])
def test_c3_size_properties(fc, f32, c):
    """138M (VGG-16-sized) gradient: size-independent properties of the exact
    top-k + error feedback (the oracle's nth_element is too slow here)."""
    g = 138_000_000
    k = fc.k_of(c, g)
    with fc.Cluster(1, g, max_cr=0.1) as cl:
        cl.fill_synthetic(0, 42, 0, 0)
        cl.fill_synthetic(0, 42, 0, 1)  # overwrite: g_o for step 1
        res0 = f32.synth(g, 42, 0, 0)
        cl.set_residual(0, res0)
        cl.ag_step(c)  # N=1: EF + top-k + residual_update + decode
        idx, val = cl.topk(0)
        res = cl.residual(0)
        agg = cl.aggregate()
    ge = f32.synth(g, 42, 0, 1) + res0  # fp32 add, same as the kernel
    assert idx.size == k
    assert np.all(np.diff(idx.astype(np.int64)) > 0)
    assert_bitwise(val, ge[idx], "values are g_e at the indices")
    # densify(g_c) + residual == g_e (SPEC exactness invariant)
    recon = res.copy()
    recon[idx] = val
    assert_bitwise(recon, ge, "densify + residual")
    assert_bitwise(agg[idx], val, "N=1 aggregate")
    # threshold separation with lowest-index tie-break
    key = ge.view(np.uint32) & 0x7FFFFFFF
    sel = np.zeros(g, bool)
    sel[idx] = True
    tmin = key[sel].min()
    assert key[~sel].max() <= tmin
    ties_out = np.nonzero((~sel) & (key == tmin))[0]
    ties_in = np.nonzero(sel & (key == tmin))[0]
    if ties_out.size:
        assert ties_in.max() < ties_out.min()


# ------------------------------------------- owed zeros / NCCL single rank --

@pytest.mark.parametrize("kind", ["star", "var", "ag"])
def test_owed_zeros_applied_by_next_pass(fc, f32, kind):
    """Residuals are NOT read between steps, so every step's residual zeroing
    travels as owed zeros into the next error-feedback pass; the aggregates of
    every step and the final residuals must still be bit-exact."""
    n, g = 3, 70_001
    with fc.Cluster(n, g) as cl:
        res = np.zeros((n, g), np.float32)
        for s in range(6):
            c = [0.01, 0.05, 0.002][s % 3]
            g_o = np.stack([f32.synth(g, 77, r, s, s % 3) for r in range(n)])
            for r in range(n):
                cl.fill_synthetic(r, 77, r, s, s % 3)
            if kind == "ag":
                cl.ag_step(c)
                agg = f32.ag_step(g_o, res, c)
            else:
                mode = fc.STAR if kind == "star" else fc.VAR
                st = cl.artopk_step(c, mode, fc.RING, s, fc.AVG)
                agg, sel, _, _ = f32.artopk_step(g_o, res, c, mode, s, 1)
                assert st.selected_rank == sel
            assert_bitwise(cl.aggregate(), agg, f"{kind} aggregate step {s}")
        for r in range(n):
            assert_bitwise(cl.residual(r), res[r], f"{kind} final residual r{r}")


@pytest.mark.parametrize("kind", ["star", "var", "ag", "dense"])
def test_nccl_single_rank_path(fc, f32, kind):
    """The one-process-per-GPU (NCCL) code path at world size 1."""
    g = 123_457
    uid = fc.get_unique_id()
    with fc.Cluster.nccl(1, 0, uid, g, device=0, max_cr=0.2) as cl:
        res = np.zeros((1, g), np.float32)
        for s in range(4):
            c = [0.01, 0.1][s % 2]
            g_o = f32.synth(g, 5, 0, s)[None, :]
            cl.fill_synthetic(0, 5, 0, s)
            if kind == "ag":
                cl.ag_step(c)
                agg = f32.ag_step(g_o, res, c)
            elif kind == "dense":
                cl.dense_step(fc.RING, fc.AVG)
                agg = f32.dense(g_o, 1)
            else:
                mode = fc.STAR if kind == "star" else fc.VAR
                st = cl.artopk_step(c, mode, fc.RING, s, fc.AVG)
                agg, sel, _, _ = f32.artopk_step(g_o, res, c, mode, s, 1)
                assert st.selected_rank == sel == 0
            assert_bitwise(cl.aggregate(), agg, f"{kind} nccl aggregate step {s}")
        if kind != "dense":
            assert_bitwise(cl.residual(0), res[0], "nccl residual")


def test_residual_pointer_and_snapshot_materialise(fc, f32):
    n, g = 2, 40_000
    with fc.Cluster(n, g) as cl:
        for r in range(n):
            cl.fill_synthetic(r, 8, r, 0)
        cl.artopk_step(0.01, fc.STAR, fc.RING, 0)
        cl.snapshot()  # must include the owed zeros
        a1 = [cl.residual(r).copy() for r in range(n)]
        cl.artopk_step(0.01, fc.STAR, fc.RING, 1)
        cl.restore()
        for r in range(n):
            assert_bitwise(cl.residual(r), a1[r], "restored residual")
