"""Layerwise and threshold compressors on the AG path:
fc_ag_step with FC_LAYERWISE / FC_THRESHOLD against the fp32 restatement of
topk_layerwise / topk_threshold / ag_step (inc/compress.hpp:67-112,
inc/artopk.hpp:113-161), bit-exact aggregates and residuals."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def random_layers(rng, g, n_max=12):
    cuts = sorted(set(int(x) for x in rng.integers(1, g, int(rng.integers(1, n_max)))))
    b = [0] + cuts + [g]
    return [(a, e - a) for a, e in zip(b, b[1:]) if e > a]


def run_traj(fc, f32, n, g, kind, crs, layers=None, rounds=25, dist=0, seed=1, max_cr=0.3, nccl=False):
    cl = fc.Cluster.nccl(1, 0, fc.get_unique_id(), g, max_cr=max_cr) if nccl else fc.Cluster(n, g, max_cr=max_cr)
    with cl:
        if layers is not None:
            cl.set_layer_map(layers)
        cl.set_threshold_rounds(rounds)
        res = np.zeros((n, g), np.float32)
        for s, c in enumerate(crs):
            g_o = np.stack([f32.synth(g, seed, r, s, dist) for r in range(n)])
            for r in range(n):
                cl.fill_synthetic(r, seed, r, s, dist)
            st = cl.ag_step(c, kind)
            agg, counts = f32.ag_step_kind(g_o, res, c, kind, layers, rounds)
            assert np.array_equal(bits(cl.aggregate()), bits(agg)), f"aggregate step {s}"
            for r in range(n):
                assert np.array_equal(bits(cl.residual(r)), bits(res[r])), f"residual r{r} step {s}"
            assert st.k == counts[0]


def test_layerwise_reference_case(fc, f32):
    """tests/test_compress.cpp:73-78 via ag_step at N=1: k=1 in each layer."""
    v = np.array([5.0, 0.1, 0.2, 0.3, 0.01, 9.0, 0.02, 0.03], np.float32)
    with fc.Cluster(1, v.size) as cl:
        cl.set_layer_map([(0, 4), (4, 4)])
        cl.set_grad(0, v)
        st = cl.ag_step(0.25, fc.LAYERWISE)
        assert st.k == 2
        want = np.zeros_like(v)
        want[[0, 5]] = [5.0, 9.0]
        np.testing.assert_array_equal(cl.aggregate(), want)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_layerwise_trajectory(fc, f32, n):
    rng = np.random.default_rng(10 + n)
    g = 60_007
    # a few one- and two-element layers, offsets that are not 4-aligned, a gap
    layers = [(0, 1), (1, 2), (3, 4)] + [(o + 8, m) for o, m in random_layers(rng, g - 8)]
    run_traj(fc, f32, n, g, fc.LAYERWISE, [0.01, 0.1, 0.25, 0.003], layers, dist=n % 3, seed=3 + n)


def test_layerwise_small_and_large_layers(fc, f32):
    """Layers above kSmallLayerMax (49152 elements) go through the segmented EF-emission
    + k_select_x path, the rest through the one-launch small-layer kernel;
    mixed maps (unaligned offsets, a tie-heavy input) stay bit-exact."""
    g = 3_200_003
    layers = [(0, 100), (100, 2_500_000), (2_500_101, 64), (2_500_165, 699_838)]
    run_traj(fc, f32, 2, g, fc.LAYERWISE, [0.01, 0.001, 0.1], layers, dist=1, seed=77, max_cr=0.1)


def test_layerwise_segment_groups(fc, f32, monkeypatch):
    """More large layers than one segmented launch holds (kMaxSegs = 16):
    two EF-emission + select groups; large layers at offsets that are not
    16-byte aligned (staged through scratch), uneven lengths (the block split
    by size), small layers between them; then the same with the sampled
    bound forced to miss (every segment's select falls back)."""
    rng = np.random.default_rng(5)
    layers, off = [], 0
    for q in range(19):
        m = int(rng.integers(1_048_577, 1_600_000)) if q != 7 else 5_000_003
        layers.append((off, m))
        off += m
        if q % 3 == 0:  # a small layer in between (shifts the next offset off 4-alignment)
            layers.append((off, 3 + q))
            off += 3 + q
    run_traj(fc, f32, 1, off, fc.LAYERWISE, [0.01, 0.002], layers, seed=21, max_cr=0.05)
    monkeypatch.setenv("FC_FORCE_FALLBACK", "1")
    run_traj(fc, f32, 1, off, fc.LAYERWISE, [0.01], layers[:9], seed=22, max_cr=0.05)


def test_layerwise_vgg16_map(fc, f32):
    """VGG-16's 32-layer map (13 conv + 3 FC, weights then biases) scaled to
    a ~27M-element gradient (convolutions at full size, FC layers shrunk),
    two workers, two steps."""
    convs = [(3, 64), (64, 64), (64, 128), (128, 128), (128, 256), (256, 256), (256, 256),
             (256, 512), (512, 512), (512, 512), (512, 512), (512, 512), (512, 512)]
    sizes = []
    for cin, cout in convs:
        sizes += [cin * cout * 9, cout]
    for fin, fout in [(2508, 4096), (4096, 409), (4096, 100)]:
        sizes += [fin * fout, fout]
    layers, off = [], 0
    for m in sizes:
        layers.append((off, m))
        off += m
    run_traj(fc, f32, 2, off, fc.LAYERWISE, [0.01, 0.05], layers, seed=16, max_cr=0.1)


def test_layerwise_without_map_is_exact(fc, f32):
    run_traj(fc, f32, 2, 30_011, fc.LAYERWISE, [0.01, 0.05], None, seed=9)


@pytest.mark.parametrize("n,rounds,dist", [(1, 25, 0), (2, 25, 1), (4, 25, 2), (3, 5, 0), (2, 1, 1)])
def test_threshold_trajectory(fc, f32, n, rounds, dist):
    run_traj(fc, f32, n, 50_021, fc.THRESHOLD, [0.01, 0.1, 0.002, 0.05], rounds=rounds, dist=dist,
             seed=20 + n, max_cr=1.0)


def test_threshold_full_ratio_keeps_everything(fc, f32):
    """tests/test_compress.cpp:93-98."""
    g = 97
    v = f32.synth(g, 3, 0, 0)
    with fc.Cluster(1, g) as cl:
        cl.set_grad(0, v)
        st = cl.ag_step(1.0, fc.THRESHOLD)
        assert st.k == g
        np.testing.assert_array_equal(bits(cl.aggregate()), bits(v))


def test_threshold_below_bound_retries(fc, f32):
    """One bisection round keeps everything >= max/2: far more than the
    sampled candidate bound admits, so the selection is redone with every
    element a candidate (still exact)."""
    g = 40_000
    rng = np.random.default_rng(5)
    v = rng.uniform(0.0, 1.0, g).astype(np.float32)
    with fc.Cluster(1, g, max_cr=1.0) as cl:
        cl.set_threshold_rounds(1)
        cl.set_grad(0, v)
        st = cl.ag_step(0.01, fc.THRESHOLD)
        idx, val = f32.topk_kind(v, 0.01, 2, None, 1)
        assert st.k == idx.size
        want = np.zeros(g, np.float32)
        want[idx] = val
        np.testing.assert_array_equal(bits(cl.aggregate()), bits(want))


def test_threshold_capacity_and_argument_errors(fc, f32):
    g = 40_000
    v = np.random.default_rng(6).uniform(0.0, 1.0, g).astype(np.float32)
    with fc.Cluster(1, g, max_cr=0.1) as cl:
        cl.set_threshold_rounds(1)
        cl.set_grad(0, v)
        with pytest.raises(fc.InvalidArgument):  # ~50 % of g > max_cr capacity
            cl.ag_step(0.01, fc.THRESHOLD)
        with pytest.raises(fc.InvalidArgument):
            cl.set_threshold_rounds(0)  # compress.hpp:84
        with pytest.raises(fc.InvalidArgument):
            cl.set_layer_map([(0, 10), (5, 10)])  # overlapping
        with pytest.raises(fc.OutOfRange):
            cl.set_layer_map([(0, g + 1)])
        with pytest.raises(fc.InvalidArgument):
            cl.set_layer_map([(0, 0)])


@pytest.mark.parametrize("kind", ["lw", "thr"])
def test_nccl_world1(fc, f32, kind):
    g = 33_333
    layers = [(0, 1000), (1001, 7), (1010, 32_000)] if kind == "lw" else None
    run_traj(fc, f32, 1, g, fc.LAYERWISE if kind == "lw" else fc.THRESHOLD, [0.01, 0.2, 0.001],
             layers, seed=7, max_cr=1.0, nccl=True)
