"""MOO controller on the device path: SyncTrainer gains vs the
oracle, checkpoint-restore exploration over device residuals, and the
reference's Controller tests (tests/test_moo.cpp:115-169) on the GPU."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2312_02493_b200 import moo
from paper_2312_02493_b200.flexcomm import Collective, NetParams

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def trainer(fc, n, g, **kw):
    sched = kw.pop("sched", None) or moo.NetworkSchedule.constant(NetParams(1e-5, 3.6e12))
    cl = fc.Cluster(n, g)
    cfg = moo.SyncConfig(**kw)
    return cl, moo.SyncTrainer(cl, cfg, sched)


@pytest.mark.parametrize("mode", [moo.SyncMode.STAR, moo.SyncMode.VAR, moo.SyncMode.AG])
def test_step_gain_matches_oracle(fc, f32, mode):
    """Gain = the reference Trainer's (inc/trainer.hpp:361-398) on the fp32
    trajectory: AR mean clamp((|g_e|^2 - |res'|^2)/|g_e|^2, 0, 1), AG mean
    |g_c|^2/|g_e|^2; rank-ordered mean, 1e-6 relative (the reference form
    cancels; the device computes the kept mass directly)."""
    n, g, c = 3, 120_000, 0.01
    cl, t = trainer(fc, n, g, c=c, mode=mode, seed=9)
    res = np.zeros((n, g), dtype=np.float32)
    with cl:
        for s in range(3):
            m = t.step()
            g_o = np.stack([f32.synth(g, 9, r, s) for r in range(n)])
            g_e = (g_o + res).astype(np.float64)
            ge2 = (g_e * g_e).sum(axis=1)
            if mode == moo.SyncMode.AG:
                kept = np.array([(f32.topk_exact((g_o + res)[r], c)[1].astype(np.float64) ** 2).sum()
                                 for r in range(n)])
                f32.ag_step(g_o, res, c)
                want = float(np.mean(kept / ge2))
            else:
                f32.artopk_step(g_o, res, c, fc.VAR if mode == moo.SyncMode.VAR else fc.STAR, s)
                r2 = (res.astype(np.float64) ** 2).sum(axis=1)
                want = float(np.mean(np.clip((ge2 - r2) / ge2, 0.0, 1.0)))
            assert m.gain == pytest.approx(want, rel=1e-6)
            assert m.t_comp_decomp > 0.0 and m.t_sync >= 0.0
            assert 0.0 < m.gain <= 1.0


def test_explore_restores_trajectory(fc):
    """tests/test_moo.cpp:115-135: explore leaves the trajectory untouched."""
    n, g = 2, 100_000
    cl, t = trainer(fc, n, g, adaptive=True, c=0.01, steps_per_epoch=4, epochs=2)
    with cl:
        t.step()
        before = [bits(cl.residual(r)).copy() for r in range(n)]
        step_before = t.step_index
        ctl = moo.Controller(moo.ControllerConfig(probe_iters=3))
        ctl.explore(t, NetParams(1e-5, 3.6e12))
        for r in range(n):
            assert np.array_equal(bits(cl.residual(r)), before[r])
        assert t.step_index == step_before
        assert not t.probe_mode()
        assert t.clock.of(moo.Category.EXPLORATION) > 0.0
        assert len(ctl.candidates) == len(moo.candidate_ladder(ctl.config()))
        for cnd in ctl.candidates:
            assert 0.0 < cnd.gain_avg <= 1.0
            assert cnd.t_comp_avg > 0.0
        # larger ratios keep more of the error-fed gradient
        gains = [cnd.gain_avg for cnd in ctl.candidates]
        assert gains == sorted(gains, reverse=True)


def test_explore_is_transparent_to_the_trajectory(fc):
    """Steps after an exploration are bit-identical to steps without one."""
    n, g = 2, 150_000

    def run(with_explore):
        cl, t = trainer(fc, n, g, adaptive=True, c=0.01)
        out = []
        with cl:
            t.set_compression(0.0111, Collective.ART_RING)
            for s in range(4):
                if with_explore and s == 2:
                    moo.Controller(moo.ControllerConfig(probe_iters=2)).explore(
                        t, NetParams(1e-5, 3.6e12))
                t.step()
                out.append(bits(cl.aggregate()).copy())
            out += [bits(cl.residual(r)).copy() for r in range(n)]
        return out

    for a, b in zip(run(False), run(True)):
        assert np.array_equal(a, b)


def test_hook_selects_on_first_step_and_on_network_change(fc):
    """tests/test_moo.cpp:137-169 on the device path."""
    sched = moo.NetworkSchedule([moo.Segment(0, NetParams(0.001, 25e9)),
                                 moo.Segment(1, NetParams(0.001, 1e9))])
    cl, t = trainer(fc, 2, 80_000, sched=sched, adaptive=True, steps_per_epoch=4, epochs=2,
                    size_bytes_override=4e7)
    with cl:
        ctl = moo.Controller()
        t.run(ctl.hook())
        net_events = [e for e in ctl.events if e.trigger == "network"]
        assert len(net_events) == 1
        assert net_events[0].step == 4
        assert 0.001 <= net_events[0].chosen_c <= 0.1
        assert net_events[0].front_size >= 1
        assert len(t.metrics) == 8
        assert t.current_c() == net_events[0].chosen_c
        # the steps after the event ran at the chosen ratio
        assert all(m.cr_used == net_events[0].chosen_c for m in t.metrics[4:])


def test_nccl_world1_metrics_match_loopback(fc):
    g = 60_000
    uid = fc.get_unique_id()
    vals = []
    for cl in (fc.Cluster(1, g), fc.Cluster.nccl(1, 0, uid, g)):
        with cl:
            t = moo.SyncTrainer(cl, moo.SyncConfig(c=0.01, seed=4),
                                moo.NetworkSchedule.constant(NetParams(1e-5, 3.6e12)))
            vals.append([t.step().gain for _ in range(3)])
    # same selection; the fp64 kept-mass partial sums run in different kernels
    assert vals[0] == pytest.approx(vals[1], rel=1e-12)


def test_degenerate_gradient_raises(fc):
    cl, t = trainer(fc, 2, 4096, c=0.01)
    with cl:
        t.grad_source = lambda tr, s: [cl.set_grad(w, np.zeros(4096, np.float32))
                                       for w in range(cl.n_local)]
        with pytest.raises(fc.RuntimeFailure):
            t.step()
