"""Adaptive-CR controller on CPU: the decision functions
bit-exact against the unmodified reference (golden vectors from
tests/golden/make_golden.py and the live reference library), the reference's
own tests/test_moo.cpp cases restated, and the Controller state machine
driven by a scripted host trainer."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2312_02493_b200 import moo
from paper_2312_02493_b200.flexcomm import (Collective, InvalidArgument, MessageSpec, NetParams,
                                            RuntimeFailure, select_collective)


def cand(c, t_comp, t_sync, inv_gain):
    return moo.CandidateCR(c, 1.0 / inv_gain, t_comp, t_sync)


# ---- tests/test_moo.cpp restated --------------------------------------------------

def test_ladder_default_rungs():  # test_moo.cpp:29-33
    assert moo.candidate_ladder(moo.ControllerConfig()) == [0.1, 0.0333, 0.0111, 0.0037, 0.001]


def test_ladder_factor_ten_and_degenerate():  # test_moo.cpp:35-46
    cfg = moo.ControllerConfig(factor=10.0)
    assert moo.candidate_ladder(cfg) == [0.1, 0.01, 0.001]
    cfg.c_low = cfg.c_high = 0.05
    assert moo.candidate_ladder(cfg) == [0.05]
    cfg.c_low = 0.2
    with pytest.raises(InvalidArgument):
        moo.candidate_ladder(cfg)
    with pytest.raises(InvalidArgument):
        moo.candidate_ladder(moo.ControllerConfig(factor=1.0))
    for bad in (dict(probe_iters=0), dict(gain_threshold=-0.1), dict(c_low=0.0)):
        with pytest.raises(InvalidArgument):
            moo.Controller(moo.ControllerConfig(**bad))


def test_round_3sig():  # test_moo.cpp:48-54
    assert moo.round_3sig(0.0333333) == pytest.approx(0.0333, rel=1e-15)
    assert moo.round_3sig(0.0111111) == pytest.approx(0.0111, rel=1e-15)
    assert moo.round_3sig(0.00370370) == pytest.approx(0.0037, rel=1e-15)
    assert moo.round_3sig(123456.0) == 123000.0
    assert moo.round_3sig(0.0) == 0.0


def test_trigger_gain():  # test_moo.cpp:56-69
    t = moo.GainTracker(10)
    t.push(0.7)
    t.push(0.7)
    assert moo.trigger_gain(0.8, t, 0.10)
    u = moo.GainTracker(10)
    u.push(0.75)
    u.push(0.75)
    assert not moo.trigger_gain(0.8, u, 0.10)
    v = moo.GainTracker(10)
    v.push(0.1)
    assert not moo.trigger_gain(0.8, v, 0.10)
    assert not moo.trigger_gain(-1.0, t, 0.10)
    with pytest.raises(InvalidArgument):
        moo.GainTracker(0)


def test_pareto_front_matches_brute_force():  # test_moo.cpp:71-95
    rng = np.random.default_rng(61)
    for _ in range(100):
        cands = [cand(0.01 * (i + 1), *rng.uniform(0.1, 10.0, 3)) for i in range(12)]
        front = moo.pareto_front(cands)
        assert front
        for f in front:
            for o in cands:
                better = (o.t_comp_avg <= f.t_comp_avg and o.t_sync_modeled <= f.t_sync_modeled
                          and 1 / o.gain_avg <= 1 / f.gain_avg
                          and (o.t_comp_avg < f.t_comp_avg or o.t_sync_modeled < f.t_sync_modeled
                               or 1 / o.gain_avg < 1 / f.gain_avg))
                assert not better
    with pytest.raises(InvalidArgument):
        moo.pareto_front([])


def test_knee_picks_balanced_candidate():  # test_moo.cpp:97-106
    front = [cand(0.1, 1.0, 9.0, 9.0), cand(0.01, 5.0, 5.0, 5.0), cand(0.001, 9.0, 9.0, 1.0)]
    net = NetParams(0.001, 10e9)
    ch = moo.choose_cr(front, net, 4e7, 8)
    assert ch.candidate.c == 0.01
    assert ch.collective == select_collective(net, MessageSpec(4e7, 0.01, 8)).collective


def test_knee_ties_go_to_larger_ratio():  # test_moo.cpp:108-113
    front = [cand(0.01, 1.0, 2.0, 2.0), cand(0.1, 2.0, 1.0, 2.0)]
    assert moo.choose_cr(front, NetParams(0.001, 10e9), 4e7, 8).candidate.c == 0.1
    with pytest.raises(InvalidArgument):
        moo.choose_cr([], NetParams(0.001, 10e9), 4e7, 8)


# ---- bit-exact against the reference (golden vectors + live library) ----------------

def test_golden_ladders(golden):
    for case in golden["moo"]["ladder"]:
        cfg = moo.ControllerConfig(case["c_low"], case["c_high"], case["factor"])
        assert moo.candidate_ladder(cfg) == case["ladder"]


def test_golden_round_3sig(golden):
    for v, want in golden["moo"]["round_3sig"]:
        assert moo.round_3sig(v) == want, v


def test_golden_knee(golden):
    for case in golden["moo"]["knee"]:
        cands = [moo.CandidateCR(*r) for r in case["rows"]]
        front = moo.pareto_front(cands)
        mask = [int(any(f is c for f in front)) for c in cands]
        assert mask == case["mask"]
        ch = moo.choose_cr(front, NetParams(case["alpha"], case["bw"]), case["m"], case["n"])
        assert ch.candidate.c == case["chosen"]
        assert int(ch.collective) == case["collective"]


def test_golden_trigger_and_network(golden):
    for case in golden["moo"]["trigger"]:
        t = moo.GainTracker(case["window"])
        for s in case["samples"]:
            t.push(s)
        assert moo.trigger_gain(case["gain_ref"], t, case["threshold"]) == case["fire"]
    for case in golden["moo"]["network"]:
        got = moo.network_changed(NetParams(case["a0"], case["b0"]), NetParams(case["a1"], case["b1"]),
                                  case["rel"])
        assert got == case["changed"]


def test_live_reference_random(ref):
    rng = np.random.default_rng(5)
    for _ in range(2000):
        m = int(rng.integers(1, 12))
        # small integer grids force exact objective ties and dominance corner cases
        grid = rng.random() < 0.5
        rows = np.empty((m, 4))
        rows[:, 0] = rng.choice([0.1, 0.0333, 0.0111, 0.0037, 0.001, 0.5], m)
        rows[:, 1] = (rng.integers(1, 4, m) / 4.0) if grid else rng.uniform(0.01, 1.0, m)
        rows[:, 2] = (rng.integers(0, 3, m) * 1e-3) if grid else 10 ** rng.uniform(-6, 0, m)
        rows[:, 3] = (rng.integers(0, 3, m) * 1e-3) if grid else 10 ** rng.uniform(-6, 0, m)
        alpha, bw = float(rng.uniform(0, 0.01)), float(10 ** rng.uniform(8, 13))
        mb, n = float(10 ** rng.uniform(3, 10)), int(rng.integers(2, 300))
        mask, chosen, coll = ref.choose_cr(rows, alpha, bw, mb, n)
        cands = [moo.CandidateCR(*map(float, r)) for r in rows]
        front = moo.pareto_front(cands)
        assert [any(f is c for f in front) for c in cands] == list(mask)
        ch = moo.choose_cr(front, NetParams(alpha, bw), mb, n)
        assert (ch.candidate.c, int(ch.collective)) == (chosen, coll)
    for _ in range(2000):
        v = float(10 ** rng.uniform(-300, 300)) * float(rng.choice([-1, 1]))
        assert moo.round_3sig(v) == ref.round_3sig(v)
        f = float(rng.uniform(1.001, 20))
        lo = float(10 ** rng.uniform(-6, 0))
        hi = float(min(1.0, lo * 10 ** rng.uniform(0, 4)))
        assert moo.candidate_ladder(moo.ControllerConfig(lo, hi, f)) == ref.candidate_ladder(lo, hi, f)


def test_params_at_matches_reference(ref):
    segs = [moo.Segment(0, NetParams(0.001, 25e9)), moo.Segment(2, NetParams(0.002, 1e9)),
            moo.Segment(5, NetParams(0.0, 3e9))]
    sched = moo.NetworkSchedule(segs)
    rows = [[s.start_epoch, s.net.alpha, s.net.bandwidth] for s in segs]
    for e in range(8):
        p = moo.params_at(sched, e)
        assert (p.alpha, p.bandwidth) == ref.params_at(rows, e)
    with pytest.raises(InvalidArgument):
        moo.params_at(sched, -1)
    with pytest.raises(InvalidArgument):
        moo.params_at(moo.NetworkSchedule([moo.Segment(1, NetParams())]), 0)


# ---- Controller state machine over a scripted trainer ---------------------------------

class ScriptedTrainer:
    """Host stand-in exposing exactly what Controller reads from the Trainer
    (inc/moo.hpp:167-263).  Gains/times are deterministic in (c, step)."""

    def __init__(self, n=4, steps_per_epoch=5, epochs=3, sched=None, gain_fn=None,
                 fail_c=(), window=50):
        self.n = n
        self.cfg = moo.SyncConfig(epochs=epochs, steps_per_epoch=steps_per_epoch, adaptive=True)
        self.sched = sched or moo.NetworkSchedule.constant(NetParams(1e-5, 400e9 * 8))
        self.gain_fn = gain_fn or (lambda c, s: 0.2 + 0.8 * c ** 0.25)
        self.fail_c = set(fail_c)
        self.window = window
        self.step_index = 0
        self._c, self._coll = 1.0, Collective.ART_RING
        self._tracker = moo.GainTracker(window)
        self._probe = False
        self.state = 0.0  # stands for the residual trajectory
        self.calls = []

    def m_eff(self):
        return 4.0 * 1e8

    def gain_tracker(self):
        return self._tracker

    def current_c(self):
        return self._c

    def current_collective(self):
        return self._coll

    def set_compression(self, c, coll):
        if c != self._c:
            self._tracker = moo.GainTracker(self.window)
        self._c, self._coll = c, coll

    def set_probe_mode(self, on):
        self._probe = on

    def snapshot(self):
        return (self.state, self.step_index, self._c, self._coll, list(self._tracker.samples))

    def restore(self, s):
        self.state, self.step_index, self._c, self._coll, samples = s
        self._tracker = moo.GainTracker(self.window)
        for x in samples:
            self._tracker.push(x)

    def step(self):
        self.calls.append((self.step_index, self._c, self._probe))
        if self._c in self.fail_c:
            raise RuntimeFailure("degenerate gradient")
        g = self.gain_fn(self._c, self.step_index)
        self._tracker.push(g)
        self.state = self.state * 0.5 + self._c
        m = moo.StepMetrics(step=self.step_index, gain=g, t_comp_decomp=1e-4 * (1 + 0.1 / self._c))
        self.step_index += 1
        return m

    def run(self, hook):
        while self.step_index < self.cfg.epochs * self.cfg.steps_per_epoch:
            e = self.step_index // self.cfg.steps_per_epoch
            hook(self, self.step_index, e, moo.params_at(self.sched, e))
            self.step()


def test_explore_restores_and_probes_every_rung():
    t = ScriptedTrainer()
    t.step()
    before = t.snapshot()
    ctl = moo.Controller()
    ctl.explore(t, NetParams(1e-5, 3.2e12))
    assert t.snapshot() == before and not t._probe
    ladder = moo.candidate_ladder(ctl.cfg)
    assert [c.c for c in ctl.candidates] == ladder
    probes = [c for c in t.calls if c[2]]
    assert len(probes) == len(ladder) * ctl.cfg.probe_iters
    assert all(s == 1 for s, _, _ in probes[:: ctl.cfg.probe_iters])  # each rung from the snapshot
    for cc in ctl.candidates:  # averages in the reference's summation order
        gs = ts = 0.0
        for i in range(ctl.cfg.probe_iters):
            gs += t.gain_fn(cc.c, 1 + i)
            ts += 1e-4 * (1 + 0.1 / cc.c)
        assert cc.gain_avg == gs / ctl.cfg.probe_iters and cc.t_comp_avg == ts / ctl.cfg.probe_iters


def test_divergent_probe_discarded_and_all_diverged_raises():
    t = ScriptedTrainer(fail_c={0.0037})
    ctl = moo.Controller()
    ctl.explore(t, NetParams(1e-5, 3.2e12))
    assert [c.c for c in ctl.candidates] == [0.1, 0.0333, 0.0111, 0.001]
    t2 = ScriptedTrainer(fail_c=set(moo.candidate_ladder(ctl.cfg)))
    with pytest.raises(RuntimeFailure):
        moo.Controller().explore(t2, NetParams(1e-5, 3.2e12))


def test_hook_selects_on_first_step_and_on_network_change(ref):
    # test_moo.cpp:137-169 with the scripted trainer: silent init, one event
    # at the epoch-1 network change, choice = the reference's choose_cr
    sched = moo.NetworkSchedule([moo.Segment(0, NetParams(0.001, 25e9)),
                                 moo.Segment(1, NetParams(0.001, 1e9))])
    t = ScriptedTrainer(sched=sched, gain_fn=lambda c, s: 0.3 + 0.7 * c ** 0.3)
    ctl = moo.Controller()
    t.run(ctl.hook())
    net_events = [e for e in ctl.events if e.trigger == "network"]
    assert len(net_events) == 1 and net_events[0].step == t.cfg.steps_per_epoch
    assert 0.001 <= net_events[0].chosen_c <= 0.1 and net_events[0].front_size >= 1
    rows = np.array([[c.c, c.gain_avg, c.t_comp_avg, c.t_sync_modeled] for c in ctl.candidates])
    _, chosen, coll = ref.choose_cr(rows, 0.001, 1e9, t.m_eff(), t.n)
    assert (net_events[0].chosen_c, int(net_events[0].collective)) == (chosen, coll)
    assert t.current_c() == chosen


def test_gain_trigger_reexplores():
    # gains drop by 30 % from step 7 on: the tracker mean leaves the 10 % band
    t = ScriptedTrainer(steps_per_epoch=20, epochs=1,
                        gain_fn=lambda c, s: (0.5 if s < 7 else 0.35) + 0.0 * c)
    ctl = moo.Controller()
    t.run(ctl.hook())
    gain_events = [e for e in ctl.events if e.trigger == "gain"]
    assert gain_events, ctl.events
    first = gain_events[0]
    # the trigger needs >= 2 samples after the first selection and a relative drift >= 10 %
    assert first.step >= 8
    assert all(e.chosen_c in moo.candidate_ladder(ctl.cfg) for e in ctl.events)


def test_refresh_sync_uses_selected_collective_cost():
    t = ScriptedTrainer()
    ctl = moo.Controller()
    net = NetParams(2e-5, 5e11)
    ctl.explore(t, net)
    ctl.refresh_sync(t, net)
    for c in ctl.candidates:
        ch = select_collective(net, MessageSpec(t.m_eff(), c.c, t.n))
        key = {Collective.AG: "ag_compressed", Collective.ART_RING: "art_ring",
               Collective.ART_TREE: "art_tree"}[ch.collective]
        assert c.t_sync_modeled == ch.costs[key]
        assert math.isfinite(c.t_sync_modeled)
