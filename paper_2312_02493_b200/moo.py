"""Adaptive compression-ratio controller over the B200 sync path.

Host mirror of the reference's MOO controller (inc/moo.hpp) and of the parts
of its Trainer the controller drives (inc/trainer.hpp:102-413), re-based on
the device path:

==========================  ===========================================  =========================
reference                   here                                         reference location
==========================  ===========================================  =========================
ControllerConfig            ``ControllerConfig``                         inc/moo.hpp:27-42
round_3sig                  ``round_3sig`` (C-ABI fc_round_3sig)         inc/moo.hpp:44-48
candidate_ladder            ``candidate_ladder``                         inc/moo.hpp:52-65
trigger_gain                ``trigger_gain``                             inc/moo.hpp:67-71
pareto_front / choose_cr    ``pareto_front`` / ``choose_cr``             inc/moo.hpp:88-146
Controller                  ``Controller``                               inc/moo.hpp:159-271
GainTracker                 ``GainTracker``                              inc/compress.hpp:145-165
NetworkSchedule, params_at  ``NetworkSchedule``, ``params_at``           inc/netsched.hpp:13-46
network_changed             ``network_changed``                          inc/netsched.hpp:50-58
Trainer (sync side)         ``SyncTrainer``                              inc/trainer.hpp:102-413
==========================  ===========================================  =========================

The decision arithmetic (ladder, dominance, knee, trigger, network change)
runs in the CUDA library's host code (csrc/fc_moo.cpp) so Python and C++
callers take identical decisions, bit-exact with the reference
(tests/test_moo.py).  What changes is the trainer underneath:

* the trajectory is the device residual store: ``SyncTrainer.snapshot`` /
  ``restore`` copy it in HBM (fc_snapshot / fc_restore) instead of copying
  model replicas on the host (inc/trainer.hpp:160-190);
* a candidate's compression time is MEASURED on the device — CUDA-event time
  of error feedback + Top-k + decode (max over ranks) — replacing the
  0.5 ns/element model (inc/trainer.hpp:344-359);
* the gain is the reference's (AR: mean clamp(kept/‖g_e‖², 0, 1); AG: mean
  ‖g_c‖²/‖g_e‖²), averaged over all ranks in rank order (fc_moo_metrics);
* gradients come from a caller-supplied source (default: the counter-based
  synthetic generator keyed by (seed, rank, step), include/fc_synth.h); the
  reference's toy model and SGD update are out of scope.
"""
from __future__ import annotations

import copy
import ctypes as C
import enum
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Optional

from . import _abi
from ._abi import check, lib
from .flexcomm import (AVG, DIST_NORMAL, RING, STAR, TREE, VAR, Cluster, Collective,
                       InvalidArgument, MessageSpec, NetParams, RuntimeFailure,
                       select_collective)

DeviceFailure = _abi.DeviceFailure


# ------------------------------------------------------------ configuration --

@dataclass
class ControllerConfig:
    """inc/moo.hpp:27-42."""

    c_low: float = 0.001
    c_high: float = 0.1
    factor: float = 3.0
    probe_iters: int = 10
    gain_threshold: float = 0.10

    def _c(self) -> _abi.fc_controller_config:
        return _abi.fc_controller_config(self.c_low, self.c_high, self.factor,
                                         self.probe_iters, self.gain_threshold)

    def validate(self) -> None:
        if lib.fc_controller_config_validate(C.byref(self._c())) != _abi.FC_OK:
            raise InvalidArgument("invalid controller config (need 0 < c_low <= c_high <= 1, "
                                  "factor > 1, probe_iters >= 1, gain_threshold >= 0)")


def round_3sig(v: float) -> float:
    out = C.c_double()
    check(lib.fc_round_3sig(float(v), C.byref(out)))
    return out.value


def candidate_ladder(cfg: ControllerConfig) -> list[float]:
    cfg.validate()
    n = C.c_int()
    check(lib.fc_candidate_ladder(C.byref(cfg._c()), None, 0, C.byref(n)))
    buf = (C.c_double * n.value)()
    check(lib.fc_candidate_ladder(C.byref(cfg._c()), buf, n.value, C.byref(n)))
    return list(buf)


class GainTracker:
    """Rolling window of per-step gains, inc/compress.hpp:145-165."""

    def __init__(self, window: int = 50):
        if window <= 0:
            raise InvalidArgument("window must be positive")
        self.window = int(window)
        self.samples: deque[float] = deque()

    def push(self, gain: float) -> None:
        self.samples.append(float(gain))
        if len(self.samples) > self.window:
            self.samples.popleft()

    def count(self) -> int:
        return len(self.samples)

    def mean(self) -> float:
        if not self.samples:
            raise RuntimeFailure("no gain samples")
        s = 0.0
        for v in self.samples:  # sequential, like std::accumulate (not math.fsum / sum())
            s += v
        return s / len(self.samples)


def trigger_gain(gain_ref: float, tracker: GainTracker, threshold: float) -> bool:
    buf = (C.c_double * max(1, tracker.count()))(*tracker.samples)
    out = C.c_int()
    check(lib.fc_trigger_gain(float(gain_ref), buf, tracker.count(), float(threshold),
                              C.byref(out)))
    return bool(out.value)


@dataclass
class CandidateCR:
    """inc/moo.hpp:20-25 (times in seconds)."""

    c: float = 1.0
    gain_avg: float = 1.0
    t_comp_avg: float = 0.0
    t_sync_modeled: float = 0.0


def _cands(cands: list[CandidateCR]):
    arr = (_abi.fc_candidate * len(cands))()
    for i, c in enumerate(cands):
        arr[i] = _abi.fc_candidate(c.c, c.gain_avg, c.t_comp_avg, c.t_sync_modeled)
    return arr


def pareto_front(cands: list[CandidateCR]) -> list[CandidateCR]:
    if not cands:
        raise InvalidArgument("empty candidate set")
    mask = (C.c_int * len(cands))()
    check(lib.fc_pareto_front(_cands(cands), len(cands), mask))
    return [c for c, m in zip(cands, mask) if m]


@dataclass
class CrChoice:
    candidate: CandidateCR
    collective: Collective = Collective.AG


def choose_cr(front: list[CandidateCR], net: NetParams, m_bytes: float, n: int) -> CrChoice:
    if not front:
        raise InvalidArgument("empty pareto front")
    MessageSpec(m_bytes, 1.0, n)  # the reference's MessageSpec validation
    if n < 2:
        raise InvalidArgument("selection undefined for single worker")
    chosen, coll = C.c_int(), C.c_int()
    check(lib.fc_choose_cr(_cands(front), len(front), net.alpha, net.bandwidth, float(m_bytes),
                           int(n), C.byref(chosen), C.byref(coll)))
    return CrChoice(front[chosen.value], Collective(coll.value))


# ------------------------------------------------------------------ network --

@dataclass
class Segment:
    start_epoch: int
    net: NetParams


@dataclass
class NetworkSchedule:
    """Piecewise-constant NetParams over epochs, inc/netsched.hpp:13-36."""

    segments: list[Segment] = field(default_factory=list)

    def validate(self) -> None:
        if not self.segments:
            raise InvalidArgument("empty network schedule")
        if self.segments[0].start_epoch != 0:
            raise InvalidArgument("first segment must start at epoch 0")
        for a, b in zip(self.segments, self.segments[1:]):
            if b.start_epoch <= a.start_epoch:
                raise InvalidArgument("segment start epochs must be strictly ascending")

    @classmethod
    def constant(cls, net: NetParams) -> "NetworkSchedule":
        return cls([Segment(0, net)])


def params_at(sched: NetworkSchedule, epoch: int) -> NetParams:
    """inc/netsched.hpp:38-46."""
    if epoch < 0:
        raise InvalidArgument("epoch must be >= 0")
    sched.validate()
    cur = sched.segments[0].net
    for seg in sched.segments:
        if seg.start_epoch <= epoch:
            cur = seg.net
    return cur


def network_changed(prev: NetParams, cur: NetParams, rel_threshold: float = 0.0) -> bool:
    out = C.c_int()
    check(lib.fc_network_changed(prev.alpha, prev.bandwidth, cur.alpha, cur.bandwidth,
                                 float(rel_threshold), C.byref(out)))
    return bool(out.value)


# ------------------------------------------------------------------ trainer --

class Category(enum.IntEnum):
    """inc/netsched.hpp:60."""

    COMPUTE = 0
    SYNC = 1
    COMPRESSION = 2
    IO = 3
    EXPLORATION = 4


class SimClock:
    """Per-category accumulated seconds (inc/netsched.hpp:60-90)."""

    def __init__(self):
        self.acc = [0.0] * 5

    def charge(self, cat: Category, seconds: float) -> None:
        if seconds < 0.0:
            raise InvalidArgument("negative duration")
        self.acc[int(cat)] += seconds

    def of(self, cat: Category) -> float:
        return self.acc[int(cat)]

    def now(self) -> float:
        return sum(self.acc)


class SyncMode(enum.Enum):
    """inc/trainer.hpp:25."""

    DENSE = "DENSE"
    AG = "AG"
    STAR = "STAR"
    VAR = "VAR"


@dataclass
class SyncConfig:
    """The TrainConfig fields the sync path and the controller read
    (inc/trainer.hpp:40-82); model/data/optimizer fields are out of scope."""

    epochs: int = 5
    steps_per_epoch: int = 10
    c: float = 1.0
    adaptive: bool = False
    mode: SyncMode = SyncMode.STAR
    reduce_algo: int = RING
    reduce_op: int = AVG
    error_feedback: bool = True
    gain_window: int = 50
    size_bytes_override: float = 0.0
    net_change_threshold: float = 0.0
    t_compute: float = 0.0  # seconds charged per step for the (external) backward pass
    t_io: float = 0.0
    seed: int = 42
    dist: int = DIST_NORMAL

    def validate(self) -> None:
        if self.epochs < 1:
            raise InvalidArgument("epochs must be >= 1")
        if self.steps_per_epoch < 1:
            raise InvalidArgument("steps_per_epoch must be >= 1")
        if not (self.c > 0.0 and self.c <= 1.0):
            raise InvalidArgument("compression ratio out of (0,1]")
        if self.t_io < 0.0 or self.t_compute < 0.0:
            raise InvalidArgument("t_io / t_compute must be >= 0")
        if self.gain_window <= 0:
            raise InvalidArgument("window must be positive")


@dataclass
class StepMetrics:
    """inc/trainer.hpp:84-96 (loss is the model's, out of scope)."""

    step: int = 0
    t_compute: float = 0.0
    t_comp_decomp: float = 0.0
    t_sync: float = 0.0
    t_io: float = 0.0
    t_step: float = 0.0
    gain: float = 1.0
    cr_used: float = 1.0
    collective_used: str = ""
    selected_rank: int = -1


@dataclass
class Snapshot:
    """Host half of Trainer::Snapshot (inc/trainer.hpp:161-172); the residual
    store half lives in HBM (fc_snapshot).  `generation` ties the two."""

    generation: int
    tracker: GainTracker
    step_index: int
    current_c: float
    current_collective: Collective


GradSource = Callable[["SyncTrainer", int], None]


def synthetic_source(trainer: "SyncTrainer", step: int) -> None:
    """Default gradient source: the counter-based N(0,1) generator keyed by
    (seed, global rank, step), filled on the device."""
    cl = trainer.cluster
    for w in range(cl.n_local):
        cl.fill_synthetic(w, trainer.cfg.seed, cl.rank + w, step, trainer.cfg.dist)


class SyncTrainer:
    """The reference Trainer's synchronisation side on the device path.

    ``step()`` fills this step's gradients (``grad_source``), runs the sync
    the current (c, collective) calls for — dense allreduce, AG-Top-k or
    AR-Top-k with STAR/VAR selection on the Ring/Tree communicator — and
    returns StepMetrics with the measured compression and exchange times.
    Works on loopback and NCCL clusters alike; under NCCL every rank must
    call it in lockstep (the metrics are rank-identical).
    """

    def __init__(self, cluster: Cluster, cfg: SyncConfig, sched: NetworkSchedule,
                 grad_source: GradSource = synthetic_source):
        cfg.validate()
        sched.validate()
        self.cluster = cluster
        self.cfg = cfg
        self.sched = sched
        self.grad_source = grad_source
        self.clock = SimClock()
        self._tracker = GainTracker(cfg.gain_window)
        self.step_index = 0
        self._c = cfg.c
        self._coll = self._initial_collective()
        self._probe = False
        self._gen = 0
        self.metrics: list[StepMetrics] = []
        self.selection_log: list[tuple[int, int]] = []

    # -- reference accessors (inc/trainer.hpp:124-158) -----------------------
    @property
    def n(self) -> int:
        return self.cluster.world

    def total_steps(self) -> int:
        return self.cfg.epochs * self.cfg.steps_per_epoch

    def epoch_of(self, step: int) -> int:
        return step // self.cfg.steps_per_epoch

    def net_at_step(self, step: int) -> NetParams:
        return params_at(self.sched, self.epoch_of(step))

    def m_eff(self) -> float:
        return (self.cfg.size_bytes_override if self.cfg.size_bytes_override > 0.0
                else 4.0 * self.cluster.grad_len)

    def gain_tracker(self) -> GainTracker:
        return self._tracker

    def current_c(self) -> float:
        return self._c

    def current_collective(self) -> Collective:
        return self._coll

    def set_compression(self, c: float, collective: Collective) -> None:
        if not (c > 0.0 and c <= 1.0):
            raise InvalidArgument("compression ratio out of (0,1]")
        if c != self._c:
            self._tracker = GainTracker(self.cfg.gain_window)
        self._c = c
        self._coll = Collective(collective)

    def probe_mode(self) -> bool:
        return self._probe

    def set_probe_mode(self, on: bool) -> None:
        self._probe = bool(on)

    # -- checkpoint / restore (inc/trainer.hpp:160-190) ------------------------
    def snapshot(self) -> Snapshot:
        self.cluster.snapshot()
        self._gen += 1
        return Snapshot(self._gen, copy.deepcopy(self._tracker), self.step_index, self._c,
                        self._coll)

    def restore(self, s: Snapshot) -> None:
        if s.generation != self._gen:
            raise RuntimeFailure("restore of a superseded snapshot (one device snapshot slot)")
        self.cluster.restore()
        self._tracker = copy.deepcopy(s.tracker)
        self.step_index = s.step_index
        self._c = s.current_c
        self._coll = s.current_collective

    # -- one synchronous step (inc/trainer.hpp:193-277) --------------------------
    def _initial_collective(self) -> Collective:
        if self.cfg.mode == SyncMode.AG:
            return Collective.AG
        return Collective.ART_RING if self.cfg.reduce_algo == RING else Collective.ART_TREE

    def _effective_mode(self) -> SyncMode:
        if not self.cfg.adaptive:
            return self.cfg.mode
        if self._coll == Collective.AG:
            return SyncMode.AG
        return SyncMode.VAR if self.cfg.mode == SyncMode.VAR else SyncMode.STAR

    def _effective_c(self) -> float:
        return self._c if self.cfg.adaptive else self.cfg.c

    def _charge(self, cat: Category, seconds: float) -> None:
        self.clock.charge(Category.EXPLORATION if self._probe else cat, seconds)

    def step(self) -> StepMetrics:
        cl = self.cluster
        m = StepMetrics(step=self.step_index, cr_used=self._effective_c(), t_io=self.cfg.t_io,
                        t_compute=self.cfg.t_compute)
        self.grad_source(self, self.step_index)
        mode = self._effective_mode()
        c = self._effective_c()
        if mode == SyncMode.DENSE:
            st = cl.dense_step(self.cfg.reduce_algo, self.cfg.reduce_op)
            gain, t_comp = 1.0, 0.0
            m.collective_used = "RING_AR" if self.cfg.reduce_algo == RING else "TREE_AR"
        elif mode == SyncMode.AG:
            st = cl.ag_step(c)
            gain, t_comp = cl.moo_metrics(st, ag=True)
            m.collective_used = "AG"
        else:
            sel = VAR if mode == SyncMode.VAR else STAR
            algo = TREE if self._coll == Collective.ART_TREE else self.cfg.reduce_algo
            if self._coll == Collective.ART_RING:
                algo = RING
            st = cl.artopk_step(c, sel, algo, self.step_index, self.cfg.reduce_op)
            gain, t_comp = cl.moo_metrics(st, ag=False)
            m.selected_rank = st.selected_rank
            m.collective_used = "ART_RING" if algo == RING else "ART_TREE"
            if not self._probe:
                self.selection_log.append((self.step_index, st.selected_rank))
        m.t_sync = st.ms_exchange * 1e-3
        m.gain = gain
        self._tracker.push(gain)
        m.t_comp_decomp = t_comp
        self._charge(Category.SYNC, m.t_sync)
        self._charge(Category.COMPRESSION, m.t_comp_decomp)
        self._charge(Category.COMPUTE, m.t_compute)
        self._charge(Category.IO, m.t_io)
        m.t_step = m.t_compute + m.t_sync + m.t_io + m.t_comp_decomp
        if not self.cfg.error_feedback:
            cl.reset_residuals()
        self.step_index += 1
        return m

    def run(self, hook: Optional[Callable[["SyncTrainer", int, int, NetParams], None]] = None):
        """inc/trainer.hpp:283-289: the hook runs before each step."""
        total = self.total_steps()
        while self.step_index < total:
            if hook:
                hook(self, self.step_index, self.epoch_of(self.step_index),
                     self.net_at_step(self.step_index))
            self.metrics.append(self.step())


# --------------------------------------------------------------- controller --

@dataclass
class ControllerEvent:
    """inc/moo.hpp:148-154."""

    step: int
    trigger: str  # "gain" or "network"
    chosen_c: float
    collective: Collective
    front_size: int


class Controller:
    """Adaptive-CR controller, inc/moo.hpp:159-271 (same state machine)."""

    def __init__(self, cfg: Optional[ControllerConfig] = None):
        self.cfg = cfg if cfg is not None else ControllerConfig()
        self.cfg.validate()
        self.candidates: list[CandidateCR] = []
        self.events: list[ControllerEvent] = []
        self._gain_ref = -1.0
        self._prev_net = NetParams()
        self._initialized = False

    def config(self) -> ControllerConfig:
        return self.cfg

    def on_step(self, trainer, step: int, epoch: int, net: NetParams) -> None:
        if not self._initialized:
            self.explore(trainer, net)
            self.refresh_sync(trainer, net)
            self._apply_selection(trainer, net)
            self._gain_ref = self._gain_of(trainer.current_c())
            self._prev_net = net
            self._initialized = True
            return
        if trigger_gain(self._gain_ref, trainer.gain_tracker(), self.cfg.gain_threshold):
            self.explore(trainer, net)
            self.refresh_sync(trainer, net)
            self._gain_ref = self._gain_of(trainer.current_c())
            self.events.append(ControllerEvent(step, "gain", trainer.current_c(),
                                               trainer.current_collective(),
                                               len(pareto_front(self.candidates))))
        if network_changed(self._prev_net, net, trainer.cfg.net_change_threshold):
            self.refresh_sync(trainer, net)
            chosen = self._apply_selection(trainer, net)
            self._gain_ref = chosen.candidate.gain_avg
            self.events.append(ControllerEvent(step, "network", chosen.candidate.c,
                                               chosen.collective,
                                               len(pareto_front(self.candidates))))
        self._prev_net = net

    def hook(self):
        return lambda t, step, epoch, net: self.on_step(t, step, epoch, net)

    def explore(self, trainer, net: NetParams) -> None:
        """Probe every rung for probe_iters steps from one snapshot; restore
        the pre-probe trajectory afterwards (inc/moo.hpp:204-236)."""
        snap = trainer.snapshot()
        trainer.set_probe_mode(True)
        fresh: list[CandidateCR] = []
        n = trainer.n
        for c in candidate_ladder(self.cfg):
            trainer.restore(snap)
            coll = (select_collective(net, MessageSpec(trainer.m_eff(), c, n)).collective
                    if n >= 2 else Collective.ART_RING)
            trainer.set_compression(c, coll)
            gain_sum = comp_sum = 0.0
            ok = True
            for _ in range(self.cfg.probe_iters):
                try:
                    mt = trainer.step()
                except DeviceFailure:
                    raise
                except RuntimeFailure:
                    ok = False  # divergent probe: candidate discarded
                    break
                gain_sum += mt.gain
                comp_sum += mt.t_comp_decomp
            if ok:
                fresh.append(CandidateCR(c, gain_sum / self.cfg.probe_iters,
                                         comp_sum / self.cfg.probe_iters, 0.0))
        trainer.restore(snap)
        trainer.set_probe_mode(False)
        if not fresh:
            raise RuntimeFailure("all exploration candidates diverged")
        self.candidates = fresh

    def refresh_sync(self, trainer, net: NetParams) -> None:
        for cand in self.candidates:
            ch = select_collective(net, MessageSpec(trainer.m_eff(), cand.c, trainer.n))
            cand.t_sync_modeled = {Collective.AG: ch.costs["ag_compressed"],
                                   Collective.ART_RING: ch.costs["art_ring"],
                                   Collective.ART_TREE: ch.costs["art_tree"]}[ch.collective]

    def _apply_selection(self, trainer, net: NetParams) -> CrChoice:
        front = pareto_front(self.candidates)
        chosen = choose_cr(front, net, trainer.m_eff(), trainer.n)
        trainer.set_compression(chosen.candidate.c, chosen.collective)
        return chosen

    def _gain_of(self, c: float) -> float:
        for cand in self.candidates:
            if cand.c == c:
                return cand.gain_avg
        return -1.0


__all__ = [
    "ControllerConfig", "round_3sig", "candidate_ladder", "GainTracker", "trigger_gain",
    "CandidateCR", "pareto_front", "CrChoice", "choose_cr", "Segment", "NetworkSchedule",
    "params_at", "network_changed", "Category", "SimClock", "SyncMode", "SyncConfig",
    "StepMetrics", "Snapshot", "SyncTrainer", "synthetic_source", "ControllerEvent",
    "Controller",
]
