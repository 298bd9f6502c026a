"""Python host mirror of the reference's hot-path API over the C-ABI.

The reference (arXiv 2312.02493 "flexcomm", /root/reference/proj/include/
flexcomm) is header-only C++; this module keeps its vocabulary and error
behaviour for Python callers (tests, bench.py, the NCCL bootstrap):

=====================  =============================================  ===========================
reference              here                                           reference location
=====================  =============================================  ===========================
CompressionRatio       ``check_cr`` (ValueError ~ invalid_argument)   inc/compress.hpp:15-24
k_of                   ``k_of``                                       inc/compress.hpp:28-33
select_star            ``select_star``                                inc/artopk.hpp:27-30
SelectionMode          ``STAR`` / ``VAR``                             inc/artopk.hpp:13
ReduceOp / ReduceAlgo  ``SUM``/``AVG``, ``RING``/``TREE``             inc/collectives.hpp:35-36
artopk_step            ``Cluster.artopk_step``                        inc/artopk.hpp:62-111
ag_step                ``Cluster.ag_step``                            inc/artopk.hpp:128-161
topk_exact             ``Cluster.topk_exact``                         inc/compress.hpp:57-65
ResidualStore          ``Cluster.residual`` / ``set_residual``        inc/core.hpp:84-95
NetParams/MessageSpec  ``NetParams`` / ``MessageSpec``                inc/costmodel.hpp:12-40
select_collective      ``select_collective``                          inc/costmodel.hpp:153-167
crossover_cr           ``crossover_cr``                               inc/costmodel.hpp:180-203
=====================  =============================================  ===========================

Every call goes to the CUDA library; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi
from ._abi import check, lib

STAR, VAR = _abi.FC_STAR, _abi.FC_VAR
RING, TREE = _abi.FC_RING, _abi.FC_TREE
SUM, AVG = _abi.FC_SUM, _abi.FC_AVG
DIST_NORMAL, DIST_TIES, DIST_LAYERED = _abi.FC_DIST_NORMAL, _abi.FC_DIST_TIES, _abi.FC_DIST_LAYERED
EXACT, LAYERWISE, THRESHOLD = _abi.FC_EXACT, _abi.FC_LAYERWISE, _abi.FC_THRESHOLD  # inc/artopk.hpp:113

InvalidArgument = _abi.InvalidArgument
OutOfRange = _abi.OutOfRange
RuntimeFailure = _abi.RuntimeFailure
NoDevice = _abi.NoDevice


class Collective(enum.IntEnum):
    """inc/costmodel.hpp:111"""

    AG = 0
    ART_RING = 1
    ART_TREE = 2


def check_cr(c: float) -> float:
    """CompressionRatio validation, inc/compress.hpp:18-22."""
    if not (c > 0.0 and c <= 1.0):
        raise InvalidArgument("compression ratio must be in (0, 1]")
    return float(c)


def k_of(c: float, grad_len: int) -> int:
    """inc/compress.hpp:28-33 (computed by the C library, same double formula)."""
    out = C.c_uint64()
    check(lib.fc_k_of(float(c), int(grad_len), C.byref(out)))
    return out.value


def select_star(step: int, n: int) -> int:
    """inc/artopk.hpp:27-30 (C semantics of % for negative steps)."""
    out = C.c_int()
    check(lib.fc_select_star(int(step), int(n), C.byref(out)))
    return out.value


def get_unique_id() -> bytes:
    buf = C.create_string_buffer(_abi.FC_NCCL_UID_BYTES)
    check(lib.fc_get_unique_id(buf))
    return buf.raw


@dataclass
class StepStats:
    selected_rank: int
    collective: int
    k: int
    ms_total: float
    ms_ef: float
    ms_select: float
    ms_exchange: float
    ms_decode: float
    hbm_bytes: float
    bus_bytes: float
    launches: int
    fallback: int

    @classmethod
    def of(cls, s: _abi.fc_step_stats) -> "StepStats":
        return cls(**{n: getattr(s, n) for n, _ in s._fields_})


@dataclass
class WorkerStats:
    ge_norm2: float
    kept_norm2: float
    topk_norm2: float
    threshold_key: int
    candidates: int
    count_above: int
    fallback: int


def _ptr(a) -> int:
    """Data pointer + memkind of a numpy array or torch tensor."""
    try:
        import torch  # noqa: F401

        if hasattr(a, "data_ptr"):
            return a.data_ptr(), (_abi.FC_DEVICE if a.is_cuda else _abi.FC_HOST)
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(a)
    return arr.ctypes.data, _abi.FC_HOST


class Cluster:
    """N data-parallel workers behind one C-ABI context.

    ``Cluster(n, G)`` is the loopback form: all N logical workers live on one
    GPU and the collectives are in-HBM, rank-ascending (the reference's
    in-process ``Cluster``, inc/collectives.hpp:15-33).
    ``Cluster.nccl(world, rank, uid, G)`` is the one-process-per-GPU form.
    """

    def __init__(self, n: int, grad_len: int, device: int = 0, max_cr: float = 1.0,
                 flags: int = 0, *, _world: Optional[int] = None, _rank: int = 0,
                 _uid: Optional[bytes] = None, _peer_only: bool = False):
        opts = _abi.fc_opts()
        opts.device = device
        opts.n_local = n
        opts.world = _world if _world is not None else n
        opts.rank = _rank
        self._uid_buf = C.create_string_buffer(_uid, _abi.FC_NCCL_UID_BYTES) if _uid else None
        opts.nccl_uid = C.cast(self._uid_buf, C.c_void_p) if _uid else None
        opts.grad_len = grad_len
        opts.max_cr = max_cr
        opts.flags = flags
        self._ctx = C.c_void_p()
        check(lib.fc_create(C.byref(self._ctx), C.byref(opts)))
        nl, w, r = C.c_int(), C.c_int(), C.c_int()
        check(lib.fc_num_workers(self._ctx, C.byref(nl), C.byref(w), C.byref(r)))
        self.n_local, self.world, self.rank = nl.value, w.value, r.value
        self.grad_len = int(grad_len)

    @classmethod
    def nccl(cls, world: int, rank: int, uid: bytes, grad_len: int, device: int = 0,
             max_cr: float = 1.0, flags: int = 0) -> "Cluster":
        return cls(1, grad_len, device, max_cr, flags, _world=world, _rank=rank, _uid=uid)

    @classmethod
    def peer_only(cls, world: int, rank: int, grad_len: int, allgather, device: int = 0,
                  max_cr: float = 1.0, flags: int = 0) -> "Cluster":
        """One worker per process over NVLink peer memory without NCCL
        (FC_FLAG_PEER_ONLY; several ranks may share a GPU).  `allgather(bytes)`
        returns every rank's bytes in rank order (e.g. over a gloo group)."""
        cl = cls(1, grad_len, device, max_cr, flags | _abi.FC_FLAG_PEER_ONLY, _world=world, _rank=rank,
                 _uid=None, _peer_only=True)
        h = (C.c_ubyte * _abi.FC_PEER_HANDLE_BYTES)()
        check(lib.fc_peer_handle(cl._ctx, h))
        parts = allgather(bytes(h))
        allh = (C.c_ubyte * (_abi.FC_PEER_HANDLE_BYTES * world)).from_buffer_copy(b"".join(parts))
        check(lib.fc_peer_attach(cl._ctx, allh))
        return cl

    # ---- lifetime ----------------------------------------------------------
    def close(self) -> None:
        if self._ctx:
            lib.fc_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        return self.world

    # ---- state I/O -----------------------------------------------------------
    def set_grad(self, worker: int, g, async_: bool = False) -> None:
        """Upload a worker's gradient.  async_=True (pinned host memory only)
        queues the copy on the upload engine and returns at once."""
        a = self._f32(g)
        p, kind = _ptr(a)
        if async_ and kind == _abi.FC_HOST:
            kind = _abi.FC_HOST_ASYNC
        check(lib.fc_set_grad(self._ctx, worker, p, kind))

    def set_grads(self, grads) -> None:
        if len(grads) != self.n_local:
            raise InvalidArgument("gradient count != worker count")
        for r, g in enumerate(grads):
            self.set_grad(r, g)

    def fill_synthetic(self, worker: int, seed: int, rank: int, step: int,
                       dist: int = DIST_NORMAL) -> None:
        check(lib.fc_fill_synthetic(self._ctx, worker, seed, rank, step, dist))

    def grad_ptr(self, worker: int = 0) -> int:
        p = C.c_void_p()
        check(lib.fc_grad_ptr(self._ctx, worker, C.byref(p)))
        return p.value

    def residual_ptr(self, worker: int = 0) -> int:
        p = C.c_void_p()
        check(lib.fc_residual_ptr(self._ctx, worker, C.byref(p)))
        return p.value

    def aggregate_ptr(self) -> int:
        p = C.c_void_p()
        check(lib.fc_aggregate_ptr(self._ctx, C.byref(p)))
        return p.value

    def set_residual(self, worker: int, r) -> None:
        a = self._f32(r)
        p, kind = _ptr(a)
        check(lib.fc_set_residual(self._ctx, worker, p, kind))

    def residual(self, worker: int) -> np.ndarray:
        out = np.empty(self.grad_len, dtype=np.float32)
        check(lib.fc_get_residual(self._ctx, worker, out.ctypes.data, _abi.FC_HOST))
        return out

    def reset_residuals(self) -> None:
        check(lib.fc_reset_residuals(self._ctx))

    def aggregate(self, out=None, async_: bool = False) -> np.ndarray:
        """Dense aggregate of the last step.  async_=True (pinned host `out`)
        queues the download; the data is valid after sync()."""
        if out is None:
            out = np.empty(self.grad_len, dtype=np.float32)
        p, kind = _ptr(out)
        if async_ and kind == _abi.FC_HOST:
            kind = _abi.FC_HOST_ASYNC
        check(lib.fc_get_aggregate(self._ctx, p, kind))
        return out

    def join(self) -> None:
        """Order the compute stream after all queued async host copies."""
        check(lib.fc_join(self._ctx))

    def topk(self, worker: int):
        k = C.c_uint64()
        check(lib.fc_get_topk(self._ctx, worker, None, None, C.byref(k)))
        idx = np.empty(k.value, dtype=np.uint32)
        val = np.empty(k.value, dtype=np.float32)
        check(lib.fc_get_topk(self._ctx, worker, idx.ctypes.data, val.ctypes.data, C.byref(k)))
        return idx, val

    def worker_stats(self, worker: int) -> WorkerStats:
        s = _abi.fc_worker_stats()
        check(lib.fc_get_worker_stats(self._ctx, worker, C.byref(s)))
        return WorkerStats(**{n: getattr(s, n) for n, _ in s._fields_})

    def snapshot(self) -> None:
        check(lib.fc_snapshot(self._ctx))

    def restore(self) -> None:
        check(lib.fc_restore(self._ctx))

    def sync(self) -> None:
        check(lib.fc_sync(self._ctx))

    def set_peer_timeout(self, seconds: float) -> None:
        """Peer-exchange waits give up (and the next call raises) after this long."""
        check(lib.fc_set_peer_timeout(self._ctx, float(seconds)))

    @property
    def peer_exchange(self) -> bool:
        """STAR steps exchange through NVLink peer memory (else NCCL)."""
        e = C.c_int()
        check(lib.fc_peer_exchange(self._ctx, C.byref(e)))
        return bool(e.value)

    @property
    def aggregate_in_place(self) -> bool:
        """The last AR-Top-k step updated the aggregate in place (same content
        as a full rewrite; FC_FLAG_DENSE_DECODE forces the rewrite)."""
        e = C.c_int()
        check(lib.fc_aggregate_in_place(self._ctx, C.byref(e)))
        return bool(e.value)

    def moo_metrics(self, st: "StepStats", ag: bool = False) -> tuple[float, float]:
        """(gain, t_comp seconds) of the last step, identical on every rank
        (the Trainer's *_with_gain, inc/trainer.hpp:361-398; t_comp measured)."""
        s = _abi.fc_step_stats()
        for n, _ in s._fields_:
            setattr(s, n, getattr(st, n))
        g, t = C.c_double(), C.c_double()
        check(lib.fc_moo_metrics(self._ctx, int(bool(ag)), C.byref(s), C.byref(g), C.byref(t)))
        return g.value, t.value

    def stream_ptr(self) -> int:
        """cudaStream_t of the context (wrap with torch.cuda.ExternalStream)."""
        p = C.c_void_p()
        check(lib.fc_stream(self._ctx, C.byref(p)))
        return p.value or 0

    def set_ef_timing_period(self, period: int) -> None:
        """Time every period-th EF launch only (fc_set_ef_timing_period)."""
        check(lib.fc_set_ef_timing_period(self._ctx, int(period)))

    def ef_kernel_timing(self, reset: bool = False):
        ms, n = C.c_double(), C.c_uint64()
        check(lib.fc_ef_kernel_timing(self._ctx, C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    # ---- the hot path ----------------------------------------------------------
    def artopk_step(self, c: float, mode: int = STAR, algo: int = RING, step: int = 0,
                    op: int = AVG, stats: bool = True) -> StepStats | None:
        """inc/artopk.hpp:62-111.  Returns step statistics (selected rank etc.)."""
        st = _abi.fc_step_stats() if stats else None
        check(lib.fc_artopk_step(self._ctx, float(c), int(mode), int(algo), int(step), int(op),
                                 C.byref(st) if st is not None else None))
        return StepStats.of(st) if st is not None else None

    def ag_step(self, c: float, compressor: int = _abi.FC_EXACT,
                stats: bool = True) -> StepStats | None:
        """inc/artopk.hpp:128-161."""
        st = _abi.fc_step_stats() if stats else None
        check(lib.fc_ag_step(self._ctx, float(c), int(compressor),
                             C.byref(st) if st is not None else None))
        return StepStats.of(st) if st is not None else None

    def set_layer_map(self, layers) -> None:
        """DenseGrad::layer_map (inc/core.hpp:11-23) as [(offset, length), ...]
        for the Layerwise compressor; [] clears it."""
        n = len(layers)
        off = (C.c_uint64 * max(1, n))(*[o for o, _ in layers])
        ln = (C.c_uint64 * max(1, n))(*[m for _, m in layers])
        check(lib.fc_set_layer_map(self._ctx, off, ln, n))

    def set_threshold_rounds(self, rounds: int) -> None:
        """ag_step's threshold_rounds (inc/artopk.hpp:131)."""
        check(lib.fc_set_threshold_rounds(self._ctx, int(rounds)))

    def dense_step(self, algo: int = RING, op: int = AVG, stats: bool = True) -> StepStats | None:
        """Dense allreduce baseline, inc/trainer.hpp:240-244."""
        st = _abi.fc_step_stats() if stats else None
        check(lib.fc_dense_step(self._ctx, int(algo), int(op),
                                C.byref(st) if st is not None else None))
        return StepStats.of(st) if st is not None else None

    def topk_exact(self, worker: int, c: float):
        """inc/compress.hpp:57-65 on the worker's gradient buffer."""
        st = _abi.fc_step_stats()
        check(lib.fc_topk_exact(self._ctx, worker, float(c), C.byref(st)))
        return self.topk(worker)

    @staticmethod
    def _f32(a):
        if hasattr(a, "data_ptr"):
            import torch

            if a.dtype != torch.float32 or not a.is_contiguous():
                raise InvalidArgument("expected a contiguous float32 tensor")
            return a
        return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- cost model --

@dataclass(frozen=True)
class NetParams:
    """inc/costmodel.hpp:12-27 (alpha seconds, bandwidth bits/s)."""

    alpha: float = 0.0
    bandwidth: float = 1e9

    def __post_init__(self):
        if self.alpha < 0.0:
            raise InvalidArgument("alpha must be >= 0")
        if not self.bandwidth > 0.0:
            raise InvalidArgument("bandwidth must be > 0")

    def beta(self) -> float:
        return 8.0 / self.bandwidth


@dataclass(frozen=True)
class MessageSpec:
    """inc/costmodel.hpp:29-40."""

    m_bytes: float = 4.0
    c: float = 1.0
    n: int = 1

    def __post_init__(self):
        if self.m_bytes < 4.0:
            raise InvalidArgument("message must be >= 4 bytes")
        if not (self.c > 0.0 and self.c <= 1.0):
            raise InvalidArgument("compression ratio out of (0,1]")
        if self.n < 1:
            raise InvalidArgument("worker count must be >= 1")


COST_FIELDS = ("ps", "ring_ar", "tree_ar", "broadcast", "allgather_dense", "ag_compressed",
               "art_ring", "art_tree")


@dataclass
class CollectiveChoice:
    collective: Collective
    costs: dict = field(default_factory=dict)


def cost_primitives(net: NetParams, msg: MessageSpec) -> dict:
    out = (C.c_double * 8)()
    check(lib.fc_cost_primitives(net.alpha, net.bandwidth, msg.m_bytes, msg.c, msg.n, out))
    return dict(zip(COST_FIELDS, list(out)))


def select_collective(net: NetParams, msg: MessageSpec) -> CollectiveChoice:
    if msg.n < 2:
        raise InvalidArgument("selection undefined for single worker")
    ch = C.c_int()
    out = (C.c_double * 8)()
    check(lib.fc_select_collective(net.alpha, net.bandwidth, msg.m_bytes, msg.c, msg.n,
                                   C.byref(ch), out))
    return CollectiveChoice(Collective(ch.value), dict(zip(COST_FIELDS, list(out))))


def prefer(net: NetParams, msg: MessageSpec, which: int) -> bool:
    out = C.c_int()
    check(lib.fc_prefer(net.alpha, net.bandwidth, msg.m_bytes, msg.c, msg.n, which, C.byref(out)))
    return bool(out.value)


def crossover_cr(net: NetParams, m_bytes: float, n: int, pair: int) -> Optional[float]:
    if n < 2:
        raise InvalidArgument("selection undefined for single worker")
    c, has = C.c_double(), C.c_int()
    check(lib.fc_crossover_cr(net.alpha, net.bandwidth, m_bytes, n, pair, C.byref(c), C.byref(has)))
    return c.value if has.value else None


def derive_m_from_ag(net: NetParams, c: float, n: int, seconds: float) -> float:
    out = C.c_double()
    check(lib.fc_derive_m_from_ag(net.alpha, net.bandwidth, c, n, seconds, C.byref(out)))
    return out.value


__all__ = [
    "STAR", "VAR", "RING", "TREE", "SUM", "AVG", "Collective", "Cluster", "StepStats",
    "WorkerStats", "k_of", "select_star", "check_cr", "get_unique_id", "NetParams",
    "MessageSpec", "cost_primitives", "select_collective", "prefer", "crossover_cr",
    "derive_m_from_ag", "InvalidArgument", "OutOfRange", "RuntimeFailure", "NoDevice",
    "DIST_NORMAL", "DIST_TIES", "DIST_LAYERED", "EXACT", "LAYERWISE", "THRESHOLD",
]
