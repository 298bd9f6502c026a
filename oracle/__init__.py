"""ORACLE — test infrastructure only.

Python access to the CPU checkers:
  * ``F32``  — liboracle_f32.so, the fp32 restatement of the reference hot path
  * ``Ref``  — _ref/libflexcomm_ref.so, the UNMODIFIED reference headers
               (/root/reference/proj/include) behind a C shim

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg may import this package, and only as the checker / the timed CPU
baseline.  The product path (``paper_2312_02493_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
F32_LIB = HERE / "liboracle_f32.so"
REF_LIB = HERE / "_ref" / "libflexcomm_ref.so"
REF_INCLUDE = Path("/root/reference/proj/include")


def build() -> None:
    """Compile the restatement and, when /root/reference exists, the reference shim."""
    res = subprocess.run(["make", "-s", "-C", str(HERE)], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + res.stdout + res.stderr)


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _u32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _f64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class F32:
    """fp32 restatement (oracle/oracle_f32.cpp)."""

    def __init__(self):
        if not F32_LIB.exists():
            build()
        lib = C.CDLL(str(F32_LIB))
        u64, d, i, P = C.c_uint64, C.c_double, C.c_int, C.c_void_p
        lib.orc_k_of.argtypes, lib.orc_k_of.restype = [d, u64], u64
        lib.orc_topk_exact.argtypes, lib.orc_topk_exact.restype = [P, u64, d, P, P], u64
        lib.orc_squared_norm.argtypes, lib.orc_squared_norm.restype = [P, u64], d
        lib.orc_artopk_step.argtypes = [i, u64, P, P, d, i, C.c_long, i, P, P, P, P]
        lib.orc_artopk_step.restype = u64
        lib.orc_ag_step.argtypes, lib.orc_ag_step.restype = [i, u64, P, P, d, P], u64
        lib.orc_dense.argtypes, lib.orc_dense.restype = [i, u64, P, i, P], None
        lib.orc_fill_synth.argtypes, lib.orc_fill_synth.restype = [P, u64, u64, C.c_uint32, u64, i], None
        lib.orc_topk_kind.argtypes = [P, u64, d, i, i, P, P, i, P, P]
        lib.orc_topk_kind.restype = u64
        lib.orc_ag_step_kind.argtypes = [i, u64, P, P, d, i, i, P, P, i, P, P]
        lib.orc_ag_step_kind.restype = u64
        lib.orc_topk_multi.argtypes, lib.orc_topk_multi.restype = [P, u64, P, i, P], i
        self.lib = lib

    def k_of(self, c, g):
        return int(self.lib.orc_k_of(c, g))

    def topk_multi(self, v, crs):
        """topk_exact index sets of one vector at several ratios (one key array)."""
        v = np.ascontiguousarray(v, dtype=np.float32)
        outs = [np.empty(self.k_of(c, v.size), dtype=np.uint32) for c in crs]
        ptrs = (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
        cs = np.asarray(crs, dtype=np.float64)
        if self.lib.orc_topk_multi(v.ctypes.data, v.size, cs.ctypes.data, len(outs), ptrs):
            raise ValueError("bad topk_multi arguments")
        return outs

    def synth(self, g, seed, rank, step, dist=0):
        out = np.empty(g, dtype=np.float32)
        self.lib.orc_fill_synth(out.ctypes.data, g, seed, rank, step, dist)
        return out

    def topk_exact(self, v, c):
        v = np.ascontiguousarray(v, dtype=np.float32)
        k = self.k_of(c, v.size)
        idx = np.empty(k, dtype=np.uint32)
        val = np.empty(k, dtype=np.float32)
        self.lib.orc_topk_exact(v.ctypes.data, v.size, c, idx.ctypes.data, val.ctypes.data)
        return idx, val

    def squared_norm(self, v):
        v = np.ascontiguousarray(v, dtype=np.float32)
        return float(self.lib.orc_squared_norm(v.ctypes.data, v.size))

    def artopk_step(self, g_o, res, c, mode, step, op=1):
        """g_o, res: (n, G) float32; res is updated in place."""
        n, g = g_o.shape
        g_o = np.ascontiguousarray(g_o, dtype=np.float32)
        assert res.dtype == np.float32 and res.flags.c_contiguous
        k = self.k_of(c, g)
        agg = np.empty(g, dtype=np.float32)
        sel = C.c_int()
        bidx = np.empty(k, dtype=np.uint32)
        norms = np.empty(n, dtype=np.float64)
        r = self.lib.orc_artopk_step(n, g, g_o.ctypes.data, res.ctypes.data, c, mode, step, op,
                                     agg.ctypes.data, C.addressof(sel), bidx.ctypes.data,
                                     norms.ctypes.data)
        if r == 0:
            raise ValueError("oracle rejected arguments")
        return agg, sel.value, bidx, norms

    def ag_step(self, g_o, res, c):
        n, g = g_o.shape
        g_o = np.ascontiguousarray(g_o, dtype=np.float32)
        agg = np.empty(g, dtype=np.float32)
        if self.lib.orc_ag_step(n, g, g_o.ctypes.data, res.ctypes.data, c, agg.ctypes.data) == 0:
            raise ValueError("oracle rejected arguments")
        return agg

    @staticmethod
    def _layers(layers):
        if not layers:
            return 0, None, None, None
        off = np.ascontiguousarray([o for o, _ in layers], dtype=np.uint64)
        ln = np.ascontiguousarray([n for _, n in layers], dtype=np.uint64)
        return len(layers), off, ln, (off, ln)

    def topk_kind(self, v, c, kind, layers=None, rounds=25):
        """kind 0 exact, 1 layerwise (layers = [(offset, length)]), 2 threshold."""
        v = np.ascontiguousarray(v, dtype=np.float32)
        nl, off, ln, _keep = self._layers(layers)
        idx = np.empty(v.size, dtype=np.uint32)
        val = np.empty(v.size, dtype=np.float32)
        m = self.lib.orc_topk_kind(v.ctypes.data, v.size, c, kind, nl,
                                   off.ctypes.data if nl else None, ln.ctypes.data if nl else None,
                                   rounds, idx.ctypes.data, val.ctypes.data)
        return idx[:m].copy(), val[:m].copy()

    def ag_step_kind(self, g_o, res, c, kind, layers=None, rounds=25):
        n, g = g_o.shape
        g_o = np.ascontiguousarray(g_o, dtype=np.float32)
        nl, off, ln, _keep = self._layers(layers)
        agg = np.empty(g, dtype=np.float32)
        counts = np.empty(n, dtype=np.uint64)
        self.lib.orc_ag_step_kind(n, g, g_o.ctypes.data, res.ctypes.data, c, kind, nl,
                                  off.ctypes.data if nl else None, ln.ctypes.data if nl else None,
                                  rounds, agg.ctypes.data, counts.ctypes.data)
        return agg, counts

    def dense(self, g_o, op=1):
        n, g = g_o.shape
        g_o = np.ascontiguousarray(g_o, dtype=np.float32)
        agg = np.empty(g, dtype=np.float32)
        self.lib.orc_dense(n, g, g_o.ctypes.data, op, agg.ctypes.data)
        return agg


def host_isa() -> str:
    """Highest x86-64 micro-architecture level this host's CPU supports
    ("x86-64-v4" AVX-512, "x86-64-v3" AVX2/FMA/BMI2, else "x86-64-v2")."""
    try:
        flags = set()
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("flags"):
                flags = set(line.split(":", 1)[1].split())
                break
    except OSError:
        return "x86-64-v2"
    v3 = {"avx", "avx2", "bmi1", "bmi2", "f16c", "fma", "movbe", "xsave"} <= flags and (
        "abm" in flags or "lzcnt" in flags)
    v4 = v3 and {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags
    return "x86-64-v4" if v4 else "x86-64-v3" if v3 else "x86-64-v2"


def ref_lib_for(isa: str) -> Path:
    return {"x86-64-v4": HERE / "_ref" / "libflexcomm_ref_v4.so",
            "x86-64-v3": HERE / "_ref" / "libflexcomm_ref_v3.so"}.get(isa, REF_LIB)


class Ref:
    """The unmodified reference (oracle/_ref/libflexcomm_ref*.so), fp64.

    isa=None loads the portable x86-64-v2 build; isa="native" the highest
    level this host supports (bench.py's reference arm)."""

    def __init__(self, isa: str | None = None):
        if not REF_LIB.exists():
            if REF_INCLUDE.exists():
                build()
            if not REF_LIB.exists():
                raise FileNotFoundError(f"{REF_LIB} not built (needs /root/reference once)")
        self.isa = "x86-64-v2"
        path = REF_LIB
        if isa == "native":
            want = host_isa()
            if ref_lib_for(want).exists():
                self.isa, path = want, ref_lib_for(want)
        lib = C.CDLL(str(path))
        u64, d, i, P, L = C.c_uint64, C.c_double, C.c_int, C.c_void_p, C.c_long
        lib.ref_k_of.argtypes, lib.ref_k_of.restype = [d, u64, P], i
        lib.ref_topk_exact.argtypes, lib.ref_topk_exact.restype = [P, u64, d, P, P, P], i
        lib.ref_artopk_step.argtypes = [i, u64, P, P, d, i, i, L, i, d, d, d, P, P, P]
        lib.ref_artopk_step.restype = i
        lib.ref_ag_step.argtypes = [i, u64, P, P, d, d, d, d, P, P]
        lib.ref_ag_step.restype = i
        lib.ref_select_collective.argtypes = [d, d, d, d, i, P, P]
        lib.ref_select_collective.restype = i
        lib.ref_crossover_cr.argtypes, lib.ref_crossover_cr.restype = [d, d, d, i, i, P, P], i
        lib.ref_candidate_ladder.argtypes, lib.ref_candidate_ladder.restype = [d, d, d, P, i], i
        lib.ref_choose_cr.argtypes = [P, i, d, d, d, i, P, P, P]
        lib.ref_choose_cr.restype = i
        lib.ref_round_3sig.argtypes, lib.ref_round_3sig.restype = [d], d
        lib.ref_trigger_gain.argtypes, lib.ref_trigger_gain.restype = [d, P, u64, u64, d], i
        lib.ref_network_changed.argtypes, lib.ref_network_changed.restype = [d, d, d, d, d], i
        lib.ref_params_at.argtypes, lib.ref_params_at.restype = [P, i, L, P, P], i
        lib.ref_topk_kind.argtypes = [P, u64, d, i, i, P, P, i, P, P]
        lib.ref_topk_kind.restype = L
        lib.ref_ag_step_kind.argtypes = [i, u64, P, P, d, i, i, P, P, i, P]
        lib.ref_ag_step_kind.restype = i
        lib.ref_state_create.argtypes, lib.ref_state_create.restype = [i, u64], P
        lib.ref_state_destroy.argtypes, lib.ref_state_destroy.restype = [P], None
        lib.ref_state_fill_synth.argtypes = [P, i, u64, C.c_uint32, u64, i]
        lib.ref_state_fill_synth.restype = None
        lib.ref_state_step.argtypes, lib.ref_state_step.restype = [P, d, i, i, L], d
        lib.ref_state_selected.argtypes, lib.ref_state_selected.restype = [P], i
        lib.ref_state_aggregate.argtypes, lib.ref_state_aggregate.restype = [P, P], None
        lib.ref_state_residual.argtypes, lib.ref_state_residual.restype = [P, i, P], None
        self.lib = lib

    def k_of(self, c, g):
        k = C.c_uint64()
        rc = self.lib.ref_k_of(c, g, C.addressof(k))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return k.value

    def topk_exact(self, v, c):
        v = np.ascontiguousarray(v, dtype=np.float64)
        kmax = max(1, v.size)
        idx = np.empty(kmax, dtype=np.uint64)
        val = np.empty(kmax, dtype=np.float64)
        k = C.c_uint64()
        rc = self.lib.ref_topk_exact(v.ctypes.data, v.size, c, idx.ctypes.data, val.ctypes.data,
                                     C.addressof(k))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return idx[: k.value].copy(), val[: k.value].copy()

    def artopk_step(self, g_o, res, c, mode, algo, step, op=1, payload_scale=1.0,
                    alpha=0.001, bandwidth=1e9):
        n, g = g_o.shape
        g_o = np.ascontiguousarray(g_o, dtype=np.float64)
        assert res.dtype == np.float64 and res.flags.c_contiguous
        agg = np.empty(g, dtype=np.float64)
        sel, charge = C.c_int(), C.c_double()
        rc = self.lib.ref_artopk_step(n, g, g_o.ctypes.data, res.ctypes.data, c, mode, algo, step,
                                      op, payload_scale, alpha, bandwidth, agg.ctypes.data,
                                      C.addressof(sel), C.addressof(charge))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return agg, sel.value, charge.value

    def ag_step(self, g_o, res, c, payload_scale=1.0, alpha=0.001, bandwidth=1e9):
        n, g = g_o.shape
        g_o = np.ascontiguousarray(g_o, dtype=np.float64)
        agg = np.empty(g, dtype=np.float64)
        charge = C.c_double()
        rc = self.lib.ref_ag_step(n, g, g_o.ctypes.data, res.ctypes.data, c, payload_scale, alpha,
                                  bandwidth, agg.ctypes.data, C.addressof(charge))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return agg, charge.value

    def select_collective(self, alpha, bandwidth, m_bytes, c, n):
        ch = C.c_int()
        costs = np.empty(8, dtype=np.float64)
        rc = self.lib.ref_select_collective(alpha, bandwidth, m_bytes, c, n, C.addressof(ch),
                                            costs.ctypes.data)
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return ch.value, costs

    def crossover_cr(self, alpha, bandwidth, m_bytes, n, pair):
        c, has = C.c_double(), C.c_int()
        rc = self.lib.ref_crossover_cr(alpha, bandwidth, m_bytes, n, pair, C.addressof(c),
                                       C.addressof(has))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return c.value if has.value else None

    def candidate_ladder(self, c_low=0.001, c_high=0.1, factor=3.0):
        out = np.empty(64, dtype=np.float64)
        m = self.lib.ref_candidate_ladder(c_low, c_high, factor, out.ctypes.data, 64)
        if m > 64:
            out = np.empty(m, dtype=np.float64)
            m = self.lib.ref_candidate_ladder(c_low, c_high, factor, out.ctypes.data, m)
        if m < 0:
            raise ValueError("reference raised")
        return [float(x) for x in out[:m]]

    def choose_cr(self, rows, alpha, bandwidth, m_bytes, n):
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        m = rows.shape[0]
        mask = np.zeros(m, dtype=np.int32)
        chosen, coll = C.c_double(), C.c_int()
        rc = self.lib.ref_choose_cr(rows.ctypes.data, m, alpha, bandwidth, m_bytes, n,
                                    mask.ctypes.data, C.addressof(chosen), C.addressof(coll))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return mask.astype(bool), chosen.value, coll.value

    def round_3sig(self, v):
        return self.lib.ref_round_3sig(v)

    def trigger_gain(self, gain_ref, samples, window, threshold):
        s = np.ascontiguousarray(samples, dtype=np.float64)
        r = self.lib.ref_trigger_gain(gain_ref, s.ctypes.data, s.size, window, threshold)
        if r < 0:
            raise ValueError(f"reference raised (code {-r})")
        return bool(r)

    def network_changed(self, a0, b0, a1, b1, rel):
        return bool(self.lib.ref_network_changed(a0, b0, a1, b1, rel))

    def params_at(self, segments, epoch):
        segs = np.ascontiguousarray(segments, dtype=np.float64).reshape(-1, 3)
        a, b = C.c_double(), C.c_double()
        rc = self.lib.ref_params_at(segs.ctypes.data, segs.shape[0], epoch, C.addressof(a),
                                    C.addressof(b))
        if rc:
            raise ValueError(f"reference raised (code {rc})")
        return a.value, b.value


def _ref_layers(layers):
    if not layers:
        return 0, None, None
    off = np.ascontiguousarray([o for o, _ in layers], dtype=np.uint64)
    ln = np.ascontiguousarray([n for _, n in layers], dtype=np.uint64)
    return len(layers), off, ln


def _ref_topk_kind(self, v, c, kind, layers=None, rounds=25):
    v = np.ascontiguousarray(v, dtype=np.float64)
    nl, off, ln = _ref_layers(layers)
    idx = np.empty(max(1, v.size), dtype=np.uint64)
    val = np.empty(max(1, v.size), dtype=np.float64)
    m = self.lib.ref_topk_kind(v.ctypes.data, v.size, c, kind, nl,
                               off.ctypes.data if nl else None, ln.ctypes.data if nl else None,
                               rounds, idx.ctypes.data, val.ctypes.data)
    if m < 0:
        raise ValueError(f"reference raised (code {-m})")
    return idx[:m].copy(), val[:m].copy()


def _ref_ag_step_kind(self, g_o, res, c, kind, layers=None, rounds=25):
    n, g = g_o.shape
    g_o = np.ascontiguousarray(g_o, dtype=np.float64)
    nl, off, ln = _ref_layers(layers)
    agg = np.empty(g, dtype=np.float64)
    rc = self.lib.ref_ag_step_kind(n, g, g_o.ctypes.data, res.ctypes.data, c, kind, nl,
                                   off.ctypes.data if nl else None, ln.ctypes.data if nl else None,
                                   rounds, agg.ctypes.data)
    if rc:
        raise ValueError(f"reference raised (code {rc})")
    return agg


Ref.topk_kind = _ref_topk_kind
Ref.ag_step_kind = _ref_ag_step_kind


class RefState:
    """Persistent reference state for timing the CPU baseline (bench.py)."""

    def __init__(self, ref: Ref, n: int, g: int):
        self.ref, self.n, self.g = ref, n, g
        self.p = ref.lib.ref_state_create(n, g)
        if not self.p:
            raise MemoryError("reference state allocation failed")

    def fill_synth(self, worker, seed, rank, step, dist=0):
        self.ref.lib.ref_state_fill_synth(self.p, worker, seed, rank, step, dist)

    def step(self, c, mode, algo, step):
        """mode 0 STAR, 1 VAR, 2 AG.  Returns seconds inside the reference call."""
        t = self.ref.lib.ref_state_step(self.p, c, mode, algo, step)
        if t < 0:
            raise RuntimeError("reference step raised")
        return t

    def selected(self):
        return self.ref.lib.ref_state_selected(self.p)

    def aggregate(self):
        out = np.empty(self.g, dtype=np.float64)
        self.ref.lib.ref_state_aggregate(self.p, out.ctypes.data)
        return out

    def residual(self, worker):
        out = np.empty(self.g, dtype=np.float64)
        self.ref.lib.ref_state_residual(self.p, worker, out.ctypes.data)
        return out

    def close(self):
        if self.p:
            self.ref.lib.ref_state_destroy(self.p)
            self.p = None

    def __del__(self):
        self.close()
