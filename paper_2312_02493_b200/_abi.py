"""ctypes binding of the C-ABI in include/flexcomm_b200.h.

Loads the in-tree ``libfc_b200.so``.  There is no fallback: if the library
is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# FC_LIB_PATH: an experimental build of the same library (tools/variants.py)
LIB_PATH = Path(os.environ["FC_LIB_PATH"]) if os.environ.get("FC_LIB_PATH") else _PKG / "libfc_b200.so"

FC_OK = 0
FC_ERR_INVALID_ARGUMENT = 1
FC_ERR_OUT_OF_RANGE = 2
FC_ERR_RUNTIME = 3
FC_ERR_CUDA = 4
FC_ERR_NCCL = 5
FC_ERR_NO_DEVICE = 6

FC_STAR, FC_VAR = 0, 1
FC_RING, FC_TREE = 0, 1
FC_SUM, FC_AVG = 0, 1
FC_EXACT, FC_LAYERWISE, FC_THRESHOLD = 0, 1, 2
FC_HOST, FC_DEVICE, FC_HOST_ASYNC = 0, 1, 2
FC_FLAG_ASYNC = 0x1
FC_FLAG_NO_TIMING = 0x2
FC_FLAG_DENSE_DECODE = 0x4
FC_FLAG_PIPELINE = 0x8
FC_FLAG_NO_COOPERATIVE = 0x10
FC_FLAG_PEER_ONLY = 0x20
FC_PEER_HANDLE_BYTES = 64
FC_NCCL_UID_BYTES = 128
FC_DIST_NORMAL, FC_DIST_TIES, FC_DIST_LAYERED = 0, 1, 2


class fc_opts(C.Structure):
    _fields_ = [
        ("device", C.c_int),
        ("n_local", C.c_int),
        ("world", C.c_int),
        ("rank", C.c_int),
        ("nccl_uid", C.c_void_p),
        ("grad_len", C.c_uint64),
        ("max_cr", C.c_double),
        ("flags", C.c_uint),
    ]


class fc_step_stats(C.Structure):
    _fields_ = [
        ("selected_rank", C.c_int),
        ("collective", C.c_int),
        ("k", C.c_uint64),
        ("ms_total", C.c_float),
        ("ms_ef", C.c_float),
        ("ms_select", C.c_float),
        ("ms_exchange", C.c_float),
        ("ms_decode", C.c_float),
        ("hbm_bytes", C.c_double),
        ("bus_bytes", C.c_double),
        ("launches", C.c_uint64),
        ("fallback", C.c_int),
    ]


class fc_worker_stats(C.Structure):
    _fields_ = [
        ("ge_norm2", C.c_double),
        ("kept_norm2", C.c_double),
        ("topk_norm2", C.c_double),
        ("threshold_key", C.c_uint32),
        ("candidates", C.c_uint64),
        ("count_above", C.c_uint64),
        ("fallback", C.c_int),
    ]


class fc_candidate(C.Structure):
    """CandidateCR, inc/moo.hpp:20-25."""
    _fields_ = [
        ("c", C.c_double),
        ("gain_avg", C.c_double),
        ("t_comp_avg", C.c_double),
        ("t_sync_modeled", C.c_double),
    ]


class fc_controller_config(C.Structure):
    """ControllerConfig, inc/moo.hpp:27-32."""
    _fields_ = [
        ("c_low", C.c_double),
        ("c_high", C.c_double),
        ("factor", C.c_double),
        ("probe_iters", C.c_int),
        ("gain_threshold", C.c_double),
    ]


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)"
        )
    lib = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    i, u64, d, f = C.c_int, C.c_uint64, C.c_double, C.c_float
    sigs = {
        "fc_status_string": ([i], C.c_char_p),
        "fc_last_error": ([], C.c_char_p),
        "fc_abi_version": ([], i),
        "fc_launch_count": ([], u64),
        "fc_k_of": ([d, u64, C.POINTER(u64)], i),
        "fc_select_star": ([C.c_long, i, C.POINTER(i)], i),
        "fc_get_unique_id": ([C.c_char_p], i),
        "fc_create": ([C.POINTER(P), C.POINTER(fc_opts)], i),
        "fc_destroy": ([P], i),
        "fc_num_workers": ([P, C.POINTER(i), C.POINTER(i), C.POINTER(i)], i),
        "fc_set_grad": ([P, i, P, i], i),
        "fc_grad_ptr": ([P, i, C.POINTER(P)], i),
        "fc_fill_synthetic": ([P, i, u64, C.c_uint32, u64, i], i),
        "fc_set_residual": ([P, i, P, i], i),
        "fc_get_residual": ([P, i, P, i], i),
        "fc_residual_ptr": ([P, i, C.POINTER(P)], i),
        "fc_reset_residuals": ([P], i),
        "fc_get_aggregate": ([P, P, i], i),
        "fc_aggregate_ptr": ([P, C.POINTER(P)], i),
        "fc_get_topk": ([P, i, P, P, C.POINTER(u64)], i),
        "fc_get_worker_stats": ([P, i, C.POINTER(fc_worker_stats)], i),
        "fc_snapshot": ([P], i),
        "fc_restore": ([P], i),
        "fc_artopk_step": ([P, d, i, i, C.c_long, i, C.POINTER(fc_step_stats)], i),
        "fc_ag_step": ([P, d, i, C.POINTER(fc_step_stats)], i),
        "fc_set_layer_map": ([P, C.POINTER(u64), C.POINTER(u64), i], i),
        "fc_set_threshold_rounds": ([P, i], i),
        "fc_dense_step": ([P, i, i, C.POINTER(fc_step_stats)], i),
        "fc_topk_exact": ([P, i, d, C.POINTER(fc_step_stats)], i),
        "fc_sync": ([P], i),
        "fc_join": ([P], i),
        "fc_stream": ([P, C.POINTER(P)], i),
        "fc_ef_kernel_timing": ([P, C.POINTER(d), C.POINTER(u64), i], i),
        "fc_set_ef_timing_period": ([P, i], i),
        "fc_diag_kernel_ms": ([P, i, i, C.POINTER(d)], i),
        "fc_diag_select_phases": ([P, i, C.POINTER(u64)], i),
        "fc_diag_collective_ms": ([P, i, u64, i, C.POINTER(d)], i),
        "fc_diag_ef_blocks": ([P, i, C.POINTER(u64), i], i),
        # host cost model (csrc/fc_costmodel.cpp)
        "fc_cost_primitives": ([d, d, d, d, i, C.POINTER(d)], i),
        "fc_select_collective": ([d, d, d, d, i, C.POINTER(i), C.POINTER(d)], i),
        "fc_prefer": ([d, d, d, d, i, i, C.POINTER(i)], i),
        "fc_crossover_cr": ([d, d, d, i, i, C.POINTER(d), C.POINTER(i)], i),
        "fc_derive_m_from_ag": ([d, d, d, i, d, C.POINTER(d)], i),
        # adaptive-CR controller (csrc/fc_moo.cpp, fc_ctx.cu)
        "fc_controller_config_validate": ([C.POINTER(fc_controller_config)], i),
        "fc_round_3sig": ([d, C.POINTER(d)], i),
        "fc_candidate_ladder": ([C.POINTER(fc_controller_config), C.POINTER(d), i, C.POINTER(i)], i),
        "fc_trigger_gain": ([d, C.POINTER(d), u64, d, C.POINTER(i)], i),
        "fc_pareto_front": ([C.POINTER(fc_candidate), i, C.POINTER(i)], i),
        "fc_choose_cr": ([C.POINTER(fc_candidate), i, d, d, d, i, C.POINTER(i), C.POINTER(i)], i),
        "fc_network_changed": ([d, d, d, d, d, C.POINTER(i)], i),
        "fc_moo_metrics": ([P, i, C.POINTER(fc_step_stats), C.POINTER(d), C.POINTER(d)], i),
        "fc_peer_exchange": ([P, C.POINTER(i)], i),
        "fc_aggregate_in_place": ([P, C.POINTER(i)], i),
        "fc_diag_seg_phases": ([P, i, C.POINTER(u64), i, C.POINTER(i)], i),
        "fc_set_peer_timeout": ([P, d], i),
        "fc_diag_exchange_ms": ([P, i, u64, i, C.POINTER(d)], i),
        "fc_set_grad_f64": ([P, i, P], i),
        "fc_set_residual_f64": ([P, i, P], i),
        "fc_get_residual_f64": ([P, i, P], i),
        "fc_get_aggregate_f64": ([P, P], i),
        "fc_peer_handle": ([P, P], i),
        "fc_peer_attach": ([P, P], i),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()

# Exported symbols the header declares (checked by tests/test_abi.py).
EXPORTS = [
    "fc_status_string", "fc_last_error", "fc_abi_version", "fc_launch_count", "fc_k_of",
    "fc_select_star", "fc_get_unique_id", "fc_create", "fc_destroy", "fc_num_workers",
    "fc_set_grad", "fc_grad_ptr", "fc_fill_synthetic", "fc_set_residual", "fc_get_residual",
    "fc_residual_ptr", "fc_reset_residuals", "fc_get_aggregate", "fc_aggregate_ptr",
    "fc_get_topk", "fc_get_worker_stats", "fc_snapshot", "fc_restore", "fc_artopk_step",
    "fc_ag_step", "fc_set_layer_map", "fc_set_threshold_rounds", "fc_dense_step", "fc_topk_exact", "fc_sync", "fc_join", "fc_stream", "fc_ef_kernel_timing", "fc_set_ef_timing_period",
    "fc_diag_kernel_ms", "fc_diag_select_phases", "fc_diag_collective_ms", "fc_diag_ef_blocks",
    "fc_cost_primitives", "fc_select_collective", "fc_prefer", "fc_crossover_cr",
    "fc_derive_m_from_ag",
    "fc_controller_config_validate", "fc_round_3sig", "fc_candidate_ladder", "fc_trigger_gain",
    "fc_pareto_front", "fc_choose_cr", "fc_network_changed", "fc_moo_metrics", "fc_peer_exchange",
    "fc_aggregate_in_place", "fc_diag_seg_phases",
    "fc_set_peer_timeout", "fc_diag_exchange_ms", "fc_set_grad_f64", "fc_set_residual_f64",
    "fc_get_residual_f64", "fc_get_aggregate_f64", "fc_peer_handle", "fc_peer_attach",
]


class FlexcommError(RuntimeError):
    """Base of the errors raised from C-ABI status codes."""


class InvalidArgument(FlexcommError, ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(FlexcommError, IndexError):
    """std::out_of_range in the reference."""


class RuntimeFailure(FlexcommError):
    """std::runtime_error in the reference (and CUDA / NCCL failures)."""


class DeviceFailure(RuntimeFailure):
    """A CUDA or NCCL failure (never a property of the data)."""


class NoDevice(FlexcommError):
    """No sm_100 device: the path never falls back to the CPU."""


_ERRS = {
    FC_ERR_INVALID_ARGUMENT: InvalidArgument,
    FC_ERR_OUT_OF_RANGE: OutOfRange,
    FC_ERR_RUNTIME: RuntimeFailure,
    FC_ERR_CUDA: DeviceFailure,
    FC_ERR_NCCL: DeviceFailure,
    FC_ERR_NO_DEVICE: NoDevice,
}


def check(status: int) -> None:
    if status != FC_OK:
        msg = lib.fc_last_error().decode(errors="replace")
        raise _ERRS.get(status, FlexcommError)(f"{lib.fc_status_string(status).decode()}: {msg}")
