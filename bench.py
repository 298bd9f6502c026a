#!/usr/bin/env python
"""Benchmark of the B200 Top-k gradient-sync path (BASELINE.json metric).

Metric: "Topk sync ms/step (compress+collective+decode), HBM GB/s & bus GB/s
vs peak".  A step is one call of the hot path (flexcomm::artopk_step /
ag_step equivalent) on every rank: error feedback, exact Top-k, the exchange
(broadcast + allreduce, or allgather) and the dense decode.

Default workload (N=1, the largest single-GPU BASELINE configuration):
config 3's per-GPU worker — a 138M-element (VGG-16-sized, 552 MB) fp32
gradient, CR 0.01, STAR AR-Top-k with a Ring allreduce — one data-parallel
worker per GPU (weak scaling: every rank holds its own 138M gradient).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--mode star|var|ag|dense]
                  [--algo ring|tree] [--grad-len G] [--cr C] [--impl ours|reference]

For N > 1 launch under torchrun (one process per GPU, NCCL over NVLink).
`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference headers, compiled) on the host.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# NCCL prints a version banner on stdout at INFO/VERSION level; the contract
# is one JSON line on stdout
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

MODES = {"star": 0, "var": 1, "ag": 2, "dense": 3}
# BASELINE.json configs (per-GPU workload; one worker per GPU):
CONFIGS = {
    "C1": dict(mode="star", grad_len=11_700_000, cr=0.01),   # ResNet-18-sized, STAR
    "C2": dict(mode="var", grad_len=25_600_000, cr=0.001),   # ResNet-50-sized, VAR
    "C3": dict(mode="star", grad_len=138_000_000, cr=0.01),  # VGG-16-sized (headline)
    "C3-ag": dict(mode="ag", grad_len=138_000_000, cr=0.01),
    "C3-tree": dict(mode="star", grad_len=138_000_000, cr=0.01, algo="tree"),
    "C3-lw": dict(mode="ag", grad_len=138_000_000, cr=0.01, compressor="layerwise"),
    "C3-thr": dict(mode="ag", grad_len=138_000_000, cr=0.01, compressor="threshold"),
    "C4": dict(mode="star", grad_len=355_000_000, cr=0.001),  # GPT-2-medium-sized
    "C5": dict(mode="star", grad_len=1_000_000_000, cr=0.001),  # 1B
}
ALGOS = {"ring": 0, "tree": 1}
COMPRESSORS = {"exact": 0, "layerwise": 1, "threshold": 2}


def vgg16_layers(G):
    """VGG-16's parameter layout (13 conv + 3 FC layers, weight then bias),
    the last layer trimmed or padded so the map covers G elements."""
    convs = [(3, 64), (64, 64), (64, 128), (128, 128), (128, 256), (256, 256), (256, 256),
             (256, 512), (512, 512), (512, 512), (512, 512), (512, 512), (512, 512)]
    sizes = []
    for cin, cout in convs:
        sizes += [cin * cout * 9, cout]
    for fin, fout in [(25088, 4096), (4096, 4096), (4096, 1000)]:
        sizes += [fin * fout, fout]
    sizes[-2] += G - sum(sizes)
    layers, off = [], 0
    for n in sizes:
        layers.append((off, n))
        off += n
    return layers
SEED = 42


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--mode", choices=list(MODES), default="star")
    p.add_argument("--algo", choices=list(ALGOS), default="ring")
    p.add_argument("--grad-len", type=int, default=138_000_000)
    p.add_argument("--cr", type=float, default=0.01)
    p.add_argument("--compressor", choices=list(COMPRESSORS), default="exact",
                   help="AG-path compressor (inc/artopk.hpp:113); layerwise uses VGG-16's layer map")
    p.add_argument("--config", choices=list(CONFIGS), default=None,
                   help="BASELINE.json configuration preset (overrides mode/grad-len/cr)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    a = p.parse_args()
    if a.config:
        for key, val in CONFIGS[a.config].items():
            setattr(a, key, val)
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def workload_name(a, world):
    mode = {"star": "STAR AR-Topk", "var": "VAR AR-Topk", "ag": "AG-Topk",
            "dense": "Dense allreduce"}[a.mode]
    algo = "" if a.mode in ("ag", "dense") and a.mode != "dense" else f" ({a.algo})"
    comp = "" if getattr(a, "compressor", "exact") == "exact" else f" [{a.compressor} compressor]"
    return (f"{mode}{algo}{comp}, {a.grad_len / 1e6:g}M fp32 gradient per GPU, CR {a.cr:g}, "
            f"{world} worker(s)")


# ------------------------------------------------------------------ clocks ---

class ClockSampler:
    """nvidia-smi sampling of SM clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- peaks ----

def ef_traffic(G):
    """DRAM bytes per EF launch from the committed ncu --set full capture
    (profiles/r02_ef_traffic.json, else round 1's), scaled to G if the capture's size differs;
    None when absent."""
    p = ROOT / "profiles" / "r02_ef_traffic.json"
    if not p.exists():
        p = ROOT / "profiles" / "r01_ef_traffic.json"
    try:
        d = json.loads(p.read_text())
        scale = G / 138_000_000
        return round((d["dram_read_bytes"] + d["dram_write_bytes"]) * scale)
    except Exception:
        return None


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------ reference (CPU) ----

def run_reference_cpu(mode: str, algo: str, grad_len: int, cr: float, n: int, steps: int,
                      warmup: int = 0):
    """Time the unmodified reference (oracle/_ref, the highest ISA level this
    host supports) on this host: `warmup` untimed then `steps` timed calls of
    flexcomm::artopk_step / ag_step on the FULL configuration (n workers x
    grad_len fp64 elements, the reference's own in-process Cluster; it loops
    over the workers serially in one thread, inc/artopk.hpp:75-102).
    Returns (median ms per step, sample description, per-step seconds, isa)."""
    import oracle

    ref = oracle.Ref("native")
    m = {"star": 0, "var": 1, "ag": 2}.get(mode, 0)
    st = oracle.RefState(ref, n, grad_len)
    try:
        for r in range(n):
            st.fill_synth(r, SEED, r, 0)
        for s in range(warmup):
            st.step(cr, m, ALGOS[algo], s)
        times = [st.step(cr, m, ALGOS[algo], warmup + s) for s in range(steps)]
    finally:
        st.close()
    ms = statistics.median(times) * 1e3
    sample = (f"full configuration: {n} worker(s) x {grad_len / 1e6:g}M fp64 elements through the "
              f"unmodified reference artopk_step/ag_step ({ref.isa} build), {warmup} untimed + "
              f"{steps} timed step(s), median")
    return ms, sample, times, ref.isa


def bench_config(a, world: int) -> dict:
    """The workload's config dict -- identical in both arms (ours / reference)."""
    k = a.grad_len if a.mode == "dense" else k_of(a.cr, a.grad_len)
    return {"workload": workload_name(a, world), "grad_len": a.grad_len, "cr": a.cr, "k": k,
            "mode": a.mode, "algo": a.algo, "workers": world, "parallelism": f"dp{world}",
            "compressor": a.compressor,
            "l2": ("inputs (2 x %.0f MB per worker) larger than the 126 MB L2" % (4 * a.grad_len / 1e6))
            if 8 * a.grad_len > 126e6 else "inputs smaller than the 126 MB L2 (not flushed)"}


def k_of(c: float, g: int) -> int:
    """inc/compress.hpp:28-33 (host arithmetic, as fc_k_of)."""
    return int(min(max(math.ceil(c * g - 1e-9), 1), g))


def reference_arm(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    mode = a.mode if a.mode != "dense" else "star"
    ms, sample, _, isa = run_reference_cpu(mode, a.algo, a.grad_len, a.cr, world, a.steps, a.warmup)
    line = {
        "metric": "Topk sync ms/step (compress+collective+decode)",
        "value": round(ms, 3), "unit": "ms/step", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": bench_config(a, world),
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/step", "cores": 1,
                         "kind": "reference", "sample": sample, "isa": isa,
                         "threads_note": "the reference's sync path is single-threaded "
                                         "(inc/artopk.hpp:75-102): 1 thread is every thread it can use",
                         "host": host_info()},
        "e2e": {"value": round(ms, 3), "unit": "ms/step", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def host_info():
    cpu = "?"
    try:
        for l in Path("/proc/cpuinfo").read_text().splitlines():
            if l.startswith("model name"):
                cpu = l.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu": cpu, "nproc": os.cpu_count()}


# ----------------------------------------------------------------- ours -----

def main():
    a = parse()
    if a.impl == "reference":
        return reference_arm(a)
    world, rank, local = dist_env()
    import numpy as np
    import torch

    from paper_2312_02493_b200 import flexcomm as fc
    from paper_2312_02493_b200 import _abi

    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist
    max_cr = min(1.0, max(a.cr, 0.1))

    def make_cluster(flags):
        # NCCL bootstrap: rank 0's unique id shipped over the gloo group
        uid = fc.get_unique_id() if rank == 0 else None
        if pg:
            obj = [uid]
            pg.broadcast_object_list(obj, src=0)
            uid = obj[0]
        # NCCL's init banner goes to fd 1; keep stdout to the one JSON line
        sys.stdout.flush()
        saved_fd = os.dup(1)
        os.dup2(2, 1)
        try:
            return fc.Cluster.nccl(world, rank, uid, a.grad_len, device=local, max_cr=max_cr,
                                   flags=flags)
        finally:
            os.dup2(saved_fd, 1)
            os.close(saved_fd)

    def make_ready(flags):
        c_ = make_cluster(flags)
        if a.compressor == "layerwise":
            c_.set_layer_map(vgg16_layers(a.grad_len))
        return c_

    cl = make_ready(_abi.FC_FLAG_ASYNC)
    G = a.grad_len
    mode = MODES[a.mode]
    algo = ALGOS[a.algo]

    def step(s):
        if mode == 2:
            cl.ag_step(a.cr, COMPRESSORS[a.compressor], stats=False)
        elif mode == 3:
            cl.dense_step(algo, fc.AVG, stats=False)
        else:
            cl.artopk_step(a.cr, mode, algo, s, fc.AVG, stats=False)

    def barrier():
        cl.sync()
        torch.cuda.synchronize()
        if pg:
            pg.barrier()

    def max_over_ranks(x):
        if not pg:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.ExternalStream(cl.stream_ptr(), device=local)
    # inputs resident in HBM before the timed region (synthetic, seed 42)
    cl.fill_synthetic(0, SEED, rank, 0)
    cl.sync()

    # ---- device-resident timing -------------------------------------------
    for s in range(a.warmup):
        step(s)
    barrier()
    t_w = time.time()
    for s in range(5):
        step(a.warmup + s)
    barrier()
    per_step = max_over_ranks((time.time() - t_w) / 5)
    clocks = ClockSampler(local)
    clocks.start()
    # the EF kernel's event pair breaks the programmatic-dependent-launch
    # overlap with its neighbours: time every 4th launch of the timed region
    cl.set_ef_timing_period(4)
    cl.ef_kernel_timing(reset=True)
    l0 = fc.lib.fc_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    for s in range(a.steps):
        step(a.warmup + 5 + s)
    ev1.record(stream)
    barrier()
    ms_local = ev0.elapsed_time(ev1) / a.steps
    launches = fc.lib.fc_launch_count() - l0
    ef_ms, ef_n = cl.ef_kernel_timing()
    in_place = mode in (0, 1) and cl.aggregate_in_place
    # the timed region is short (K steps of well under a millisecond): keep the
    # same load running ~1.5 s longer so nvidia-smi samples the clocks under it
    # (same step count on every rank; not part of the timed number)
    n_soak = int(min(20_000, max(50, 1.5 / max(per_step, 1e-5))))
    for s in range(n_soak):
        step(10_000 + s)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(ms_local)

    # ---- phase split from one synchronous step (diagnostic) ---------------
    phase = None
    try:
        cl.sync()
        stt = _abi.fc_step_stats()
        import ctypes as C

        if mode == 2:
            rc = fc.lib.fc_ag_step(cl._ctx, a.cr, COMPRESSORS[a.compressor], C.byref(stt))
        elif mode == 3:
            rc = fc.lib.fc_dense_step(cl._ctx, algo, fc.AVG, C.byref(stt))
        else:
            rc = fc.lib.fc_artopk_step(cl._ctx, a.cr, mode, algo, 1000, fc.AVG, C.byref(stt))
        cl.sync()
        if rc == 0:
            phase = {"k": stt.k, "hbm_bytes_alg": stt.hbm_bytes, "bus_bytes": stt.bus_bytes,
                     "launches_per_step": stt.launches}
    except Exception:
        pass

    # ---- exchange phase alone (N > 1): bus GB/s of the collective ----------
    # The product's own exchange kernels timed back to back with the lists in
    # place (fc_diag_exchange_ms: from the selections' publish to the point
    # where the decode could start), max over ranks; bus bytes follow the
    # NCCL-tests convention (broadcast 4k + allreduce 2(N-1)/N 4k for ART,
    # (N-1) 8k for AG, 2(N-1)/N 4G for the dense allreduce).
    exchange = None
    if world > 1:
        try:
            import ctypes as C

            k_ex = fc.k_of(a.cr, G)
            if mode == 3:
                ex_ms = ms  # the dense step is the allreduce
                ex_bus = 2.0 * (world - 1) / world * 4.0 * G
                how = "the dense step (one ncclAllReduce of 4G bytes, ncclAvg)"
            else:
                which = 0 if mode == 2 else (2 if algo == 1 else 1)
                out = C.c_double()
                barrier()
                rc = fc.lib.fc_diag_exchange_ms(cl._ctx, which, k_ex, 20, C.byref(out))
                if rc != 0:
                    raise RuntimeError(fc.lib.fc_last_error().decode())
                ex_ms = max_over_ranks(out.value)
                ex_bus = (world - 1) * 8.0 * k_ex if mode == 2 else 4.0 * k_ex + 2.0 * (world - 1) / world * 4.0 * k_ex
                how = ("fc_diag_exchange_ms: the step's exchange kernels (" +
                       ("list publish + k_collect_packs" if mode == 2 else
                        "list publish + k_fetch_gather + " + ("k_reduce_root" if algo == 1 else
                                                             ("k_reduce_slice" if world > 2 else "direct push")))
                       + ") back to back, max over ranks; peer memory" if cl.peer_exchange else
                       "fc_diag_exchange_ms (NCCL collectives)")
                # the diagnostic leaves no selection behind: re-run one step
                step(20_000)
                barrier()
            exchange = {"ms": round(ex_ms, 4), "bus_bytes": ex_bus,
                        "bus_gbs": round(ex_bus / (ex_ms * 1e-3) / 1e9, 1), "bus_peak_gbs": 900.0,
                        "frac": round(ex_bus / (ex_ms * 1e-3) / 1e9 / 900.0, 3), "timing": how}
        except Exception as e:  # diagnostics never fail the bench
            exchange = {"unavailable": str(e)[:200]}

    # ---- end-to-end through the public API with host buffers --------------
    # A host-fed user creates the context with FC_FLAG_PIPELINE (two gradient
    # and two aggregate buffers).  Every step: upload of the step's gradient
    # from pinned host memory, the sync step, download of the dense aggregate
    # (the reference returns it by value).  The copies run on the copy
    # engines: step s+1's upload and step s's download overlap each other and
    # the compute (PCIe is full duplex).
    e2e = None
    if not a.no_e2e:
        host_g = torch.empty(G, dtype=torch.float32, pin_memory=True)
        host_agg = torch.empty(G, dtype=torch.float32, pin_memory=True)
        host_g.copy_(_tensor_from_ptr(cl.grad_ptr(0), G, local))  # setup only
        torch.cuda.synchronize()
        cl.close()
        cl = make_ready(_abi.FC_FLAG_ASYNC | _abi.FC_FLAG_PIPELINE)
        stream = torch.cuda.ExternalStream(cl.stream_ptr(), device=local)
        # (a long enough run that the pipeline's fill and drain -- one upload and one
        # download not overlapped -- are amortised: steady-state throughput)
        e2e_steps = max(40, a.steps)
        for s in range(2):
            cl.set_grad(0, host_g, async_=True)
            step(s)
            cl.aggregate(host_agg, async_=True)
        cl.sync()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(e2e_steps):
            cl.set_grad(0, host_g, async_=True)
            step(100 + s)
            cl.aggregate(host_agg, async_=True)
        cl.join()
        e1.record(stream)
        barrier()
        cl.sync()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
        e2e = {"value": round(e2e_ms, 4), "unit": "ms/step",
               "h2d_bytes_per_step": 4 * G, "d2h_bytes_per_step": 4 * G, "steps": e2e_steps,
               "context": "FC_FLAG_ASYNC | FC_FLAG_PIPELINE, FC_HOST_ASYNC copies"}

    # ---- roofline of the dominant kernel (error feedback) -----------------
    peak, peak_src = hbm_peak()
    ef_bytes = 12.0 * G  # read g_o + residual, write g_e
    achieved = ef_bytes / (ef_ms * 1e-3) / 1e9 if ef_ms > 0 else None
    k = fc.k_of(a.cr, G) if mode != 3 else G
    if mode in (0, 1):
        # dense aggregate: 4G written; in place: <= 2 x 32-byte sectors per
        # index (the previous support cleared, this one written) + the lists
        agg_bytes = 80.0 * k if in_place else 4.0 * G
        step_bytes = 12.0 * G + agg_bytes + 32.0 * k + (8.0 * world if mode == 1 else 0.0)
        bus = 4.0 * k + 2.0 * (world - 1) / world * 4.0 * k if world > 1 else 0.0
    elif mode == 2:
        step_bytes = 16.0 * G + 8.0 * k + 12.0 * world * k
        bus = (world - 1) * 8.0 * k
    else:
        step_bytes = 12.0 * G
        bus = 2.0 * (world - 1) / world * 4.0 * G if world > 1 else 0.0
    step_gbs = step_bytes / (ms * 1e-3) / 1e9

    # ---- CPU baseline (rank 0, N=1 only): the reference itself -------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and a.compressor == "exact":
        try:
            # bounded: 2 timed steps of the full configuration (~6-10 s of CPU work)
            ms_cpu, sample, _, isa = run_reference_cpu(a.mode if a.mode != "dense" else "star", a.algo,
                                                       G, a.cr, 1, 2, 0)
            cpu = {"value": round(ms_cpu, 2), "unit": "ms/step", "cores": 1, "kind": "reference",
                   "sample": sample, "isa": isa, "host": host_info()}
        except Exception as e:  # the baseline is reported, never a dependency
            cpu = {"value": None, "unit": "ms/step", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "Topk sync ms/step (compress+collective+decode)",
            "value": round(ms, 4), "unit": "ms/step", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(a, world),
            "hbm_gbs_step": round(step_gbs, 1),
            "bus_gbs_step": round(bus / (ms * 1e-3) / 1e9, 2) if bus else 0.0,
            "exchange": exchange,
            "aggregate": ("in place: the previous support's 32-byte sectors zeroed, this step's rewritten "
                          "(same dense content; FC_FLAG_DENSE_DECODE / FC_INCR_DIV=0 rewrite it whole)"
                          if in_place else "dense rewrite (4G bytes)") if mode in (0, 1) else None,
            "bus_peak_gbs": 900.0,
            "roofline": {"kernel": "k_ef (error feedback + candidate emission)", "bound": "hbm",
                         "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None,
                         "traffic": ef_traffic(G), "bytes_per_launch": ef_bytes,
                         "mean_launch_ms": round(ef_ms, 5), "launches_timed": ef_n,
                         "timing": "CUDA events around every 4th EF launch of the timed region",
                         "peak_source": peak_src},
            "step_roofline": {"alg_bytes": step_bytes, "achieved_gbs": round(step_gbs, 1),
                              "frac": round(step_gbs / peak, 4),
                              "lower_bound_ms": round(step_bytes / peak / 1e6, 4)},
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "cpu_baseline": cpu,
            "phase": phase,
        }
        print(json.dumps(line), flush=True)
    cl.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def _tensor_from_ptr(ptr: int, n: int, device: int):
    """Zero-copy torch view of a library-owned device buffer (setup/readback only)."""
    import torch

    class _CudaArray:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (p, False),
                                             "version": 3, "strides": None}

    return torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{device}")


if __name__ == "__main__":
    sys.exit(main())
