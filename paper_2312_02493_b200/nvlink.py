"""NetParams calibrated on this pool's B200 NVLink/NVSwitch fabric.

The reference's selector (`select_collective`, inc/costmodel.hpp:153-167) is
kept unchanged; only its NetParams input is recalibrated (BASELINE north
star).  `tools/calibrate.py` measured AG-compressed / ART-Ring / ART-Tree
through this library's NCCL communicators at N = 2 and 4 and fitted one
(alpha, bandwidth) per N by least squares on log time; the measurements and
fits live in fixtures/nvlink_grid_n{N}.csv and fixtures/nvlink_fit_n{N}.json.
"""
from __future__ import annotations

import json
from pathlib import Path

from .flexcomm import NetParams

FIXTURES = Path(__file__).resolve().parents[1] / "fixtures"


def fitted(n: int) -> dict:
    """The stored fit for world size n (N >= 4 uses the largest measured fit)."""
    avail = sorted(int(p.stem.split("_n")[-1]) for p in FIXTURES.glob("nvlink_fit_n*.json"))
    if not avail:
        raise FileNotFoundError("no NVLink calibration fixtures (run tools/calibrate.py)")
    m = max([a for a in avail if a <= n] or [avail[0]])
    return json.loads((FIXTURES / f"nvlink_fit_n{m}.json").read_text())


def net_params(n: int) -> NetParams:
    d = fitted(n)
    return NetParams(d["alpha_s"], d["bandwidth_bps"])
