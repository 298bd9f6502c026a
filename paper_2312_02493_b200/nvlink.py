"""NetParams calibrated on this pool's B200 NVLink/NVSwitch fabric.

The reference's selector (`select_collective`, inc/costmodel.hpp:153-167) is
kept unchanged; only its NetParams input is recalibrated (BASELINE north
star).  Two calibrations exist:

* peer memory (the product's exchange, used whenever the context maps its
  peers): `tools/calibrate_peer.py` timed whole AR-Ring / AR-Tree / AG steps
  at ten (G, CR) points and `tools/fit_peer.py` fitted one (alpha,
  bandwidth) per N to their sync times -- fixtures/peer_fit_n{N}.json;
* NCCL (round 1, contexts created with FC_NO_P2P=1): `tools/calibrate.py`
  over the library's NCCL communicators -- fixtures/nvlink_fit_n{N}.json.
"""
from __future__ import annotations

import json
from pathlib import Path

from .flexcomm import NetParams

FIXTURES = Path(__file__).resolve().parents[1] / "fixtures"


def _pick(prefix: str, n: int):
    avail = sorted(int(p.stem.split("_n")[-1]) for p in FIXTURES.glob(f"{prefix}_n*.json"))
    if not avail:
        return None
    m = max([a for a in avail if a <= n] or [avail[0]])
    return json.loads((FIXTURES / f"{prefix}_n{m}.json").read_text())


def fitted(n: int, peer: bool = True) -> dict:
    """The stored fit for world size n (the largest measured N <= n): the
    peer-memory fit when `peer` and present, else the NCCL one."""
    d = _pick("peer_fit", n) if peer else None
    if d is None:
        d = _pick("nvlink_fit", n)
    if d is None:
        raise FileNotFoundError("no NVLink calibration fixtures (run tools/calibrate_peer.py)")
    return d


def net_params(n: int, peer: bool = True) -> NetParams:
    d = fitted(n, peer)
    return NetParams(d["alpha_s"], d["bandwidth_bps"])
