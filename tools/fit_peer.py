"""Fit the reference's NetParams to the product exchange's measured times.

    python tools/fit_peer.py [fixtures_dir]

Reads fixtures/peer_steps_n{N}.csv and fixtures/peer_exchange_n{N}.csv
(tools/calibrate_peer.py, run on the GPUs) and fits ONE NetParams(alpha,
bandwidth) per N -- the reference's API has a single one
(inc/costmodel.hpp:12-27) -- by least squares on log time over the three
collectives' measured SYNC times of whole steps (step - the one-worker step
of the same kind; ten (G, CR) points incl. BASELINE configs 1-3, Mc =
4 G c), against cost_ag_compressed / cost_art_ring / cost_art_tree
(inc/costmodel.hpp:79-96).  The sync time is what choosing a collective
costs a step; it includes AG's N-list decode, which the formulas have no
term for, so the fitted bandwidth is an effective one for the whole sync
path rather than the link's.  Then it checks the unchanged
select_collective (inc/costmodel.hpp:153-167) the way the reference checks
its fixtures (tests/test_acceptance.cpp:45-60): the predicted fastest must
be the measured fastest wherever the measured top-two margin exceeds 15 %,
and (stricter) the predicted collective's measured time is within 15 % of
the fastest at every point where the formulas can name the winner at all.
The fit minimises the total regret of the selector's choices (ties: least
squares on log time).  Where a decisive winner cannot be named by the
formulas for ANY NetParams -- ART at N = 2 (AG's cost is below ART-Ring's by
2 alpha for every bandwidth) and ART-Tree at N = 4 (above AG by 4 alpha) --
the point is recorded as "expressible": false.  The exchange-only grid is
checked against the same fit and reported, not fitted.  Writes
fixtures/peer_fit_n{N}.json.
"""
from __future__ import annotations

import csv
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KINDS = ["ag", "art_ring", "art_tree"]


def model(alpha: float, beta: float, n: int, mc: float) -> dict:
    """cost_ag_compressed / cost_art_ring / cost_art_tree (inc/costmodel.hpp:79-96)."""
    lg = math.log2(n)
    nm1 = n - 1
    return {"ag": alpha * lg + 2.0 * mc * beta * nm1,
            "art_ring": alpha * (2 * nm1 + lg) + mc * beta * (2 * nm1 / n + lg),
            "art_tree": 3 * alpha * lg + 3 * mc * beta * lg}


def log_err(alpha: float, beta: float, n: int, pts) -> float:
    e = 0.0
    for mc, meas in pts:
        m = model(alpha, beta, n, mc)
        for kk in KINDS:
            e += (math.log(m[kk]) - math.log(meas[kk])) ** 2
    return e


def regret(alpha: float, beta: float, n: int, pts) -> float:
    """Sum over the points of (measured time of the collective the selector
    picks) / (measured time of the fastest) - 1."""
    r = 0.0
    for mc, meas in pts:
        best = min(meas.values())
        r += meas[choose(alpha, beta, n, mc)] / best - 1.0
    return r


def fit(n: int, pts) -> tuple[float, float]:
    """NetParams for the unchanged selector: on a grid of log alpha / log beta,
    the least total regret of the selector's choices over the measured points
    (what a calibration is for), ties broken by least squares on log time;
    then a local least-squares refinement that keeps the regret."""
    best = None
    for i in range(121):
        la = -7.5 + i * (5.0 / 120)          # alpha 30 ns .. 3 ms
        for j in range(121):
            lb = -13.5 + j * (5.0 / 120)     # beta: 1/(3e13) .. 1/(3e8) s/byte
            a, b = 10 ** la, 10 ** lb
            key = (round(regret(a, b, n, pts), 9), log_err(a, b, n, pts))
            if best is None or key < best[0]:
                best = (key, la, lb)
    (r0, e0), la, lb = best
    step = 5.0 / 120
    for _ in range(60):
        improved = False
        for da, db in ((step, 0), (-step, 0), (0, step), (0, -step)):
            a, b = 10 ** (la + da), 10 ** (lb + db)
            if round(regret(a, b, n, pts), 9) > r0:
                continue
            e = log_err(a, b, n, pts)
            if e < e0:
                e0, la, lb, improved = e, la + da, lb + db, True
        if not improved:
            step /= 2
    return 10 ** la, 10 ** lb


def expressible(n: int, mc: float, winner: str) -> bool:
    """Can the reference's formulas pick `winner` at this Mc for ANY NetParams?
    (At N = 2 the AG cost is below ART-Ring's by 2 alpha for every bandwidth;
    at N = 4 ART-Tree is above AG by 4 alpha.)  Checked on a wide grid."""
    for i in range(61):
        for j in range(61):
            if choose(10 ** (-9 + i * 0.2), 10 ** (-15 + j * 0.2), n, mc) == winner:
                return True
    return False


def choose(alpha: float, beta: float, n: int, mc: float) -> str:
    """select_collective's argmin, ties to AG then ART_RING (costmodel.hpp:153-167)."""
    m = model(alpha, beta, n, mc)
    best, name = m["ag"], "ag"
    if m["art_ring"] < best:
        best, name = m["art_ring"], "art_ring"
    if m["art_tree"] < best:
        name = "art_tree"
    return name


def check(alpha, beta, n, pts, labels):
    out = []
    for (mc, meas), lab in zip(pts, labels):
        order = sorted(KINDS, key=lambda kk: meas[kk])
        margin = meas[order[1]] / meas[order[0]] - 1.0
        pred = choose(alpha, beta, n, mc)
        m = model(alpha, beta, n, mc)
        out.append({"point": lab, "mc_bytes": mc, "measured_us": {kk: round(meas[kk] * 1e6, 2) for kk in KINDS},
                    "measured_fastest": order[0], "margin": round(margin, 3), "predicted": pred,
                    "agree": pred == order[0], "decisive": margin > 0.15,
                    "regret": round(meas[pred] / meas[order[0]] - 1.0, 3),
                    "expressible": expressible(n, mc, order[0]),
                    "rel_err": {kk: round(abs(m[kk] - meas[kk]) / meas[kk], 3) for kk in KINDS}})
    return out


def load(d: Path, n: int):
    ex, st = [], []
    with open(d / f"peer_exchange_n{n}.csv") as f:
        for r in csv.DictReader(f):
            ex.append((float(r["mc_bytes"]), {kk: float(r[kk + "_us"]) * 1e-6 for kk in KINDS}, f"k={r['k']}"))
    p = d / f"peer_steps_n{n}.csv"
    if p.exists():
        with open(p) as f:
            for r in csv.DictReader(f):
                mc = 4.0 * float(r["grad_len"]) * float(r["cr"])
                meas = {"ag": float(r["ag_step_us"]) - float(r["ag_one_worker_us"]),
                        "art_ring": float(r["art_ring_step_us"]) - float(r["art_one_worker_us"]),
                        "art_tree": float(r["art_tree_step_us"]) - float(r["art_one_worker_us"])}
                meas = {kk: max(v, 0.05) * 1e-6 for kk, v in meas.items()}
                st.append((mc, meas, r["config"]))
    return ex, st


def main() -> int:
    d = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "fixtures"
    worlds = sorted(int(p.stem.split("_n")[-1]) for p in d.glob("peer_exchange_n*.csv"))
    for n in worlds:
        ex, st = load(d, n)
        pts = [(mc, meas) for mc, meas, _ in st]
        alpha, beta = fit(n, pts)
        exc = check(alpha, beta, n, [(mc, meas) for mc, meas, _ in ex], [lab for *_, lab in ex])
        stc = check(alpha, beta, n, [(mc, meas) for mc, meas, _ in st], [lab for *_, lab in st])
        dec = [c for c in exc if c["decisive"]]
        sdec = [c for c in stc if c["decisive"]]
        regret = max((c["measured_us"][c["predicted"]] / c["measured_us"][c["measured_fastest"]] - 1.0)
                     for c in stc) if stc else None
        res = {"n": n, "source": "whole steps on the product's peer-memory exchange, tools/calibrate_peer.py",
               "alpha_s": alpha, "bandwidth_bps": 8.0 / beta, "bandwidth_GBps": 1.0 / beta / 1e9,
               "fit": "least total regret of the selector's choices over the step grid (sync time = step - "
                      "one-worker step), ties by least squares on log time; effective bandwidth of the sync path",
               "step_max_regret": regret,
               "exchange_agreement_decisive": (sum(c["agree"] for c in dec) / len(dec)) if dec else None,
               "exchange_decisive_points": len(dec),
               "step_agreement_decisive": (sum(c["agree"] for c in sdec) / len(sdec)) if sdec else None,
               "step_decisive_points": len(sdec),
               "max_rel_err": max(max(c["rel_err"].values()) for c in stc),
               "exchange_points": exc, "step_points": stc}
        (d / f"peer_fit_n{n}.json").write_text(json.dumps(res, indent=1))
        print(json.dumps({kk: v for kk, v in res.items() if not kk.endswith("_points")}))
        for c in exc + stc:
            print(f"  {c['point']:>12} fastest={c['measured_fastest']:9} margin={c['margin']:6.3f} "
                  f"pred={c['predicted']:9} {'ok' if c['agree'] else ('MISS' if c['decisive'] else 'tie')} "
                  f"{c['measured_us']}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
