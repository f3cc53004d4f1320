"""Fit the tile chooser's launch model (tools/tile_model.py, tb_launch.cuh
choose_tile) to a kernel-only sweep of every configuration under both
schedules (tooling):

    python tools/tile_model_fit.py profiles/r02_tile_sched_sweep.jsonl

Input lines: {"sched": "auto"|"dp", "tile": "<bm>x<bn>", "n": N, "us": t}
(tools/tile_sweep.py with TB_TILE / TB_SCHED=dp). Fits one steady-state
efficiency per configuration plus the fixup (F), epilogue (E) and launch (R)
constants by least squares on log time, then reports how far the model's
(configuration, schedule) pick is from the fastest measured one per N."""
import collections
import json
import math
import os
import sys

import numpy as np
from scipy.optimize import least_squares

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import tile_model as tm  # noqa: E402


def load(path):
    pts = []
    for line in open(path):
        if line.startswith("{"):
            r = json.loads(line)
            pts.append((r["tile"], r["sched"] == "dp", r["n"], r["us"] * 1e-6))
    return pts


def features(tile, dp, n):
    """(w * t_stage at eff=1, fixups * s, units * s) for a square n."""
    bm, bn, sub, _ = tm.CFG[tile]
    tiles = -(-n // bm) * -(-n // bn)
    grid, dpt, sk, ipc, num_k = tm.plan_schedule(tiles, -(-n // (16 * sub)), tm.P, dp)
    t_stage = bm * bn * 16 * sub / tm.SM_FMA_PER_S
    s = bm * bn / 8192
    if sk == 0:
        units = -(-tiles // grid)
        return units * num_k * t_stage, 0.0, units * s
    dpw = dpt // grid
    return (dpw * num_k + ipc) * t_stage, 2 * s, (dpw + -(-ipc // num_k) + 1) * s


def fit(pts):
    tiles = sorted(tm.CFG)
    feats = np.array([features(t, dp, n) for t, dp, n, _ in pts])
    idx = np.array([tiles.index(t) for t, _, _, _ in pts])
    y = np.log(np.array([p[3] for p in pts]))

    def pred(x):
        eff, (F, E, R) = x[:len(tiles)], x[len(tiles):]
        return feats[:, 0] / eff[idx] + F * feats[:, 1] + E * feats[:, 2] + R

    x0 = np.r_[[0.95] * len(tiles), 5e-6, 0.2e-6, 4e-6]
    lo = np.r_[[0.5] * len(tiles), 0, 0, 0]
    hi = np.r_[[1.0] * len(tiles), 1e-4, 1e-4, 1e-4]
    res = least_squares(lambda x: np.log(pred(x)) - y, x0, bounds=(lo, hi), x_scale=np.abs(x0))
    return dict(zip(tiles, res.x[:len(tiles)])), tuple(res.x[len(tiles):]), float(np.sqrt(np.mean(res.fun ** 2)))


def evaluate(pts):
    by = collections.defaultdict(dict)
    for t, dp, n, sec in pts:
        by[n][(t, dp)] = sec
    rows = []
    for n, d in sorted(by.items()):
        p = tm.choose(n, n, n, sorted({t for t, _ in d}))
        b = min(d, key=d.get)
        rows.append((n, p, b, d.get(p, float("nan")) / d[b]))
    return rows


if __name__ == "__main__":
    pts = load(sys.argv[1])
    effs, (F, E, R), rms = fit(pts)
    print(f"# rms log error {rms:.4f}; F = {F * 1e6:.2f} us, E = {E * 1e6:.3f} us, R = {R * 1e6:.2f} us")
    for t in sorted(effs, key=lambda t: -effs[t]):
        print(f"#   {t:8s} eff {effs[t]:.4f}")
    for t, e in effs.items():
        tm.CFG[t] = tm.CFG[t][:3] + (e,)
    tm.F, tm.E, tm.R = F, E, R
    rows = evaluate(pts)
    print(f"# pick vs fastest: worst {max(r[3] for r in rows):.4f}, "
          f"geomean {math.exp(sum(math.log(r[3]) for r in rows) / len(rows)):.4f}")
    for n, p, b, loss in rows:
        print(f"{n:6d} picked {p[0]:8s}{' dp' if p[1] else ' sk'}  fastest {b[0]:8s}{' dp' if b[1] else ' sk'}  "
              f"loss {loss:.4f}")
