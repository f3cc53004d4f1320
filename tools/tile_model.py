"""Replay of the tile-shape chooser's launch model (tb_launch.cuh
choose_tile / model_seconds) against measured kernel-only sweeps (tooling;
tests/test_tile_model.py runs it on the committed sweeps).

    python tools/tile_model.py [profiles/r02_tile_sweep_1000_3000_50.jsonl ...]

For every N of a sweep (one JSON line per (tile, n): kernel-only us, from
tools/tile_sweep.py) it prints the configuration the model picks, the
fastest measured one and the time lost by the pick."""
import collections
import json
import math
import os
import sys

P = 148
# name: (bm, bn, sub, steady-state efficiency) — kTileCfgs in tb_launch.cuh
CFG = {  # largest tiles first (the chooser's tie-break order)
    "128x128": (128, 128, 1, 0.9691), "128x96": (128, 96, 1, 0.9701), "96x128": (96, 128, 1, 0.9705),
    "128x64": (128, 64, 2, 0.9710), "64x128d": (64, 128, 2, 0.9670), "64x128": (64, 128, 1, 0.9530),
    "96x96t": (96, 96, 3, 0.9776), "96x96": (96, 96, 2, 0.9731), "64x96": (64, 96, 2, 0.9688),
    "64x64d": (64, 64, 4, 0.9632), "64x64": (64, 64, 2, 0.9480),
}
PREFER_LARGER = 2e-3
F, E, R = 2.31e-6, 0.344e-6, 4e-6
SM_FMA_PER_S = 64 * 1.965e9


def plan_schedule(tiles, num_k, sms=P, dp_only=False):
    """tb_launch.cuh plan_schedule: (grid, dp, sk, ipc, num_k)."""
    rem = tiles % sms
    if rem == 0 or dp_only or (tiles < sms and 4 * tiles >= 3 * sms):
        return min(tiles, sms), tiles, 0, 1, num_k
    min_seg = min(num_k, 8)
    if 2 * tiles <= sms:
        split = min(sms // tiles, num_k // min_seg)
        if split >= 2:
            ipc = -(-num_k // split)
            return split * tiles, 0, tiles, ipc, ipc * split
    sk = rem + sms if tiles > sms else tiles
    ipc = max(-(-sk * num_k // sms), min_seg)
    return sms, tiles - sk, sk, ipc, num_k


def model_seconds(m, n, k, bm, bn, sub, eff, sms=P, dp_only=False):
    tiles = -(-m // bm) * -(-n // bn)
    grid, dp, sk, ipc, num_k = plan_schedule(tiles, -(-k // (16 * sub)), sms, dp_only)
    t_stage = bm * bn * 16 * sub / (SM_FMA_PER_S * eff)
    s = bm * bn / 8192
    if sk == 0:
        units = -(-tiles // grid)
        w, fix = units * num_k, 0
    else:
        dpw = dp // grid
        w = dpw * num_k + ipc
        units = dpw + -(-ipc // num_k) + 1
        fix = 2
    return w * t_stage + fix * F * s + units * E * s + R


def choose(m, n, k, cands=None):
    """(config, dp_only) the model picks among single launches: in CFG order
    (largest tiles first), a different shape must be faster by PREFER_LARGER."""
    best, best_t = None, float("inf")
    for c in [c for c in CFG if c in (cands or CFG)]:
        for dp in (False, True):
            t = model_seconds(m, n, k, *CFG[c], dp_only=dp)
            if t < best_t * (1.0 if best and best[0] == c else 1.0 - PREFER_LARGER):
                best, best_t = (c, dp), t
    return best


def pick(m, n, k, cands=None):
    return choose(m, n, k, cands)[0]


def load(path):
    """{n: {(tile, dp_only): us}} from tools/tile_sweep.py lines tagged with "sched"."""
    by = collections.defaultdict(dict)
    for line in open(path):
        if line.startswith("{"):
            r = json.loads(line)
            by[r["n"]][(r["tile"], r.get("sched") == "dp")] = r["us"]
    return by


def replay(path):
    """[(n, picked, fastest, picked_us / fastest_us), ...]; picks are (tile, dp_only)."""
    out = []
    for n, d in sorted(load(path).items()):
        p = choose(n, n, n, sorted({t for t, _ in d}))
        b = min(d, key=d.get)
        out.append((n, p, b, d[p] / d[b]))
    return out


if __name__ == "__main__":
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    paths = sys.argv[1:] or [os.path.join(root, "profiles", "r02_tile_sched_sweep.jsonl")]
    for path in paths:
        rows = replay(path)
        print(f"# {os.path.basename(path)}: worst loss {max(r[3] for r in rows):.4f}, "
              f"geomean {math.exp(sum(math.log(r[3]) for r in rows) / len(rows)):.4f}")
        for r in rows:
            print(f"{r[0]:6d} picked {r[1][0]:8s}{' dp' if r[1][1] else ' sk'} "
                  f"fastest {r[2][0]:8s}{' dp' if r[2][1] else ' sk'} loss {r[3]:.4f}")
