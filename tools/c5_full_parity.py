"""Whole-batch parity of the C5 workload: every scene of one batch against the
CPU oracle (multiprocessing over the host cores).  Reports how many scenes
match the test contract (status / winner bit-exact, FP64 outputs <= 1e-9).
Usage: python tools/c5_full_parity.py [scenes] [first_scene]"""
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def _check(args):
    lo, hi, data, out, cfg_dict = args
    from oracle_py import Oracle
    from paper_2509_17340_b200.workloads import plan_config

    oracle = Oracle()
    cfg = plan_config()
    ocfg = oracle.config(cfg)
    off = data["offsets"]
    bad = []
    for s in range(lo, hi):
        pts = data["xyz"][off[s]:off[s + 1]].astype(np.float64)
        snap = oracle.snapshot(pts, data["poses"][s], cfg.r_max)
        g = data["goals"][s]
        o = oracle.plan(snap, ocfg, data["states"][s], g[0:3], g[3:6], g[6:10], None, data["last"][s],
                        int(data["cycles"][s]), int(data["seeds"][s]))
        why = None
        if out["status"][s] != o["rc"]:
            why = f"status {out['status'][s]} vs {o['rc']}"
        elif o["rc"] == 0:
            if out["winner"][s] != o["winner"]:
                why = f"winner {out['winner'][s]} vs {o['winner']}"
            else:
                r = max(_rel(out["control"][s], o["control"]),
                        _rel(out["winner_nominal"][s], o["nominal"][o["winner"]]),
                        _rel(out["breakdown"][s], o["breakdown"]))
                fin = np.isfinite(o["stage2"])
                r = max(r, _rel(out["stage2"][s][fin], o["stage2"][fin]))
                if r > 1e-9:
                    why = f"rel {r:.3e}"
        if why:
            bad.append((s, why))
    return bad


def main():
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    cfg = plan_config()
    data = scenes(S, points=20000, frames=20, first=first)
    planner = Planner(cfg, precision=32, max_scenes=S, max_points=int(data["offsets"][-1]))
    out = planner.cycle_batch(data["offsets"], data["xyz"], data["poses"], data["states"], data["goals"],
                              data["last"], data["cycles"], data["seeds"])
    planner.close()
    workers = max(1, (os.cpu_count() or 2) - 1)
    step = (S + workers * 4 - 1) // (workers * 4)
    jobs = [(lo, min(S, lo + step), data, out, None) for lo in range(0, S, step)]
    with mp.get_context("fork").Pool(workers) as pool:
        bad = [b for part in pool.map(_check, jobs) for b in part]
    print(f"scenes {S} (first {first}): {S - len(bad)} match, {len(bad)} differ")
    for s, why in bad[:40]:
        print(f"  scene {s}: {why}")


if __name__ == "__main__":
    main()
