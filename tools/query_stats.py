"""Collision-query statistics of the FP32 screening kernel (stats build:
AMPPI_LIB_PATH=build_stats/libamppi_b200.so) per scene family."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17340_b200 import Planner, load  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

lib = load()
lib.amppi_query_stats.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
SLOTS = 8 + 64 + 8
cfg = plan_config()
out = {}
for kind in (1, 2, 3):
    d = scenes(256, kinds=kind)
    p = Planner(cfg, max_scenes=256, max_points=int(d["offsets"][-1]) + 1)
    st = (ctypes.c_ulonglong * SLOTS)()
    lib.amppi_query_stats(st, 1)
    p.cycle_batch(d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"], d["seeds"])
    lib.amppi_query_stats(st, 1)
    q = st[0]
    out[{1: "forest", 2: "verticals", 3: "inclines"}[kind]] = {
        "queries": q, "past_occupancy": st[1] / q, "cells_tested_per_query": st[2] / q,
        "cells_scanned_per_query": st[3] / q, "points_per_query": st[4] / q,
        "points_per_scanned_cell": st[4] / max(st[3], 1),
        "hit_queries": st[5] / q, "scanned_miss_queries": st[6] / q,
        "points_per_hit_query": (st[4] - st[7]) / max(st[5], 1), "points_per_miss_query": st[7] / max(st[6], 1),
        "d_max_band_steps_per_query": st[72] / q,
        "main_pass_flagged_of_completed": st[73] / max(st[74], 1),
        "main_pass_live_fraction_by_step": [round(st[8 + j] / max(st[8], 1), 3) for j in range(cfg.mppi.horizon)]}
    p.close()
print(json.dumps(out, indent=1))
