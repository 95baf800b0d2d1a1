"""Per-phase cycle split of the few-scene finalize kernel (C1 snapshot, stats build:
AMPPI_LIB_PATH=build_stats/libamppi_b200.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17340_b200 import Planner, State, load  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

NAMES = ["table init", "pass A keying", "pass B ties", "pool+compact+bbox", "grid meta", "sort", "scatter+flags",
         "leaf boxes", "cell records", "neighbour masks"]
lib = load()
lib.amppi_snapshot_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
cfg = plan_config()
one = scenes(1, points=20000, frames=20, first=0, kinds=1)
p = Planner(cfg, precision=32, max_scenes=1, max_points=1 << 16)
x = State.from_array(one["states"][0])
st = (ctypes.c_ulonglong * 10)()
for i in range(20):
    p.build_snapshot(one["xyz"], x, cfg.r_max)
p.synchronize()
lib.amppi_snapshot_phase_cycles(st, 1)
for i in range(100):
    p.build_snapshot(one["xyz"], x, cfg.r_max)
p.synchronize()
lib.amppi_snapshot_phase_cycles(st, 1)
tot = sum(st)
for n, v in zip(NAMES, st):
    print(f"{n:20s} {v / 100:10.0f} cycles {100 * v / max(tot, 1):5.1f}%")
