"""Per-phase cycle split of the fused per-scene snapshot (k_snapshot_scene) over
one C5 host batch (stats build: AMPPI_LIB_PATH=build_stats/libamppi_b200.so).
Cycles are summed over all CTAs; the shares are what matters."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17340_b200 import Planner, load  # noqa: E402
from paper_2509_17340_b200.workloads import plan_config, scenes  # noqa: E402

NAMES = ["table init", "pass A keying", "pass B ties", "pool+compact+bbox", "grid meta", "sort", "scatter+flags",
         "leaf boxes", "cell records", "neighbour masks"]
lib = load()
lib.amppi_snapshot_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
cfg = plan_config()
S = 4096
d = scenes(S, points=20000, frames=20)
p = Planner(cfg, precision=32, max_scenes=S, max_points=int(d["offsets"][-1]))
st = (ctypes.c_ulonglong * 10)()
args = [d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"], d["seeds"]]
p.cycle_batch(*args)
p.synchronize()
lib.amppi_snapshot_phase_cycles(st, 1)
p.cycle_batch(*args)
p.synchronize()
lib.amppi_snapshot_phase_cycles(st, 1)
tot = sum(st)
for n, v in zip(NAMES, st):
    print(f"{n:20s} {v / S:10.0f} cycles/scene {100 * v / max(tot, 1):5.1f}%")
