import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, "tests")
import numpy as np
from oracle_py import Oracle, RandomStream, random_cloud
from paper_2509_17340_b200 import EnsembleConfig, Planner, State
o = Oracle()
p = Planner(EnsembleConfig(), max_points=1 << 21)
IDENT = np.array([0, 0, 0, 1, 0, 0, 0, 0, 0, 0], dtype=np.float64)
for n, spread in ((10000, 8.0), (300, 8.0), (20000, 12.0)):
    pts = random_cloud(RandomStream(101), n, spread)
    for f64 in (True, False):
        q = pts if f64 else pts.astype(np.float32).astype(np.float64)
        snap = p.build_snapshot(q, State.from_array(IDENT), 10.0, f64=f64)
        d = snap.download()
        r = o.snapshot(q, IDENT, 10.0).get()
        bad = np.nonzero(d["ranges"] != r["ranges"])[0]
        print(n, f64, "bad cells", len(bad), [(int(c), d["ranges"][c], r["ranges"][c]) for c in bad[:5]])
