"""Step-count agreement of mode R with the oracle in step-hint-binding
regimes (developer check; see tests/test_gpu_geodesic.py)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from oracle_lib import orc_trace_reference
from paper_2507_16165_b200 import geodesic as G
from test_gpu_geodesic import random_rays, cfg
for eps, rt, at in [(0.1, 1e-10, 1e-12), (1.0, 1e-10, 1e-12), (5.0, 1e-13, 1e-15)]:
    o, d = random_rays(600, 21, 10.0, 80.0)
    rec, _ = G.trace_batch(o, d, G.BlackHole(1.0), cfg(eps=eps, esc=300.0, rt=rt, at=at))
    diff = sum(int(rec[i]["steps"] != orc_trace_reference(o[i], d[i], 1.0, (0, 0, 0), eps, 300.0, 10, rt, at)[5]) for i in range(len(o)))
    print(eps, rt, "steps differ on", diff, "of", len(o), "mean steps", rec["steps"].mean())
