"""Small cases for compute-sanitizer (racecheck / memcheck / synccheck): one INT8, FP64 and dense step
and an apply on a ragged grid, plus a 2-slab overlapped step and a damped 2-slab step.  The INT8
kernel keeps its A operand in TMEM: racecheck covers the shared-memory traffic; the TMEM hand-over
between the two M-tiles is ordered by the MMA-completion mbarriers (synccheck)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2404_13683_b200 import Ovx, dist as D  # noqa: E402

m = wl.small_random(40, 8, 70, ds=0.01, dt=1e-6)
wl.point_source(m, 17, 3, 35, 1, 1e5, 2e-5, 4, scale=1.0)
u = wl.random_field(m) * 1e-3
for path in (0, 1, 2, 3):
    s = Ovx(0)
    s.load_model(m, path)
    s.set_state(u, u, 0)
    s.step(2)
    s.apply_K(u)
    s.sync()
    print("path", path, "ok", flush=True)
m2 = wl.small_random(33, 8, 60, ds=0.5, dt=1e-5)
g = D.SlabGroup(m2, 2, lambda lm, sl: D.OvxCompute(lm, sl, 0, 0))
u2 = wl.random_field(m2) * 1e-6
g.set_state(u2, u2, 0)
g.step(2, overlap=True)
m2.alpha, m2.beta = 0.02 / m2.dt, 0.03 * m2.dt      # damped z-slab step (third buffer rotation)
g2 = D.SlabGroup(m2, 2, lambda lm, sl: D.OvxCompute(lm, sl, 0, 0))
g2.set_state(u2, u2, 0)
g2.step(2)
import torch  # noqa: E402
torch.cuda.synchronize()
print("slabs ok", flush=True)
