"""Small cases for compute-sanitizer (racecheck / memcheck / synccheck): one INT8, FP64 and dense step
and an apply on a ragged grid, plus a 2-slab overlapped step and a damped 2-slab step; round 2 adds
the direct N-stage path (OVX_INT8_DIRECT), the library-driven distributed schedule on a loopback
group (ovx_create_group / ovx_step_group) and, with OVX_I8_KERNEL=x, the step_i8x kernels.  The INT8
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
for path in (0, 1, 2, 3, 5):
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
from paper_2404_13683_b200 import ovx as O  # noqa: E402
ranks = O.Ovx.create_group(2, [0, 0])
nn2 = (m2.nx + 1) * (m2.ny + 1)
for r, s in enumerate(ranks):
    ez0, ez1 = O.get_partition(m2.nz, 2, r)
    s.set_grid(m2.nx, m2.ny, m2.nz, m2.ds)
    s.set_materials(m2.rho, m2.kappa, m2.G)
    s.set_element_materials(m2.mat[max(ez0 - 1, 0) * m2.nx * m2.ny: ez1 * m2.nx * m2.ny])
    s.set_dirichlet(m2.dirichlet[ez0 * nn2:(ez1 + 1) * nn2])
    s.setup_elements(0, 8)
    s.set_dt(m2.dt)
    s.set_state(u2[3 * nn2 * ez0:3 * nn2 * (ez1 + 1)], u2[3 * nn2 * ez0:3 * nn2 * (ez1 + 1)], 0)
O.step_group(ranks, 2)
for s in ranks:
    s.sync()
print("library group ok", flush=True)
