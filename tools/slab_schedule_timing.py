"""Serial vs overlapped z-slab step schedule, all ranks of a C5-like grid on one GPU (loopback
exchange): per-step device time of both schedules (the ranks' kernels share the one device, so this
measures the schedule's launch / wave behaviour, not multi-GPU scaling)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2404_13683_b200 import dist as D  # noqa: E402

world, n, steps = 3, 256, 10
m = wl.c2_block(8)
m.nx, m.ny, m.nz = n, n, n * world
m.mat = np.zeros(n * n * n * world, np.uint8)
m.dirichlet = wl.roller_mask(n, n, n * world)
u0 = wl.standing_wave(m, mvec=(16, 0, 0))
for path in (0, 1):
    g = D.SlabGroup(m, world, lambda lm, s: D.OvxCompute(lm, s, 0, path))
    for overlap in (False, True, False, True):
        g.set_state(u0, u0, 0)
        g.step(2, overlap=overlap)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.step(steps, overlap=overlap)
        e1.record()
        torch.cuda.synchronize()
        print(f"path {path} overlap {overlap}: {e0.elapsed_time(e1) / steps:.3f} ms per step ({world} slabs of {n}^3)")
