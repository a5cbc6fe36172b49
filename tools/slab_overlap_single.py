"""One z-slab rank as on a real multi-GPU run (the middle rank of three: both interfaces), alone on
one GPU, the exchange replaced by a no-op: serial schedule (one launch, then the interface update)
vs the overlapped schedule (edge z-chunks on a high-priority stream, interior chunks concurrently,
the interface update after the edge chunks).  Measures each schedule's own cost per GPU."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2404_13683_b200 import dist as D  # noqa: E402


class NoExchange:
    def exchange_up(self, slab, send, recv):
        pass

    def exchange_down(self, slab, send, recv):
        pass


world, n, steps = 3, 256, 20
m = wl.c2_block(8)
m.nx, m.ny, m.nz = n, n, n * world
m.mat = np.zeros(n * n * n * world, np.uint8)
m.dirichlet = wl.roller_mask(n, n, n * world)
u0 = wl.standing_wave(m, mvec=(16, 0, 0))
for path in (0, 1):
    run = D.SlabRun(m, 1, world, lambda lm, s: D.OvxCompute(lm, s, 0, path), NoExchange())
    run._comm = None
    for overlap in (False, True, False, True):
        run.set_state(u0, u0, 0)
        run.step(3, overlap=overlap)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run.step(steps, overlap=overlap)
        e1.record()
        torch.cuda.synchronize()
        print(f"path {path} overlap {overlap}: {e0.elapsed_time(e1) / steps:.4f} ms per step (one 256^3 slab, both interfaces)")
