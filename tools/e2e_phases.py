"""Host-timed phases of the bench's end-to-end region (C2 256³): pinned upload, K steps, pinned readback."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2404_13683_b200 import Ovx, OVX_INT8  # noqa: E402

m = wl.c2_block(256)
u0 = wl.standing_wave(m, mvec=(16, 0, 0))
s = Ovx(0)
s.load_model(m, OVX_INT8)
uh = torch.from_numpy(u0).pin_memory().numpy()
uout = torch.empty(u0.size, dtype=torch.float64).pin_memory().numpy()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.set_state(uh, uh, 0)
    t1 = time.perf_counter()
    s.step(20)
    s.sync()
    t2 = time.perf_counter()
    s.get_state(out_u=uout, with_prev=False)
    t3 = time.perf_counter()
    gb = u0.nbytes / 1e9
    print(f"rep {rep}: set_state {1e3*(t1-t0):.1f} ms ({2*gb/(t1-t0):.1f} GB/s)  step(20) {1e3*(t2-t1):.1f} ms  "
          f"get_state {1e3*(t3-t2):.1f} ms ({gb/(t3-t2):.1f} GB/s)")
x = torch.empty(u0.size, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
x.copy_(torch.from_numpy(uh), non_blocking=True)
torch.cuda.synchronize()
print(f"torch pinned H2D {u0.nbytes/1e9/(time.perf_counter()-t0):.1f} GB/s")
