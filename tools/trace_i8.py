"""Per-warp phase timeline of one CTA of the INT8 step (tools/abl/libovx_trace.so, clock64 stamps):
points 0 loop top, 1 converted, 2 past the M-tile barrier, 3 MMAs issued, 4 post-phase done,
5 MMA complete (epilogue wait), 6 epilogue done, 7 before __syncthreads, 8 after,
9 post-phase face sums read, 10 update start (T read), 11 update stored."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2404_13683_b200 import build as B
B.LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "abl", "libovx_trace.so")
B._stale = lambda: False
import bench
from paper_2404_13683_b200 import Ovx, OVX_INT8
from paper_2404_13683_b200 import ovx as O
m, u0 = bench._workload(256)
s = Ovx(0)
s.set_stream(torch.cuda.current_stream())
s.load_model(m, OVX_INT8)
s.set_state(u0, u0, 0)
s.step(5)
torch.cuda.synchronize()
tr = np.zeros(16 * 16 * 16, dtype=np.uint64)
L = O.lib()
L.ovx_trace_read(tr.ctypes.data_as(ctypes.c_void_p))
tr = tr.reshape(16, 16, 16).astype(np.int64)
t0 = tr[tr > 0].min()
np.save("gpurun_out/trace_i8.npy", tr)
for hh in range(16):
    print(f"--- half-iteration {hh}")
    for w in range(16):
        row = tr[hh, w]
        print(f"w{w:2d} " + " ".join(f"{(x - t0) if x else -1:7d}" for x in row))
