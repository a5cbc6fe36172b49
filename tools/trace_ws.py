"""Per-warp phase timeline of one CTA of the warp-specialised INT8 step (step_i8ws built with
-DOVX_TRACE=<block>: tools/build_variant.sh trace -DOVX_TRACE=600 → tools/abl/libovx_trace.so;
clock64 stamps of layers 20-35 of that CTA on the C2 workload).
Converter warps 0-7: 0 loop top, 1 planes ready, 11 s_e scalars done, 2 gather done, 3 A stored,
4 past the group barrier, issuer (warps 0, 4): 5 D free, 6 MMAs issued; 10 plane L+3 finished,
9 plane L+4 issued.  Epilogue warps 8-15: 0 top, 1 MMAs complete, 2 D read (limbs done),
6 face sums exchanged, 7 update done."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2404_13683_b200 import build as B
B.LIB = os.environ.get("OVX_TRACE_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "abl", "libovx_trace.so")
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
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/trace_ws.npy", tr)
for k in range(16):
    print(f"--- layer {k + 20}")
    for w in range(16):
        print(f"w{w:2d} " + " ".join(f"{(x - t0) if x else -1:7d}" for x in tr[k, w]))


def d(w, a, b):
    v = [tr[k, w, b] - tr[k, w, a] for k in range(1, 16) if tr[k, w, a] and tr[k, w, b]]
    return float(np.mean(v)) if v else float("nan")


print("layer period (warp 0):", np.mean([tr[k, 0, 0] - tr[k - 1, 0, 0] for k in range(1, 16)]))
for w in (0, 1, 4, 5):
    print(f"conv w{w}: plane-wait {d(w,0,1):.0f} s_e {d(w,1,11):.0f} gather {d(w,11,2):.0f} convert+store {d(w,2,3):.0f} "
          f"bar {d(w,3,4):.0f} | issue: D-free wait {d(w,4,5):.0f} MMAs {d(w,5,6):.0f} | finish_plane {d(w,6 if w in (0, 4) else 4,10):.0f} "
          f"issue_plane {d(w,10,9):.0f}")
for w in (8, 9, 12, 13):
    print(f"epi w{w}: MMA wait {d(w,0,1):.0f} D read+limbs {d(w,1,2):.0f} face sums {d(w,2,6):.0f} update {d(w,6,7):.0f}")
