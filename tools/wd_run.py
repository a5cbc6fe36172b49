"""Run C2 INT8 steps on the watchdog build (tools/abl/libovx_wd.so): a stuck mbarrier wait prints its
block / thread / source line and traps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_13683_b200 import build as B
B.LIB = os.environ.get("OVX_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "abl", "libovx_wd.so")
B._stale = lambda: False
import bench
from paper_2404_13683_b200 import Ovx, OVX_INT8
m, u0 = bench._workload(256)
s = Ovx(0)
s.load_model(m, OVX_INT8)
s.set_state(u0, u0, 0)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 50):
    s.step(1)
    s.sync()
print("done", flush=True)
