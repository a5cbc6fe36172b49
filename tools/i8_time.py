"""Time the C2 INT8 step (256³, the bench workload) of the kernel variant selected by the environment
(OVX_I8_KERNEL, OVX_I8X_LAYOUT, OVX_ZCHUNKS): ms per step over 40 steps after 5 warm-up steps,
CUDA events on the launching stream; prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if os.environ.get("OVX_LIB_PATH"):       # an ablation / variant build (tools/build_variant.sh)
    from paper_2404_13683_b200 import build as B
    B.LIB = os.environ["OVX_LIB_PATH"]
    B._stale = lambda: False
import bench
from paper_2404_13683_b200 import Ovx, OVX_INT8
m, u0 = bench._workload(256)
s = Ovx(0)
st = torch.cuda.current_stream()
s.set_stream(st)
s.load_model(m, int(os.environ.get("OVX_PATH", OVX_INT8)), stages=int(os.environ.get("OVX_STAGES", "8")))
s.set_state(u0, u0, 0)
s.step(5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); s.step(40); e1.record(st); torch.cuda.synchronize()
env = {k: os.environ[k] for k in ("OVX_I8_KERNEL", "OVX_I8X_LAYOUT", "OVX_ZCHUNKS", "OVX_STAGES", "OVX_LIB_PATH", "OVX_PATH")
       if k in os.environ}
print(json.dumps({"env": env, "ms_per_step": e0.elapsed_time(e1) / 40}))
