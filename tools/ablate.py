"""Time the C2 INT8 step with ablated libovx builds (tools/abl/libovx_abl<k>.so).

The numbers in DESIGN.md §6.1 came from a copy of the shared-memory-A kernel of commit c550195
patched under `#if OVX_ABLATE == k` (built with tools/build_variant.sh abl<k> -DOVX_ABLATE=k):
1 the 3 main-block MMAs per array skipped, 2 the conversion's DMUL/F2I replaced by a bit move,
3 the limb recombination replaced by an XOR, 4 the update-operand loads skipped, 5 the A stores
skipped, 7 the 2 identity-fold MMAs per array skipped.  The results are wrong by construction; only
the timing is of interest."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_13683_b200 import build as B
k = int(sys.argv[1])
B.LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "abl", f"libovx_abl{k}.so")
B._stale = lambda: False
import bench
from paper_2404_13683_b200 import Ovx, OVX_INT8
m, u0 = bench._workload(256)
s = Ovx(0)
s.set_stream(torch.cuda.current_stream())
s.load_model(m, OVX_INT8)
s.set_state(u0, u0, 0)
s.step(5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); s.step(20); e1.record(); torch.cuda.synchronize()
print(f"ablate {k}: {e0.elapsed_time(e1) / 20:.4f} ms/step")
