"""NEXT-4 on the GPU: C2 256³ INT8 step time for M = 8, 6, 4 INT8 stages (a = 2^{7M}; byte slices of
v + 2^{7M}: 4, 3, 2 half-word arrays -> 20, 15, 10 MMAs per M-tile and layer) and each variant's
relative L2 distance to the FP64 path after 20 steps from the same field (Table 3's ordering)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2404_13683_b200 import OVX_FP64, OVX_INT8, Ovx  # noqa: E402

m, u0 = bench._workload(256)
out = {}


def run(path, stages, steps=20, warm=5):
    s = Ovx(0)
    s.set_stream(torch.cuda.current_stream())
    s.load_model(m, path, stages)
    s.set_state(u0, u0, 0)
    s.step(warm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.step(steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    s.set_state(u0, u0, 0)
    s.step(steps)
    u, _, _ = s.get_state()
    return ms, u


ms64, u64 = run(OVX_FP64, 8)
out["fp64"] = {"ms_per_step": ms64}
for M in (8, 6, 4):
    ms, u = run(OVX_INT8, M)
    out[f"int8_M{M}"] = {"ms_per_step": ms, "element_updates_per_s": m.n_elems / (ms / 1e3),
                         "rel_l2_vs_fp64_20_steps": float(np.linalg.norm(u - u64) / np.linalg.norm(u64))}
    print(M, json.dumps(out[f"int8_M{M}"]), flush=True)
json.dump(out, open("gpurun_out/stages_timing.json", "w"), indent=1)
