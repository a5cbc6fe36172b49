"""BASELINE configs 3 and 4 on ONE B200 (context for the z-slab runs): C3 512³ two-layer soil over
bedrock with a Ricker source, C4 891×352×1056 multi-layer ground + stiff cylinder (1.0e9 DOF).
Per config and path: device time per step (CUDA events over K steps after W warm-up steps),
element-updates/s, DOF-steps/s, finiteness, and the INT8-vs-FP64 relative L2 of the final field."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2404_13683_b200 import OVX_FP64, OVX_INT8, Ovx  # noqa: E402


def run(m, path, steps, warm):
    s = Ovx(0)
    s.set_stream(torch.cuda.current_stream())
    s.load_model(m, path)
    z = np.zeros(3 * m.n_nodes)
    s.set_state(z, z, 0)
    s.step(warm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.step(steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    s.check_finite()
    u, _, it = s.get_state(with_prev=False)
    del s
    torch.cuda.empty_cache()
    return ms, u


out = {}
for name, m, steps, warm in (("C3 512^3 two-layer", wl.c3_two_layer(512, steps=400), 300, 20),
                             ("C4 891x352x1056 ground (1.0e9 DOF)", wl.c4_ground(steps=200), 150, 10)):
    r = {"elements": m.n_elems, "dof": 3 * m.n_nodes, "steps_timed": steps, "after_warmup": warm}
    us = {}
    for pname, path in (("int8", OVX_INT8), ("fp64", OVX_FP64)):
        ms, u = run(m, path, steps, warm)
        us[pname] = u
        r[pname] = {"ms_per_step": ms, "element_updates_per_s": m.n_elems / (ms / 1e3),
                    "dof_steps_per_s": 3 * m.n_nodes / (ms / 1e3)}
    n64 = np.linalg.norm(us["fp64"])
    r["l2_int8_vs_fp64"] = float(np.linalg.norm(us["int8"] - us["fp64"]) / n64) if n64 > 0 else None
    r["field_norm"] = float(n64)
    out[name] = r
    print(name, json.dumps(r), flush=True)
with open("gpurun_out/configs_run.json", "w") as f:
    json.dump(out, f, indent=1)
