"""E1 (NEXT-2): the paper's rebar experiment at ds = 2 mm on one B200 — the like-for-like workload of
PAPER.md Table 4 (A100 80 GB: TCOVFEM INT8 M=8 loop 14.2 s / matvec kernel 9.62 s; OVFEM FP64
48.3 s / 43.3 s for 16,384 steps; context only, other hardware).

Runs 162×64×192 elements (steel rebar in concrete), the Table 1 source and 8 receivers (24 channels),
Rayleigh damping (ζ input, default 0.01), 16,384 steps, on the INT8, factored FP64 and factored VFEM
paths; reports device time of the step kernels (CUDA events), the loop's wall time (host enqueue +
device, state resident), and the paper's Err metric of the INT8 traces against the FP64
traces.  Product path only (libovx.so); no oracle.

    python tools/e1_table4.py [--steps 16384] [--zeta 0.01] [--out gpurun_out/e1_table4.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as wl  # noqa: E402
from paper_2404_13683_b200 import OVX_FP64, OVX_INT8, OVX_VFEM, Ovx  # noqa: E402


def err_metric(obs, ref):
    """Err = (1/n_c) Σ_channels Σ_t (u_obs − u_ref)² / Σ_t u_ref²."""
    den = np.sum(ref * ref, axis=1)
    live = den > 0
    return float(np.mean(np.sum((obs[live] - ref[live]) ** 2, axis=1) / den[live]))


def run(path, m, steps):
    s = Ovx(0)
    s.load_model(m, path)
    s.set_receivers(m.receivers, steps)
    z = np.zeros(3 * m.n_nodes)
    s.set_state(z, z, 0)
    s.step(8)                        # warm-up (module load, constants)
    s.sync()
    s.set_state(z, z, 0)
    s.set_receivers(m.receivers, steps)
    s.sync()
    s.get_timers(reset=True)
    t0 = time.perf_counter()
    s.step(steps)
    s.sync()
    wall = time.perf_counter() - t0
    ms, n = s.get_timers()
    s.check_finite()
    return {"kernel_s": ms / 1e3, "loop_s": wall, "launches": n,
            "elem_updates_per_s": m.n_elems * steps / (ms / 1e3)}, s.get_traces()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=16384)
    ap.add_argument("--zeta", type=float, default=0.01)
    ap.add_argument("--out", default="gpurun_out/e1_table4.json")
    a = ap.parse_args()
    m = wl.e1_rebar(2.0, steps=a.steps, zeta=a.zeta)
    out = {"workload": "E1 rebar model, ds = 2 mm, 162x64x192 elements (1.99 M), 16,384 steps at dt = 5e-8 s"
                       if a.steps == 16384 else f"E1 rebar model, ds = 2 mm, {a.steps} steps",
           "zeta": a.zeta, "paper_a100_table4_s": {"int8_loop": 14.2, "int8_kernel": 9.62,
                                                    "fp64_loop": 48.3, "fp64_kernel": 43.3}}
    tr = {}
    for name, path in (("int8", OVX_INT8), ("fp64", OVX_FP64), ("vfem", OVX_VFEM)):
        out[name], tr[name] = run(path, m, a.steps)
    n = tr["int8"].shape[-1]
    out["err_int8_vs_fp64"] = err_metric(tr["int8"].reshape(-1, n), tr["fp64"].reshape(-1, n))
    out["err_vfem_vs_ovfem_fp64"] = err_metric(tr["vfem"].reshape(-1, n), tr["fp64"].reshape(-1, n))
    out["peak_trace_amplitude"] = float(np.abs(tr["fp64"]).max())
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
