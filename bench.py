#!/usr/bin/env python
"""Benchmark of the OVFEM / TCOVFEM explicit time step on B200 (BASELINE.json metric:
element-updates/s; INT8 tensor-pipe use; error vs FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--path int8|fp64] [--impl ovx|reference]

A "step" is one full time step of the hot path (EBE product Σ_e K_e u_e through the INT8
tcgen05 path + fused central-difference update) over the C2 workload (256³ voxels,
BASELINE.json configs[1]).  Timing: W warm-up steps, then K steps bracketed by
barrier + cuda.synchronize, CUDA events on the launching stream, max over ranks.
Inputs are far larger than L2 (≈1.4 GB touched per step), so no L2 flush is needed.
`--impl reference` times the CPU oracle (oracle/, the only other implementation) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "element-updates/s"


def _peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def _workload(n: int):
    import workloads as wl
    m = wl.c2_block(n)
    u0 = wl.standing_wave(m, mvec=(16, 0, 0), U=(1.0, 0.0, 0.0))
    return m, u0


def _algorithmic_bytes(m) -> int:
    """u^{it} 24 B + u^{it-1} 24 B + u^{it+1} 24 B + w 8 B per node,
    1 B material per element, 1 B Dirichlet mask per node."""
    return 80 * m.n_nodes + m.n_elems + m.n_nodes


def cpu_oracle_sample(path_int8: bool, steps: int, n: int = 64) -> dict:
    """Time the oracle as it stands (single thread) on an n³ block of the C2 workload."""
    import oracle
    m, u0 = _workload(n)
    t0 = time.perf_counter()
    oracle.run(m.as_dict(), u0, u0, 0, steps, path=oracle.PATH_INT8 if path_int8 else oracle.PATH_FP64)
    dt = time.perf_counter() - t0
    return {"value": m.n_elems * steps / dt, "unit": METRIC, "cores": 1, "kind": "oracle",
            "sample": f"{n}^3 block of the C2 workload (ν=0.25 roller box, standing P wave), {steps} steps, "
                      f"{'INT8-path emulation (int128)' if path_int8 else 'FP64 path'}, 1 thread, "
                      f"{dt:.1f} s"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = 48
    import oracle
    m, u0 = _workload(n)
    po = oracle.PATH_INT8 if args.path == "int8" else oracle.PATH_FP64
    u, up = u0, u0
    for _ in range(args.warmup):
        u, up, _, _ = oracle.run(m.as_dict(), u, up, 0, 1, path=po)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        u, up, _, _ = oracle.run(m.as_dict(), u, up, 0, 1, path=po)
    dt = time.perf_counter() - t0
    value = m.n_elems * args.steps / dt
    sample = f"{n}^3 block of the C2 workload per step ({m.n_elems} elements), oracle {args.path} path, 1 thread"
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": "C2 256^3 homogeneous block (sampled: %d^3)" % n,
                                            "path": args.path},
           "cpu_baseline": {"value": value, "unit": METRIC, "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ovx", choices=["ovx", "reference"])
    ap.add_argument("--path", default="int8", choices=["int8", "fp64", "fp64_dense"])
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    from paper_2404_13683_b200 import Ovx, OVX_INT8, OVX_FP64, OVX_FP64_DENSE

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")

    m, u0 = _workload(args.n)
    path = {"int8": OVX_INT8, "fp64": OVX_FP64, "fp64_dense": OVX_FP64_DENSE}[args.path]
    stream = torch.cuda.Stream()
    s = Ovx(local)
    s.set_stream(stream)
    s.load_model(m, path)
    s.set_state(u0, u0, 0)
    s.step(args.warmup)
    s.sync()
    s.get_timers(reset=True)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    s.step(args.steps)
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    ms_kernel, launches = s.get_timers(reset=True)
    clocks = sampler.stop()
    s.check_finite()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    E = m.n_elems
    value = world * E * args.steps / (ms / 1e3)
    bytes_launch = _algorithmic_bytes(m)
    t_launch = ms_kernel / max(launches, 1) / 1e3
    achieved = bytes_launch / t_launch / 1e9
    pk = _peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{args.path}_{args.n}")

    # end to end through the public API with pinned host buffers (upload state, K steps, download)
    uh = torch.from_numpy(u0).pin_memory().numpy()
    uph = torch.from_numpy(u0).pin_memory().numpy()
    oh = torch.empty(3 * m.n_nodes, dtype=torch.float64).pin_memory().numpy()
    oph = torch.empty(3 * m.n_nodes, dtype=torch.float64).pin_memory().numpy()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.set_state(uh, uph, 0)
    s.step(args.steps)
    u_out, up_out, _ = s.get_state()
    e1.record(stream)
    barrier()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    del oh, oph, u_out, up_out

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    ops = 18432 * E / t_launch / 1e12 if path == OVX_INT8 else None
    out = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8xs8->s32 + f64" if path == OVX_INT8 else "f64",
        "data": "synthetic (seeded; C2 roller box with a standing P wave)",
        "config": {"workload": f"C2: {args.n}^3 homogeneous block (kappa=5/3, G=1, rho=1, ds=1), rollers",
                   "path": args.path, "elements": E, "nodes": m.n_nodes,
                   "parallelism": "single GPU" if world == 1 else f"replicas x{world} (no z-slab exchange yet)",
                   "l2": "inputs larger than L2 (%.2f GB touched per step)" % (bytes_launch / 1e9)},
        "dof_steps_per_s": 3 * m.n_nodes * world * args.steps / (ms / 1e3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                     "peak_src": pk["src"], "bytes_per_launch": bytes_launch,
                     "kernel_ms_per_launch": t_launch * 1e3},
        "int8_tops_useful": ops,
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": {"value": world * E * args.steps / (ms_e2e / 1e3), "unit": METRIC,
                "h2d_bytes_per_step": 2 * 24 * m.n_nodes / args.steps,
                "d2h_bytes_per_step": 2 * 24 * m.n_nodes / args.steps,
                "note": f"set_state(host pinned) + {args.steps} steps + get_state(host) per run"},
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_oracle_sample(path == OVX_INT8, steps=3)
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
