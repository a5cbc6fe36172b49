#!/usr/bin/env python
"""Benchmark of the OVFEM / TCOVFEM explicit time step on B200 (BASELINE.json metric:
element-updates/s at 1/2/4/8 B200; INT8 tensor-pipe use; error vs FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--path int8|fp64|fp64_dense|vfem|vfem_dense] [--impl ovx|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A "step" is one full time step of the hot path (element-by-element product Σ_e K_e u_e through
the INT8 tcgen05 path, fused scatter + central-difference update) over the whole grid.
  N = 1: C2 (BASELINE.json configs[1]): 256³ voxels, homogeneous roller box, standing P wave.
  N > 1: C5 (configs[4]) weak scaling: 256 × 256 × 256·N voxels, one 256³ z-slab per GPU,
         interface forces exchanged with NCCL point-to-point every step.
Timing: W warm-up steps, then K steps bracketed by barrier + cuda.synchronize, CUDA events on the
launching stream, max over ranks.  Inputs are far larger than L2 (≈1.4 GB touched per step per
GPU), so no L2 flush is needed.  `--impl reference` times the CPU oracle (oracle/) on a bounded
sample of the same workload (the reference is a paper; there is no other implementation).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "element-updates/s"
N_EDGE = 256


def _peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback (B200_PROFILING.md)"}


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


def _slab_workload(n: int, world: int, rank: int):
    """This rank's z-slab of the C5 weak-scaling grid (BASELINE configs[4]):
    n × n × (n·world) elements, ds = 1 m, soil / rock alternating every 64 element layers (C3
    materials), the 4 bottom corners fixed, a Ricker z-force (f0 = 25 Hz) at the top-surface
    centre, dt = 1e-4 s; the initial field is a smooth standing wave along x (so that every element
    carries data from the first step).  Built locally per rank: (local model, Slab, u0 of planes
    ez0..ez1)."""
    import workloads as wl
    from paper_2404_13683_b200 import dist as D
    from types import SimpleNamespace
    nz = n * world
    ez0, ez1 = D.partition(nz, world, rank)
    slab = D.Slab(rank, world, ez0, ez1)
    rho, kappa, G = wl._materials(wl.SOIL, wl.ROCK)
    nzl = ez1 - ez0
    lay = ((np.arange(ez0 - (1 if rank > 0 else 0), ez1) // 64) % 2).astype(np.uint8)
    mats = np.broadcast_to(lay[:, None], (lay.size, n * n)).reshape(-1)
    nn2 = (n + 1) * (n + 1)
    mask = np.zeros((nzl + 1) * nn2, np.uint8)
    if rank == 0:
        for ix, iy in ((0, 0), (n, 0), (0, n), (n, n)):
            mask[ix + (n + 1) * iy] = 7
    dt, f0 = 1e-4, 25.0
    steps = 1 << 14
    if rank == world - 1:
        src = np.array([(n // 2) + (n + 1) * (n // 2) + nzl * nn2], dtype=np.int64)
        amp = (1.0e6 * wl.ricker(np.arange(steps) * dt, f0, 1.2 / f0)).reshape(1, -1)
        axis = np.array([2], dtype=np.int32)
    else:
        src, amp, axis = np.zeros(0, np.int64), np.zeros((0, 1)), np.zeros(0, np.int32)
    lm = SimpleNamespace(nx=n, ny=n, nz=nzl, ds=1.0, rho=rho, kappa=kappa, G=G, dt=dt,
                         mat=np.ascontiguousarray(mats[(n * n if rank > 0 else 0):]),
                         mat_below=np.ascontiguousarray(mats[:n * n]) if rank > 0 else None,
                         dirichlet=mask, src_node=src, src_axis=axis, amp=amp)
    k = math.pi * 16 / n
    x = np.arange(n + 1, dtype=np.float64)
    u = np.zeros((nzl + 1, n + 1, n + 1, 3))
    u[..., 0] = 1e-3 * np.sin(k * x)[None, None, :]
    return lm, slab, u.reshape(-1)


def _algorithmic_bytes(nn: int, ne: int) -> int:
    """u^{it} 24 B + u^{it-1} 24 B + u^{it+1} 24 B + w 8 B per node,
    1 B material per element, 1 B Dirichlet mask per node."""
    return 80 * nn + ne + nn


def _cpu_info() -> dict:
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def _oracle_path(path_name: str):
    import oracle
    po = {"int8": oracle.PATH_INT8, "vfem": oracle.PATH_VFEM, "vfem_dense": oracle.PATH_VFEM}.get(path_name, oracle.PATH_FP64)
    what = {"int8": "INT8-path emulation (int128)", "vfem": "VFEM path", "vfem_dense": "VFEM path"}.get(path_name, "FP64 path")
    return po, what


def _set_omp_threads(n: int) -> None:
    """Thread count of the oracle's OpenMP element loop (libgomp reads it per parallel region via
    omp_set_num_threads; results are bit-identical for any count)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


def _oracle_rate(path_name: str, n: int, steps: int, threads: int) -> tuple[float, float]:
    """(element-updates/s, seconds) of the oracle as it stands on an n³ block of the C2 workload."""
    import oracle
    po, _ = _oracle_path(path_name)
    m, u0 = _workload(n)
    _set_omp_threads(threads)
    t0 = time.perf_counter()
    oracle.run(m.as_dict(), u0, u0, 0, steps, path=po)
    dt = time.perf_counter() - t0
    return m.n_elems * steps / dt, dt


def _sample_edge(path_name: str, threads: int, budget_s: float, steps: int) -> int:
    """Largest n ≤ 256 (the C2 edge) whose `steps` oracle steps fit the time budget, from a 64³
    calibration step (the oracle's cost is linear in the element count)."""
    rate, _ = _oracle_rate(path_name, 64, 1, threads)
    n = int((budget_s * rate / steps) ** (1.0 / 3.0))
    return max(16, min(N_EDGE, n))


def cpu_oracle_sample(path_name: str, budget_s: float = 20.0) -> dict:
    """The oracle as it stands, timed on this host: (i) all cores (OpenMP over the independent
    element forces; SURVEY §8(d) "oracle timing"), on the largest block of the C2 workload whose 2
    steps fit ~budget_s (the full 256³ grid on a large host), and (ii) one thread on a 64³ block."""
    info = _cpu_info()
    cores = info["nproc"] or 1
    _, what = _oracle_path(path_name)
    n = _sample_edge(path_name, cores, budget_s, 2)
    v_all, t_all = _oracle_rate(path_name, n, 2, cores)
    v_one, t_one = _oracle_rate(path_name, 64, 2, 1)
    return {"value": v_all, "unit": METRIC, "cores": cores, "kind": "oracle",
            "sample": f"{n}^3 block of the C2 workload (ν=0.25 roller box, standing P wave; full C2 = 256^3), "
                      f"2 steps, {what}, OpenMP over element forces on {cores} threads, {t_all:.1f} s",
            "cpu_model": info["cpu_model"], "nproc": info["nproc"], "same_config": n == N_EDGE,
            "single_thread": {"value": v_one, "unit": METRIC, "cores": 1,
                              "sample": f"64^3 block, 2 steps, 1 thread, {t_one:.1f} s"}}


def run_reference(args) -> None:
    """The base contract's reference arm for this tier: the CPU oracle as it stands, on all host
    cores, timed per step on the largest block of the C2 workload that keeps the whole
    --steps/--warmup run within a few minutes (the full 256³ grid when the host is large enough)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    info = _cpu_info()
    cores = info["nproc"] or 1
    po, what = _oracle_path(args.path)
    n = _sample_edge(args.path, cores, args.ref_budget, args.steps + args.warmup)
    m, u0 = _workload(n)
    _set_omp_threads(cores)
    u, up = u0, u0
    for _ in range(args.warmup):
        u, up, _, _ = oracle.run(m.as_dict(), u, up, 0, 1, path=po)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        u, up, _, _ = oracle.run(m.as_dict(), u, up, 0, 1, path=po)
    dt = time.perf_counter() - t0
    value = m.n_elems * args.steps / dt
    sample = (f"{n}^3 block of the C2 workload per step ({m.n_elems} elements; full C2 = 256^3), oracle {what}, "
              f"OpenMP over element forces on {cores} threads")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": f"C2 256^3 homogeneous block (sampled: {n}^3)",
                                            "path": args.path, "same_config": n == N_EDGE},
           "cpu_baseline": {"value": value, "unit": METRIC, "cores": cores, "kind": "oracle", "sample": sample,
                            "cpu_model": info["cpu_model"], "nproc": info["nproc"]},
           "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


class Single:
    """One GPU: the whole C2 grid in one context."""

    def __init__(self, n, path, local, stream):
        from paper_2404_13683_b200 import Ovx
        self.m, self.u0 = _workload(n)
        self.s = Ovx(local)
        self.s.set_stream(stream)
        self.s.load_model(self.m, path)
        self.nn, self.ne = self.m.n_nodes, self.m.n_elems
        self.launches_per_step = 1

    def set_state(self, u, up):
        self.s.set_state(u, up, 0)

    def step(self, k):
        self.s.step(k)

    def get_state(self, out_u=None):
        """The step's result: the final displacement field u^{K} (into out_u, e.g. pinned)."""
        return self.s.get_state(out_u=out_u, with_prev=False)[0]


class ShardedLib:
    """One rank of the C5 z-slab decomposition, stepped by the library (ovx_create_dist: a
    library-owned NCCL communicator; ovx_step runs the overlapped schedule — edge z-chunks on a
    high-priority stream, interior chunks concurrently, NCCL P2P interface exchange, interface
    update).  The NCCL unique id travels through torch.distributed."""

    def __init__(self, n, path, local, stream, world, rank):
        import torch.distributed as dist
        from paper_2404_13683_b200 import ovx as O
        lm, slab, self.u0 = _slab_workload(n, world, rank)
        uid = [O.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        s = O.Ovx.create_dist(local, rank, world, uid[0])
        s.set_stream(stream)
        s.set_grid(n, n, n * world, lm.ds)               # global layer count; the library derives the slab
        assert (s.ez0, s.nz) == (slab.ez0, slab.nzl)
        s.set_materials(lm.rho, lm.kappa, lm.G)
        s.set_element_materials(lm.mat if lm.mat_below is None else np.concatenate([lm.mat_below, lm.mat]))
        s.set_dirichlet(lm.dirichlet)
        s.setup_elements(path, 8)
        s.set_dt(lm.dt)
        nn2 = (n + 1) * (n + 1)
        s.set_sources(lm.src_node + slab.ez0 * nn2, lm.src_axis, lm.amp)   # global node ids
        self.s = s
        self.nn = (n + 1) * (n + 1) * (slab.nzl + 1)
        self.ne = n * n * slab.nzl
        self.launches_per_step = None

    def set_state(self, u, up):
        self.s.set_state(u, up, 0)

    def step(self, k):
        if self.launches_per_step is None and k > 0:
            _, n0 = self.s.get_timers()
            self.s.step(1)
            _, n1 = self.s.get_timers()
            self.launches_per_step = n1 - n0
            k -= 1
        self.s.step(k)

    def get_state(self, out_u=None):
        return self.s.get_state(out_u=out_u, with_prev=False)[0]


class Sharded:
    """One rank of the C5 z-slab decomposition driven from Python (dist.py; the test hook with
    several ranks on one device and a gloo host-staged exchange, or OVX_BENCH_DIST=python)."""

    def __init__(self, n, path, local, stream, world, rank):
        from paper_2404_13683_b200 import dist as D
        self.lm, self.slab, self.u0 = _slab_workload(n, world, rank)
        self.c = D.OvxCompute(self.lm, self.slab, local, path, stream=stream)
        self.t = D.TorchTransport() if os.environ.get("OVX_BENCH_BACKEND", "nccl") == "nccl" else D.HostStagedTransport()
        self.s = self.c.ovx
        self.nn = (n + 1) * (n + 1) * (self.slab.nzl + 1)
        self.ne = n * n * self.slab.nzl
        self.run = D.SlabRun.__new__(D.SlabRun)       # the overlapped schedule of dist.SlabRun
        self.run.slab, self.run.compute, self.run.transport = self.slab, self.c, self.t
        self.run._comm = None
        self.launches_per_step = None                    # counted on the first step

    def set_state(self, u, up):
        self.c.set_state(u, up, 0)

    OVERLAP = os.environ.get("OVX_BENCH_SCHEDULE", "overlap") == "overlap"

    def step(self, k):
        """Overlapped schedule (default; OVX_BENCH_SCHEDULE=serial for the other): the edge
        z-chunks on a high-priority stream, the interior chunks concurrently, the NCCL exchange and
        the interface update after the edge chunks.  Measured for one 256³ slab alone on a GPU: 13 µs
        per step more than one launch, against a 30-60 µs serial exchange."""
        if self.launches_per_step is None and k > 0:
            _, n0 = self.s.get_timers()
            self.run.step(1, overlap=self.OVERLAP)
            _, n1 = self.s.get_timers()
            self.launches_per_step = n1 - n0
            k -= 1
        self.run.step(k, overlap=self.OVERLAP)

    def get_state(self, out_u=None):
        return self.s.get_state(out_u=out_u, with_prev=False)[0]


def _spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: relaunch this command as N ranks (one process
    per GPU, torch.distributed.run on 127.0.0.1); refuse (exit 2) when fewer than N GPUs exist."""
    import socket
    import torch
    if os.environ.get("OVX_BENCH_DEVICE") is None and torch.cuda.device_count() < n:
        print(f"bench.py: --gpus {n} needs {n} GPUs, {torch.cuda.device_count()} visible", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ovx", choices=["ovx", "reference"])
    ap.add_argument("--path", default="int8", choices=["int8", "fp64", "fp64_dense", "vfem", "vfem_dense"])
    ap.add_argument("--n", type=int, default=N_EDGE)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp64-companion", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: seconds of oracle work the whole run may take (sets the sample size)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args.gpus))

    import torch
    import torch.distributed as dist
    from paper_2404_13683_b200 import OVX_INT8, OVX_FP64, OVX_FP64_DENSE, OVX_VFEM, OVX_VFEM_DENSE

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("OVX_BENCH_DEVICE") is not None:   # test hook: all ranks on one device
        local = int(os.environ["OVX_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    # OVX_BENCH_BACKEND=gloo (test hook, with OVX_BENCH_DEVICE): several ranks on one GPU, the
    # interface messages staged through host memory; the benchmark itself uses NCCL
    backend = os.environ.get("OVX_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    paths = {"int8": OVX_INT8, "fp64": OVX_FP64, "fp64_dense": OVX_FP64_DENSE, "vfem": OVX_VFEM,
             "vfem_dense": OVX_VFEM_DENSE}
    path = paths[args.path]
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_run(path_id: int, steps: int, warmup: int, sample_clocks: bool):
        if world == 1:
            R = Single(args.n, path_id, local, stream)
        elif backend == "nccl" and os.environ.get("OVX_BENCH_DIST", "library") == "library":
            try:
                R = ShardedLib(args.n, path_id, local, stream, world, rank)
            except Exception as ex:   # e.g. OVX_ENCCL: fall back to the Python-driven schedule
                print(f"bench.py: library z-slab path unavailable ({ex}); using dist.py", file=sys.stderr)
                os.environ["OVX_BENCH_DIST"] = "python"
                R = Sharded(args.n, path_id, local, stream, world, rank)
        else:
            R = Sharded(args.n, path_id, local, stream, world, rank)
        R.set_state(R.u0, R.u0)
        try:
            R.step(warmup)
        except Exception as ex:   # the library's NCCL schedule failed at run time: the Python-driven one
            if not isinstance(R, ShardedLib):
                raise
            print(f"bench.py: library z-slab step failed ({ex}); using dist.py", file=sys.stderr)
            os.environ["OVX_BENCH_DIST"] = "python"
            R = Sharded(args.n, path_id, local, stream, world, rank)
            R.set_state(R.u0, R.u0)
            R.step(warmup)
        barrier()
        R.s.get_timers(reset=True)
        sampler = ClockSampler(local) if sample_clocks else None
        if sampler:
            sampler.start()
            time.sleep(0.3)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record(stream)
        R.step(steps)
        ev1.record(stream)
        barrier()
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        clocks = sampler.stop() if sampler else None
        return R, ms, clocks

    R, ms, clocks = timed_run(path, args.steps, args.warmup, True)
    R.s.check_finite()
    # dominant kernel: the step kernel's own CUDA-event time (Single: events bracket the launches)
    kernel_ms = None
    if world == 1:
        k_ms, launches = R.s.get_timers(reset=True)
        kernel_ms = k_ms / max(launches, 1)
    E_total = R.ne * world
    value = E_total * args.steps / (ms / 1e3)

    # end to end through the public API with pinned host buffers (upload state, K steps, download)
    uh = torch.from_numpy(R.u0).pin_memory().numpy()
    uout = torch.empty(R.u0.size, dtype=torch.float64).pin_memory().numpy()   # pinned result buffer
    def e2e_once():
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        th0 = time.perf_counter()
        e0.record(stream)
        R.set_state(uh, uh)
        th1 = time.perf_counter()
        R.step(args.steps)
        u_fin = R.get_state(out_u=uout)
        e1.record(stream)
        barrier()
        th2 = time.perf_counter()
        return u_fin, max_over_ranks(e0.elapsed_time(e1)), {"set_state": 1e3 * (th1 - th0), "total": 1e3 * (th2 - th0)}

    # two passes over the same region: the first touches the freshly pinned pages (the first upload
    # from a new pinned buffer measured 15-420 ms on different boxes); the second is reported
    e2e_once()
    u_final, ms_e2e, e2e_host_ms = e2e_once()

    # FP64 CUDA-core path measured beside the INT8 path (same workload, same clock record)
    R_nn, R_ne, R_lps = R.nn, R.ne, R.launches_per_step
    # INT8 MMA work actually issued per launch (padding, ⊗I₂ structure, the Eq. 9 diagonal K-steps and
    # the recomputed halo elements included): tiles × computed layers × 2 M-tiles × 20 MMAs of
    # M128·N48·K32 (393,216 ops each); computed layers = nz + (z-chunks − 1)
    issued_ops = None
    if world == 1 and path == OVX_INT8:
        ctas = R.s.get_launch_config()[0]
        txy = -(-(args.n + 1) // 31) * -(-(args.n + 1) // 7)
        issued_ops = txy * (args.n + ctas // txy - 1) * 2 * 20 * 393216
    if world > 1:   # the job's launches: step kernels of every rank + the interface updates
        t = torch.tensor([float(R_lps)], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        R_lps = int(t.item())
    fp64 = None
    if path == OVX_INT8 and not args.no_fp64_companion:
        del R
        torch.cuda.empty_cache()
        R64, ms64, _ = timed_run(OVX_FP64, args.steps, args.warmup, False)
        fp64 = {"value": E_total * args.steps / (ms64 / 1e3), "ms_per_step": ms64 / args.steps}
        if world == 1:   # BASELINE "L2 err vs FP64": the same K steps from the same field on both paths
            R64.set_state(uh, uh)
            R64.step(args.steps)
            u64 = R64.get_state()
            fp64["l2_err_int8_vs_fp64"] = float(np.linalg.norm(u_final - u64) / np.linalg.norm(u64))
            fp64["l2_err_steps"] = args.steps
            del u64
        del R64

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    bytes_launch = _algorithmic_bytes(R_nn, R_ne) if world == 1 else None
    pk = _peaks()
    roof = None
    if world == 1:
        achieved = bytes_launch / (kernel_ms / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"{args.path}_{args.n}")
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_src": pk["src"],
                "bytes_per_launch": bytes_launch, "kernel_ms_per_launch": kernel_ms,
                "kernel": {0: "step_i8ws<M=8> (warp-specialised)", 1: "step_f64", 2: "step_v1<FP64_DENSE>", 3: "step_f64<VF>",
                           4: "step_v1<FP64_DENSE> (VFEM matrices)"}[path]}
    # SURVEY §8(d)'s per-run ncu figures for the dominant kernel, from the committed capture of the
    # same command (profiles/; ncu numbers are never taken inside this timed run)
    ncu = None
    prof = {0: "r2_int8_ws_final", 1: "r2_fp64_final"}.get(path)
    if world == 1 and prof and os.path.exists(os.path.join(ROOT, "profiles", prof + ".json")):
        try:
            l0 = json.load(open(os.path.join(ROOT, "profiles", prof + ".json")))["launches"][0]
            g = lambda k: l0.get(k, [None])[0]
            _scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6}
            gu = lambda k: l0[k][0] * _scale[l0[k][1]]   # ncu picks the unit per value: GB / ms
            ncu = {"source": f"profiles/{prof}.md", "kernel_ms": gu("gpu__time_duration.sum"),
                   "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "tensor_pipe_active_pct": g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                   "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                   "dram_gbytes_per_launch": gu("dram__bytes_read.sum") + gu("dram__bytes_write.sum"),
                   "warp_instructions": g("smsp__inst_executed.sum")}
        except Exception:
            ncu = None
    # the issue-slot roofline of the same kernel (the INT8 path is CUDA-core issue bound, DESIGN.md
    # §6.1): warp-instructions per launch (the committed ncu capture of this launch configuration)
    # over the live kernel time, against 4 warp-instructions per clock per SM at the max SM clock
    issue_roof = None
    if ncu and ncu.get("warp_instructions") and kernel_ms:
        mhz = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0) \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
        import torch as _t
        sms = _t.cuda.get_device_properties(local).multi_processor_count
        peak = 4.0 * sms * mhz * 1e6
        ach = ncu["warp_instructions"] / (kernel_ms / 1e3)
        issue_roof = {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-instructions/s",
                      "frac": ach / peak, "instructions_src": ncu["source"],
                      "note": "secondary: the HBM roofline above is the SURVEY §8(d) binding one"}
    nodes_total = (args.n + 1) ** 2 * (args.n * world + 1)
    out = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8xs8->s32 + f64" if path == OVX_INT8 else "f64",
        "data": ("synthetic (seeded; roller box with a standing P wave)" if world == 1 else
                 "synthetic (layered soil/rock, Ricker source, smooth initial field)"),
        "config": {"workload": (f"C2: {args.n}^3 homogeneous block" if world == 1 else
                                f"C5: {args.n}x{args.n}x{args.n * world} layered soil/rock (64-layer period), "
                                f"{args.n}^3 z-slab per GPU"),
                   "material": ("kappa=5/3, G=1, rho=1, ds=1, rollers" if world == 1 else
                                "soil (1800, 1000, 300) / rock (2500, 4000, 2000), ds=1 m, 4 bottom corners fixed"),
                   "path": args.path,
                   "elements": E_total, "nodes": nodes_total,
                   "parallelism": "single GPU" if world == 1 else
                   (f"z-slabs x{world}, NCCL P2P interface exchange, overlapped schedule in the library (ovx_step)"
                    if backend == "nccl" and os.environ.get("OVX_BENCH_DIST", "library") == "library" else
                    f"z-slabs x{world}, NCCL P2P interface exchange, {'overlapped' if Sharded.OVERLAP else 'serial'} schedule (dist.py)" if backend == "nccl" else
                    f"z-slabs x{world} on one device, {backend} host-staged interface exchange (test hook)"),
                   "l2": "inputs larger than L2 (%.2f GB touched per step per GPU)" % (_algorithmic_bytes(R_nn, R_ne) / 1e9)},
        "dof_steps_per_s": 3 * nodes_total * args.steps / (ms / 1e3),
        "roofline": roof,
        "roofline_issue": issue_roof,
        "int8_tops_useful": (18432 * R_ne / (kernel_ms / 1e3) / 1e12) if (path == OVX_INT8 and kernel_ms) else None,
        "int8_tops_issued": (issued_ops / (kernel_ms / 1e3) / 1e12) if (issued_ops and kernel_ms) else None,
        # BASELINE "INT8 tensor-pipe % peak": useful INT8 MACs×2 per second over the INT8 dense peak
        # (2 × the measured bf16 TF/s, the guide's nominal int8:bf16 ratio); ncu pipe activity in
        # profiles/r1_int8_v*.md (sm__pipe_tensor_cycles_active)
        "int8_tensor_pct_of_peak": (100.0 * 18432 * R_ne / (kernel_ms / 1e3) / 1e12 / (2.0 * pk["bf16_tflops"]))
                                   if (path == OVX_INT8 and kernel_ms) else None,
        "fp64_path": fp64,
        "ncu_profile": ncu,
        "clocks": clocks,
        "gpu_launches": R_lps * args.steps,
        "e2e": {"value": E_total * args.steps / (ms_e2e / 1e3), "unit": METRIC,
                "h2d_bytes_per_step": 2 * 24 * R_nn / args.steps,
                "d2h_bytes_per_step": 24 * R_nn / args.steps,
                "note": f"per GPU: set_state(u, u_prev from pinned host) + {args.steps} steps + the result u^K "
                        f"into a pinned host buffer (get_state)", "host_ms": e2e_host_ms},
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_oracle_sample(args.path)   # ~20-30 s of oracle work
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
