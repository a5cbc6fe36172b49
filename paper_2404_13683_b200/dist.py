"""z-slab decomposition of the time step over several GPUs.

Rank r owns element layers [ez0, ez1) (balanced to ±1 layer) and node planes ez0..ez1.  The
rank ABOVE owns (updates) each interface plane, which keeps the result bit-identical to a
single-GPU run: per step
    begin : fused step kernel over the slab (all planes but the interfaces updated); the top
            interface's top-face force sum T is left in a_send, plane 0's bottom-face sum B
            (layer 0) is kept on the device
    xchg A: a_send(r) -> a_recv(r+1)                                 (NCCL P2P over NVLink)
    (overlap=True: the edge z-chunks run on a second, high-priority stream concurrently with the
     interior chunks; the exchanges and the interface update follow them on that stream)
    iface : owner forms f = T + B (the single-GPU order, reading U2), updates plane 0
    xchg u: u_send(r) -> u_recv(r-1)
    end   : the rank below installs the updated plane, swaps u / u_prev
Only plumbing lives here: partitioning, slicing the model, and the transport (torch.distributed
process group, any backend; or an in-process loopback).  All arithmetic runs in libovx.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition(nz: int, world: int, rank: int) -> tuple[int, int]:
    """Element layers [ez0, ez1) of `rank`: contiguous, balanced to within one layer."""
    base, rem = divmod(nz, world)
    ez0 = rank * base + min(rank, rem)
    return ez0, ez0 + base + (1 if rank < rem else 0)


@dataclass
class Slab:
    rank: int
    world: int
    ez0: int
    ez1: int

    @property
    def nzl(self) -> int:
        return self.ez1 - self.ez0

    @property
    def flags(self) -> int:
        return (1 if self.rank > 0 else 0) | (2 if self.rank < self.world - 1 else 0)

    def owned_planes(self, nz: int) -> tuple[int, int]:
        """Global node planes [p0, p1) this rank updates (interfaces belong to the rank above)."""
        return self.ez0, (self.ez1 if self.rank < self.world - 1 else nz + 1)


def local_model(m, slab: Slab):
    """The slab's sub-model: local grid, materials, mask, sources (global -> local ids)."""
    from types import SimpleNamespace
    nx, ny = m.nx, m.ny
    nn2 = (nx + 1) * (ny + 1)
    ne2 = nx * ny
    lm = SimpleNamespace(nx=nx, ny=ny, nz=slab.nzl, ds=m.ds, rho=m.rho, kappa=m.kappa, G=m.G, dt=m.dt,
                         alpha=getattr(m, "alpha", 0.0), beta=getattr(m, "beta", 0.0))
    lm.mat = np.ascontiguousarray(m.mat[slab.ez0 * ne2: slab.ez1 * ne2])
    lm.mat_below = np.ascontiguousarray(m.mat[(slab.ez0 - 1) * ne2: slab.ez0 * ne2]) if slab.rank > 0 else None
    lm.dirichlet = None if m.dirichlet is None else np.ascontiguousarray(
        m.dirichlet[slab.ez0 * nn2: (slab.ez1 + 1) * nn2])
    p0, p1 = slab.owned_planes(m.nz)
    keep = [k for k in range(len(m.src_node)) if p0 <= m.src_node[k] // nn2 < p1]
    lm.src_node = np.array([m.src_node[k] - slab.ez0 * nn2 for k in keep], dtype=np.int64)
    lm.src_axis = np.array([m.src_axis[k] for k in keep], dtype=np.int32)
    lm.amp = m.amp[keep] if len(keep) else np.zeros((0, 1))
    return lm


class TorchTransport:
    """Interface exchange through a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def _run(self, ops):
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def exchange_up(self, slab: Slab, send, recv):
        d = self.dist
        ops = []
        if slab.rank < slab.world - 1:
            ops.append(d.P2POp(d.isend, send, slab.rank + 1, self.group))
        if slab.rank > 0:
            ops.append(d.P2POp(d.irecv, recv, slab.rank - 1, self.group))
        self._run(ops)

    def exchange_down(self, slab: Slab, send, recv):
        d = self.dist
        ops = []
        if slab.rank > 0:
            ops.append(d.P2POp(d.isend, send, slab.rank - 1, self.group))
        if slab.rank < slab.world - 1:
            ops.append(d.P2POp(d.irecv, recv, slab.rank + 1, self.group))
        self._run(ops)


class HostStagedTransport(TorchTransport):
    """TorchTransport for a CPU-only backend (gloo) with device buffers: each message is staged
    through host memory.  A test hook (several ranks sharing one GPU, which NCCL refuses); the
    NCCL transport moves device buffers directly."""

    def _run(self, ops):
        if not ops:
            return
        staged = []
        for op in ops:
            h = op.tensor.detach().to("cpu")
            staged.append((op, h))
        reqs = self.dist.batch_isend_irecv([self.dist.P2POp(op.op, h, op.peer, op.group) for op, h in staged])
        for req in reqs:
            req.wait()
        for op, h in staged:
            if op.op is self.dist.irecv:
                op.tensor.copy_(h)


class LoopbackTransport:
    """All ranks in one process (tests on one device): exchanges are plain tensor copies.
    Use with SlabGroup, which runs the per-rank phases in lock step."""

    def exchange_all_up(self, runs):
        for r in range(len(runs) - 1):
            runs[r + 1].a_recv.copy_(runs[r].a_send)

    def exchange_all_down(self, runs):
        for r in range(1, len(runs)):
            runs[r - 1].u_recv.copy_(runs[r].u_send)


class OvxCompute:
    """The CUDA compute of one slab (libovx.so context)."""

    def __init__(self, lm, slab: Slab, device: int, path: int, stream=None):
        import torch
        from .ovx import Ovx
        self.ovx = Ovx(device)
        # the interface exchange (torch copies / NCCL P2P) is ordered against torch's current
        # stream, so the slab's kernels must run on that same stream
        self._stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.ovx.set_stream(self._stream)
        o = self.ovx
        o.set_grid(lm.nx, lm.ny, lm.nz, lm.ds)
        o.set_materials(lm.rho, lm.kappa, lm.G)
        o.set_element_materials(lm.mat)
        o.set_dirichlet(lm.dirichlet)
        o.set_slab(slab.flags, lm.mat_below)
        o.setup_elements(path, 8)
        o.set_dt(lm.dt)
        if getattr(lm, "alpha", 0.0) or getattr(lm, "beta", 0.0):   # Rayleigh damping (reading R1)
            o.set_damping(lm.alpha, lm.beta)
        if len(lm.src_node):
            o.set_sources(lm.src_node, lm.src_axis, lm.amp)
        n = 3 * (lm.nx + 1) * (lm.ny + 1)
        mk = lambda: torch.zeros(n, dtype=torch.float64, device=f"cuda:{device}")
        self.a_send, self.a_recv, self.u_send, self.u_recv = mk(), mk(), mk(), mk()
        o.set_iface_buffers(self.a_send, self.a_recv, self.u_send, self.u_recv)

    def set_state(self, u, up, it):
        self.ovx.set_state(u, up, it)

    def get_state(self):
        return self.ovx.get_state()

    def begin(self):
        self.ovx.step_begin()

    def begin_edges(self, stream=None):
        """The first and last z-chunk: they produce a_send and the plane-0 partial.  stream: launch
        them on another stream (so they share the SMs with the interior launch instead of adding a
        wave tail in front of it); the context stream is restored afterwards."""
        if stream is None:
            self.ovx.step_begin_part(0)
            return
        self.ovx.set_stream(stream)
        try:
            self.ovx.step_begin_part(0)
        finally:
            self.ovx.set_stream(self._stream)

    def begin_interior(self):
        self.ovx.step_begin_part(1)

    def iface(self):
        self.ovx.step_iface()

    def iface_on(self, stream):
        self.ovx.step_iface_stream(stream)

    def end(self):
        self.ovx.step_end()

    def sync(self):
        self.ovx.sync()


class SlabRun:
    """One rank of a z-slab run."""

    def __init__(self, model, rank: int, world: int, compute_factory, transport=None):
        self.model = model
        ez0, ez1 = partition(model.nz, world, rank)
        self.slab = Slab(rank, world, ez0, ez1)
        self.lm = local_model(model, self.slab)
        self.compute = compute_factory(self.lm, self.slab)
        self.transport = transport

    # interface buffers live on the compute object
    a_send = property(lambda self: self.compute.a_send)
    a_recv = property(lambda self: self.compute.a_recv)
    u_send = property(lambda self: self.compute.u_send)
    u_recv = property(lambda self: self.compute.u_recv)

    def _planes(self, arr):
        nn2 = (self.model.nx + 1) * (self.model.ny + 1)
        return np.ascontiguousarray(np.asarray(arr).reshape(-1)[3 * nn2 * self.slab.ez0: 3 * nn2 * (self.slab.ez1 + 1)])

    def set_state(self, u_global, up_global, it: int = 0):
        self.compute.set_state(self._planes(u_global), self._planes(up_global), it)

    def step(self, n: int = 1, overlap: bool = False):
        """overlap (CUDA compute only): the edge z-chunks run first; the exchange and the interface
        update then run on a second stream while the interior chunks compute."""
        s, t, c = self.slab, self.transport, self.compute
        if overlap and hasattr(c, "begin_edges"):
            import torch
            comp = torch.cuda.current_stream()
            if getattr(self, "_comm", None) is None:
                self._comm = torch.cuda.Stream(priority=-1)   # edge chunks first when SMs free up
            comm = self._comm
            for _ in range(n):
                comm.wait_stream(comp)                # after the previous step's end
                c.begin_edges(comm)                   # edge chunks on the high-priority stream
                c.begin_interior()                    # interior chunks, concurrently, on comp
                with torch.cuda.stream(comm):         # ordered after the edge chunks only
                    t.exchange_up(s, c.a_send, c.a_recv)
                    c.iface_on(comm)
                    t.exchange_down(s, c.u_send, c.u_recv)
                comp.wait_stream(comm)
                c.end()
            return
        for _ in range(n):
            c.begin()
            t.exchange_up(s, c.a_send, c.a_recv)
            c.iface()
            t.exchange_down(s, c.u_send, c.u_recv)
            c.end()

    def owned_state(self):
        """(first global plane, u and u_prev of the planes this rank owns)."""
        u, up, it = self.compute.get_state()
        nn2 = (self.model.nx + 1) * (self.model.ny + 1)
        p0, p1 = self.slab.owned_planes(self.model.nz)
        a, b = 3 * nn2 * (p0 - self.slab.ez0), 3 * nn2 * (p1 - self.slab.ez0)
        return p0, u[a:b], up[a:b], it


class SlabGroup:
    """All ranks of a decomposition in one process, stepped in lock step (loopback transport)."""

    def __init__(self, model, world: int, compute_factory):
        self.runs = [SlabRun(model, r, world, compute_factory) for r in range(world)]
        self.lb = LoopbackTransport()

    def set_state(self, u, up, it=0):
        for r in self.runs:
            r.set_state(u, up, it)

    def step(self, n=1, overlap: bool = False):
        if overlap:                    # the overlapped schedule of SlabRun.step, all ranks in lock step
            import torch
            comp = torch.cuda.current_stream()
            if getattr(self, "_comm", None) is None:
                self._comm = torch.cuda.Stream(priority=-1)
            comm = self._comm
            for _ in range(n):
                comm.wait_stream(comp)
                for r in self.runs:
                    r.compute.begin_edges(comm)
                for r in self.runs:
                    r.compute.begin_interior()
                with torch.cuda.stream(comm):
                    self.lb.exchange_all_up(self.runs)
                    for r in self.runs:
                        r.compute.iface_on(comm)
                    self.lb.exchange_all_down(self.runs)
                comp.wait_stream(comm)
                for r in self.runs:
                    r.compute.end()
            return
        for _ in range(n):
            for r in self.runs:
                r.compute.begin()
            self.lb.exchange_all_up(self.runs)
            for r in self.runs:
                r.compute.iface()
            self.lb.exchange_all_down(self.runs)
            for r in self.runs:
                r.compute.end()

    def get_state(self):
        parts = [r.owned_state() for r in self.runs]
        u = np.concatenate([p[1] for p in parts])
        up = np.concatenate([p[2] for p in parts])
        return u, up, parts[0][3]


def gather_state(run: SlabRun, group=None):
    """Assemble the global (u, u_prev) on rank 0 via torch.distributed (None on other ranks)."""
    import torch
    import torch.distributed as dist
    p0, u, up, it = run.owned_state()
    payload = [None] * run.slab.world if run.slab.rank == 0 else None
    dist.gather_object((p0, u, up), payload, dst=0, group=group)
    if run.slab.rank != 0:
        return None
    payload.sort(key=lambda x: x[0])
    return np.concatenate([x[1] for x in payload]), np.concatenate([x[2] for x in payload]), it
