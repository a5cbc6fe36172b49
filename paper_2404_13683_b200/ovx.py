"""Thin ctypes binding of the C ABI in include/ovx.h (argument marshalling only).

Every step of the method runs inside libovx.so (hand-written sm_100a kernels).  There is no
CPU fallback: if the library cannot be loaded, importing this module's `lib()` raises.
Method names are the C names without the `ovx_` prefix.
"""
from __future__ import annotations

import ctypes
import os
from functools import lru_cache

import numpy as np

from . import build as _build

OVX_OK, OVX_EINVAL, OVX_EUNSTABLE, OVX_ESTATE, OVX_ECUDA, OVX_ENCCL, OVX_ENOMEM = 0, 2, 3, 6, 7, 8, 9
OVX_INT8, OVX_FP64, OVX_FP64_DENSE, OVX_VFEM, OVX_VFEM_DENSE = 0, 1, 2, 3, 4   # VFEM: NEXT-3
OVX_INT8_DIRECT = 5   # NEXT-4: the direct N-stage FP64→INT8 conversion (Fig. 2 left)

_c = ctypes
_vp = _c.c_void_p
_i64 = _c.c_int64
_int = _c.c_int
_d = _c.c_double


class OvxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"ovx status {status}: {msg}")
        self.status = status


_SIGS = {
    "ovx_create": [_int, _c.POINTER(_vp)],
    "ovx_destroy": [_vp],
    "ovx_set_stream": [_vp, _vp],
    "ovx_set_grid": [_vp, _i64, _i64, _i64, _d],
    "ovx_set_materials": [_vp, _int, _vp, _vp, _vp],
    "ovx_set_element_materials": [_vp, _vp],
    "ovx_set_dirichlet": [_vp, _vp],
    "ovx_set_dt": [_vp, _d],
    "ovx_set_damping": [_vp, _d, _d],
    "ovx_setup_elements": [_vp, _int, _int],
    "ovx_get_int8_matrix": [_vp, _vp],
    "ovx_critical_dt": [_vp, _vp, _vp],
    "ovx_get_phase_timers": [_vp, _vp, _vp, _vp, _int],
    "ovx_get_partition": [_i64, _int, _int, _vp, _vp],
    "ovx_nccl_unique_id": [_vp],
    "ovx_create_dist": [_int, _int, _int, _vp, _vp],
    "ovx_create_group": [_int, _vp, _vp],
    "ovx_step_group": [_vp, _int, _i64],
    "ovx_set_sources": [_vp, _int, _vp, _vp, _i64, _vp],
    "ovx_set_state": [_vp, _vp, _vp, _i64],
    "ovx_get_state": [_vp, _vp, _vp, _vp],
    "ovx_set_state_device": [_vp, _vp, _vp, _i64],
    "ovx_get_state_device": [_vp, _vp, _vp, _vp],
    "ovx_step": [_vp, _i64],
    "ovx_sync": [_vp],
    "ovx_check_finite": [_vp],
    "ovx_apply_K": [_vp, _vp, _vp],
    "ovx_apply_K_device": [_vp, _vp, _vp],
    "ovx_debug_element_ints": [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "ovx_get_node_w": [_vp, _vp],
    "ovx_get_timers": [_vp, _vp, _vp, _int],
    "ovx_get_launch_config": [_vp, _vp, _vp, _vp],
    "ovx_set_slab": [_vp, _int, _vp],
    "ovx_set_iface_buffers": [_vp, _vp, _vp, _vp, _vp],
    "ovx_step_begin": [_vp],
    "ovx_step_iface": [_vp],
    "ovx_step_begin_part": [_vp, _int],
    "ovx_step_iface_stream": [_vp, _vp],
    "ovx_step_end": [_vp],
    "ovx_set_receivers": [_vp, _int, _vp, _i64],
    "ovx_get_traces": [_vp, _vp],
}
EXPORTS = tuple(_SIGS) + ("ovx_last_error", "ovx_version")


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    """Load (building in-tree if stale) libovx.so; raises if it cannot be loaded."""
    path = _build.LIB if os.path.exists(_build.LIB) and not _build._stale() else _build.build()
    L = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _int
    L.ovx_last_error.argtypes = [_vp]
    L.ovx_last_error.restype = _c.c_char_p
    L.ovx_version.argtypes = []
    L.ovx_version.restype = _c.c_char_p
    return L


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _host(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def _dev_ptr(t) -> int:
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous() and t.dtype == torch.float64):
        raise TypeError("expected a contiguous CUDA float64 tensor")
    return t.data_ptr()


def get_partition(nz: int, world: int, rank: int) -> tuple[int, int]:
    """Element layers [ez0, ez1) of `rank` (ovx_get_partition)."""
    a, b = np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
    L = lib()
    if L.ovx_get_partition(int(nz), int(world), int(rank), _np_ptr(a), _np_ptr(b)) != OVX_OK:
        raise OvxError(OVX_EINVAL, L.ovx_last_error(None).decode())
    return int(a[0]), int(b[0])


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes; ovx_nccl_unique_id)."""
    out = np.zeros(128, dtype=np.uint8)
    L = lib()
    st = L.ovx_nccl_unique_id(_np_ptr(out))
    if st != OVX_OK:
        raise OvxError(st, L.ovx_last_error(None).decode())
    return out.tobytes()


class Ovx:
    """One context on one GPU.  Methods mirror `ovx_*` of include/ovx.h."""

    def __init__(self, device: int = 0, _handle=None, rank: int = 0, world: int = 1):
        self._L = lib()
        if _handle is None:
            h = _vp()
            self._check(self._L.ovx_create(device, _c.byref(h)), None)
        else:
            h = _handle
        self.h = h
        self.device = device
        self.rank, self.world = rank, world
        self.nx = self.ny = self.nz = 0
        self.ez0 = 0

    @classmethod
    def create_dist(cls, device: int, rank: int, world: int, uid: bytes) -> "Ovx":
        """Rank `rank` of `world` with a library-owned NCCL communicator (ovx_create_dist; collective)."""
        L = lib()
        idb = np.frombuffer(bytes(uid), dtype=np.uint8).copy()
        h = _vp()
        st = L.ovx_create_dist(device, rank, world, _np_ptr(idb), _c.byref(h))
        if st != OVX_OK:
            raise OvxError(st, L.ovx_last_error(None).decode())
        return cls(device, _handle=h, rank=rank, world=world)

    @classmethod
    def create_group(cls, world: int, devices) -> list:
        """`world` loopback-linked ranks in this process (ovx_create_group); step with step_group."""
        L = lib()
        dev = np.asarray(devices, dtype=np.int32)
        hs = (_vp * world)()
        st = L.ovx_create_group(world, _np_ptr(dev), hs)
        if st != OVX_OK:
            raise OvxError(st, L.ovx_last_error(None).decode())
        return [cls(int(dev[r]), _handle=_vp(hs[r]), rank=r, world=world) for r in range(world)]

    # -- helpers ---------------------------------------------------------------
    def _check(self, st: int, h) -> None:
        if st != OVX_OK:
            msg = self._L.ovx_last_error(h).decode()
            raise OvxError(st, msg)

    def _call(self, name: str, *args) -> None:
        self._check(getattr(self._L, name)(self.h, *args), self.h)

    @property
    def n_nodes(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def n_elems(self) -> int:
        return self.nx * self.ny * self.nz

    def close(self) -> None:
        if getattr(self, "h", None):
            self._L.ovx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- C ABI -------------------------------------------------------------------
    def set_stream(self, stream) -> None:
        """stream: a torch.cuda.Stream (its handle may be 0, the default stream), a raw
        cudaStream_t int, or None for a library-owned stream."""
        if stream is None:
            self._call("ovx_set_stream", _vp(-1 & 0xFFFFFFFFFFFFFFFF))
            return
        raw = int(getattr(stream, "cuda_stream", stream))
        self._call("ovx_set_stream", _vp(raw) if raw else None)

    def set_grid(self, nx: int, ny: int, nz: int, ds: float) -> None:
        """nz: the global element-layer count; a distributed rank keeps its slab [ez0, ez1)."""
        self._call("ovx_set_grid", nx, ny, nz, ds)
        ez0, ez1 = get_partition(nz, self.world, self.rank) if self.world > 1 else (0, nz)
        self.nx, self.ny, self.nz, self.ez0 = nx, ny, ez1 - ez0, ez0

    def set_materials(self, rho, kappa, G) -> None:
        r, k, g = _host(rho, np.float64), _host(kappa, np.float64), _host(G, np.float64)
        self._call("ovx_set_materials", len(r), _np_ptr(r), _np_ptr(k), _np_ptr(g))

    def set_element_materials(self, mat) -> None:
        """Material id per element; a distributed rank > 0 passes the layer below its slab first."""
        m = _host(mat, np.uint8)
        halo = self.nx * self.ny if (self.world > 1 and self.rank > 0) else 0
        if m.size != self.n_elems + halo:
            raise OvxError(OVX_EINVAL, "element material array size mismatch")
        self._call("ovx_set_element_materials", _np_ptr(m))

    def set_dirichlet(self, mask) -> None:
        if mask is None:
            self._call("ovx_set_dirichlet", None)
            return
        m = _host(mask, np.uint8)
        if m.size != self.n_nodes:
            raise OvxError(OVX_EINVAL, "Dirichlet mask size mismatch")
        self._call("ovx_set_dirichlet", _np_ptr(m))

    def set_dt(self, dt: float) -> None:
        self._call("ovx_set_dt", dt)

    def set_damping(self, alpha: float, beta: float) -> None:
        """Rayleigh damping C = alpha M + beta K (ovx_set_damping; reading R1)."""
        self._call("ovx_set_damping", float(alpha), float(beta))

    def setup_elements(self, path: int = OVX_INT8, stages: int = 8) -> None:
        self._call("ovx_setup_elements", path, stages)

    def get_int8_matrix(self) -> np.ndarray:
        out = np.zeros((24, 48), dtype=np.int8)
        self._call("ovx_get_int8_matrix", _np_ptr(out))
        return out

    def critical_dt(self, power_iter: bool = False):
        """The element bound (float); with power_iter, (element bound, power-iteration dt)."""
        a, b = np.zeros(1), np.zeros(1)
        self._call("ovx_critical_dt", _np_ptr(a), _np_ptr(b) if power_iter else None)
        return (float(a[0]), float(b[0])) if power_iter else float(a[0])

    def get_phase_timers(self, reset: bool = False):
        """(ms_ebe, ms_halo, ms_update) since the last reset (ovx_get_phase_timers)."""
        a, b, c = np.zeros(1), np.zeros(1), np.zeros(1)
        self._call("ovx_get_phase_timers", _np_ptr(a), _np_ptr(b), _np_ptr(c), 1 if reset else 0)
        return float(a[0]), float(b[0]), float(c[0])

    def set_sources(self, node, axis, amp) -> None:
        node = _host(node, np.int64)
        axis = _host(axis, np.int32)
        amp = _host(amp, np.float64).reshape(len(node), -1) if len(node) else np.zeros((0, 0))
        self._call("ovx_set_sources", len(node), _np_ptr(node), _np_ptr(axis), amp.shape[1] if len(node) else 0,
                   _np_ptr(amp))

    def set_state(self, u, u_prev, it: int = 0) -> None:
        u, up = _host(u, np.float64), _host(u_prev, np.float64)
        if u.size != 3 * self.n_nodes or up.size != 3 * self.n_nodes:
            raise OvxError(OVX_EINVAL, "state size mismatch")
        self._call("ovx_set_state", _np_ptr(u), _np_ptr(up), it)

    def get_state(self, out_u=None, out_up=None, with_prev: bool = True):
        """(u, u_prev, it) on the host.  out_u / out_up: optional preallocated float64 arrays (e.g.
        pinned); with_prev=False skips u_prev (returned as None)."""
        n = 3 * self.n_nodes
        u = np.empty(n) if out_u is None else out_u
        up = (np.empty(n) if out_up is None else out_up) if with_prev else None
        for a in (u, up):
            if a is not None and (a.dtype != np.float64 or a.size != n or not a.flags.c_contiguous):
                raise OvxError(OVX_EINVAL, "output arrays must be contiguous float64 of 3*n_nodes")
        it = np.zeros(1, dtype=np.int64)
        self._call("ovx_get_state", _np_ptr(u), _np_ptr(up) if up is not None else None, _np_ptr(it))
        return u, up, int(it[0])

    def set_state_device(self, u, u_prev, it: int = 0) -> None:
        self._call("ovx_set_state_device", _vp(_dev_ptr(u)), _vp(_dev_ptr(u_prev)), it)

    def get_state_device(self, u, u_prev) -> int:
        it = np.zeros(1, dtype=np.int64)
        self._call("ovx_get_state_device", _vp(_dev_ptr(u)), _vp(_dev_ptr(u_prev)), _np_ptr(it))
        return int(it[0])

    def step(self, n: int = 1) -> None:
        self._call("ovx_step", n)

    def sync(self) -> None:
        self._call("ovx_sync")

    def check_finite(self) -> None:
        self._call("ovx_check_finite")

    def apply_K(self, u) -> np.ndarray:
        u = _host(u, np.float64)
        f = np.zeros_like(u)
        self._call("ovx_apply_K", _np_ptr(u), _np_ptr(f))
        return f

    def apply_K_device(self, u, f) -> None:
        self._call("ovx_apply_K_device", _vp(_dev_ptr(u)), _vp(_dev_ptr(f)))

    def debug_element_ints(self, u, e0: int, ne: int) -> dict:
        u = _host(u, np.float64)
        s = np.zeros(ne)
        v = np.zeros((ne, 48), dtype=np.int64)
        d = np.zeros((ne, 8, 48), dtype=np.uint8)
        C = np.zeros((ne, 8, 24), dtype=np.int32)
        yh = np.zeros((ne, 24), dtype=np.int64)
        yl = np.zeros((ne, 24), dtype=np.int64)
        fe = np.zeros((ne, 24))
        self._call("ovx_debug_element_ints", _np_ptr(u), e0, ne, _np_ptr(s), _np_ptr(v), _np_ptr(d), _np_ptr(C),
                   _np_ptr(yh), _np_ptr(yl), _np_ptr(fe))
        y = [[(int(h) << 64) + (int(l) & ((1 << 64) - 1)) for h, l in zip(yh[j], yl[j])] for j in range(ne)]
        return dict(s=s, v=v, d=d, C=C, y=y, fe=fe)

    def debug_element_forces(self, u, e0: int, ne: int) -> np.ndarray:
        u = _host(u, np.float64)
        fe = np.zeros((ne, 24))
        self._call("ovx_debug_element_ints", _np_ptr(u), e0, ne, None, None, None, None, None, None, _np_ptr(fe))
        return fe

    def get_node_w(self) -> np.ndarray:
        w = np.zeros(self.n_nodes)
        self._call("ovx_get_node_w", _np_ptr(w))
        return w

    def get_timers(self, reset: bool = False):
        ms = np.zeros(1)
        n = np.zeros(1, dtype=np.int64)
        self._call("ovx_get_timers", _np_ptr(ms), _np_ptr(n), 1 if reset else 0)
        return float(ms[0]), int(n[0])

    def get_launch_config(self):
        c = np.zeros(1, dtype=np.int64)
        t = np.zeros(1, dtype=np.int32)
        s = np.zeros(1, dtype=np.int32)
        self._call("ovx_get_launch_config", _np_ptr(c), _np_ptr(t), _np_ptr(s))
        return int(c[0]), int(t[0]), int(s[0])

    def set_receivers(self, node, n_t: int) -> None:
        node = _host(node, np.int64)
        self._nrec, self._rec_nt = len(node), int(n_t)
        self._call("ovx_set_receivers", len(node), _np_ptr(node), int(n_t))

    def get_traces(self) -> np.ndarray:
        out = np.zeros((getattr(self, "_nrec", 0), 3, getattr(self, "_rec_nt", 0)))
        self._call("ovx_get_traces", _np_ptr(out))
        return out

    def set_slab(self, flags: int, mat_below=None) -> None:
        mb = None if mat_below is None else _host(mat_below, np.uint8)
        if mb is not None and mb.size != self.nx * self.ny:
            raise OvxError(OVX_EINVAL, "halo material layer size mismatch")
        self._call("ovx_set_slab", flags, None if mb is None else _np_ptr(mb))

    def set_iface_buffers(self, a_send=None, a_recv=None, u_send=None, u_recv=None) -> None:
        ptr = lambda t: None if t is None else _vp(_dev_ptr(t))
        self._iface = (a_send, a_recv, u_send, u_recv)   # keep the tensors alive
        self._call("ovx_set_iface_buffers", ptr(a_send), ptr(a_recv), ptr(u_send), ptr(u_recv))

    def step_begin(self) -> None:
        self._call("ovx_step_begin")

    def step_iface(self) -> None:
        self._call("ovx_step_iface")

    def step_begin_part(self, part: int) -> None:
        """0: the edge z-chunks (interface producers), 1: the interior chunks (ovx_step_begin_part)."""
        self._call("ovx_step_begin_part", int(part))

    def step_iface_stream(self, stream) -> None:
        """Interface update on another stream (torch.cuda.Stream or raw handle; 0 = default)."""
        raw = int(getattr(stream, "cuda_stream", stream))
        self._call("ovx_step_iface_stream", _vp(raw) if raw else None)

    def step_end(self) -> None:
        self._call("ovx_step_end")

    # -- convenience ---------------------------------------------------------------
    def load_model(self, m, path: int = OVX_INT8, stages: int = 8) -> None:
        """Upload a workloads.Model-like object (grid, materials, mask, dt, sources) and set up."""
        self.set_grid(m.nx, m.ny, m.nz, m.ds)
        self.set_materials(m.rho, m.kappa, m.G)
        self.set_element_materials(m.mat)
        self.set_dirichlet(m.dirichlet)
        self.setup_elements(path, stages)
        self.set_dt(m.dt)
        self.set_sources(m.src_node, m.src_axis, m.amp)   # also when empty: no stale sources
        if getattr(m, "alpha", 0.0) or getattr(m, "beta", 0.0):
            self.set_damping(m.alpha, m.beta)


def step_group(ranks, n: int = 1) -> None:
    """n steps of all ranks of a loopback group in lock step (ovx_step_group)."""
    L = lib()
    hs = (_vp * len(ranks))(*[r.h for r in ranks])
    st = L.ovx_step_group(hs, len(ranks), int(n))
    if st != OVX_OK:
        raise OvxError(st, L.ovx_last_error(ranks[0].h).decode())


def version() -> str:
    return lib().ovx_version().decode()
