"""CPU oracle for the OVFEM / TCOVFEM explicit time step (arxiv 2404.13683).

TEST INFRASTRUCTURE.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything under `oracle/`.
The product package (`paper_2404_13683_b200`) never imports it, links it or
shares code with it; the two meet only on inputs produced by `workloads/`.

Contents
  element.py     exact-rational derivation of B, Gram, A_κ, A_G, K_e^INT8 (Eqs. 5-8)
  ovx_oracle.c   plain-C FP64 EBE product, integer-path emulation (Eqs. 10-17, int128),
                 central-difference stepper (Eq. 3)
  assemble.py    dense global K / M assembly for tiny meshes (brute force)
  physics.py     closed forms used as pins: 1-D dispersion, leapfrog energy, Err metric

"Parity unpinned" items are listed in DESIGN.md §Oracle.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ovx_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no fast-math, no FMA contraction; OpenMP over the independent
    element forces only — results are bit-identical for any OMP_NUM_THREADS)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11",
                               "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i8p = ctypes.POINTER(ctypes.c_int8)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64
_d = ctypes.c_double
_int = ctypes.c_int


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    L = ctypes.CDLL(build())
    L.oracle_node_w.argtypes = [_i64, _i64, _i64, _d, _u8p, _dp, _d, _dp]
    L.oracle_element_fp64.argtypes = [_dp, _d, _d, _d, _i32p, _i32p, _dp]
    L.oracle_element_vfem.argtypes = [_dp, _d, _d, _d, _i32p, _i32p, _dp]
    L.oracle_element_int8.argtypes = [_dp, _d, _d, _d, _i8p, _int, _int,
                                      _dp, _i64p, _i32p, _i64p, _i64p, _i64p, _dp]
    L.oracle_element_int8.restype = _int
    L.oracle_apply_K.argtypes = [_i64, _i64, _i64, _d, _u8p, _dp, _dp, _int,
                                 _i32p, _i32p, _i8p, _int, _int, _int, _dp, _dp]
    L.oracle_apply_K3.argtypes = [_i64, _i64, _i64, _d, _u8p, _dp, _dp, _int,
                                  _i32p, _i32p, _i8p, _int, _int, _dp, _dp, _dp, _dp]
    L.oracle_run.argtypes = [_i64, _i64, _i64, _d, _u8p, _dp, _dp, _dp, _u8p,
                             _int, _i32p, _i32p, _i8p, _int, _int, _int,
                             _int, _i64p, _i32p, _i64, _dp, _d, _d, _d, _dp, _dp, _i64p, _i64]
    L.oracle_run.restype = _int
    L.oracle_element_nodes.argtypes = [_i64, _i64, _i64, _i64p]
    L.oracle_digits.argtypes = [_i64, _int, _int, _i32p]
    L.oracle_update_dofs.argtypes = [_i64, _dp, _dp, _dp, _dp, _dp]
    return L


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@lru_cache(maxsize=1)
def int_matrices():
    """(K8 24×48 int8, Kk 24×24 int32, Kg 24×24 int32) from the exact derivation."""
    from .element import k_int8, k_int8_split
    K8 = np.array(k_int8(), dtype=np.int8)
    Kk, Kg = k_int8_split()
    return K8, np.array(Kk, dtype=np.int32), np.array(Kg, dtype=np.int32)


PATH_FP64, PATH_INT8, PATH_VFEM = 0, 1, 2     # VFEM: the paper's conventional element (NEXT-3)


@lru_cache(maxsize=1)
def vfem_matrices():
    """(Vk, Vg) int32 24×24: K_e^V = κ ds Vk/72 + G ds Vg/216 (oracle/element.py, exact)."""
    from .element import vfem_int_matrices
    Vk, Vg = vfem_int_matrices()
    return np.array(Vk, dtype=np.int32), np.array(Vg, dtype=np.int32)


def element_vfem(ue, kappa: float, G: float, ds: float) -> np.ndarray:
    """VFEM element force K_e^V u_e, the C oracle's operation order."""
    Vk, Vg = vfem_matrices()
    ue = np.ascontiguousarray(ue, dtype=np.float64)
    fe = np.zeros(24)
    lib().oracle_element_vfem(_p(ue, _dp), float(kappa), float(G), float(ds), _p(Vk, _i32p), _p(Vg, _i32p),
                              _p(fe, _dp))
    return fe
DIGITS_PAPER, DIGITS_BYTES = 0, 1
# Summation order of f_n = Σ_e f_e[n] (ovx_oracle.c, oracle_apply_K):
#   ORDER_ELEMENT — the definition: plain scatter in element id order;
#   ORDER_U2      — MIRROR VARIANT of the B200 kernels' per-node pairwise tree (reading U2),
#                   used only where a test wants the kernels' bits; never the reference physics.
#   ORDER_ABS     — not a product: Σ_e |f_e[n]|, the scale of the cross-order rounding bound.
ORDER_ELEMENT, ORDER_U2, ORDER_ABS = 0, 1, 2
DIGITS_BYTES_FOLD = 3      # byte slices + Eq. 9 diagonal term in the integer product (variant D)
DIGITS_DIRECT = 4          # the direct N-stage FP64→INT8 conversion (Fig. 2 left, Eqs. 11-14, a = 2^7)
DIGITS_DIRECT_FOLD = 6     # direct conversion + variant D


def element_nodes(nx: int, ny: int, e: int) -> np.ndarray:
    out = np.zeros(8, dtype=np.int64)
    lib().oracle_element_nodes(nx, ny, e, _p(out, _i64p))
    return out


def digits(v: int, M: int = 8, scheme: int = DIGITS_BYTES) -> list[int]:
    """Digit expansion of one INT64 value (Eq. 16; variant B for scheme=1)."""
    nd = (7 * M + 1 + 7) // 8 if scheme else M
    out = np.zeros(8, dtype=np.int32)
    lib().oracle_digits(int(v), M, scheme, _p(out, _i32p))
    return [int(x) for x in out[:nd]]


def update_dofs(w, F, f, u, up) -> None:
    """up <- fma(w, F - f, 2u - up) elementwise (Eq. 3), in place."""
    args = [np.ascontiguousarray(a, dtype=np.float64) for a in (w, F, f, u)]
    assert up.flags["C_CONTIGUOUS"] and up.dtype == np.float64
    lib().oracle_update_dofs(len(up), *[_p(a, _dp) for a in args], _p(up, _dp))


def node_w(nx, ny, nz, ds, mat, rho, dt) -> np.ndarray:
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    w = np.zeros(nn)
    mat = np.ascontiguousarray(mat, dtype=np.uint8)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    lib().oracle_node_w(nx, ny, nz, ds, _p(mat, _u8p), _p(rho, _dp), dt, _p(w, _dp))
    return w


def element_fp64(ue, kappa, G, ds) -> np.ndarray:
    _, Kk, Kg = int_matrices()
    ue = np.ascontiguousarray(ue, dtype=np.float64)
    fe = np.zeros(24)
    lib().oracle_element_fp64(_p(ue, _dp), kappa, G, ds, _p(Kk, _i32p), _p(Kg, _i32p), _p(fe, _dp))
    return fe


def element_int8(ue, kappa, G, ds, M: int = 8, digits: int = DIGITS_BYTES_FOLD) -> dict:
    """Bit-level integer path for one element; returns s, v, d, C, y (python ints), fe."""
    K8, _, _ = int_matrices()
    ue = np.ascontiguousarray(ue, dtype=np.float64)
    nd = (7 * M + 1 + 7) // 8 if (digits & 1) and not (digits & 4) else M
    s = np.zeros(1)
    v = np.zeros(48, dtype=np.int64)
    d = np.zeros(nd * 48, dtype=np.int32)
    C = np.zeros(nd * 24, dtype=np.int64)
    yh = np.zeros(24, dtype=np.int64)
    yl = np.zeros(24, dtype=np.int64)
    fe = np.zeros(24)
    deg = lib().oracle_element_int8(_p(ue, _dp), kappa, G, ds, _p(K8, _i8p), M, digits,
                                    _p(s, _dp), _p(v, _i64p), _p(d, _i32p), _p(C, _i64p),
                                    _p(yh, _i64p), _p(yl, _i64p), _p(fe, _dp))
    y = [(int(h) << 64) + (int(l) & ((1 << 64) - 1)) for h, l in zip(yh, yl)]
    return dict(s=float(s[0]), v=v, d=d.reshape(nd, 48), C=C.reshape(nd, 24), y=y, fe=fe,
                degenerate=bool(deg))


def _path_matrices(path):
    """(K8, Kk, Kg) for the C oracle: for PATH_VFEM, Kk / Kg carry the VFEM matrices Vk / Vg."""
    K8, Kk, Kg = int_matrices()
    if path == PATH_VFEM:
        Kk, Kg = vfem_matrices()
    return K8, Kk, Kg


def apply_K(nx, ny, nz, ds, mat, kappa, G, u, path=PATH_FP64, M=8, digits=DIGITS_BYTES_FOLD,
            order=ORDER_ELEMENT) -> np.ndarray:
    K8, Kk, Kg = _path_matrices(path)
    mat = np.ascontiguousarray(mat, dtype=np.uint8)
    kappa = np.ascontiguousarray(kappa, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    f = np.zeros_like(u)
    lib().oracle_apply_K(nx, ny, nz, ds, _p(mat, _u8p), _p(kappa, _dp), _p(G, _dp), path,
                         _p(Kk, _i32p), _p(Kg, _i32p), _p(K8, _i8p), M, digits, int(order),
                         _p(u, _dp), _p(f, _dp))
    return f


def apply_K_orders(nx, ny, nz, ds, mat, kappa, G, u, path=PATH_FP64, M=8, digits=DIGITS_BYTES_FOLD):
    """One element pass, three scatters: (f in element order = the definition, f in the U2 mirror
    order, Σ_e |f_e[n]| = the cross-order rounding-bound scale)."""
    K8, Kk, Kg = _path_matrices(path)
    mat = np.ascontiguousarray(mat, dtype=np.uint8)
    kappa = np.ascontiguousarray(kappa, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    fa, fb, fc = np.zeros_like(u), np.zeros_like(u), np.zeros_like(u)
    lib().oracle_apply_K3(nx, ny, nz, ds, _p(mat, _u8p), _p(kappa, _dp), _p(G, _dp), path,
                          _p(Kk, _i32p), _p(Kg, _i32p), _p(K8, _i8p), M, digits,
                          _p(u, _dp), _p(fa, _dp), _p(fb, _dp), _p(fc, _dp))
    return fa, fb, fc


def run(model, u, u_prev, it: int, nsteps: int, path=PATH_FP64, M=8, digits=DIGITS_BYTES_FOLD,
        order=ORDER_ELEMENT):
    """Advance (u, u_prev, it) by nsteps with the model dict produced by workloads.

    model keys: nx, ny, nz, ds, mat (uint8 per element), rho/kappa/G (per material),
    dt, dirichlet (uint8 per node or None), src_node, src_axis, amp (nsrc × n_t),
    alpha, beta (Rayleigh damping C = alpha M + beta K, reading R1; default 0).
    Returns (u, u_prev, it, status) with new arrays (inputs are not modified).
    """
    K8, Kk, Kg = _path_matrices(path)
    nx, ny, nz, ds = model["nx"], model["ny"], model["nz"], model["ds"]
    mat = np.ascontiguousarray(model["mat"], dtype=np.uint8)
    kappa = np.ascontiguousarray(model["kappa"], dtype=np.float64)
    G = np.ascontiguousarray(model["G"], dtype=np.float64)
    w = node_w(nx, ny, nz, ds, mat, model["rho"], model["dt"])
    dm = model.get("dirichlet")
    dm = None if dm is None else np.ascontiguousarray(dm, dtype=np.uint8)
    src_node = np.ascontiguousarray(model.get("src_node", np.zeros(0)), dtype=np.int64)
    src_axis = np.ascontiguousarray(model.get("src_axis", np.zeros(0)), dtype=np.int32)
    amp = np.ascontiguousarray(model.get("amp", np.zeros((0, 1))), dtype=np.float64)
    n_t = amp.shape[1] if amp.ndim == 2 else 0
    u = np.array(u, dtype=np.float64, copy=True).reshape(-1)
    up = np.array(u_prev, dtype=np.float64, copy=True).reshape(-1)
    itp = np.array([it], dtype=np.int64)
    st = lib().oracle_run(nx, ny, nz, ds, _p(mat, _u8p), _p(kappa, _dp), _p(G, _dp), _p(w, _dp),
                          None if dm is None else _p(dm, _u8p),
                          path, _p(Kk, _i32p), _p(Kg, _i32p), _p(K8, _i8p), M, digits, int(order),
                          len(src_node), _p(src_node, _i64p), _p(src_axis, _i32p), n_t,
                          _p(amp, _dp), float(model["dt"]), float(model.get("alpha", 0.0)),
                          float(model.get("beta", 0.0)), _p(u, _dp), _p(up, _dp), _p(itp, _i64p), nsteps)
    return u, up, int(itp[0]), st
