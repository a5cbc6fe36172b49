"""Tolerances for comparing the CUDA path with the oracle when the two sum in different orders
(TEST INFRASTRUCTURE; DESIGN.md §3 "parity bars").

* Same element forces, different summation order of the ≤ 8 terms of a node force (the INT8 and
  dense paths against the oracle's element-order definition):
      |f_a − f_b|_n ≤ 2·γ_7·Σ_e |f_e[n]|,  γ_7 = 7u/(1 − 7u),  u = 2^-53
  (Higham, Accuracy and Stability, Lemma 3.1 / Eq. 4.4 for recursive summation, applied to both
  orders).  Σ_e |f_e[n]| comes from the oracle (ORDER_ABS).
* Factored FP64 forms (Walsh-Hadamard, OVX_FP64 / OVX_VFEM) against the dense definition: every
  intermediate of the factored element product is a signed sum of corner values weighted by
  coefficients of magnitude ≤ (κ_e + G_e)·ds, so the element-force error is ≤ c·u·(κ_e + G_e)·ds·Σ_b |u_e,b|
  with c a small operation count; the node bound sums it over the ≤ 8 elements of the node
  (reading P1 of DESIGN.md: a per-node, not a per-field, bound; c = 64).
"""
import numpy as np

import oracle

U = 2.0 ** -53
GAMMA7 = 7 * U / (1 - 7 * U)
FACTORED_C = 64


def element_nodes_all(nx, ny, ez0, ez1):
    """(E_chunk, 8) node ids of the elements of layers [ez0, ez1), local order of reading Q1."""
    ex, ey, ez = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(ez0, ez1), indexing="ij")
    ex, ey, ez = (a.transpose(2, 1, 0).reshape(-1) for a in (ex, ey, ez))   # element id order
    cx = np.array([0, 1, 1, 0, 0, 1, 1, 0])
    cy = np.array([0, 0, 1, 1, 0, 0, 1, 1])
    cz = np.array([0, 0, 0, 0, 1, 1, 1, 1])
    return (ex[:, None] + cx) + (nx + 1) * ((ey[:, None] + cy) + (ny + 1) * (ez[:, None] + cz))


def order_bound(m, u, path):
    """2·γ_7·Σ_e |f_e[n]| per DOF (+ the smallest subnormal, for exactly-zero nodes)."""
    s = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=path, order=oracle.ORDER_ABS)
    return 2 * GAMMA7 * s + 5e-324


def factored_bound(m, u):
    """c·u·Σ_{e∋n} (κ_e + G_e)·ds·Σ_b |u_e,b| per DOF (all three components of a node alike)."""
    au = np.abs(np.asarray(u).reshape(-1, 3)).sum(1)
    nn = (m.nx + 1) * (m.ny + 1) * (m.nz + 1)
    acc = np.zeros(nn)
    kg = (np.asarray(m.kappa) + np.asarray(m.G)) * m.ds
    step = max(1, (1 << 22) // max(1, m.nx * m.ny))
    for z0 in range(0, m.nz, step):
        z1 = min(m.nz, z0 + step)
        nodes = element_nodes_all(m.nx, m.ny, z0, z1)
        e0, e1 = z0 * m.nx * m.ny, z1 * m.nx * m.ny
        se = kg[np.asarray(m.mat[e0:e1])] * au[nodes].sum(1)
        np.add.at(acc, nodes.reshape(-1), np.repeat(se, 8))
    return np.repeat(FACTORED_C * U * acc, 3) + 5e-324


def within(a, ref, bound):
    """Element-wise |a − ref| ≤ bound; returns (ok, worst ratio)."""
    d = np.abs(np.asarray(a) - np.asarray(ref))
    r = d / bound
    return bool(np.all(d <= bound)), float(r.max()) if r.size else 0.0
