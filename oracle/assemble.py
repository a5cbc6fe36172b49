"""Brute-force dense assembly of the global OVFEM K and M for tiny meshes.

TEST INFRASTRUCTURE (oracle).  PAPER.md L31-L36 (Eq. 2): "K and M are ... assembled
using the element stiffness matrix K_e and the element mass matrix M_e".
Element matrices come from the exact derivation in element.py (Eq. 5, Eq. 6);
assembly is the textbook  K = Σ_e P_eᵀ K_e P_e  with explicit index loops, used to
check the EBE product and to compute spectra on meshes of a few hundred nodes.
"""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np

from .element import element_stiffness, CORNERS


def element_matrix_float(kappa: float, G: float, ds: float) -> np.ndarray:
    Ke = element_stiffness(Fr(kappa), Fr(G), Fr(ds))
    return np.array([[float(x) for x in row] for row in Ke])


def node_of(nx, ny, ix, iy, iz):
    return ix + (nx + 1) * (iy + (ny + 1) * iz)


def assemble_K(nx, ny, nz, ds, mat, kappa, G) -> np.ndarray:
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    K = np.zeros((3 * nn, 3 * nn))
    cache = {}
    for ez in range(nz):
        for ey in range(ny):
            for ex in range(nx):
                e = ex + nx * (ey + ny * ez)
                m = int(mat[e])
                if m not in cache:
                    cache[m] = element_matrix_float(kappa[m], G[m], ds)
                Ke = cache[m]
                dofs = []
                for (sx, sy, sz) in CORNERS:
                    n = node_of(nx, ny, ex + (sx > 0), ey + (sy > 0), ez + (sz > 0))
                    dofs += [3 * n, 3 * n + 1, 3 * n + 2]
                for a in range(24):
                    for b in range(24):
                        K[dofs[a], dofs[b]] += Ke[a, b]
    return K


def assemble_M_diag(nx, ny, nz, ds, mat, rho) -> np.ndarray:
    """Diagonal global mass: Σ_e ρ_e ds³/8 per node and axis (Eq. 6)."""
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    m = np.zeros(nn)
    for ez in range(nz):
        for ey in range(ny):
            for ex in range(nx):
                e = ex + nx * (ey + ny * ez)
                for (sx, sy, sz) in CORNERS:
                    m[node_of(nx, ny, ex + (sx > 0), ey + (sy > 0), ez + (sz > 0))] += rho[int(mat[e])] * ds ** 3 / 8
    return np.repeat(m, 3)
