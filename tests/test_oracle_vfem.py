"""Pins for the oracle's VFEM element (NEXT-3, the paper's conventional method).

Pinned against: the stiffness spectrum of a full-integration trilinear hex (symmetric, exactly the 6
rigid-body zero modes); translation invariance (integer row sums 0); the lumped mass as the row sum
of the consistent mass; brute-force global assembly; the patch test; the closed-form
lattice dispersion of an axis-aligned mode (identical to OVFEM); and the [111]
Bloch-symbol phase velocities at 5 points per wavelength derived independently in SURVEY App. B
(OVFEM S 0.9777 / P 0.9267, VFEM S 0.9097 / P 0.8869, ν = 0.25) — the paper's lower-dispersion
claim for OVFEM.
"""
import math
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
import workloads as wl
from oracle import element as E
from oracle import physics


def _kv(kappa=Fr(5, 3), G=Fr(1), ds=Fr(1)):
    return np.array([[float(x) for x in r] for r in E.vfem_element_stiffness(kappa, G, ds)])


def test_vfem_element_spectrum_rigid_modes():
    K = _kv()
    assert np.array_equal(K, K.T)
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == 6
    assert np.all(ev[np.abs(ev) >= 1e-12 * ev.max()] > 0)


def test_vfem_integer_matrices_translation_invariant():
    Vk, Vg = oracle.vfem_matrices()
    for M in (Vk, Vg):
        for ax in range(3):
            assert np.all(M[:, ax::3].sum(axis=1) == 0)
    Ak, Ag = E.vfem_stiffness_parts(Fr(1))
    assert Fr(int(Vk[0, 0]), 72) == Ak[0][0] and Fr(int(Vg[5, 7]), 216) == Ag[5][7]


def test_vfem_lumped_mass_is_consistent_row_sum():
    # consistent ∫ φ^a φ^b dv = (ds/2)³ Π_j (1 + r̄_j^a r̄_j^b / 3)/2; its row sum is ds³/8
    for a in range(8):
        row = Fr(0)
        for b in range(8):
            v = Fr(1, 64)
            for j in range(3):
                v *= 1 + Fr(E.CORNERS[a][j] * E.CORNERS[b][j], 3)
            row += v
        assert row == Fr(1, 8)            # = ρ/8 (1)_e for ρ = ds = 1


@pytest.mark.parametrize("dims", [(1, 1, 1), (3, 2, 2), (4, 3, 2)])
def test_vfem_matches_dense_assembly(dims):
    m = wl.small_random(*dims, ds=0.01)
    u = wl.random_field(m)
    nx, ny, nz = m.nx, m.ny, m.nz
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    K = np.zeros((3 * nn, 3 * nn))
    cache = {}
    for e in range(nx * ny * nz):
        k = int(m.mat[e])
        if k not in cache:
            cache[k] = _kv(Fr(m.kappa[k]), Fr(m.G[k]), Fr(m.ds))
        nodes = oracle.element_nodes(nx, ny, e)
        dofs = np.concatenate([np.arange(3 * q, 3 * q + 3) for q in nodes])
        K[np.ix_(dofs, dofs)] += cache[k]
    ref = K @ u
    f = oracle.apply_K(nx, ny, nz, m.ds, m.mat, m.kappa, m.G, u, path=oracle.PATH_VFEM)
    assert np.linalg.norm(f - ref) <= 1e-14 * np.linalg.norm(ref)


def test_vfem_patch_test():
    m = wl.c1_cube(4)
    m.ds = 1.0
    n = m.nx + 1
    grid = np.stack(np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij"), -1)[..., ::-1]
    x = grid.reshape(-1, 3).astype(np.float64)
    A = np.array([[0.3, -0.2, 0.5], [0.1, 0.7, -0.4], [0.25, 0.05, -0.6]])
    u = (x @ A.T + np.array([1.0, 2.0, 3.0])).reshape(-1)
    f = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=oracle.PATH_VFEM).reshape(-1, 3)
    inner = [(ix + n * (iy + n * iz)) for iz in range(1, n - 1) for iy in range(1, n - 1) for ix in range(1, n - 1)]
    assert np.abs(f[inner]).max() <= 1e-13 * np.abs(f).max()


def _bloch_speeds(K, kvec):
    X = (np.array(E.CORNERS, dtype=float) + 1) / 2
    S = np.zeros((3, 3), complex)
    for a in range(8):
        for b in range(8):
            S += K[3 * a:3 * a + 3, 3 * b:3 * b + 3] * np.exp(1j * np.dot(kvec, X[b] - X[a]))
    ev = np.sort(np.linalg.eigvalsh(S).real)
    return np.sqrt(ev) / np.linalg.norm(kvec)


def test_bloch_dispersion_111_matches_survey_appendix_b():
    kap, G = Fr(5, 3), Fr(1)                     # ν = 0.25, ρ = ds = 1
    Vp, Vs = math.sqrt(5 / 3 + 4 / 3), 1.0
    k111 = 2 * math.pi / 5 * np.ones(3) / math.sqrt(3)
    ko = np.array([[float(x) for x in r] for r in E.element_stiffness(kap, G, Fr(1))])
    co, cv = _bloch_speeds(ko, k111), _bloch_speeds(_kv(kap, G), k111)
    assert co[0] / Vs == pytest.approx(0.9777, abs=6e-5) and co[2] / Vp == pytest.approx(0.9267, abs=6e-5)
    assert cv[0] / Vs == pytest.approx(0.9097, abs=6e-5) and cv[2] / Vp == pytest.approx(0.8869, abs=6e-5)
    kx = np.array([2 * math.pi / 5, 0.0, 0.0])   # axis-aligned: identical, 0.9355 of V
    for c in (_bloch_speeds(ko, kx), _bloch_speeds(_kv(kap, G), kx)):
        assert c[0] / Vs == pytest.approx(0.9355, abs=6e-5) and c[2] / Vp == pytest.approx(0.9355, abs=6e-5)


def test_vfem_axis_standing_wave_closed_form():
    m = wl.c2_block(8)
    m.nx, m.ny, m.nz = 12, 4, 4
    m.mat = np.zeros(m.nx * m.ny * m.nz, np.uint8)
    m.dirichlet = wl.roller_mask(m.nx, m.ny, m.nz)
    u0 = wl.standing_wave(m, mvec=(3, 0, 0), U=(1.0, 0.0, 0.0))
    k = math.pi * 3 / (m.nx * m.ds)
    V = math.sqrt((m.kappa[0] + 4 * m.G[0] / 3) / m.rho[0])
    lam = physics.lattice_lambda_axis(V, k, m.ds)
    u, _, it, st = oracle.run(m.as_dict(), u0, u0, 0, 200, path=oracle.PATH_VFEM)
    assert st == 0 and it == 200
    assert np.abs(u - physics.mode_amplitude(lam, m.dt, 200) * u0).max() <= 1e-12 * np.abs(u0).max()
