"""Pins for the exact-rational element derivation (oracle/element.py).

Each test checks the oracle against something other than itself: the paper's
statements (integer range of K_e^INT8, diagonal mass, Eq. 9), an independent
integration-by-parts evaluation of (ψ∇φ)_e, an independent 4-index tensor
route to Eq. 5 (no Voigt / engineering-shear convention involved), and exact
rigid-body mechanics.
"""
from fractions import Fraction as Fr
import random

import numpy as np
import pytest

from oracle import element as el


def _surface_by_parts(ds):
    """(ψ^β ∂_i φ^α)_e = ∮ ψ φ n_i dA − ∫ φ ∂_i ψ dv  (Gauss; SPEC's by-parts reading).

    Surface: φ^α = 1 only on the outer face r_i = r̄_i^α quadrant; n_i = r̄_i^α.
    Volume: ∂_{x_i} ψ = (2/ds) ∂_{r_i} ψ integrated over octant α.
    Polynomial integrals are done by exact antiderivatives, independent of element.py.
    """
    def half(e, sgn):  # ∫ over [0,1] or [-1,0] of r^e
        lo, hi = (Fr(0), Fr(1)) if sgn > 0 else (Fr(-1), Fr(0))
        return (hi ** (e + 1) - lo ** (e + 1)) / (e + 1)

    P = {}
    for b, ex in enumerate(el.PSI):
        for i in range(3):
            for a, rb in enumerate(el.CORNERS):
                # surface term: ψ evaluated at r_i = r̄_i (value r̄_i^{e_i}), times quadrant integral
                q = Fr(rb[i]) ** ex[i]
                for j in range(3):
                    if j != i:
                        q *= half(ex[j], rb[j])
                surf = (Fr(ds) / 2) ** 2 * rb[i] * q
                # volume term: ∂_{r_i} r_i^{e_i} = e_i r_i^{e_i - 1}
                vol = Fr(0)
                if ex[i] > 0:
                    v = Fr(ex[i]) * half(ex[i] - 1, rb[i])
                    for j in range(3):
                        if j != i:
                            v *= half(ex[j], rb[j])
                    vol = (Fr(ds) / 2) ** 3 * (2 / Fr(ds)) * v
                P[(b, i, a)] = surf - vol
    return P


@pytest.mark.parametrize("ds", [Fr(1), Fr(1, 500), Fr(7, 3)])
def test_psi_grad_phi_matches_integration_by_parts(ds):
    P = el.psi_grad_phi(ds)
    Q = _surface_by_parts(ds)
    for b in range(7):
        for i in range(3):
            for a in range(8):
                assert P[b][i][a] == Q[(b, i, a)], (b, i, a)


def test_gram_is_diagonal_with_closed_form_entries():
    ds = Fr(3, 2)
    Gm = el.psi_gram_full(ds)
    expect = [1, Fr(1, 3), Fr(1, 3), Fr(1, 3), Fr(1, 9), Fr(1, 9), Fr(1, 9)]
    for b1 in range(7):
        for b2 in range(7):
            assert Gm[b1][b2] == (ds ** 3 * expect[b1] if b1 == b2 else 0)


def test_k_int8_is_int8_integer_matrix_paper_L110():
    K = el.k_int8()
    assert len(K) == 24 and all(len(r) == 48 for r in K)
    flat = [x for r in K for x in r]
    assert all(isinstance(x, int) and -128 <= x <= 127 for x in flat)
    # "constant": independent of ds and of the material
    for ds in (Fr(1, 500), Fr(2, 1000), Fr(13, 7)):
        Ak, Ag = el.stiffness_parts(ds)
        for r in range(24):
            for c in range(24):
                assert 256 * Ak[r][c] / ds == K[r][c]
                assert 384 * Ag[r][c] / ds - (128 if r == c else 0) == K[r][24 + c]


def _tensor_route_K(kappa, G, ds):
    """K_e^o via Eq. 5 in 4-index form with c_pqrs = λδpqδrs + μ(δprδqs + δpsδqr)."""
    lam, mu = Fr(kappa) - Fr(2, 3) * Fr(G), Fr(G)
    d = lambda a, b: 1 if a == b else 0
    cten = [[[[lam * d(p, q) * d(r, s) + mu * (d(p, r) * d(q, s) + d(p, s) * d(q, r))
               for s in range(3)] for r in range(3)] for q in range(3)] for p in range(3)]
    P = el.psi_grad_phi(ds)
    g = el.psi_gram(ds)
    K = [[Fr(0)] * 24 for _ in range(24)]
    for b in range(7):
        for a1 in range(8):
            for p in range(3):          # displacement component of row DOF
                for a2 in range(8):
                    for r in range(3):  # displacement component of column DOF
                        acc = Fr(0)
                        for q in range(3):
                            if P[b][q][a1] == 0:
                                continue
                            for s in range(3):
                                acc += P[b][q][a1] * cten[p][q][r][s] * P[b][s][a2]
                        K[3 * a1 + p][3 * a2 + r] += acc / g[b]
    return K


def test_eq5_voigt_matches_tensor_route():
    kappa, G, ds = Fr(7, 3), Fr(5, 4), Fr(2, 1000)
    Kv = el.element_stiffness(kappa, G, ds)
    Kt = _tensor_route_K(kappa, G, ds)
    assert Kv == Kt


def test_eq9_identity_exact():
    """Eq. 9: K_e^o u_e = (κ ds/256)(K_e^INT8 ū_e + (256/3)(G/κ) u_e), ū_e = (u_e, (2/3)(G/κ)u_e)."""
    K8 = el.k_int8()
    rnd = random.Random(13683)
    for _ in range(5):
        kappa = Fr(rnd.randint(1, 10 ** 6), rnd.randint(1, 1000))
        G = Fr(rnd.randint(1, 10 ** 6), rnd.randint(1, 1000))
        ds = Fr(rnd.randint(1, 100), rnd.randint(1, 1000))
        u = [Fr(rnd.randint(-10 ** 9, 10 ** 9), rnd.randint(1, 10 ** 6)) for _ in range(24)]
        Ke = _tensor_route_K(kappa, G, ds)
        lhs = [sum(Ke[r][c] * u[c] for c in range(24)) for r in range(24)]
        ub = u + [Fr(2, 3) * G / kappa * x for x in u]
        rhs = [kappa * ds / 256 * (sum(K8[r][k] * ub[k] for k in range(48)) + Fr(256, 3) * G / kappa * u[r])
               for r in range(24)]
        assert lhs == rhs


def test_rigid_body_modes_are_the_exact_null_space():
    kappa, G, ds = Fr(3), Fr(2), Fr(1, 2)
    K = el.element_stiffness(kappa, G, ds)
    # symmetric
    assert all(K[r][c] == K[c][r] for r in range(24) for c in range(24))
    X = [[Fr(c) * ds for c in (sx > 0, sy > 0, sz > 0)] for (sx, sy, sz) in el.CORNERS]
    modes = []
    for ax in range(3):           # translations
        modes.append([Fr(1) if c == ax else Fr(0) for a in range(8) for c in range(3)])
    for ax in range(3):           # infinitesimal rotations u = e_ax × x
        v = []
        for a in range(8):
            x = X[a]
            w = [0, 0, 0]
            w[ax] = 1
            v += [w[1] * x[2] - w[2] * x[1], w[2] * x[0] - w[0] * x[2], w[0] * x[1] - w[1] * x[0]]
        modes.append([Fr(t) for t in v])
    for m in modes:
        assert all(sum(K[r][c] * m[c] for c in range(24)) == 0 for r in range(24))
    Kf = np.array([[float(x) for x in row] for row in K])
    ev = np.linalg.eigvalsh(Kf)
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == 6     # exactly 6 zero modes
    assert ev.min() > -1e-12 * ev.max()                   # PSD


def test_stiffness_linear_in_ds():
    Ka = el.element_stiffness(Fr(2), Fr(1), Fr(1))
    Kb = el.element_stiffness(Fr(2), Fr(1), Fr(1, 3))
    assert all(Kb[r][c] * 3 == Ka[r][c] for r in range(24) for c in range(24))


def test_mass_is_diagonal_without_lumping_paper_L90():
    rho, ds = Fr(2400), Fr(1, 500)
    M = el.element_mass_full(rho, ds)
    for a in range(8):
        for b in range(8):
            assert M[a][b] == (rho * ds ** 3 / 8 if a == b else 0)
    # equals the VFEM lumped value ρ/8 (1)_e exactly
    assert el.element_mass_diag(rho, ds)[0] == rho * ds ** 3 / 8
