"""Pins for the oracle's Rayleigh-damped time step (NEXT-1, reading R1).

Pinned against: the two-point fit's defining property; the closed-form solution of the damped
modal recurrence for an exact lattice eigenmode (α only, β only, both — a dropped term, a wrong
sign or swapped roles fails one of them); the continuous-time decay rate exp(−ζ(ω) ω t) in the
small-dt limit; monotone decay of the discrete energy.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as wl
from oracle import assemble, physics


def test_rayleigh_two_point_fit():
    a, b = wl.rayleigh_coeffs(100e3, 125e3, 0.01)
    for f in (100e3, 125e3):
        assert physics.rayleigh_zeta(a, b, 2 * math.pi * f) == pytest.approx(0.01, rel=1e-12)
    grid = np.linspace(2 * math.pi * 100e3, 2 * math.pi * 125e3, 101)
    assert max(physics.rayleigh_zeta(a, b, w) for w in grid) <= 0.01 * (1 + 1e-12)   # interior dip
    assert wl.rayleigh_coeffs(100e3, 125e3, 0.0) == (0.0, 0.0)
    with pytest.raises(ValueError):
        wl.rayleigh_coeffs(125e3, 100e3, 0.01)


def _mode_box():
    m = wl.c2_block(8)
    m.nx, m.ny, m.nz = 12, 4, 4
    m.mat = np.zeros(m.nx * m.ny * m.nz, np.uint8)
    m.dirichlet = wl.roller_mask(m.nx, m.ny, m.nz)
    u0 = wl.standing_wave(m, mvec=(3, 0, 0), U=(1.0, 0.0, 0.0))
    k = math.pi * 3 / (m.nx * m.ds)
    V = math.sqrt((m.kappa[0] + 4 * m.G[0] / 3) / m.rho[0])
    return m, u0, physics.lattice_lambda_axis(V, k, m.ds)


@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8])
@pytest.mark.parametrize("ab", [(0.02, 0.0), (0.0, 0.03), (0.015, 0.02)])
def test_damped_mode_follows_closed_form(path, ab):
    m, u0, lam = _mode_box()
    w = math.sqrt(lam)
    m.alpha, m.beta = ab[0] * w, ab[1] / w        # α ~ ω, β ~ 1/ω so both terms matter
    nsteps = 200
    u, _, it, st = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=path)
    assert st == 0 and it == nsteps
    a = physics.mode_amplitude_damped(lam, m.dt, m.alpha, m.beta, nsteps)
    assert np.abs(u - a * u0).max() <= 1e-11 * np.abs(u0).max()
    a_undamped = physics.mode_amplitude(lam, m.dt, nsteps)
    assert abs(a) < abs(a_undamped) or abs(a_undamped) < 0.2   # the mode lost amplitude


def test_damped_decay_rate_matches_zeta():
    """Small dt: the modal envelope decays as exp(−ζ(ω) ω t) with ζ = α/(2ω) + βω/2."""
    m, u0, lam = _mode_box()
    w = math.sqrt(lam)
    m.dt = 0.02 / w                                # 314 steps per period
    m.alpha, m.beta = wl.rayleigh_coeffs(0.8 * w / (2 * math.pi), 1.25 * w / (2 * math.pi), 0.02)
    zeta = physics.rayleigh_zeta(m.alpha, m.beta, w)
    per = int(round(2 * math.pi / (w * m.dt)))
    n = 5 * per
    u, up, _, st = oracle.run(m.as_dict(), u0, u0, 0, n, path=oracle.PATH_FP64)
    assert st == 0
    # envelope from the discrete modal energy ~ a_n² + (a_n − a_{n−1})²/(ω dt)²
    i = int(np.argmax(np.abs(u0)))
    a_n, a_m = u[i] / u0[i], up[i] / u0[i]
    env = math.sqrt(a_n ** 2 + ((a_n - a_m) / (w * m.dt)) ** 2)
    rate = -math.log(env) / (n * m.dt)
    assert rate == pytest.approx(zeta * w, rel=0.03)


def test_damped_energy_decreases():
    m = wl.small_random(4, 4, 4, ds=1.0, dt=1e-4)
    m.dirichlet = None
    rng = np.random.default_rng(13683)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-3
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    md = assemble.assemble_M_diag(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho)
    ev = np.linalg.eigvalsh((K / np.sqrt(md)[:, None]) / np.sqrt(md)[None, :]).max()
    m.dt = 0.5 * 2.0 / math.sqrt(ev)
    m.alpha, m.beta = 0.05 * math.sqrt(ev), 0.02 / math.sqrt(ev)
    u, up = u0.copy(), u0.copy()
    E = []
    for _ in range(80):
        un, u2, _, st = oracle.run(m.as_dict(), u, up, 0, 1)
        assert st == 0
        E.append(physics.leapfrog_energy(K, md, u, un, m.dt))
        u, up = un, u2
    E = np.array(E)
    assert np.all(np.diff(E) <= 1e-14 * E[0])
    assert E[-1] < 0.5 * E[0]


def test_zero_damping_is_the_undamped_step():
    m = wl.small_random(5, 3, 4, ds=0.01, dt=1e-6)
    wl.point_source(m, 2, 1, 4, 2, 2e5, 1e-5, 30, scale=1.0)
    z = np.zeros(3 * m.n_nodes)
    u1, up1, _, _ = oracle.run(m.as_dict(), z, z, 0, 30, path=oracle.PATH_INT8)
    d = m.as_dict()
    d["alpha"], d["beta"] = 0.0, 0.0
    u2, up2, _, _ = oracle.run(d, z, z, 0, 30, path=oracle.PATH_INT8)
    assert np.array_equal(u1, u2) and np.array_equal(up1, up2)
