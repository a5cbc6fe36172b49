"""Pins for the oracle's global EBE product, node mass and time integrator.

Pinned against: closed-form numbering (D1) and shared-face counts; brute-force
dense assembly (Eq. 2); exact rigid-mode null space of the free mesh; the
patch test; the textbook central-difference recurrence for an exact lattice
eigenmode with the 1-D lattice dispersion relation; the leapfrog energy
invariant; the Err metric's closed-form cases.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as wl
from oracle import assemble, physics


def test_numbering_closed_form_and_shared_face():
    nx, ny = 2, 1
    n0 = oracle.element_nodes(nx, ny, 0)
    n1 = oracle.element_nodes(nx, ny, 1)
    assert len(set(n0) & set(n1)) == 4
    nx, ny, nz = 5, 4, 3
    seen = set()
    for e in range(nx * ny * nz):
        ex, ey, ez = e % nx, (e // nx) % ny, e // (nx * ny)
        nodes = oracle.element_nodes(nx, ny, e)
        assert nodes[0] == ex + (nx + 1) * (ey + (ny + 1) * ez)
        assert nodes[6] == (ex + 1) + (nx + 1) * ((ey + 1) + (ny + 1) * (ez + 1))
        seen.update(int(x) for x in nodes)
    assert seen == set(range((nx + 1) * (ny + 1) * (nz + 1)))


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (3, 3, 3), (4, 2, 3)])
def test_ebe_matches_dense_assembly(dims):
    m = wl.small_random(*dims, ds=0.01)
    u = wl.random_field(m)
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    assert np.allclose(K, K.T, rtol=0, atol=1e-12 * np.abs(K).max())
    ref = K @ u
    for path in (oracle.PATH_FP64, oracle.PATH_INT8):
        f = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=path)
        assert np.linalg.norm(f - ref) <= 1e-14 * np.linalg.norm(ref)


@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8])
def test_summation_order_is_the_u2_tree(path):
    """Reading U2: f_n = T_n + B_n with face(ez) = P(iy) + P(iy-1), P = x-pair of corner values
    (missing elements 0.0), rebuilt here from the per-element forces one node at a time."""
    m = wl.small_random(3, 2, 2, ds=0.01)
    u = wl.random_field(m) * np.exp(np.random.default_rng(5).uniform(-8, 8, 3 * m.n_nodes))
    nx, ny, nz = m.nx, m.ny, m.nz
    fe = {}
    for e in range(nx * ny * nz):
        nodes = oracle.element_nodes(nx, ny, e)
        ue = np.concatenate([u[3 * q:3 * q + 3] for q in nodes])
        k = m.mat[e]
        fe[(e % nx, (e // nx) % ny, e // (nx * ny))] = (
            oracle.element_fp64(ue, m.kappa[k], m.G[k], m.ds) if path == oracle.PATH_FP64
            else oracle.element_int8(ue, m.kappa[k], m.G[k], m.ds)["fe"])
    corner = {(0, 0): 0, (0, 1): 1, (1, 1): 2, (1, 0): 3}   # (dy, dx) -> local node of e(ix-dx, iy-dy)

    def val(ix, iy, ez, dx, dy, top, c):
        e = (ix - dx, iy - dy, ez)
        return fe[e][3 * (corner[(dy, dx)] + 4 * top) + c] if e in fe else 0.0

    ref = np.zeros(3 * m.n_nodes)
    for iz in range(nz + 1):
        for iy in range(ny + 1):
            for ix in range(nx + 1):
                n = ix + (nx + 1) * (iy + (ny + 1) * iz)
                for c in range(3):
                    face = [(val(ix, iy, ez, 0, 0, top, c) + val(ix, iy, ez, 1, 0, top, c)) +
                            (val(ix, iy, ez, 0, 1, top, c) + val(ix, iy, ez, 1, 1, top, c))
                            for ez, top in ((iz - 1, 1), (iz, 0))]
                    ref[3 * n + c] = face[0] + face[1]
    f = oracle.apply_K(nx, ny, nz, m.ds, m.mat, m.kappa, m.G, u, path=path)
    assert np.array_equal(f, ref)


def test_free_cube_has_exactly_six_zero_modes():
    m = wl.small_random(3, 3, 3, ds=1.0)
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    Mi = 1.0 / np.sqrt(assemble.assemble_M_diag(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho))
    ev = np.linalg.eigvalsh(Mi[:, None] * K * Mi[None, :])
    assert np.sum(np.abs(ev) < 1e-9 * ev.max()) == 6


def test_patch_test_linear_field_gives_zero_interior_force():
    m = wl.c1_cube(4)
    m.ds = 1.0
    n = m.nx + 1
    grid = np.stack(np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij"), -1)[..., ::-1]
    x = grid.reshape(-1, 3).astype(np.float64)   # node order z, y, x -> (x, y, z) coordinates
    A = np.array([[0.3, -0.2, 0.5], [0.1, 0.7, -0.4], [0.25, 0.05, -0.6]])
    u = (x @ A.T + np.array([1.0, 2.0, 3.0])).reshape(-1)
    f = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u).reshape(-1, 3)
    inner = [(ix + n * (iy + n * iz)) for iz in range(1, n - 1) for iy in range(1, n - 1) for ix in range(1, n - 1)]
    assert np.abs(f[inner]).max() <= 1e-13 * np.abs(f).max()
    assert np.abs(f).max() > 0


def test_node_mass_matches_assembly():
    m = wl.small_random(4, 3, 2)
    w = oracle.node_w(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho, m.dt)
    md = assemble.assemble_M_diag(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho)[::3]
    assert np.allclose(w, m.dt ** 2 / md, rtol=1e-15, atol=0)


@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8])
@pytest.mark.parametrize("wave", ["Px", "Py"])
def test_standing_wave_follows_closed_form_dispersion(path, wave):
    """Axis-aligned P mode on a roller box: u^n = a_n u^0 with λ = 4V²/ds² sin²(k ds/2).

    (An axis-aligned S mode is not compatible with rollers on the side faces.)"""
    m = wl.c2_block(8)
    m.nx, m.ny, m.nz = 12, 4, 4
    m.mat = np.zeros(m.nx * m.ny * m.nz, np.uint8)
    m.dirichlet = wl.roller_mask(m.nx, m.ny, m.nz)
    U = (1.0, 0.0, 0.0) if wave == "Px" else (0.0, 1.0, 0.0)
    mvec = (3, 0, 0) if wave == "Px" else (0, 2, 0)
    u0 = wl.standing_wave(m, mvec=mvec, U=U)
    k = math.pi * max(mvec) / (m.nx * m.ds if wave == "Px" else m.ny * m.ds)
    kap, G, rho = m.kappa[0], m.G[0], m.rho[0]
    V = math.sqrt((kap + 4 * G / 3) / rho)
    lam = physics.lattice_lambda_axis(V, k, m.ds)
    nsteps = 200
    u, up, it, st = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=path)
    assert st == 0 and it == nsteps
    a = physics.mode_amplitude(lam, m.dt, nsteps)
    assert np.abs(u - a * u0).max() <= 1e-12 * np.abs(u0).max()


def test_leapfrog_energy_is_conserved():
    m = wl.small_random(4, 4, 4, ds=1.0, dt=1e-4)
    m.dirichlet = None
    rng = np.random.default_rng(13683)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-3
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    md = assemble.assemble_M_diag(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho)
    ev = np.linalg.eigvalsh((K / np.sqrt(md)[:, None]) / np.sqrt(md)[None, :]).max()
    m.dt = 0.8 * 2.0 / math.sqrt(ev)
    u, up = u0.copy(), u0.copy()
    E = []
    for _ in range(60):
        un, u2, _, st = oracle.run(m.as_dict(), u, up, 0, 1)
        assert st == 0
        E.append(physics.leapfrog_energy(K, md, u, un, m.dt))
        u, up = un, u2
    E = np.array(E)
    assert np.abs(E - E[0]).max() <= 1e-12 * abs(E[0])


def test_zero_state_is_a_fixed_point_and_source_linearity():
    m = wl.c1_cube(4, steps=30)
    z = np.zeros(3 * m.n_nodes)
    d = m.as_dict()
    d["amp"] = np.zeros_like(m.amp)
    u, up, it, st = oracle.run(d, z, z, 0, 30)
    assert np.all(u == 0) and np.all(up == 0)
    u1, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 30)
    d["amp"] = 2.0 * m.amp
    u2, _, _, _ = oracle.run(d, z, z, 0, 30)
    assert np.abs(u2 - 2 * u1).max() <= 1e-12 * np.abs(u1).max()


def test_err_metric_closed_forms():
    rng = np.random.default_rng(0)
    ref = rng.standard_normal((24, 100))
    assert physics.err_metric(ref, ref) == 0.0
    assert physics.err_metric(np.zeros_like(ref), ref) == 1.0
    assert abs(physics.err_metric(1.1 * ref, ref) - 0.01) < 1e-14


def test_int8_and_fp64_trajectories_agree():
    """The paper's claim that the INT8 path matches FP64 (L245-L258), over a run with a source."""
    m = wl.c1_cube(6, steps=300)
    z = np.zeros(3 * m.n_nodes)
    a, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 300, path=oracle.PATH_FP64)
    b, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 300, path=oracle.PATH_INT8)
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)
