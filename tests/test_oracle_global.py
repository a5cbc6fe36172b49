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


@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8, oracle.PATH_VFEM])
@pytest.mark.parametrize("order", [oracle.ORDER_ELEMENT, oracle.ORDER_U2])
def test_scatter_exact_arithmetic_equals_dense_assembly(path, order):
    """Pin of the scatter that does not restate it: with κ = 256, G = 384,
    ds = 1 the element matrices are integer (A_κ·256 + A_G·384 = K^κ + K̄^G + 128 I; VFEM: Vk·256/72 +
    Vg·384/216 is not integer, so VFEM uses κ = 72, G = 216) and u ∈ {−2..2}, so every element force
    and every partial sum is an exact integer: f must equal the brute-force dense assembly K @ u bit
    for bit in ANY summation order.  A transposed corner, a wrong node id, a dropped or duplicated
    element fails.  INT8: every s_e ∈ {1, 2} is a power of two and cG = 1, so ū/s_e·2^56 is exact,
    no truncation happens and f_e = K_e u_e exactly (Eqs. 10-17 reduce to the exact product)."""
    m = wl.small_random(3, 4, 2, ds=1.0)
    if path == oracle.PATH_VFEM:
        m.kappa = np.full_like(m.kappa, 72.0)
        m.G = np.full_like(m.G, 216.0)
        from fractions import Fraction as Fr
        from oracle.element import vfem_element_stiffness
        K = np.zeros((3 * m.n_nodes, 3 * m.n_nodes))
        Ke = np.array([[float(x) for x in r] for r in vfem_element_stiffness(Fr(72), Fr(216), Fr(1))])
        for e in range(m.n_elems):
            d = np.concatenate([[3 * n, 3 * n + 1, 3 * n + 2] for n in oracle.element_nodes(m.nx, m.ny, e)])
            K[np.ix_(d, d)] += Ke
    else:
        m.kappa = np.full_like(m.kappa, 256.0)
        m.G = np.full_like(m.G, 384.0)
        K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    assert np.array_equal(K, np.round(K))
    rng = np.random.default_rng(11)
    u = rng.integers(-2, 3, size=3 * m.n_nodes).astype(np.float64)
    f = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=path, order=order)
    assert np.array_equal(f, K @ u)
    assert np.abs(f).max() > 0


@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8])
def test_u2_mirror_differs_from_the_definition_only_by_summation_rounding(path):
    """The mirror variant (ORDER_U2, the kernels' tree) and the definition (element order) sum the
    same 8 terms per node: |f_U2 − f_elem| ≤ 2·γ_7·Σ_e |f_e[n]| ≤ 2·γ_7·(|K| |u|)_n (γ_7 = 7u/(1−7u))."""
    m = wl.small_random(5, 4, 3, ds=0.01)
    u = wl.random_field(m) * np.exp(np.random.default_rng(5).uniform(-8, 8, 3 * m.n_nodes))
    fa = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=path)
    fb = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=path, order=oracle.ORDER_U2)
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    bound = 2 * 8 * 2.0 ** -53 * 1.001 * (np.abs(K) @ np.abs(u))
    assert np.all(np.abs(fa - fb) <= bound)
    assert not np.array_equal(fa, fb)          # the two orders are really different


def test_u2_mirror_variant_is_the_documented_tree():
    """Implementation check of the MIRROR variant (not a pin of the definition): the oracle's
    ORDER_U2 equals reading U2 rebuilt node by node from the per-element forces."""
    path = oracle.PATH_INT8
    m = wl.small_random(3, 2, 2, ds=0.01)
    u = wl.random_field(m) * np.exp(np.random.default_rng(5).uniform(-8, 8, 3 * m.n_nodes))
    nx, ny, nz = m.nx, m.ny, m.nz
    fe = {}
    for e in range(nx * ny * nz):
        nodes = oracle.element_nodes(nx, ny, e)
        ue = np.concatenate([u[3 * q:3 * q + 3] for q in nodes])
        k = m.mat[e]
        fe[(e % nx, (e // nx) % ny, e // (nx * ny))] = oracle.element_int8(ue, m.kappa[k], m.G[k], m.ds)["fe"]
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
    f = oracle.apply_K(nx, ny, nz, m.ds, m.mat, m.kappa, m.G, u, path=path, order=oracle.ORDER_U2)
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


def _impulse_model(amp_series, node=(2, 1, 3), axis=1):
    m = wl.small_random(4, 3, 4, ds=0.01, dt=1e-6)
    m.dirichlet = wl.corner_mask(m.nx, m.ny, m.nz)
    n = m.node(*node)
    m.src_node = np.array([n], dtype=np.int64)
    m.src_axis = np.array([axis], dtype=np.int32)
    m.amp = np.array(amp_series, dtype=np.float64).reshape(1, -1)
    return m, 3 * n + axis


@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8])
def test_source_impulse_enters_at_its_dof_and_step(path):
    """Source term of Eq. 3 (M ü + K u = F, F^{it} at t = it·dt):
    from u^0 = u^{-1} = 0 a single impulse amp[0] = a gives u^1 = w_n·a at exactly that DOF and 0
    elsewhere (K·0 = 0); u^2 = 2u^1 − w ⊙ (K u^1) (brute-force K); an impulse at amp[1] leaves u^1 = 0
    and gives u^2 = w_n·a; a run started at it = 5 uses amp[5]; it ≥ n_t contributes nothing.
    A wrong sign of F, an amp[it+1] index or a wrong DOF fails here."""
    a = 3.25e3
    m, dof = _impulse_model([a, 0.0, 0.0, 0.0])
    z = np.zeros(3 * m.n_nodes)
    w = oracle.node_w(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho, m.dt)
    u1, u0, it, st = oracle.run(m.as_dict(), z, z, 0, 1, path=path)
    assert st == 0 and it == 1 and np.all(u0 == 0)
    exp1 = np.zeros_like(z)
    exp1[dof] = w[dof // 3] * a
    assert np.array_equal(u1, exp1)
    u2, u1b, _, _ = oracle.run(m.as_dict(), u1, u0, 1, 1, path=path)
    assert np.array_equal(u1b, u1)
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    ref2 = 2 * u1 - np.repeat(w, 3) * (K @ u1)
    ref2[(np.tile([1, 2, 4], m.n_nodes) & np.repeat(m.dirichlet, 3)) > 0] = 0.0   # fixed components
    assert np.abs(u2 - ref2).max() <= 1e-13 * np.abs(ref2).max()
    # impulse one step later
    m, dof = _impulse_model([0.0, a, 0.0])
    u1, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 1, path=path)
    assert np.all(u1 == 0)
    u2, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 2, path=path)
    assert u2[dof] == w[dof // 3] * a and np.count_nonzero(u2) == 1
    # start at it = 5: amp[5] is used; beyond n_t nothing
    m, dof = _impulse_model([0, 0, 0, 0, 0, -a])
    u6, _, it, _ = oracle.run(m.as_dict(), z, z, 5, 1, path=path)
    assert it == 6 and u6[dof] == -w[dof // 3] * a and np.count_nonzero(u6) == 1
    u7, _, _, _ = oracle.run(m.as_dict(), z, z, 6, 1, path=path)
    assert np.all(u7 == 0)


@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8])
def test_energy_balance_with_a_ricker_source(path):
    """Discrete work-energy balance of Eq. 3 with a source (derived by multiplying the scheme by
    (u^{n+1} − u^{n−1})/2, M and K symmetric):
        E_{n+½} − E_{n−½} = F^nᵀ (u^{n+1} − u^{n−1}) / 2,
        E_{n+½} = ½ v_{n+½}ᵀ M v_{n+½} + ½ u^nᵀ K u^{n+1},  v_{n+½} = (u^{n+1} − u^n)/dt,
    with M and K assembled by brute force, checked at every step of a Ricker run."""
    m = wl.small_random(4, 3, 3, ds=1.0, dt=1e-4)
    m.dirichlet = None
    f0 = 400.0
    wl.point_source(m, 2, 1, 3, 2, f0, 1.2 / f0, 80, scale=1e9)
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    md = assemble.assemble_M_diag(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho)
    F = np.zeros(3 * m.n_nodes)
    dof = 3 * int(m.src_node[0]) + int(m.src_axis[0])
    u = [np.zeros(3 * m.n_nodes), np.zeros(3 * m.n_nodes)]     # u^{-1}, u^0
    for n in range(80):
        un, _, _, st = oracle.run(m.as_dict(), u[-1], u[-2], n, 1, path=path)
        assert st == 0
        u.append(un)
    E = [physics.leapfrog_energy(K, md, u[k], u[k + 1], m.dt) for k in range(1, 81)]   # E_{n+½}, n = 0..79
    scale = max(abs(e) for e in E)
    assert scale > 0
    worst = 0.0
    for n in range(1, 80):
        F[:] = 0.0
        F[dof] = m.amp[0, n]
        work = F @ (u[n + 2] - u[n]) / 2.0     # u[k] = u^{k-1}
        worst = max(worst, abs((E[n] - E[n - 1]) - work))
    assert worst <= 1e-12 * scale
    # the same balance with the amplitude one step late is violated (the index pin is sharp)
    late = max(abs((E[n] - E[n - 1]) - m.amp[0, n + 1] * (u[n + 2] - u[n])[dof] / 2.0) for n in range(1, 79))
    assert late > 1e3 * max(worst, 1e-300)


def test_bloch_symbol_axis_aligned_reduces_to_the_bar():
    """Ŝ(k e_x) has the textbook 1-D lattice eigenvalues 4V²/ds² sin²(k ds/2) for V = Vp (×1) and
    V = Vs (×2) — the closed form the axis-aligned GPU test uses."""
    kap, G, rho, ds = 5.0 / 3.0, 1.0, 1.3, 0.7
    for kk in (0.1, 1.0, 2.5):
        lam, _ = physics.bloch_modes(kap, G, rho, ds, (kk, 0.0, 0.0))
        vp, vs = math.sqrt((kap + 4 * G / 3) / rho), math.sqrt(G / rho)
        ref = sorted([physics.lattice_lambda_axis(vs, kk, ds)] * 2 + [physics.lattice_lambda_axis(vp, kk, ds)])
        assert np.allclose(lam, ref, rtol=1e-14, atol=0)


@pytest.mark.parametrize("nu", ["0.25", "0.35"])
@pytest.mark.parametrize("mvec", [(1, 2, 3), (3, 3, 3), (5, 1, 0), (4, 4, 0)])
def test_oblique_roller_box_modes_are_exact_eigenvectors(nu, mvec):
    """on a roller box, u_a = U_a sin(k_a x_a) Π_{b≠a} cos(k_b x_b) with U an
    eigenvector of Ŝ(k) satisfies K u = λ M u exactly at every free DOF (the oracle's product,
    independent of the symbol's derivation); then the time stepper follows cos(nθ),
    cos θ = 1 − λ dt²/2 (Eq. 3 recurrence)."""
    m = wl.c2_block(8, nu=nu)
    k = [math.pi * mv / (8 * m.ds) for mv in mvec]
    lam, U = physics.bloch_modes(m.kappa[0], m.G[0], m.rho[0], m.ds, k)
    free = (np.tile([1, 2, 4], m.n_nodes) & np.repeat(m.dirichlet, 3)) == 0
    md = assemble.assemble_M_diag(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho)
    for i in range(3):
        u0 = wl.standing_wave(m, mvec=mvec, U=tuple(U[:, i]))
        f = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u0)
        res = f[free] - lam[i] * md[free] * u0[free]
        assert np.linalg.norm(res) <= 1e-13 * np.linalg.norm(f[free])
    th = math.acos(1 - lam[-1] * m.dt ** 2 / 2)
    u0 = wl.standing_wave(m, mvec=mvec, U=tuple(U[:, -1]))
    u, _, _, st = oracle.run(m.as_dict(), u0, math.cos(th) * u0, 0, 60)
    assert st == 0
    assert np.linalg.norm(u - math.cos(60 * th) * u0) <= 1e-12 * np.linalg.norm(u0)
