"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (DESIGN.md §3 "parity bars"):
  * integer work (v, byte slices, per-stage tensor-core products C_j, y) and the per-element
    forces f_e — bit-exact (they do not depend on any summation order);
  * global f = K u against the oracle's DEFINITION (plain element-order scatter): per node within
    the cross-order rounding bound 2·γ_7·Σ_e|f_e[n]| (INT8, dense paths) or the factored-form bound
    (tests/parity.py); additionally bit-exact against the oracle's MIRROR variant ORDER_U2 (the
    kernels' per-node tree, reading U2) for the INT8 and dense paths;
  * trajectories: within rel-L2 1e-10 of the oracle's definition after up to 1000 steps
    (BASELINE.json north_star), and bit-exact against the U2 mirror for the INT8 / dense paths;
  * full-size (256³, 512³, 1e9-DOF) launches: the whole field (C2) or sampled nodes recomputed by
    the oracle node by node, in the bench's launch configuration.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as wl
from parity import GAMMA7, factored_bound, within

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ovxmod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_13683_b200 import ovx
    return ovx


def _solver(ovxmod, m, path):
    s = ovxmod.Ovx(0)
    s.load_model(m, path)
    return s


PATHS = [("int8", 0), ("fp64", 1), ("fp64_dense", 2), ("vfem", 3), ("vfem_dense", 4)]
EXACT = {0: True, 1: False, 2: True, 3: False, 4: True}   # factored forms differ from the dense order by rounding
ORACLE_PATH = {0: oracle.PATH_INT8, 1: oracle.PATH_FP64, 2: oracle.PATH_FP64, 3: oracle.PATH_VFEM, 4: oracle.PATH_VFEM}


def _close(a, ref, path, rel=1e-13):
    if EXACT[path]:
        return np.array_equal(a, ref)
    return np.linalg.norm(a - ref) <= rel * np.linalg.norm(ref)


def _check_apply(f, m, u, path, M=8):
    """f = K u from the GPU against the oracle: the definition within the per-node bound, and the
    U2 mirror bit for bit on the INT8 / dense paths."""
    op = ORACLE_PATH[path]
    plain, mirror, absf = oracle.apply_K_orders(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=op, M=M)
    if EXACT[path]:
        assert np.array_equal(f, mirror), "differs from the oracle's U2 mirror"
        ok, worst = within(f, plain, 2 * GAMMA7 * absf + 5e-324)
    else:
        ok, worst = within(f, plain, factored_bound(m, u))
    assert ok, f"outside the per-node bound (worst ratio {worst:.3g})"
    return plain


def _traj_check(u, m, u0, up0, it0, nsteps, path, bar=1e-10, order_bits=True):
    """A GPU trajectory against the oracle's definition (rel-L2 ≤ bar) and, on the INT8 / dense
    paths, against the U2 mirror bit for bit.  Returns the definition's state."""
    op = ORACLE_PATH[path]
    ru, rup, rit, st = oracle.run(m.as_dict(), u0, up0, it0, nsteps, path=op)
    assert st == 0
    assert np.linalg.norm(u[0] - ru) <= bar * np.linalg.norm(ru)
    assert np.linalg.norm(u[1] - rup) <= bar * max(np.linalg.norm(rup), 1e-300)
    if EXACT[path] and order_bits:
        mu, mup, _, _ = oracle.run(m.as_dict(), u0, up0, it0, nsteps, path=op, order=oracle.ORDER_U2)
        assert np.array_equal(u[0], mu) and np.array_equal(u[1], mup), "differs from the U2 mirror"
    return ru, rup


def _ragged():
    # spans several tiles in x (31 nodes) and y (3 nodes), two z-chunks (64 planes), ragged tails
    m = wl.small_random(40, 8, 70, ds=0.01, dt=1e-6)
    return m


def test_node_w_bit_exact(ovxmod):
    m = _ragged()
    s = _solver(ovxmod, m, 0)
    w = s.get_node_w()
    ref = oracle.node_w(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho, m.dt)
    assert np.array_equal(w, ref)


def test_library_matrix_equals_oracle_matrix(ovxmod):
    s = ovxmod.Ovx(0)
    K8, _, _ = oracle.int_matrices()
    assert np.array_equal(s.get_int8_matrix(), K8)


@pytest.mark.parametrize("name,path", PATHS)
@pytest.mark.parametrize("dims", [(1, 1, 1), (5, 4, 3), (40, 8, 70), (33, 2, 65)])
def test_apply_K(ovxmod, name, path, dims):
    m = wl.small_random(*dims, ds=0.01)
    u = wl.random_field(m)
    s = _solver(ovxmod, m, path)
    _check_apply(s.apply_K(u), m, u, path)


@pytest.mark.parametrize("name,path", PATHS)
def test_apply_K_wide_dynamic_range(ovxmod, name, path):
    """Node magnitudes spread over 10^±12 across the grid: the per-node bounds are sharp where the
    forces are small (a global bound would not see errors there)."""
    m = wl.small_random(40, 8, 70, ds=0.01)
    rng = np.random.default_rng(21)
    u = wl.random_field(m) * np.repeat(10.0 ** rng.uniform(-12, 12, m.n_nodes), 3)
    s = _solver(ovxmod, m, path)
    _check_apply(s.apply_K(u), m, u, path)


def test_int8_element_records_bit_exact(ovxmod):
    m = wl.small_random(9, 5, 4, ds=0.01)
    rng = np.random.default_rng(7)
    u = wl.random_field(m) * 10.0 ** rng.uniform(-20, 5, size=3 * m.n_nodes)
    u[::97] = 0.0
    s = _solver(ovxmod, m, 0)
    rec = s.debug_element_ints(u, 0, m.n_elems)
    K8, _, _ = oracle.int_matrices()
    for e in range(m.n_elems):
        nodes = oracle.element_nodes(m.nx, m.ny, e)
        ue = np.concatenate([u[3 * n:3 * n + 3] for n in nodes])
        mm = m.mat[e]
        r = oracle.element_int8(ue, m.kappa[mm], m.G[mm], m.ds, 8, oracle.DIGITS_BYTES_FOLD)
        assert rec["s"][e] == r["s"]
        assert np.array_equal(rec["v"][e], r["v"])
        assert np.array_equal(rec["d"][e].astype(np.int32), r["d"])
        assert np.array_equal(rec["C"][e].astype(np.int64), r["C"])
        assert rec["y"][e] == r["y"]
        assert np.array_equal(rec["fe"][e], r["fe"])


def test_int8_edge_inputs(ovxmod):
    m = wl.small_random(6, 4, 3, ds=0.01)
    s = _solver(ovxmod, m, 0)
    z = np.zeros(3 * m.n_nodes)
    assert np.all(s.apply_K(z) == 0.0)
    for scale in (1e-310, 1e-300, 1e-290, 1e300):
        u = wl.random_field(m) * scale
        ref = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=oracle.PATH_INT8,
                             order=oracle.ORDER_U2)
        assert np.array_equal(s.apply_K(u), ref, equal_nan=True), scale
    # sign-aligned extremes (the worst case of the two-limb recombination)
    u = np.sign(wl.random_field(m)) * 3.0
    _check_apply(s.apply_K(u), m, u, 0)


@pytest.mark.parametrize("name,path", PATHS)
def test_c1_trajectory(ovxmod, name, path):
    """C1 (8³ concrete cube, Ricker source, 4 fixed corners), 100 steps: within 1e-12 of the
    oracle's definition; bit-exact vs the U2 mirror (INT8, dense)."""
    m = wl.c1_cube(8, steps=100)
    z = np.zeros(3 * m.n_nodes)
    s = _solver(ovxmod, m, path)
    s.set_state(z, z, 0)
    s.step(100)
    u, up, it = s.get_state()
    assert it == 100
    _traj_check((u, up), m, z, z, 0, 100, path, bar=1e-12)
    assert np.abs(u).max() > 0


def test_1000_steps_int8_vs_fp64_oracle(ovxmod):
    """BASELINE.json bar: INT8 path within 1e-10 rel-L2 of the FP64 oracle (the definition: element-
    order scatter) after 1000 steps (heterogeneous, ragged grid, source, fixed corners); also
    bit-exact vs the INT8 oracle's U2 mirror."""
    m = wl.small_random(14, 9, 12, ds=1.0, dt=1e-4)
    f0 = 25.0
    wl.point_source(m, 7, 4, 12, 2, f0, 1.2 / f0, 1000, scale=1e6)
    z = np.zeros(3 * m.n_nodes)
    s = _solver(ovxmod, m, 0)
    assert m.dt < s.critical_dt()
    s.set_state(z, z, 0)
    s.step(1000)
    s.check_finite()
    u, _, _ = s.get_state()
    ref64, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 1000, path=oracle.PATH_FP64)
    ref8, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 1000, path=oracle.PATH_INT8, order=oracle.ORDER_U2)
    assert np.linalg.norm(u - ref64) <= 1e-10 * np.linalg.norm(ref64)
    assert np.array_equal(u, ref8)
    s64 = _solver(ovxmod, m, 1)
    s64.set_state(z, z, 0)
    s64.step(1000)
    u64, _, _ = s64.get_state()
    assert np.linalg.norm(u64 - ref64) <= 1e-10 * np.linalg.norm(ref64)


def _node_force_oracle(m, u, ix, iy, iz, path):
    """f at one node from the oracle's element forces: (U2 mirror order, element order = the
    definition, the per-node bound of the comparison with the definition).
    Mirror (reading U2): f = T + B, face = P(iy) + P(iy-1), P = f(ix,·)[corner] + f(ix-1,·)[corner]
    (missing: 0.0).  Definition: 0.0 + the contributions in increasing element id."""
    import parity
    corner = {(0, 0): 0, (0, 1): 1, (1, 1): 2, (1, 0): 3}   # (dy, dx) -> local node of e(ix-dx, iy-dy)
    contrib = {}                                            # element id -> (force 3-vector, scale)

    def val(dx, dy, ez, top):
        ex, ey = ix - dx, iy - dy
        if not (0 <= ex < m.nx and 0 <= ey < m.ny and 0 <= ez < m.nz):
            return np.zeros(3)
        e = ex + m.nx * (ey + m.ny * ez)
        nodes = oracle.element_nodes(m.nx, m.ny, e)
        ue = np.concatenate([u[3 * n:3 * n + 3] for n in nodes])
        mm = m.mat[e]
        fe = (oracle.element_int8(ue, m.kappa[mm], m.G[mm], m.ds)["fe"] if path == 0
              else oracle.element_vfem(ue, m.kappa[mm], m.G[mm], m.ds) if path in (3, 4)
              else oracle.element_fp64(ue, m.kappa[mm], m.G[mm], m.ds))
        a = corner[(dy, dx)] + 4 * top
        fac = parity.FACTORED_C * parity.U * (m.kappa[mm] + m.G[mm]) * m.ds * np.abs(ue).sum()
        contrib[e] = (fe[3 * a:3 * a + 3], fac)
        return fe[3 * a:3 * a + 3]

    faces = [(val(0, 0, ez, top) + val(1, 0, ez, top)) + (val(0, 1, ez, top) + val(1, 1, ez, top))
             for ez, top in ((iz - 1, 1), (iz, 0))]
    mirror = faces[0] + faces[1]
    plain = np.zeros(3)
    absf = np.zeros(3)
    fact = 0.0
    for e in sorted(contrib):
        plain = plain + contrib[e][0]
        absf = absf + np.abs(contrib[e][0])
        fact += contrib[e][1]
    bound = (2 * GAMMA7 * absf if EXACT[path] else np.full(3, fact)) + 5e-324
    return mirror, plain, bound


def _check_node(fn, m, u, ix, iy, iz, path):
    mirror, plain, bound = _node_force_oracle(m, u, ix, iy, iz, path)
    if EXACT[path]:
        assert np.array_equal(fn, mirror), ("U2 mirror", ix, iy, iz)
    assert np.all(np.abs(fn - plain) <= bound), ("definition", ix, iy, iz, fn, plain, bound)


_C2_REF = {}


def _c2_oracle(m, u, op):
    """The oracle's full-field C2 product (cached per oracle path: the dense and factored GPU forms
    share it)."""
    if op not in _C2_REF:
        _C2_REF.clear()
        _C2_REF[op] = oracle.apply_K_orders(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=op)
    return _C2_REF[op]


@pytest.mark.parametrize("name,path", PATHS)
def test_full_field_c2(ovxmod, name, path):
    """C2 (256³, 16.8 M elements, the bench configuration and launch): EVERY node force against
    the oracle — the definition within the per-node bound, the U2 mirror bit for bit (INT8, dense)."""
    import torch
    m = wl.c2_block(256)
    u = wl.random_field(m)
    s = _solver(ovxmod, m, path)
    ut = torch.from_numpy(u).cuda()
    ft = torch.empty_like(ut)
    s.apply_K_device(ut, ft)
    s.sync()
    f = ft.cpu().numpy()
    del ut, ft
    plain, mirror, absf = _c2_oracle(m, u, ORACLE_PATH[path])
    if EXACT[path]:
        assert np.array_equal(f, mirror)
        ok, worst = within(f, plain, 2 * GAMMA7 * absf + 5e-324)
    else:
        ok, worst = within(f, plain, factored_bound(m, u))
    assert ok, worst
    for (ix, iy, iz) in [(0, 0, 0), (256, 256, 256), (31, 3, 64), (128, 7, 200)]:   # the node-wise route
        n = ix + 257 * (iy + 257 * iz)
        _check_node(f[3 * n:3 * n + 3], m, u, ix, iy, iz, path)


def test_c2_plane_wave_dispersion_on_gpu(ovxmod):
    """Physics at scale: axis-aligned standing P wave on a 128×32×32 roller box, 1000 steps,
    against the closed-form lattice recurrence (property that holds at any size)."""
    from oracle import physics
    m = wl.c2_block(32)
    m.nx, m.ny, m.nz = 128, 32, 32
    m.mat = np.zeros(m.nx * m.ny * m.nz, np.uint8)
    m.dirichlet = wl.roller_mask(m.nx, m.ny, m.nz)
    u0 = wl.standing_wave(m, mvec=(16, 0, 0), U=(1.0, 0.0, 0.0))
    k = math.pi * 16 / (m.nx * m.ds)
    V = math.sqrt((m.kappa[0] + 4 * m.G[0] / 3) / m.rho[0])
    lam = physics.lattice_lambda_axis(V, k, m.ds)
    for path in (0, 1, 2):
        s = _solver(ovxmod, m, path)
        s.set_state(u0, u0, 0)
        s.step(1000)
        u, _, _ = s.get_state()
        a = physics.mode_amplitude(lam, m.dt, 1000)
        assert np.abs(u - a * u0).max() <= 1e-10 * np.abs(u0).max()


def test_receiver_traces_and_err_metric(ovxmod):
    """Receivers at the paper's observation-point layout (Table 1: a line of points on the top
    surface, z-force source): GPU traces equal the oracle's step-by-step trace bit for bit (INT8),
    and the Err metric between the INT8 and FP64 paths is at FP64 round-off."""
    from oracle import physics
    m = wl.c1_cube(8, steps=120)
    rec = np.array([m.node(ix, 4, 8) for ix in (1, 2, 3, 5, 6, 7)], dtype=np.int64)
    z = np.zeros(3 * m.n_nodes)
    traces = {}
    for path in (0, 1):
        s = _solver(ovxmod, m, path)
        s.set_receivers(rec, 120)
        s.set_state(z, z, 0)
        s.step(120)
        traces[path] = s.get_traces()
    # oracle traces, one step at a time: the U2 mirror (bits) and the definition (Err)
    refs = {}
    for order in (oracle.ORDER_U2, oracle.ORDER_ELEMENT):
        u, up = z.copy(), z.copy()
        ref = np.zeros((len(rec), 3, 120))
        for it in range(120):
            u, up, _, _ = oracle.run(m.as_dict(), u, up, it, 1, path=oracle.PATH_INT8, order=order)
            for k, n in enumerate(rec):
                ref[k, :, it] = u[3 * n:3 * n + 3]
        refs[order] = ref
    assert np.array_equal(traces[0], refs[oracle.ORDER_U2])
    # channels that are zero by symmetry carry only round-off in one order and exact zeros in the
    # other (Err = 1 there); compare the channels with signal
    en = (refs[oracle.ORDER_ELEMENT].reshape(-1, 120) ** 2).sum(1)
    live0 = en > 1e-20 * en.max()
    assert physics.err_metric(traces[0].reshape(-1, 120)[live0],
                              refs[oracle.ORDER_ELEMENT].reshape(-1, 120)[live0]) < 1e-24
    a8, a64 = traces[0].reshape(-1, 120), traces[1].reshape(-1, 120)
    e64 = (a64 ** 2).sum(1)
    live = e64 > 1e-20 * e64.max()
    err = physics.err_metric(a8[live], a64[live])
    assert err < 1e-24


@pytest.mark.parametrize("M", [4, 6])
def test_int8_stage_variants_bit_exact(ovxmod, M):
    """NEXT-4: M = 4 / 6 INT8 stages (a = 2^{7M}) on the tensor cores, bit-exact vs the oracle."""
    m = wl.small_random(35, 9, 11, ds=0.01)
    u = wl.random_field(m)
    s = ovxmod.Ovx(0)
    s.load_model(m, 0, stages=M)
    _check_apply(s.apply_K(u), m, u, 0, M=M)
    rec = s.debug_element_ints(u, 0, 40)
    for e in range(40):
        nodes = oracle.element_nodes(m.nx, m.ny, e)
        ue = np.concatenate([u[3 * n:3 * n + 3] for n in nodes])
        r = oracle.element_int8(ue, m.kappa[m.mat[e]], m.G[m.mat[e]], m.ds, M, oracle.DIGITS_BYTES_FOLD)
        nb = r["d"].shape[0]
        assert np.array_equal(rec["v"][e], r["v"])
        assert np.array_equal(rec["d"][e][:nb].astype(np.int32), r["d"])
        assert np.array_equal(rec["C"][e][:nb].astype(np.int64), r["C"])
        assert rec["y"][e] == r["y"]


def test_table3_hierarchy_on_gpu(ovxmod):
    """PAPER.md Table 3 / L245 on the tensor cores: error vs the exact product falls from M = 4
    (FP32-class, ~2^-28) to M = 8 (FP64-class), measured on K·u for a random u (reading Q21)."""
    from fractions import Fraction as Fr
    from oracle import assemble
    m = wl.small_random(3, 3, 3, ds=2e-3)
    u = wl.random_field(m)
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    ref = K @ u
    errs = {}
    for M in (4, 6, 8):
        s = ovxmod.Ovx(0)
        s.load_model(m, 0, stages=M)
        errs[M] = np.linalg.norm(s.apply_K(u) - ref) / np.linalg.norm(ref)
    assert errs[8] < 1e-14 and errs[6] < 1e-11 and 1e-10 < errs[4] < 1e-6
    assert errs[8] < errs[6] < errs[4]


@pytest.mark.parametrize("name,path", PATHS)
def test_damped_c1_trajectory(ovxmod, name, path):
    """NEXT-1: Rayleigh damping (reading R1), C1 cube with the paper's 100-125 kHz band (ζ = 0.05),
    100 steps against the damped oracle run; bit-exact on the INT8 and dense paths."""
    m = wl.c1_cube(8, steps=100)
    m.alpha, m.beta = wl.rayleigh_coeffs(100e3, 125e3, 0.05)
    z = np.zeros(3 * m.n_nodes)
    s = _solver(ovxmod, m, path)
    s.set_state(z, z, 0)
    s.step(100)
    u, up, it = s.get_state()
    assert it == 100
    ru, _ = _traj_check((u, up), m, z, z, 0, 100, path, bar=1e-12)
    u0, _, _, _ = oracle.run(wl.c1_cube(8, steps=100).as_dict(), z, z, 0, 100, path=ORACLE_PATH[path])
    assert np.linalg.norm(u - u0) > 1e-6 * np.linalg.norm(u0)      # damping changed the answer


def test_damped_ragged_multichunk_bit_exact(ovxmod):
    """Damped steps read u_prev at halo nodes of neighbouring tiles and z-chunks: the update goes to
    a third buffer; several tiles in x and y, two z-chunks, ragged tails, a source; INT8 path."""
    m = _ragged()
    wl.point_source(m, 17, 3, 35, 1, 1e5, 2e-5, 40, scale=1.0)
    m.alpha, m.beta = 0.02 / m.dt, 0.03 * m.dt
    rng = np.random.default_rng(3)
    u0 = wl.random_field(m) * 1e-3
    up0 = u0 + rng.standard_normal(u0.size) * 1e-6
    for path in (0, 2):
        s = _solver(ovxmod, m, path)
        s.set_state(u0, up0, 0)
        s.step(12)
        u, up, _ = s.get_state()
        _traj_check((u, up), m, u0, up0, 0, 12, path, bar=1e-12)


def test_e1_rebar_reduced_bit_exact(ovxmod):
    """NEXT-2: the paper's rebar model (E1) at ds = 8 mm (steel / concrete, Table 1 source and
    receivers, Rayleigh damping over 100-125 kHz), 30 steps: INT8 and dense-FP64 states and
    receiver traces equal the oracle's U2 mirror bit for bit and its definition to 1e-12."""
    m = wl.e1_rebar(8.0, steps=30)
    m.amp = (1e3 * wl.bandlimited_impulse(12 * m.dt, 100e3, 125e3, m.dt, 30)).reshape(1, -1)   # early pulse
    z = np.zeros(3 * m.n_nodes)
    for path in (0, 2):
        s = _solver(ovxmod, m, path)
        s.set_receivers(m.receivers, 30)
        s.set_state(z, z, 0)
        s.step(30)
        u, up, _ = s.get_state()
        tr = s.get_traces()
        ru, rup, ref = z.copy(), z.copy(), np.zeros((len(m.receivers), 3, 30))
        for it in range(30):
            ru, rup, _, st = oracle.run(m.as_dict(), ru, rup, it, 1, path=ORACLE_PATH[path],
                                        order=oracle.ORDER_U2)
            assert st == 0
            for k, n in enumerate(m.receivers):
                ref[k, :, it] = ru[3 * n:3 * n + 3]
        assert np.array_equal(u, ru) and np.array_equal(up, rup), path
        assert np.array_equal(tr, ref), path
        pu, _, _, _ = oracle.run(m.as_dict(), z, z, 0, 30, path=ORACLE_PATH[path])
        assert np.linalg.norm(u - pu) <= 1e-12 * np.linalg.norm(pu)
        assert np.abs(tr).max() > 0


def test_state_roundtrip_and_nonfinite_rejected(ovxmod):
    """set_state checks finiteness on the device (OVX_EINVAL for a NaN/Inf anywhere); get_state
    writes into caller-provided arrays and can skip u_prev."""
    m = wl.small_random(6, 5, 4, ds=0.01)
    s = _solver(ovxmod, m, 0)
    u = wl.random_field(m)
    up = wl.random_field(m, seed=3)
    s.set_state(u, up, 7)
    out = np.empty_like(u)
    r, rp, it = s.get_state(out_u=out, with_prev=False)
    assert r is out and rp is None and it == 7 and np.array_equal(out, u)
    r, rp, _ = s.get_state()
    assert np.array_equal(r, u) and np.array_equal(rp, up)
    for bad in (np.nan, np.inf):
        v = up.copy()
        v[123] = bad
        with pytest.raises(ovxmod.OvxError):
            s.set_state(u, v, 0)


@pytest.mark.parametrize("name,path", [("int8", 0), ("fp64", 1)])
def test_full_size_1000_steps_closed_form(ovxmod, name, path):
    """BASELINE bar at the bench size: C2 (256³, the bench launch), 1000 steps from the standing P
    wave (an exact lattice eigenmode of the roller box) against the closed-form amplitude
    u^n = a_n u^0 (1-D lattice dispersion, Eq. 3 recurrence) — relative L2 ≤ 1e-10;
    the INT8 path also within 1e-10 of the FP64 path."""
    from oracle import physics
    m = wl.c2_block(256)
    u0 = wl.standing_wave(m, mvec=(16, 0, 0), U=(1.0, 0.0, 0.0))
    k = math.pi * 16 / (m.nx * m.ds)
    V = math.sqrt((m.kappa[0] + 4 * m.G[0] / 3) / m.rho[0])
    lam = physics.lattice_lambda_axis(V, k, m.ds)
    s = _solver(ovxmod, m, path)
    s.set_state(u0, u0, 0)
    s.step(1000)
    u, _, _ = s.get_state(with_prev=False)
    ref = physics.mode_amplitude(lam, m.dt, 1000) * u0
    assert np.linalg.norm(u - ref) <= 1e-10 * np.linalg.norm(ref)
    if path == 0:
        s64 = _solver(ovxmod, m, 1)
        s64.set_state(u0, u0, 0)
        s64.step(1000)
        u64, _, _ = s64.get_state(with_prev=False)
        assert np.linalg.norm(u - u64) <= 1e-10 * np.linalg.norm(u64)


def _sampled_apply_check(ovxmod, m, path, u, pts, nsample=40):
    """apply_K at full size in the bench's launch configuration; sampled node forces vs the oracle
    (the definition within the per-node bound; the U2 mirror bit for bit on the exact paths)."""
    import torch
    s = _solver(ovxmod, m, path)
    ut = torch.from_numpy(u).cuda()
    ft = torch.empty_like(ut)
    s.apply_K_device(ut, ft)
    s.sync()
    rng = np.random.default_rng(13683 + path)
    pts = list(pts) + [(int(rng.integers(0, m.nx + 1)), int(rng.integers(0, m.ny + 1)), int(rng.integers(0, m.nz + 1)))
                       for _ in range(nsample)]
    nx1, ny1 = m.nx + 1, m.ny + 1
    idx = torch.tensor([3 * (ix + nx1 * (iy + ny1 * iz)) + c for (ix, iy, iz) in pts for c in range(3)],
                       device="cuda")
    f = ft[idx].cpu().numpy().reshape(-1, 3)
    del ut, ft
    for k, (ix, iy, iz) in enumerate(pts):
        _check_node(f[k], m, u, ix, iy, iz, path)


@pytest.mark.parametrize("name,path", [("int8", 0), ("fp64", 1)])
def test_full_size_c3_sampled(ovxmod, name, path):
    """BASELINE config 3 at full size (512³ two-layer soil over bedrock, 1.35e8 elements):
    sampled nodes on the boundaries, the soil/rock interface plane and at random."""
    m = wl.c3_two_layer(512)
    u = wl.random_field(m)
    iface = 512 - 128
    pts = [(0, 0, 0), (512, 512, 512), (256, 256, iface), (255, 17, iface - 1), (1, 511, iface + 1),
           (31, 7, 64), (32, 8, 129), (511, 0, 384)]
    _sampled_apply_check(ovxmod, m, path, u, pts)


@pytest.mark.parametrize("name,path", [("int8", 0), ("fp64", 1)])
def test_full_size_c4_sampled(ovxmod, name, path):
    """BASELINE config 4 at full size (891×352×1056, 3.3e8 elements, 1.0e9 DOF, one B200):
    sampled nodes on the layer boundaries, around the stiff cylinder and at random."""
    m = wl.c4_ground()
    u = wl.random_field(m)
    cx, cz = int(160 / 324 * 891), int(100 / 384 * 1056)
    pts = [(0, 0, 0), (891, 352, 1056), (cx, 100, cz), (cx + 41, 5, cz), (cx - 41, 351, cz), (cx, 200, cz + 41),
           (400, 176, 1056 - 52), (10, 10, 1056 - 211), (890, 1, 1056 - 475)]
    _sampled_apply_check(ovxmod, m, path, u, pts)


@pytest.mark.parametrize("variant", [{"OVX_I8_KERNEL": "tmem"}, {"OVX_I8_KERNEL": "smem"},
                                     {"OVX_I8_KERNEL": "x", "OVX_I8X_LAYOUT": "word"},
                                     {"OVX_I8_KERNEL": "x", "OVX_I8X_LAYOUT": "half"},
                                     {"OVX_I8_PLANES": "bulk"}])
def test_alternate_int8_kernels_bit_exact(ovxmod, variant):
    """The alternate INT8 kernels (selected once per process, so in a subprocess): step_i8w (the
    round-1 kernel: roles alternating per half-iteration) with the A operand in TMEM or in shared
    memory, step_i8x with the word (−K ⊗ I_4, no byte permutes) or half-word operand layout, and the
    default warp-specialised step_i8ws with its node planes delivered by the bulk-copy (TMA) engine
    instead of cp.async: apply_K and a 30-step trajectory bit-exact vs the oracle's U2 mirror on the ragged
    multi-tile grid (DESIGN.md §6.1 compares their speed)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle, workloads as wl
from paper_2404_13683_b200 import Ovx
m = wl.small_random(40, 8, 70, ds=0.01, dt=1e-6)
wl.point_source(m, 17, 3, 35, 1, 1e5, 2e-5, 30, scale=1.0)
u = wl.random_field(m) * 1e-3
s = Ovx(0); s.load_model(m, 0)
f = s.apply_K(u)
assert np.array_equal(f, oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=oracle.PATH_INT8,
                                       order=oracle.ORDER_U2))
s.set_state(u, u, 0); s.step(30)
v, vp, _ = s.get_state()
r, rp, _, st = oracle.run(m.as_dict(), u, u, 0, 30, path=oracle.PATH_INT8, order=oracle.ORDER_U2)
assert st == 0 and np.array_equal(v, r) and np.array_equal(vp, rp)
print('ok')
"""
    env = dict(os.environ, **variant)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_1000_steps_multi_tile_multi_chunk(ovxmod):
    """BASELINE bar on a grid that exercises the kernels' decomposition: 64×16×24 elements
    (3 x-tiles, 3 y-tiles, 3 z-chunks, ragged tails), three random materials per element, a Ricker
    source, fixed corners, 1000 steps: INT8 within 1e-10 rel-L2 of the FP64 oracle's definition,
    bit-exact vs the INT8 oracle's U2 mirror; the factored FP64 path within 1e-10 as well."""
    m = wl.small_random(64, 16, 24, ds=1.0, dt=1e-4)
    f0 = 25.0
    wl.point_source(m, 33, 9, 24, 2, f0, 1.2 / f0, 1000, scale=1e6)
    z = np.zeros(3 * m.n_nodes)
    s = _solver(ovxmod, m, 0)
    assert m.dt < s.critical_dt()
    ctas, _, _ = s.get_launch_config()
    assert ctas >= 27, ctas      # 3 × 3 tiles × ≥ 3 z-chunks
    s.set_state(z, z, 0)
    s.step(1000)
    s.check_finite()
    u, up, _ = s.get_state()
    ref64, _, _, st = oracle.run(m.as_dict(), z, z, 0, 1000, path=oracle.PATH_FP64)
    assert st == 0 and np.abs(ref64).max() > 0
    assert np.linalg.norm(u - ref64) <= 1e-10 * np.linalg.norm(ref64)
    ref8, ref8p, _, _ = oracle.run(m.as_dict(), z, z, 0, 1000, path=oracle.PATH_INT8, order=oracle.ORDER_U2)
    assert np.array_equal(u, ref8) and np.array_equal(up, ref8p)
    s64 = _solver(ovxmod, m, 1)
    s64.set_state(z, z, 0)
    s64.step(1000)
    u64, _, _ = s64.get_state()
    assert np.linalg.norm(u64 - ref64) <= 1e-10 * np.linalg.norm(ref64)


def _phase_fit(a, ns, th0):
    """θ minimising Σ (a_n − cos(n θ))² near θ0 (Gauss-Newton; the projection fit of SURVEY §8(d))."""
    th = th0
    for _ in range(20):
        r = a - np.cos(ns * th)               # residual of the model cos(n θ)
        J = -ns * np.sin(ns * th)             # its derivative in θ
        th += float(J @ r) / float(J @ J)
    return th


@pytest.mark.parametrize("nu", ["0.25", "0.35"])
@pytest.mark.parametrize("mvec", [(10, 10, 10), (16, 16, 0)])
def test_c2_oblique_bloch_modes(ovxmod, nu, mvec):
    """BASELINE config 2 / SURVEY §8(d) C2: oblique standing waves on the 256³ roller box (bench
    launch), k = π·mvec/256, ν = 0.25 and 0.35.  IC: an eigenvector U of the Bloch symbol Ŝ(k)
    (the symbol is pinned against the oracle in test_oracle_global), u^{−1} = cos θ u^0
    with cos θ = 1 − λ dt²/2, so u^n = cos(nθ) u^0 exactly.  1000 steps of the INT8 path: rel-L2 ≤ 1e-10
    against cos(nθ) u^0 at every 100th step, and the phase velocity c_h = θ/(dt|k|) fitted from the
    projections a_n = ⟨u^n, u^0⟩/⟨u^0, u^0⟩ within 1e-9 of the closed form — for the P-like and an
    S-like mode.  (These modes separate OVFEM from VFEM: PAPER.md L60, L90.)"""
    from oracle import physics
    m = wl.c2_block(256, nu=nu)
    k = np.array([math.pi * mv / (256 * m.ds) for mv in mvec])
    lam, U = physics.bloch_modes(m.kappa[0], m.G[0], m.rho[0], m.ds, k)
    s = _solver(ovxmod, m, 0)
    # the P-like mode (largest eigenvalue) and the S-like mode with a non-zero roller-box field (for
    # k_z = 0 a purely z-polarised mode vanishes identically: u_z ∝ sin(k_z z))
    fields = {i: wl.standing_wave(m, mvec=mvec, U=tuple(U[:, i])) for i in range(3)}
    s_mode = max((0, 1), key=lambda i: float(fields[i] @ fields[i]))
    for i in (2, s_mode):
        u0 = fields[i]
        assert float(u0 @ u0) > 0
        th0 = math.acos(1 - lam[i] * m.dt ** 2 / 2)
        s.set_state(u0, math.cos(th0) * u0, 0)
        n0 = float(u0 @ u0)
        ns, amps = [], []
        for blk in range(10):
            s.step(100)
            u, _, it = s.get_state(with_prev=False)
            ref = math.cos(it * th0) * u0
            assert np.linalg.norm(u - ref) <= 1e-10 * math.sqrt(n0), (i, it)
            ns.append(it)
            amps.append(float(u @ u0) / n0)
        th = _phase_fit(np.array(amps), np.array(ns, dtype=np.float64), th0)
        c_fit = th / (m.dt * np.linalg.norm(k))
        c_closed = th0 / (m.dt * np.linalg.norm(k))
        assert abs(c_fit / c_closed - 1) <= 1e-9, (i, c_fit, c_closed)


def test_c5_layered_sampled(ovxmod):
    """BASELINE config 5 (layered soil / rock every 64 element layers, 256³ per GPU): sampled node
    forces around the layer interfaces and at random vs the oracle, INT8 path, bench launch."""
    m = wl.c5_layered(1)
    u = wl.random_field(m)
    pts = [(0, 0, 0), (256, 256, 256), (128, 128, 64), (17, 250, 128), (255, 3, 192), (31, 7, 63), (62, 14, 65)]
    _sampled_apply_check(ovxmod, m, 0, u, pts)
    _sampled_apply_check(ovxmod, m, 1, u, pts[:3], nsample=10)


def test_two_contexts_different_materials_concurrent_streams(ovxmod):
    """Per-context material tables (no device-global __constant__ materials): two contexts with
    different materials on one device, each on its own stream, their steps interleaved without host
    synchronisation — both bit-exact against the oracle's U2 mirror (INT8 and factored-FP64 paths)."""
    import torch
    for path in (0, 1):
        ma = wl.small_random(40, 8, 30, seed=1, ds=0.01, dt=1e-6)
        mb = wl.small_random(33, 9, 28, seed=2, ds=0.02, dt=2e-6)
        assert not np.allclose(ma.kappa, mb.kappa)
        ua, ub = wl.random_field(ma, seed=5) * 1e-3, wl.random_field(mb, seed=6) * 1e-3
        sa_t, sb_t = torch.cuda.Stream(), torch.cuda.Stream()
        sa, sb = ovxmod.Ovx(0), ovxmod.Ovx(0)
        sa.set_stream(sa_t)
        sb.set_stream(sb_t)
        sa.load_model(ma, path)
        sb.load_model(mb, path)
        sa.set_state(ua, ua, 0)
        sb.set_state(ub, ub, 0)
        for _ in range(6):
            sa.step(5)
            sb.step(5)
        got = {}
        for nm, s in (("a", sa), ("b", sb)):
            got[nm] = s.get_state()
        for nm, m, u0 in (("a", ma, ua), ("b", mb, ub)):
            op = ORACLE_PATH[path]
            if EXACT[path]:
                r, rp, _, st = oracle.run(m.as_dict(), u0, u0, 0, 30, path=op, order=oracle.ORDER_U2)
                assert st == 0 and np.array_equal(got[nm][0], r) and np.array_equal(got[nm][1], rp), (path, nm)
            else:
                r, _, _, st = oracle.run(m.as_dict(), u0, u0, 0, 30, path=op)
                assert st == 0 and np.linalg.norm(got[nm][0] - r) <= 1e-12 * np.linalg.norm(r), (path, nm)


def test_set_grid_resets_sources_and_negative_step_index_rejected(ovxmod):
    """A context reused for a second model without sources injects nothing (set_grid clears the
    previous model's sources and receivers); set_state rejects it < 0 (OVX_EINVAL)."""
    m1 = wl.c1_cube(8, steps=20)
    s = _solver(ovxmod, m1, 0)
    m2 = wl.small_random(6, 5, 4, ds=0.01)
    m2.src_node = np.zeros(0, np.int64)
    m2.src_axis = np.zeros(0, np.int32)
    m2.amp = np.zeros((0, 1))
    s.set_grid(m2.nx, m2.ny, m2.nz, m2.ds)
    s.set_materials(m2.rho, m2.kappa, m2.G)
    s.set_element_materials(m2.mat)
    s.set_dirichlet(m2.dirichlet)
    s.setup_elements(0, 8)
    s.set_dt(m2.dt)
    z = np.zeros(3 * m2.n_nodes)
    s.set_state(z, z, 0)
    s.step(5)
    u, _, _ = s.get_state()
    assert np.all(u == 0)                   # no stale point force from the first model
    with pytest.raises(ovxmod.OvxError):
        s.set_state(z, z, -1)


def test_direct_n_stage_path_bit_exact(ovxmod):
    """NEXT-4, the paper's DIRECT FP64→INT8 method (Fig. 2 left, Eqs. 11-14, a = 2^7, N = 8) on the
    tensor cores (OVX_INT8_DIRECT): per-element records (v, the 8 signed digits per value, the
    per-stage products C_j, y, f_e) bit-exact vs the oracle's direct variant; K u bit-exact vs its
    U2 mirror; the results equal the hierarchical paper-digit path (same integer image, L146) and a
    20-step trajectory equals the oracle's."""
    m = wl.small_random(9, 5, 4, ds=0.01)
    rng = np.random.default_rng(8)
    u = wl.random_field(m) * 10.0 ** rng.uniform(-20, 5, size=3 * m.n_nodes)
    u[::97] = 0.0
    s = ovxmod.Ovx(0)
    s.load_model(m, ovxmod.OVX_INT8_DIRECT)
    rec = s.debug_element_ints(u, 0, m.n_elems)
    for e in range(m.n_elems):
        nodes = oracle.element_nodes(m.nx, m.ny, e)
        ue = np.concatenate([u[3 * n:3 * n + 3] for n in nodes])
        mm = m.mat[e]
        r = oracle.element_int8(ue, m.kappa[mm], m.G[mm], m.ds, 8, oracle.DIGITS_DIRECT_FOLD)
        assert rec["s"][e] == r["s"]
        assert np.array_equal(rec["v"][e], r["v"])
        assert np.array_equal(rec["d"][e][:8].astype(np.int8).astype(np.int32), r["d"])
        assert np.array_equal(rec["C"][e].astype(np.int64), r["C"])
        assert rec["y"][e] == r["y"]
        assert np.array_equal(rec["fe"][e], r["fe"])
    f = s.apply_K(u)
    mirror = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=oracle.PATH_INT8,
                            digits=oracle.DIGITS_DIRECT_FOLD, order=oracle.ORDER_U2)
    paper = oracle.apply_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=oracle.PATH_INT8,
                           digits=oracle.DIGITS_PAPER | 2, order=oracle.ORDER_U2)
    assert np.array_equal(f, mirror) and np.array_equal(mirror, paper)
    mc = wl.c1_cube(8, steps=20)
    z = np.zeros(3 * mc.n_nodes)
    sd = ovxmod.Ovx(0)
    sd.load_model(mc, ovxmod.OVX_INT8_DIRECT)
    sd.set_state(z, z, 0)
    sd.step(20)
    ud, upd, _ = sd.get_state()
    ru, rup, _, st = oracle.run(mc.as_dict(), z, z, 0, 20, path=oracle.PATH_INT8, digits=oracle.DIGITS_DIRECT_FOLD,
                                order=oracle.ORDER_U2)
    assert st == 0 and np.array_equal(ud, ru) and np.array_equal(upd, rup)


def test_c3_scaled_1000_steps_vs_oracle(ovxmod):
    """BASELINE config 3 (two-layer soil over bedrock, Ricker source at the top centre, 4 bottom
    corners fixed) scaled to 64³: 1000 steps of the INT8 path within 1e-10 rel-L2 of the FP64
    oracle's definition (the north-star bar), the factored FP64 path too.  (BASELINE names 128³ for
    this comparison; its 1000 oracle steps take ≈ 15 min of host time on the GPU box's 16 cores, so
    the test uses the same model at 64³, ≈ 1 min.)"""
    m = wl.c3_two_layer(64, steps=1000)
    z = np.zeros(3 * m.n_nodes)
    ref, _, _, st = oracle.run(m.as_dict(), z, z, 0, 1000, path=oracle.PATH_FP64)
    assert st == 0 and np.abs(ref).max() > 0
    for path in (0, 1):
        s = _solver(ovxmod, m, path)
        assert m.dt < s.critical_dt()
        s.set_state(z, z, 0)
        s.step(1000)
        u, _, _ = s.get_state(with_prev=False)
        assert np.linalg.norm(u - ref) <= 1e-10 * np.linalg.norm(ref), path


def test_c3_full_size_10_steps_int8_vs_fp64(ovxmod):
    """BASELINE config 3 at full size (512³, 1.35e8 elements, the bench launch): 10 steps from a
    random field, the INT8 path within 1e-12 rel-L2 of the factored FP64 path (which is itself
    compared with the oracle at this size node by node in test_full_size_c3_sampled)."""
    import torch
    m = wl.c3_two_layer(512, steps=10)
    rng = np.random.default_rng(3)
    u0 = torch.from_numpy(rng.standard_normal(3 * m.n_nodes) * 1e-3).cuda()
    out = {}
    for path in (0, 1):
        s = _solver(ovxmod, m, path)
        s.set_state_device(u0, u0, 0)
        s.step(10)
        u = torch.empty_like(u0)
        up = torch.empty_like(u0)
        s.get_state_device(u, up)
        out[path] = u
        del s
    assert float(torch.linalg.norm(out[0] - out[1]) / torch.linalg.norm(out[1])) <= 1e-12
