"""z-slab CUDA path on one GPU: several slab contexts (world 2, 3, 4) stepped in lock step with an
in-process loopback exchange — the same kernels and interface buffers the NCCL transport uses.
The assembled field must equal the single-context GPU run and the oracle bit for bit."""
import numpy as np
import pytest

import oracle
import workloads as wl

pytestmark = pytest.mark.gpu


def _model():
    m = wl.small_random(40, 9, 21, ds=0.5, dt=1e-5)
    t = np.arange(80) * m.dt
    m.src_node = np.array([m.node(20, 4, 10), m.node(7, 2, 11), m.node(33, 8, 21)], dtype=np.int64)
    m.src_axis = np.array([2, 0, 1], dtype=np.int32)
    m.amp = np.stack([1e3 * wl.ricker(t, 2e4, 5e-5), 5e2 * wl.ricker(t, 3e4, 4e-5), -7e2 * wl.ricker(t, 2.5e4, 6e-5)])
    return m


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("path", [0, 1, 3])
def test_slabs_on_one_gpu_equal_monolithic(world, path, overlap):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_13683_b200 import Ovx, dist as D
    m = _model()
    rng = np.random.default_rng(11)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    nsteps = 60
    g = D.SlabGroup(m, world, lambda lm, s: D.OvxCompute(lm, s, 0, path))
    g.set_state(u0, u0, 0)
    g.step(nsteps, overlap=overlap)
    torch.cuda.synchronize()
    u, up, it = g.get_state()
    s = Ovx(0)
    s.load_model(m, path)
    s.set_state(u0, u0, 0)
    s.step(nsteps)
    mu, mup, _ = s.get_state()
    # same kernel (step_i8w / step_f64) and summation order on slabs and on one context -> bit-identical
    assert np.array_equal(u, mu) and np.array_equal(up, mup)
    if path == 0:
        ru, rup, _, _ = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=oracle.PATH_INT8, order=oracle.ORDER_U2)
        assert np.array_equal(u, ru)
        pu, _, _, _ = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=oracle.PATH_INT8)   # the definition
        assert np.linalg.norm(u - pu) <= 1e-12 * np.linalg.norm(pu)


@pytest.mark.parametrize("path", [0, 1])
def test_overlapped_slabs_with_interior_chunks(path):
    """Slabs tall enough for several z-chunks, so the interior launch really runs while the
    exchange and the interface update proceed on the second stream; equal to the serial schedule
    bit for bit (and, on the INT8 path, to the monolithic run)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_13683_b200 import Ovx, dist as D
    m = wl.small_random(33, 8, 120, ds=0.5, dt=1e-5)
    t = np.arange(40) * m.dt
    m.src_node = np.array([m.node(16, 4, 60), m.node(5, 2, 61)], dtype=np.int64)
    m.src_axis = np.array([2, 0], dtype=np.int32)
    m.amp = np.stack([1e3 * wl.ricker(t, 2e4, 5e-5), 5e2 * wl.ricker(t, 3e4, 4e-5)])
    rng = np.random.default_rng(5)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    res = {}
    for overlap in (False, True):
        g = D.SlabGroup(m, 2, lambda lm, s: D.OvxCompute(lm, s, 0, path))
        g.set_state(u0, u0, 0)
        g.step(40, overlap=overlap)
        torch.cuda.synchronize()
        res[overlap] = g.get_state()
    assert np.array_equal(res[False][0], res[True][0]) and np.array_equal(res[False][1], res[True][1])
    if path == 0:
        s = Ovx(0)
        s.load_model(m, 0)
        s.set_state(u0, u0, 0)
        s.step(40)
        mu, mup, _ = s.get_state()
        assert np.array_equal(res[True][0], mu) and np.array_equal(res[True][1], mup)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("path", [0, 2, 1])
def test_damped_slabs_equal_monolithic(world, path):
    """Rayleigh damping (reading R1) on z-slabs: the interface update applies the same damped
    recurrence and the third state buffer rotates on every rank.  Bit-identical to the single-context
    run on every path (INT8 and dense FP64 also to the oracle)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_13683_b200 import Ovx, dist as D
    m = _model()
    m.alpha, m.beta = 0.02 / m.dt, 0.03 * m.dt
    rng = np.random.default_rng(17)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    up0 = u0 + rng.standard_normal(u0.size) * 1e-9
    nsteps = 40
    g = D.SlabGroup(m, world, lambda lm, s: D.OvxCompute(lm, s, 0, path))
    g.set_state(u0, up0, 0)
    g.step(nsteps)
    torch.cuda.synchronize()
    u, up, it = g.get_state()
    s = Ovx(0)
    s.load_model(m, path)
    s.set_state(u0, up0, 0)
    s.step(nsteps)
    mu, mup, _ = s.get_state()
    assert np.array_equal(u, mu) and np.array_equal(up, mup)
    if path in (0, 2):
        ru, rup, _, st = oracle.run(m.as_dict(), u0, up0, 0, nsteps,
                                    path=oracle.PATH_INT8 if path == 0 else oracle.PATH_FP64, order=oracle.ORDER_U2)
        assert st == 0 and np.array_equal(u, ru) and np.array_equal(up, rup)
    ud, _, _, _ = oracle.run(m.as_dict() | {"alpha": 0.0, "beta": 0.0}, u0, up0, 0, nsteps, path=oracle.PATH_FP64)
    assert np.linalg.norm(u - ud) > 1e-6 * np.linalg.norm(ud)   # the damping acts


def _group_run(m, world, path, u0, up0, nsteps, rec=None):
    """The library-driven distributed schedule (ovx_create_group + ovx_step_group: the kernels,
    streams and events of a NCCL ovx_step with device copies in place of ncclSend/Recv), all
    ranks on device 0; returns the assembled owned planes (u, u_prev) and the summed traces."""
    from paper_2404_13683_b200 import ovx as O
    ranks = O.Ovx.create_group(world, [0] * world)
    nn2 = (m.nx + 1) * (m.ny + 1)
    ne2 = m.nx * m.ny
    for r, s in enumerate(ranks):
        ez0, ez1 = O.get_partition(m.nz, world, r)
        s.set_grid(m.nx, m.ny, m.nz, m.ds)                 # global counts
        assert (s.ez0, s.nz) == (ez0, ez1 - ez0)
        s.set_materials(m.rho, m.kappa, m.G)
        s.set_element_materials(m.mat[max(ez0 - 1, 0) * ne2: ez1 * ne2])   # halo layer first (r > 0)
        s.set_dirichlet(None if m.dirichlet is None else m.dirichlet[ez0 * nn2:(ez1 + 1) * nn2])
        s.setup_elements(path, 8)
        s.set_dt(m.dt)
        if getattr(m, "alpha", 0.0) or getattr(m, "beta", 0.0):
            s.set_damping(m.alpha, m.beta)
        s.set_sources(m.src_node, m.src_axis, m.amp)        # global node ids
        if rec is not None:
            s.set_receivers(rec, nsteps)
        s.set_state(u0[3 * nn2 * ez0: 3 * nn2 * (ez1 + 1)], up0[3 * nn2 * ez0: 3 * nn2 * (ez1 + 1)], 0)
    O.step_group(ranks, nsteps)
    us, ups, tr = [], [], None
    for r, s in enumerate(ranks):
        u, up, it = s.get_state()
        assert it == nsteps
        ez0, ez1 = O.get_partition(m.nz, world, r)
        own = (ez1 - ez0) if r < world - 1 else (ez1 - ez0 + 1)   # interface planes belong to the rank above
        us.append(u[:3 * nn2 * own])
        ups.append(up[:3 * nn2 * own])
        if rec is not None:
            t = s.get_traces()
            tr = t if tr is None else tr + t
        ebe, halo, upd = s.get_phase_timers()
        assert ebe > 0 and upd == 0.0 and (halo > 0 or world == 1)
    for s in ranks:
        s.close()
    return np.concatenate(us), np.concatenate(ups), tr


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("path", [0, 1])
def test_library_distributed_schedule_equals_one_gpu(world, path):
    """SURVEY §8(b) distributed boundary: the multi-GPU step runs inside the library (edge chunks
    on a high-priority stream, interior chunks concurrently, exchange, interface update), global
    ids for sources and receivers; the assembled result equals one context bit for bit."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_13683_b200 import Ovx
    m = wl.small_random(33, 8, 90, ds=0.5, dt=1e-5)        # tall enough for interior z-chunks per slab
    t = np.arange(60) * m.dt
    m.src_node = np.array([m.node(20, 4, 45), m.node(7, 2, 90), m.node(3, 3, 30)], dtype=np.int64)
    m.src_axis = np.array([2, 0, 1], dtype=np.int32)
    m.amp = np.stack([1e3 * wl.ricker(t, 2e4, 5e-5), 5e2 * wl.ricker(t, 3e4, 4e-5), -7e2 * wl.ricker(t, 2.5e4, 6e-5)])
    rec = np.array([m.node(20, 4, 44), m.node(5, 5, 90), m.node(1, 1, 31)], dtype=np.int64)
    rng = np.random.default_rng(23)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    nsteps = 30
    u, up, tr = _group_run(m, world, path, u0, u0, nsteps, rec)
    s = Ovx(0)
    s.load_model(m, path)
    s.set_receivers(rec, nsteps)
    s.set_state(u0, u0, 0)
    s.step(nsteps)
    mu, mup, _ = s.get_state()
    assert np.array_equal(u, mu) and np.array_equal(up, mup)
    assert np.array_equal(tr, s.get_traces())
    if path == 0:
        ru, _, _, st = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=oracle.PATH_INT8, order=oracle.ORDER_U2)
        assert st == 0 and np.array_equal(u, ru)


def test_library_distributed_damped():
    """The library schedule with Rayleigh damping (three rotating state buffers on every rank)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_13683_b200 import Ovx
    m = _model()
    m.alpha, m.beta = 0.02 / m.dt, 0.03 * m.dt
    rng = np.random.default_rng(17)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    up0 = u0 + rng.standard_normal(u0.size) * 1e-9
    u, up, _ = _group_run(m, 3, 0, u0, up0, 25)
    s = Ovx(0)
    s.load_model(m, 0)
    s.set_state(u0, up0, 0)
    s.step(25)
    mu, mup, _ = s.get_state()
    assert np.array_equal(u, mu) and np.array_equal(up, mup)


def test_power_iteration_critical_dt():
    """ovx_critical_dt's power iteration on M⁻¹K (the device EBE product): below the element bound
    (the element bound is conservative) and, on a free cube, within 1e-4 of the dense eigenvalue."""
    import math
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from oracle import assemble
    from paper_2404_13683_b200 import Ovx
    m = wl.small_random(4, 3, 3, ds=1.0, dt=1e-4)
    m.dirichlet = None
    s = Ovx(0)
    s.load_model(m, 1)
    de, dp = s.critical_dt(power_iter=True)
    K = assemble.assemble_K(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G)
    md = assemble.assemble_M_diag(m.nx, m.ny, m.nz, m.ds, m.mat, m.rho)
    lam = np.linalg.eigvalsh(K / np.sqrt(np.outer(md, md))).max()
    assert abs(dp / (2 / math.sqrt(lam)) - 1) < 1e-4
    assert dp > de


def test_nccl_communicator_of_one():
    """The library's NCCL plumbing on one GPU: libnccl.so.2 loads (dlopen, the copy torch uses if
    already loaded), ovx_nccl_unique_id and ovx_create_dist (ncclCommInitRank) succeed for a world of
    one, and the context then runs like a plain one (NCCL refuses two ranks on one device, so the
    multi-rank exchange itself is covered by the loopback-group tests and the driver's multi-GPU runs)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_13683_b200 import ovx as O
    uid = O.nccl_unique_id()
    assert len(uid) == 128
    s = O.Ovx.create_dist(0, 0, 1, uid)
    m = wl.c1_cube(8, steps=10)
    s.load_model(m, 0)
    z = np.zeros(3 * m.n_nodes)
    s.set_state(z, z, 0)
    s.step(10)
    u, _, _ = s.get_state()
    r = O.Ovx(0)
    r.load_model(m, 0)
    r.set_state(z, z, 0)
    r.step(10)
    assert np.array_equal(u, r.get_state()[0])
    s.close()
