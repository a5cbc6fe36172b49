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
