"""z-slab protocol (paper_2404_13683_b200/dist.py) on CPU: partitioning, slicing, and the
interface exchange over a real torch.distributed gloo process group (world sizes 2 and 3),
with the oracle as the per-slab compute.  The assembled field must equal the monolithic
oracle run bit for bit (the owner-computes interface forms f = T + B, the order of reading U2)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import workloads as wl
from paper_2404_13683_b200 import dist as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_partition_is_balanced_and_covering():
    for nz in (1, 7, 64, 1056):
        for world in (1, 2, 3, 4, 8):
            if world > nz:
                continue
            parts = [D.partition(nz, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == nz
            assert all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def _model():
    m = wl.small_random(5, 4, 9, ds=0.5, dt=1e-5)
    m.dirichlet = wl.corner_mask(m.nx, m.ny, m.nz)
    # sources on an interface plane (global plane 3 / 4 / 6 are interfaces for world 2, 3) and inside
    t = np.arange(60) * m.dt
    m.src_node = np.array([m.node(2, 2, 3), m.node(1, 3, 5), m.node(3, 1, 6)], dtype=np.int64)
    m.src_axis = np.array([2, 0, 1], dtype=np.int32)
    m.amp = np.stack([1e3 * wl.ricker(t, 2e4, 5e-5), 5e2 * wl.ricker(t, 3e4, 4e-5), -7e2 * wl.ricker(t, 2.5e4, 6e-5)])
    return m


def test_local_model_slices():
    m = _model()
    for world in (2, 3):
        tot_src = 0
        for r in range(world):
            s = D.Slab(r, world, *D.partition(m.nz, world, r))
            lm = D.local_model(m, s)
            assert lm.mat.size == m.nx * m.ny * s.nzl
            assert (lm.mat_below is None) == (r == 0)
            tot_src += len(lm.src_node)
        assert tot_src == len(m.src_node)      # every source owned by exactly one rank


def _worker(rank, world, port, path, nsteps, out, staged=False):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from slab_emulation import OracleSlabCompute
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    m = _model()
    rng = np.random.default_rng(5)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    tr = D.HostStagedTransport() if staged else D.TorchTransport()
    run = D.SlabRun(m, rank, world, lambda lm, s: OracleSlabCompute(lm, s, path), tr)
    run.set_state(u0, u0, 0)
    run.step(nsteps)
    g = D.gather_state(run)
    if rank == 0:
        np.save(out, np.stack([g[0], g[1]]))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("path", [oracle.PATH_FP64, oracle.PATH_INT8])
def test_gloo_slabs_equal_monolithic_run(tmp_path, world, path):
    nsteps = 40
    out = str(tmp_path / "u.npy")
    mp.spawn(_worker, args=(world, _free_port(), path, nsteps, out), nprocs=world, join=True)
    got = np.load(out)
    m = _model()
    rng = np.random.default_rng(5)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    ru, rup, _, st = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=path, order=oracle.ORDER_U2)
    assert st == 0
    assert np.array_equal(got[0], ru) and np.array_equal(got[1], rup)
    pu, _, _, _ = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=path)   # the definition's order
    assert np.linalg.norm(got[0] - pu) <= 1e-12 * np.linalg.norm(pu)


def test_host_staged_transport_equals_monolithic(tmp_path):
    """The bench's one-GPU test hook (dist.HostStagedTransport: messages staged through host
    memory over gloo) carries the same protocol: world 2, INT8 emulation, bit-exact."""
    nsteps = 20
    out = str(tmp_path / "u.npy")
    mp.spawn(_worker, args=(2, _free_port(), oracle.PATH_INT8, nsteps, out, True), nprocs=2, join=True)
    got = np.load(out)
    m = _model()
    rng = np.random.default_rng(5)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    ru, rup, _, st = oracle.run(m.as_dict(), u0, u0, 0, nsteps, path=oracle.PATH_INT8, order=oracle.ORDER_U2)
    assert st == 0
    assert np.array_equal(got[0], ru) and np.array_equal(got[1], rup)
