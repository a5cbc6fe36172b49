"""Repeat the one-GPU z-slab comparison (tests/test_gpu_dist.py) and report where mismatches land."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as wl  # noqa: E402
from paper_2404_13683_b200 import Ovx, dist as D  # noqa: E402


def model():
    m = wl.small_random(40, 9, 21, ds=0.5, dt=1e-5)
    t = np.arange(80) * m.dt
    m.src_node = np.array([m.node(20, 4, 10), m.node(7, 2, 11), m.node(33, 8, 21)], dtype=np.int64)
    m.src_axis = np.array([2, 0, 1], dtype=np.int32)
    m.amp = np.stack([1e3 * wl.ricker(t, 2e4, 5e-5), 5e2 * wl.ricker(t, 3e4, 4e-5), -7e2 * wl.ricker(t, 2.5e4, 6e-5)])
    return m


def main(reps=int(sys.argv[1]) if len(sys.argv) > 1 else 20, world=int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    m = model()
    rng = np.random.default_rng(11)
    u0 = rng.standard_normal(3 * m.n_nodes) * 1e-6
    s = Ovx(0)
    s.load_model(m, 0)
    s.set_state(u0, u0, 0)
    s.step(60)
    mu, _, _ = s.get_state()
    bad = 0
    for r in range(reps):
        g = D.SlabGroup(m, world, lambda lm, sl: D.OvxCompute(lm, sl, 0, 0))
        g.set_state(u0, u0, 0)
        g.step(60)
        torch.cuda.synchronize()
        u, _, _ = g.get_state()
        d = np.nonzero(u != mu)[0]
        if d.size:
            bad += 1
            n = d // 3
            ix, iy, iz = n % (m.nx + 1), (n // (m.nx + 1)) % (m.ny + 1), n // ((m.nx + 1) * (m.ny + 1))
            print(f"rep {r}: {d.size} dofs differ; z planes {sorted(set(iz.tolist()))[:10]} "
                  f"x {sorted(set(ix.tolist()))[:10]} y {sorted(set(iy.tolist()))[:10]}")
        # monolithic repeat as well
        s.set_state(u0, u0, 0)
        s.step(60)
        mu2, _, _ = s.get_state()
        if not np.array_equal(mu2, mu):
            print(f"rep {r}: MONOLITHIC run differs from its first run ({np.count_nonzero(mu2 != mu)} dofs)")
    print(f"world {world}: {bad}/{reps} slab runs differ")


if __name__ == "__main__":
    main()
