"""Bit-exactness of a variant build (OVX_LIB_PATH) on the ragged multi-tile grid: INT8 apply_K and a
30-step trajectory against the oracle's U2 mirror (the same check as the alternate-kernel GPU test)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
if os.environ.get("OVX_LIB_PATH"):
    from paper_2404_13683_b200 import build as B
    B.LIB = os.environ["OVX_LIB_PATH"]
    B._stale = lambda: False
import numpy as np
import oracle
import workloads as wl
from paper_2404_13683_b200 import Ovx
m = wl.small_random(40, 8, 70, ds=0.01, dt=1e-6)
u = wl.random_field(m)
s = Ovx(0)
s.load_model(m, 0)
f = s.apply_K(u)
plain, mirror, absf = oracle.apply_K_orders(m.nx, m.ny, m.nz, m.ds, m.mat, m.kappa, m.G, u, path=oracle.PATH_INT8, M=8)
ok1 = np.array_equal(f, mirror)
print("apply bit-exact:", ok1, flush=True)
sys.exit(0 if ok1 else 1)
