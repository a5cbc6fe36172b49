"""CPU emulation of one z-slab's compute (test infrastructure for the gloo protocol tests).

Implements the same begin / iface / end contract as paper_2404_13683_b200.dist.OvxCompute,
with the oracle's element forces and update, so the distributed protocol in dist.py can be
checked bit-for-bit against the monolithic oracle run in the same summation order (the mirror
variant ORDER_U2) on CPU, and within round-off of the plain element-order definition (world size 2, 3 over gloo)."""
import numpy as np
import torch

import oracle


class OracleSlabCompute:
    def __init__(self, lm, slab, path=oracle.PATH_FP64):
        self.lm, self.slab, self.path = lm, slab, path
        nx, ny, nz = lm.nx, lm.ny, lm.nz
        self.nn2 = (nx + 1) * (ny + 1)
        if lm.mat_below is not None:   # nodal mass of plane 0 includes the layer below
            w = oracle.node_w(nx, ny, nz + 1, lm.ds, np.concatenate([lm.mat_below, lm.mat]), lm.rho, lm.dt)
            self.w = w[self.nn2:]
        else:
            self.w = oracle.node_w(nx, ny, nz, lm.ds, lm.mat, lm.rho, lm.dt)
        self.w3 = np.repeat(self.w, 3)
        n = 3 * self.nn2
        self.a_send, self.a_recv = torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)
        self.u_send, self.u_recv = torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)

    def set_state(self, u, up, it):
        self.u, self.up, self.it = np.array(u, dtype=np.float64), np.array(up, dtype=np.float64), it

    def get_state(self):
        return self.u.copy(), self.up.copy(), self.it

    def _forces(self):
        lm = self.lm
        F = np.zeros_like(self.u)
        for k in range(len(lm.src_node)):
            F[3 * lm.src_node[k] + lm.src_axis[k]] += lm.amp[k, self.it] if self.it < lm.amp.shape[1] else 0.0
        return F

    def begin(self):
        lm, nn2 = self.lm, self.nn2
        # the z-slab protocol reproduces the kernels' per-node tree f = T + B (mirror order U2)
        f = oracle.apply_K(lm.nx, lm.ny, lm.nz, lm.ds, lm.mat, lm.kappa, lm.G, self.u, path=self.path,
                           order=oracle.ORDER_U2)
        F = self._forces()
        self.F = F
        if self.slab.flags & 2:
            self.a_send.copy_(torch.from_numpy(f[3 * nn2 * lm.nz:]))
        if self.slab.flags & 1:   # B: the bottom-face tree sum of layer 0 (no layer below locally)
            self.b = f[:3 * nn2].copy()
        lo = 3 * nn2 if self.slab.flags & 1 else 0
        hi = 3 * nn2 * lm.nz if self.slab.flags & 2 else len(self.u)
        seg = slice(lo, hi)
        up = np.ascontiguousarray(self.up[seg])
        oracle.update_dofs(self.w3[seg], F[seg], f[seg], self.u[seg], up)
        self.up[seg] = up
        self._mask(seg)

    def _mask(self, seg):
        if self.lm.dirichlet is None:
            return
        m = np.repeat(self.lm.dirichlet, 3)
        bit = np.tile(np.array([1, 2, 4], dtype=np.uint8), len(self.lm.dirichlet))
        z = (m & bit) != 0
        idx = np.arange(len(self.up))[seg]
        self.up[idx[z[seg]]] = 0.0

    def iface(self):
        if not self.slab.flags & 1:
            return
        nn2 = self.nn2
        f0 = self.a_recv.numpy() + self.b          # f_n = T_n + B_n (reading U2)
        seg = slice(0, 3 * nn2)
        up = np.ascontiguousarray(self.up[seg])
        oracle.update_dofs(self.w3[seg], self.F[seg], f0, self.u[seg], up)
        self.up[seg] = up
        self._mask(seg)
        self.u_send.copy_(torch.from_numpy(self.up[seg].copy()))

    def end(self):
        if self.slab.flags & 2:
            self.up[3 * self.nn2 * self.lm.nz:] = self.u_recv.numpy()
        self.u, self.up = self.up, self.u
        self.it += 1
