"""CPU emulation of one z-slab's compute (test infrastructure for the gloo protocol tests).

Implements the same begin / iface / end contract as paper_2404_13683_b200.dist.OvxCompute,
with the oracle's element forces and update, so the distributed protocol in dist.py can be
checked bit-for-bit against the monolithic oracle run on CPU (world size 2, 3 over gloo)."""
import numpy as np
import torch

import oracle

CORNER = {(1, 1): 2, (0, 1): 3, (1, 0): 1, (0, 0): 0}   # (node is +x corner, +y corner) -> local node


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

    def _layer0_contribs(self):
        lm, nx, ny = self.lm, self.lm.nx, self.lm.ny
        b = np.zeros((self.nn2, 4, 3))
        for ey in range(ny):
            for ex in range(nx):
                e = ex + nx * ey
                nodes = oracle.element_nodes(nx, ny, e)
                ue = np.concatenate([self.u[3 * q:3 * q + 3] for q in nodes])
                m = lm.mat[e]
                fe = (oracle.element_fp64(ue, lm.kappa[m], lm.G[m], lm.ds) if self.path == oracle.PATH_FP64
                      else oracle.element_int8(ue, lm.kappa[m], lm.G[m], lm.ds)["fe"])
                for dy in (0, 1):
                    for dx in (0, 1):
                        j = (ex + dx) + (nx + 1) * (ey + dy)
                        # order: e(ix-1,iy-1), e(ix,iy-1), e(ix-1,iy), e(ix,iy)  ->  k = 2*(1-dy) + (1-dx)
                        k = 2 * (1 - dy) + (1 - dx)
                        a = CORNER[(dx, dy)]
                        b[j, k, :] = fe[3 * a:3 * a + 3]
        return b

    def begin(self):
        lm, nn2 = self.lm, self.nn2
        f = oracle.apply_K(lm.nx, lm.ny, lm.nz, lm.ds, lm.mat, lm.kappa, lm.G, self.u, path=self.path)
        F = self._forces()
        self.F = F
        if self.slab.flags & 2:
            self.a_send.copy_(torch.from_numpy(f[3 * nn2 * lm.nz:]))
        if self.slab.flags & 1:
            self.b = self._layer0_contribs()
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
        f0 = self.a_recv.numpy().copy()
        b = self.b.reshape(nn2, 4, 3)
        for k in range(4):
            f0 = f0 + b[:, k, :].reshape(-1)
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
