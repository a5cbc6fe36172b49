// step_f64.cuh — fused time step for the factored FP64 path (OVX_FP64); included by kernels.cu.
//
// Same tiling and z-march as step_v1 (32×8 elements per layer, owned nodes 31×7, one halo ring),
// but no per-element force staging in shared memory:
//   * thread (lane = lx, warp = ly) computes element (lx, ly) with the Walsh-Hadamard factored
//     K_e^o u_e (element_force_wht, ≈180 FP64 ops);
//   * contributions are summed along x with one warp shuffle (the +x corners of lane lx-1 meet
//     the -x corners of lane lx), along y through a 6-double-per-thread smem row exchange;
//   * thread (lx, ly) owns node (lx, ly) of the tile (lx, ly >= 1) and keeps its plane-L and
//     plane-(L+1) force accumulators in registers across the z-march; the completed plane is
//     updated in place (Eq. 3 / L263-L266 with the sign of Eq. 3).
// Node sums follow the oracle's order (reading U2); the factored element force differs from the
// dense one in rounding (parity: tolerance).

struct F2 {
    static constexpr int EY = 8;
    static constexpr int NT = EX * EY;                 // 256 threads = elements per layer
    static constexpr int TY = EY - 1;
    static constexpr int PY = EY + 1;
    static constexpr int PLANE = PX * PY * 3;          // 891 doubles
    static constexpr int PF = (PLANE + NT - 1) / NT;   // 4
};

// the material constants of the factored force, staged in shared memory once per CTA (a
// per-lane indexed constant-bank load serialises and misses the constant cache)
struct MatW {
    double L0, M0, M0x2, L1, M1, M1x3, C2, pad;
};

// factored VFEM constants (OVX_VFEM): w_T λ, w_T μ for |T| = 0, 1, 2
struct MatV {
    double vl[3], vm[3], pad[2];
};
union MatU {
    MatW w;
    MatV v;
};

struct SmemF2 {
    double up[5][F2::PLANE];          // ring: L-1 (its update may still run), L, L+1 in use, L+2, L+3 in flight
    double ysum[2][F2::EY][EX][6];    // +y-corner x-sums of each element row (double-buffered)
    MatU mw[kMaxMat];                 // [0, nmat) and the zero material kZeroMat
};

// DAMP (MODE_STEP only): Rayleigh damping, reading R1 — the planes hold ũ = u + cb·(u − u_prev),
// the update reads u and u_prev from global memory and writes u^{it+1} to p.un.
// VF: the factored VFEM element (OVX_VFEM, NEXT-3) instead of the factored OVFEM element.
template <int MODE, bool DAMP, bool VF = false>
__global__ void __launch_bounds__(F2::NT, 2) step_f64(const StepParams p) {
    constexpr int NT = F2::NT, TY = F2::TY, PLANE = F2::PLANE, PF = F2::PF;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SmemF2 &S = *reinterpret_cast<SmemF2 *>(smem_raw);
    const int t = threadIdx.x;
    const int lx = t & 31, ly = t >> 5;

    int bid = blockIdx.x;
    const int tx = bid % p.tiles_x;
    bid /= p.tiles_x;
    const int ty = bid % p.tiles_y;
    const int tz = p.tz0 + bid / p.tiles_y;            // z-chunk (a launch may cover a subrange)
    const int64_t X0 = (int64_t)tx * TX, Y0 = (int64_t)ty * TY;
    const int Z0 = tz * p.zchunk;
    const int Z1 = (int)min((int64_t)Z0 + p.zchunk, p.nz + 1);
    const int nz = (int)p.nz;
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1, PSTRIDE = NX1 * NY1;

    const int64_t ex = X0 - 1 + lx, ey = Y0 - 1 + ly;
    const bool ein = (ex >= 0 && ex < p.nx && ey >= 0 && ey < p.ny);
    const uint8_t *matcol = p.mat + (ein ? ex + p.nx * ey : 0);
    const int64_t mstride = p.nx * p.ny;

    int pfoff[PF];
    bool pfok[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        const int idx = t + j * NT;
        const int py = idx / (PX * 3);
        const int rem = idx - py * (PX * 3);
        const int px = rem / 3, c = rem - px * 3;
        const int64_t ix = X0 - 1 + px, iy = Y0 - 1 + py;
        pfok[j] = idx < PLANE && ix >= 0 && ix < NX1 && iy >= 0 && iy < NY1;
        pfoff[j] = pfok[j] ? 3 * (ix + NX1 * iy) + c : 0;
    }
    // owned node of this thread: tile node (lx, ly) = global (X0-1+lx, Y0-1+ly), lx, ly >= 1
    const int64_t uix = X0 - 1 + lx, uiy = Y0 - 1 + ly;
    const bool own = lx >= 1 && ly >= 1 && uix < NX1 && uiy < NY1;
    const int64_t ucol = own ? uix + NX1 * uiy : 0;

    bool has_src = false;
    if (MODE == MODE_STEP)
        for (int k = 0; k < p.nsrc; ++k) {
            const int64_t n = p.src_dof[k] / 3;
            const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
            has_src |= (ix >= X0 && ix < X0 + TX && iy >= Y0 && iy < Y0 + TY);
        }

    // does any receiver fall on this tile's owned columns?
    bool has_rec = false;
    if (MODE == MODE_STEP && p.it < p.rec_nt)
        for (int k = 0; k < p.nrec; ++k) {
            const int64_t n = p.rec_node[k];
            const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
            has_rec |= (ix >= X0 && ix < X0 + TX && iy >= Y0 && iy < Y0 + TY);
        }

    // u (undamped) or ũ = u + cb·(u − u_prev) (damped) at global offset o
    auto load_in = [&](int64_t o) {
        const double uu = __ldg(p.u + o);
        if constexpr (DAMP) {
            const double pp = __ldg(p.uo + o);    // u_prev is read-only in a damped step
            return __dadd_rn(uu, __dmul_rn(p.cb, __dsub_rn(uu, pp)));
        } else {
            return uu;
        }
    };
    for (int i = t; i < p.nmat + 1; i += NT) {
        const int id = i < p.nmat ? i : kZeroMat;
        const MatConst &m = p.mc[id];
        if (VF) S.mw[id].v = MatV{{m.vl[0], m.vl[1], m.vl[2]}, {m.vm[0], m.vm[1], m.vm[2]}, {0.0, 0.0}};
        else S.mw[id].w = MatW{m.L0, m.M0, m.M0x2, m.L1, m.M1, m.M1x3, m.C2, 0.0};
    }
    const int Lfirst = max(Z0 - 1, 0);
    // synchronous first three planes (the loop prefetches three planes ahead); the other two ring
    // slots are zeroed for the damped register path
    auto r5 = [](int z) { return (z + 10) % 5; };        // ring slot of plane z >= -10
    for (int idx = t; idx < PLANE; idx += NT) {   // the damped park never writes out-of-domain entries
        S.up[r5(Lfirst + 3)][idx] = 0.0;
        S.up[r5(Lfirst + 4)][idx] = 0.0;
    }
    {   // all loads of the three planes first (one DRAM round trip per CTA), then the stores
        double v0[3][PF];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int iz = Lfirst + j;
#pragma unroll
            for (int k = 0; k < PF; ++k)
                v0[j][k] = (pfok[k] && iz <= nz) ? load_in(3 * PSTRIDE * (int64_t)iz + pfoff[k]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < PF; ++k)
                if (t + k * NT < PLANE) S.up[r5(Lfirst + j)][t + k * NT] = v0[j][k];
    }
    __syncthreads();

    // Plane L+3 is fetched at layer L into the ring slot of plane L-2 (no thread reads it any more:
    // the slowest thread is past this layer's predecessor barrier, after which only planes L-1 .. L+1
    // are read).  Undamped: cp.async straight into shared memory (zero-fill outside the domain),
    // waited for one layer later before the barrier.  Damped (ũ needs arithmetic): registers, parked
    // into the slot one layer later before the barrier.
    double pend[PF];
    int pend_z = -1;
    auto park_prev = [&]() {
        if constexpr (DAMP) {
            if (pend_z >= 0) {
                double *dst = S.up[r5(pend_z)];
#pragma unroll
                for (int j = 0; j < PF; ++j) {
                    const int idx = t + j * NT;
                    if (pfok[j]) dst[idx] = pend[j];
                }
            }
        } else {
            ptx::cp_async_wait<1>();   // the copies issued one layer ago (plane L+2) have landed
        }
    };
    double facc[3] = {0.0, 0.0, 0.0};   // plane L (receives layer L-1 top + layer L bottom)
    // material ids of layers L, L+1, L+2; the one after is fetched three layers ahead
    int mcur = (ein && Lfirst < nz) ? (int)__ldg(matcol + mstride * Lfirst) : kZeroMat;
    int mnxt = (ein && Lfirst + 1 < nz) ? (int)__ldg(matcol + mstride * (Lfirst + 1)) : kZeroMat;
    int mnx2 = (ein && Lfirst + 2 < nz) ? (int)__ldg(matcol + mstride * (Lfirst + 2)) : kZeroMat;
    double nupv[3] = {0.0, 0.0, 0.0}, nwn = 0.0, nuv[3] = {0.0, 0.0, 0.0};
    uint8_t ndm = 0;
    // running offsets (advanced once per layer instead of 64-bit products per use)
    const uint8_t *mfar_p = matcol + mstride * (int64_t)(Z0 + 2);      // material of layer L+3
    int64_t uplane = 3 * PSTRIDE * (int64_t)(Z0 + 2);                  // plane L+3 of u
    int64_t un_id = ucol + PSTRIDE * (int64_t)(Z0 - 1);                // node of plane L
    for (int L = Z0 - 1; L < Z1; ++L, mfar_p += mstride, uplane += 3 * PSTRIDE, un_id += PSTRIDE) {
        const bool layer_ok = (L >= 0 && L < nz);
        const bool plane_done = (L >= Z0 && L <= nz);
        // material of layer L+3 (three layers ahead: the register rotation at the end of the layer
        // waits on a load issued one layer earlier)
        const int mfar = (ein && L >= Lfirst && L + 3 < nz) ? (int)__ldg(mfar_p) : kZeroMat;
        // ---- prefetch plane L+3 (parked next iteration) and the update operands of plane L ----
        const int pz = L + 3;
        const bool pf = (pz > Lfirst + 2) && (L + 2 < Z1) && (L + 2 < nz);
        double pfv[PF];
        if constexpr (DAMP) {
#pragma unroll
            for (int j = 0; j < PF; ++j)
                if (pf && pfok[j]) pfv[j] = load_in(uplane + pfoff[j]);
        } else {
            if (pf) {
                double *dst = S.up[r5(pz)];
#pragma unroll
                for (int j = 0; j < PF; ++j)
                    if (t + j * NT < PLANE) ptx::cp_async8(dst + t + j * NT, p.u + uplane + pfoff[j], pfok[j]);
            }
            ptx::cp_async_commit();
        }
        const bool upd = plane_done && own;
        // update operands of plane L were loaded one layer ahead; fetch those of plane L+1
        double upv[3] = {nupv[0], nupv[1], nupv[2]};
        const double uv[3] = {nuv[0], nuv[1], nuv[2]};
        const double wn = nwn;
        const uint8_t dm = ndm;
        if (MODE == MODE_STEP) {
            const int L1 = L + 1;
            if (own && L1 >= Z0 && L1 < Z1 && L1 <= nz) {
                const int64_t nid = un_id + PSTRIDE;
                nupv[0] = p.uo[3 * nid];
                nupv[1] = p.uo[3 * nid + 1];
                nupv[2] = p.uo[3 * nid + 2];
                if constexpr (DAMP) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) nuv[c] = __ldg(p.u + 3 * nid + c);
                }
                nwn = __ldg(p.w + nid);
                ndm = p.dmask ? __ldg(p.dmask + nid) : (uint8_t)0;
            }
        }

        double nbot[3] = {0.0, 0.0, 0.0}, ntop[3] = {0.0, 0.0, 0.0};
        double(*ys)[EX][6] = S.ysum[L & 1];
        if (layer_ok) {
            double ue[24], fe[24];
            gather<F2::PY>(ue, S.up[r5(L)], S.up[r5(L + 1)], lx, ly);
            if constexpr (VF) element_force_vfem_wht(ue, S.mw[mcur].v, fe);   // zero material outside
            else element_force_wht(ue, S.mw[mcur].w, fe);                    // the domain -> fe = 0
            // x-sums at this element's -x node column: own -x corners + lane lx-1's +x corners
            // local nodes: (-x,-y)=0,4  (+x,-y)=1,5  (+x,+y)=2,6  (-x,+y)=3,7   (bottom, top)
            double xs[12];   // [dy][dz][c]
#pragma unroll
            for (int dz = 0; dz < 2; ++dz)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double pm = __shfl_up_sync(0xffffffffu, fe[3 * (1 + 4 * dz) + c], 1);  // (+x,-y) of lx-1
                    const double pp = __shfl_up_sync(0xffffffffu, fe[3 * (2 + 4 * dz) + c], 1);  // (+x,+y) of lx-1
                    // (lane 0 adds its own value here; it owns no node, so the sum is never used)
                    xs[0 * 6 + dz * 3 + c] = fe[3 * (0 + 4 * dz) + c] + pm;
                    xs[1 * 6 + dz * 3 + c] = fe[3 * (3 + 4 * dz) + c] + pp;
                }
#pragma unroll
            for (int q = 0; q < 6; ++q) ys[ly][lx][q] = xs[6 + q];
            park_prev();
            __syncthreads();   // the only barrier of the layer
            if (ly > 0) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    nbot[c] = xs[c] + ys[ly - 1][lx][c];
                    ntop[c] = xs[3 + c] + ys[ly - 1][lx][3 + c];
                }
            }
        } else {
            park_prev();
            __syncthreads();
        }
        if (L >= Z0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) facc[c] += nbot[c];
        }
        // ---- plane L complete: update ----
        // z-slab interfaces: plane 0 owned here, its partial from below arrives later
        // (keep the bottom-face sum B); the top plane is owned by the rank above (send T + B = T + 0)
        const bool bot_iface = (p.slab_flags & 1) && L == 0;
        const bool top_iface = (p.slab_flags & 2) && L == nz;
        if (upd && bot_iface) {
#pragma unroll
            for (int c = 0; c < 3; ++c) p.iface_bot_b[3 * ucol + c] = nbot[c];
        } else if (upd && top_iface) {
#pragma unroll
            for (int c = 0; c < 3; ++c) p.iface_top_A[3 * ucol + c] = facc[c];
        } else if (upd) {
            const double *up = &S.up[r5(L)][(ly * PX + lx) * 3];
            if (MODE == MODE_STEP) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int64_t dof = 3 * un_id + c;
                    double F = 0.0;
                    if (has_src)
                        for (int k = 0; k < p.nsrc; ++k)
                            if (p.src_dof[k] == dof) F += p.src_val[k];
                    const double uc = DAMP ? uv[c] : up[c];
                    double b = __dsub_rn(__dmul_rn(2.0, uc), upv[c]);
                    if constexpr (DAMP) b = __dsub_rn(b, __dmul_rn(p.ca, __dsub_rn(uc, upv[c])));
                    double un = __fma_rn(wn, __dsub_rn(F, facc[c]), b);
                    if ((dm >> c) & 1) un = 0.0;
                    (DAMP ? p.un : p.uo)[dof] = un;
                    if (has_rec)
                        for (int k = 0; k < p.nrec; ++k)
                            if (p.rec_node[k] == un_id) p.traces[(3 * k + c) * p.rec_nt + p.it] = un;
                }
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) p.fout[3 * un_id + c] = facc[c];
            }
        }
        if (L + 1 < Z1) {
#pragma unroll
            for (int c = 0; c < 3; ++c) facc[c] = ntop[c];
        }
        if (L >= Lfirst) {
            mcur = mnxt;
            mnxt = mnx2;
            mnx2 = mfar;
        }
#pragma unroll
        if constexpr (DAMP) {
#pragma unroll
            for (int j = 0; j < PF; ++j) pend[j] = pfv[j];
            pend_z = pf ? pz : -1;
        }
    }
}
