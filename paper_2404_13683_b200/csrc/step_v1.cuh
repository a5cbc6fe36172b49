// step_v1.cuh — the fused time-step kernel (included by kernels.cu inside ovx::{anon}).
//
// CTA = 32×8 elements per layer (one halo ring recomputed by the neighbour tiles: owned
// nodes 31×7, element-work redundancy 256/217 = 1.18), marching in z over a chunk of node
// planes.  Per layer L:
//   (1) prefetch node plane L+2 of u^{it} and the update operands of plane L (u^{it-1}, w, mask)
//       into registers — their latency hides under (2);
//   (2) element forces of layer L (path-specific) -> smem fe[24][256];
//   (3) scatter into two smem force planes, node sums in the U2 tree order; plane L is then complete
//       and is updated in place (Eq. 3 / L263-L266 with the sign of Eq. 3);
//   (4) park the prefetched plane in the 3-slot smem ring.
// Paths: OVX_FP64_DENSE (the literal dense form, bit-exact mirror of the oracle's FP64
// definition) and OVX_FP64 when z-slab interfaces or debug records are requested.

template <int PATH>
struct V1 {
    static constexpr int EY = 8;
    static constexpr int NE = EX * EY;                 // 256 elements per layer
    static constexpr int NT = NE;                      // threads, one per element
    static constexpr int TY = EY - 1;                  // 7 owned node rows
    static constexpr int PY = EY + 1;                  // 9 node rows per smem plane
    static constexpr int NOWN = TX * TY;               // 217 owned nodes per plane
    static constexpr int PLANE = PX * PY * 3;          // 891 doubles per plane
    static constexpr int PF = (PLANE + NT - 1) / NT;   // prefetched doubles per thread
    static constexpr int MINB = 2;
};

struct SmemV1F64 {
    double up[3][V1<OVX_FP64>::PLANE];
    double fe[24][256];
    double facc[2][V1<OVX_FP64>::NOWN * 3];
};

template <int PATH>
using SmemV1 = SmemV1F64;

// u (undamped) or the damped EBE input ũ = u + cb·(u − u_prev) (reading R1) at global offset o
template <bool DAMP>
__device__ __forceinline__ double v1_load_in(const StepParams &p, int64_t o) {
    const double uu = __ldg(p.u + o);
    if constexpr (DAMP) {
        const double pp = __ldg(p.uo + o);    // u_prev is read-only in a damped step
        return __dadd_rn(uu, __dmul_rn(p.cb, __dsub_rn(uu, pp)));
    } else {
        return uu;
    }
}

template <int PATH, bool DAMP>
__device__ __forceinline__ void v1_load_plane_sync(double *dst, const StepParams &p, int64_t X0, int64_t Y0,
                                                   int64_t iz) {
    using C = V1<PATH>;
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;
    for (int idx = threadIdx.x; idx < C::PLANE; idx += C::NT) {
        const int py = idx / (PX * 3);
        const int rem = idx - py * (PX * 3);
        const int px = rem / 3, c = rem - px * 3;
        const int64_t ix = X0 - 1 + px, iy = Y0 - 1 + py;
        double v = 0.0;
        if (iz <= p.nz && ix >= 0 && ix < NX1 && iy >= 0 && iy < NY1) v = v1_load_in<DAMP>(p, 3 * (ix + NX1 * (iy + NY1 * iz)) + c);
        dst[idx] = v;
    }
}

// DAMP (MODE_STEP only): Rayleigh damping, reading R1 (planes hold ũ; update reads u, u_prev from
// global memory and writes u^{it+1} to p.un).
template <int PATH, int MODE, bool DAMP>
__global__ void __launch_bounds__(V1<PATH>::NT, V1<PATH>::MINB) step_v1(const StepParams p) {
    using C = V1<PATH>;
    constexpr int NT = C::NT, TY = C::TY, NOWN = C::NOWN, PLANE = C::PLANE, PF = C::PF;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SmemV1<PATH> &S = *reinterpret_cast<SmemV1<PATH> *>(smem_raw);
    const int t = threadIdx.x;

    int bid = blockIdx.x;
    const int tx = bid % p.tiles_x;
    bid /= p.tiles_x;
    const int ty = bid % p.tiles_y;
    const int tz = p.tz0 + bid / p.tiles_y;            // z-chunk (a launch may cover a subrange)
    const int64_t X0 = (int64_t)tx * TX, Y0 = (int64_t)ty * TY;
    const int64_t Z0 = (int64_t)tz * p.zchunk;
    const int64_t Z1 = min(Z0 + (int64_t)p.zchunk, p.nz + 1);
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;
    const int64_t PSTRIDE = NX1 * NY1;        // nodes per plane

    const int el = t;                          // element of this thread
    const int lx = el % EX, ly = el / EX;
    const int64_t ex = X0 - 1 + lx, ey = Y0 - 1 + ly;
    const bool ein = (ex >= 0 && ex < p.nx && ey >= 0 && ey < p.ny);
    const uint8_t *matcol = p.mat + (ein ? ex + p.nx * ey : 0);   // + nx*ny*L per layer
    const int64_t mstride = p.nx * p.ny;

    // loop-invariant prefetch sources of this thread (offsets within a plane of u)
    int64_t pfoff[PF];
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
    // update role: owned node (nxl, nyl) of the tile
    const int nxl = t % TX, nyl = t / TX;
    const int64_t uix = X0 + nxl, uiy = Y0 + nyl;
    const bool own = t < NOWN && uix < NX1 && uiy < NY1;
    const int64_t ucol = own ? uix + NX1 * uiy : 0;

    // does any point source fall on this tile's owned columns?
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

    for (int i = t; i < 2 * NOWN * 3; i += NT) (&S.facc[0][0])[i] = 0.0;
    const int64_t Lfirst = max(Z0 - 1, (int64_t)0);
    v1_load_plane_sync<PATH, DAMP>(S.up[Lfirst % 3], p, X0, Y0, Lfirst);
    v1_load_plane_sync<PATH, DAMP>(S.up[(Lfirst + 1) % 3], p, X0, Y0, Lfirst + 1);
    __syncthreads();

    // material of this thread's element in the current layer (prefetched one layer ahead;
    // elements outside the domain use the reserved zero material)
    int mcur = (ein && Lfirst < p.nz) ? (int)__ldg(matcol + mstride * Lfirst) : kZeroMat;
    for (int64_t L = Z0 - 1; L < Z1; ++L) {
        const bool layer_ok = (L >= 0 && L < p.nz);
        const bool plane_done = (L >= Z0 && L <= p.nz);
        const int mnext = (ein && L + 1 > Lfirst && L + 1 < p.nz) ? (int)__ldg(matcol + mstride * (L + 1)) : kZeroMat;
        // ---- (1) prefetch: plane L+2 (needed by layer L+1) and the update operands of plane L ----
        const int64_t pz = L + 2;
        const bool pf = (pz > Lfirst + 1) && (L + 1 < Z1) && (L + 1 < p.nz);
        double pfv[PF];
        const int64_t uplane = 3 * PSTRIDE * pz;
#pragma unroll
        for (int j = 0; j < PF; ++j) pfv[j] = (pf && pfok[j]) ? v1_load_in<DAMP>(p, uplane + pfoff[j]) : 0.0;
        const bool upd = plane_done && own;
        const int64_t un_id = ucol + PSTRIDE * L;
        double upv[3] = {0.0, 0.0, 0.0}, wn = 0.0, uv[3] = {0.0, 0.0, 0.0};
        uint8_t dm = 0;
        if (MODE == MODE_STEP && upd) {
            upv[0] = p.uo[3 * un_id];
            upv[1] = p.uo[3 * un_id + 1];
            upv[2] = p.uo[3 * un_id + 2];
            if constexpr (DAMP) {
#pragma unroll
                for (int c = 0; c < 3; ++c) uv[c] = __ldg(p.u + 3 * un_id + c);
            }
            wn = __ldg(p.w + un_id);
            dm = p.dmask ? __ldg(p.dmask + un_id) : (uint8_t)0;
        }

        // ---- (2) element forces of layer L ----
        if (layer_ok) {
            const double *plo = S.up[L % 3], *phi = S.up[(L + 1) % 3];
            const int m = mcur;
            const int64_t eid = ex + p.nx * (ey + p.ny * L);
            const int64_t dj = eid - p.dbg_e0;
            const bool dbg = (MODE == MODE_DEBUG) && ein && lx < TX && ly < TY && (L + 1 >= Z0) && (L + 1 < Z1) &&
                             dj >= 0 && dj < p.dbg_ne;
            double ue[24];
            gather<C::PY>(ue, plo, phi, lx, ly);
            if constexpr (PATH == OVX_FP64 || PATH == OVX_VFEM) {
                double fe[24];
                if constexpr (PATH == OVX_VFEM) element_force_vfem_wht(ue, p.mc[m], fe);
                else element_force_wht(ue, p.mc[m], fe);   // zero material -> fe = 0 exactly
#pragma unroll
                for (int r = 0; r < 24; ++r) {
                    S.fe[r][el] = fe[r];
                    if (MODE == MODE_DEBUG && dbg && p.dbg_fe) p.dbg_fe[dj * 24 + r] = fe[r];
                }
            } else if constexpr (PATH == OVX_FP64_DENSE) {
                const double ck = p.mc[m].ck, cg = p.mc[m].cg;
#pragma unroll 1
                for (int r = 0; r < 24; ++r) {
                    double a = 0.0, b = 0.0;
#pragma unroll
                    for (int c = 0; c < 24; ++c) {
                        a = __dadd_rn(a, __dmul_rn(c_Kk[p.kset][r * 24 + c], ue[c]));
                        b = __dadd_rn(b, __dmul_rn(c_Kg[p.kset][r * 24 + c], ue[c]));
                    }
                    const double f = __dadd_rn(__dmul_rn(ck, a), __dmul_rn(cg, b));
                    S.fe[r][el] = ein ? f : 0.0;
                    if (MODE == MODE_DEBUG && dbg && p.dbg_fe) p.dbg_fe[dj * 24 + r] = f;
                }
            }
        }
        __syncthreads();

        // ---- (3) scatter (U2 tree order) + update of the completed plane L ----
        if (t < NOWN) {
            auto fe = S.fe;
            const int e00 = nxl + EX * nyl, e10 = e00 + 1, e01 = e00 + EX, e11 = e01 + 1;
            double *fl = &S.facc[L & 1][t * 3];
            double *fh = &S.facc[(L + 1) & 1][t * 3];
            const bool bot_iface = (p.slab_flags & 1) && L == 0;             // plane 0 owned, partial from below
            const bool top_iface = (p.slab_flags & 2) && L == p.nz;          // plane owned by the rank above
            // node force f_n = T_n + B_n, face sums (x-pair row iy) + (x-pair row iy-1) (reading U2)
            if (layer_ok && L >= Z0) {     // bottom face of layer L -> plane L
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double B = __dadd_rn(__dadd_rn(fe[3 * 0 + c][e11], fe[3 * 1 + c][e01]),
                                               __dadd_rn(fe[3 * 3 + c][e10], fe[3 * 2 + c][e00]));
                    if (bot_iface) {       // interface plane: B waits for T from the rank below
                        if (own) p.iface_bot_b[3 * ucol + c] = B;
                    } else {
                        fl[c] = __dadd_rn(fl[c], B);
                    }
                }
            }
            if (layer_ok && L + 1 < Z1) {  // top face of layer L -> plane L+1
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    fh[c] = __dadd_rn(__dadd_rn(fe[3 * 4 + c][e11], fe[3 * 5 + c][e01]),
                                      __dadd_rn(fe[3 * 7 + c][e10], fe[3 * 6 + c][e00]));
            }
            if (upd && top_iface) {
#pragma unroll
                for (int c = 0; c < 3; ++c) p.iface_top_A[3 * ucol + c] = fl[c];
            } else if (upd && !bot_iface) {
                const double *up = &S.up[L % 3][((nyl + 1) * PX + (nxl + 1)) * 3];
                if (MODE == MODE_STEP) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int64_t dof = 3 * un_id + c;
                        double F = 0.0;
                        if (has_src)
                            for (int k = 0; k < p.nsrc; ++k)
                                if (p.src_dof[k] == dof) F = __dadd_rn(F, p.src_val[k]);
                        const double uc = DAMP ? uv[c] : up[c];
                        double b = __dsub_rn(__dmul_rn(2.0, uc), upv[c]);
                        if constexpr (DAMP) b = __dsub_rn(b, __dmul_rn(p.ca, __dsub_rn(uc, upv[c])));
                        double un = __fma_rn(wn, __dsub_rn(F, fl[c]), b);
                        if ((dm >> c) & 1) un = 0.0;
                        (DAMP ? p.un : p.uo)[dof] = un;
                        if (has_rec)
                            for (int k = 0; k < p.nrec; ++k)
                                if (p.rec_node[k] == un_id) p.traces[(3 * k + c) * p.rec_nt + p.it] = un;
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 3; ++c) p.fout[3 * un_id + c] = fl[c];
                }
            }
            if (plane_done) fl[0] = fl[1] = fl[2] = 0.0;
        }
        if (L >= Lfirst) mcur = mnext;
        // ---- (4) park the prefetched plane L+2 (slot of plane L-1, no longer read) ----
        if (pf) {
            double *dst = S.up[pz % 3];
#pragma unroll
            for (int j = 0; j < PF; ++j) {
                const int idx = t + j * NT;
                if (idx < PLANE) dst[idx] = pfv[j];
            }
        }
        __syncthreads();
    }
}
