// step_i8c.cuh — INT8 tensor-core time step with three threads per element (one per displacement
// component); included by kernels.cu after step_i8w.cuh (shares its A/B layout constants).
//
// Same tiling, z-march, skewed M-tiles, integer arithmetic and summation order (reading U2) as
// step_i8w, bit-identical results, but 768 threads (24 warps/SM) for latency hiding.  The MMA's K
// (values) and N (outputs) orders are permuted by component — value k' = 8c + node (u part) and
// 24 + 8c + node (G part), output r' = 8c + node — with B = −K_e^INT8 ⊗ I₂ permuted to match, so
// the work of component c is contiguous everywhere:
//   * conversion: thread c gathers the 8 corner values of u_c and writes A chunks c (ū_u) and 3+c
//     (ū_G = RN(cG u_c));  s_e is recomputed by each of the three threads from the node maxima;
//   * epilogue: thread c reads 16 contiguous TMEM columns per array (its 8 outputs) and forms both
//     face sums of component c (x-pairs by shuffle, y-pairs through SMEM), so the top-face sum T of
//     layer L-1 stays in a register until the node force f = T + B of plane L is complete;
//   * update: component c of the owned node.
// Warp w: M-tile w/12, component (w/4)%3, TMEM lane quadrant w%4.

struct I8C {
    static constexpr int EY = 8;
    static constexpr int NE = EX * EY;                 // elements per layer
    static constexpr int NT = 3 * NE;                  // threads
    static constexpr int MT = NE / 128;                // M=128 MMA tiles per layer
    static constexpr int TPM = NT / MT;                // threads per M-tile (384)
    static constexpr int TY = EY - 1;
    static constexpr int PY = EY + 1;
    static constexpr int NODES = PX * PY;              // nodes of one u plane held in smem
    static constexpr int PLANE = NODES * 3;
    static constexpr int TMEM_COLS = MT * 256;
};

struct SmemI8C {
    uint8_t A[I8C::MT][4][A1_BYTES];      // [M-tile][half-word array], K-major, component-permuted K
    alignas(128) uint8_t B[6 * B1_PITCH];
    alignas(128) uint8_t BI[2][6 * BI_PITCH];
    double up[5][I8C::PLANE];                       // ring: L-2, L-1 (updates), L, L+1 (gather), L+2
    unsigned long long nmax[5][I8C::NODES];         // max_c |u_c| of each node (bit patterns)
    double ysum[3][2][I8C::EY][EX][3];              // [layer mod 3][face][row][x][component]
    double2 mc[kMaxMat];                            // (cG, c1) per material
    uint64_t mbar[I8C::MT];
    uint32_t tmem;
};

// value index k (0..47, reading Q1 order 3·node + axis, G part + 24) of permuted position k'
__host__ __device__ constexpr int i8c_kval(int kp) {
    return kp < 24 ? 3 * (kp & 7) + (kp >> 3) : 24 + 3 * ((kp - 24) & 7) + ((kp - 24) >> 3);
}

template <int MODE, int M, bool FAST>
__device__ __forceinline__ void i8c_chunks(const StepParams &p, const double (&ue)[8], int cc, double cG,
                                           double r, double R, bool deg, uint8_t *Ab, uint32_t rowoff,
                                           bool dbg, int64_t dj) {
    constexpr int NB = (7 * M + 1 + 7) / 8;
    constexpr int NA = (NB + 1) / 2;
    constexpr double SCALE = (double)(1ull << (7 * M));
    constexpr unsigned long long AOFF = 1ull << (7 * M);
#pragma unroll
    for (int g = 0; g < 2; ++g) {                   // g = 0: u part (chunk cc), 1: G part (chunk 3+cc)
        const int ch = cc + 3 * g;
        long long v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double ub = g ? __dmul_rn(cG, ue[q]) : ue[q];
            if (FAST)
                v[q] = __double2ll_rz(__dmul_rn(ub, R));
            else
                v[q] = deg ? 0ll : __double2ll_rz(__dmul_rn(__dmul_rn(ub, r), SCALE));
        }
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if constexpr (7 * M >= 32) {
                lo[q] = (uint32_t)(unsigned long long)v[q];
                hi[q] = (uint32_t)((unsigned long long)v[q] >> 32) + (uint32_t)(AOFF >> 32);
            } else {
                lo[q] = (uint32_t)(unsigned long long)v[q] + (uint32_t)AOFF;
                hi[q] = 0;
            }
            if (MODE == MODE_DEBUG && dbg) {
                const unsigned long long vp = ((unsigned long long)hi[q] << 32) | lo[q];
                const int k = i8c_kval(ch * 8 + q);
                if (p.dbg_v) p.dbg_v[dj * 48 + k] = v[q];
                if (p.dbg_d)
#pragma unroll
                    for (int j = 0; j < 8; ++j) p.dbg_d[dj * 384 + j * 48 + k] = j < NB ? (uint8_t)(vp >> (8 * j)) : 0;
            }
        }
        const uint32_t off = rowoff + (uint32_t)ch * 128;
#pragma unroll
        for (int pa = 0; pa < NA; ++pa) {
            const uint32_t *src = pa < 2 ? lo : hi;
            const uint32_t sel = (pa & 1) ? 0x7632u : 0x5410u;
            uint4 wv;
            wv.x = __byte_perm(src[0], src[1], sel);
            wv.y = __byte_perm(src[2], src[3], sel);
            wv.z = __byte_perm(src[4], src[5], sel);
            wv.w = __byte_perm(src[6], src[7], sel);
            *reinterpret_cast<uint4 *>(Ab + pa * A1_BYTES + off) = wv;
        }
    }
}

template <int MODE, int M, bool DAMP>
__global__ void __launch_bounds__(I8C::NT, 1) step_i8c(const StepParams p) {
    using C = I8C;
    constexpr int NB = (7 * M + 1 + 7) / 8;
    constexpr int NA = (NB + 1) / 2;
    constexpr double SCALE = (double)(1ull << (7 * M));
    constexpr double ISCALE = 1.0 / SCALE;                         // exact power of two
    constexpr int NT = C::NT, NODES = C::NODES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SmemI8C &S = *reinterpret_cast<SmemI8C *>(smem_raw);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int wu = __shfl_sync(0xffffffffu, warp, 0);   // the warp index as a uniform value
    const int mt = wu / 12, cc = (wu >> 2) % 3, qd = wu & 3;   // warp-uniform roles
    const int row = 32 * qd + lane;                      // MMA row = TMEM lane

    int bid = blockIdx.x;
    const int tx = bid % p.tiles_x;
    bid /= p.tiles_x;
    const int ty = bid % p.tiles_y;
    const int tz = bid / p.tiles_y;
    const int64_t X0 = (int64_t)tx * TX, Y0 = (int64_t)ty * C::TY;
    const int Z0 = tz * p.zchunk;
    const int Z1 = (int)min((int64_t)Z0 + p.zchunk, p.nz + 1);
    const int nz = (int)p.nz;
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;
    const int64_t PSTRIDE = NX1 * NY1;
    const int Lfirst = max(Z0 - 1, 0);
    const int Lend = min(nz, Z1);
    auto layer_ok = [&](int x) { return x >= Lfirst && x < Lend; };

    const int lx = lane, ly = 4 * mt + qd;
    const int64_t ex = X0 - 1 + lx, ey = Y0 - 1 + ly;
    const bool ein = (ex >= 0 && ex < p.nx && ey >= 0 && ey < p.ny);
    const uint8_t *matp = p.mat + (ein ? ex + p.nx * ey : 0);
    const int64_t mstride = p.nx * p.ny;
    const bool tnode = lx >= 1 && ly >= 1;
    const bool own = tnode && ex < NX1 && ey < NY1;
    const int64_t ucol = own ? ex + NX1 * ey : 0;

    auto load_in = [&](int64_t o) {
        const double uu = __ldg(p.u + o);
        if constexpr (DAMP) {
            const double pp = __ldg(p.uo + o);
            return __dadd_rn(uu, __dmul_rn(p.cb, __dsub_rn(uu, pp)));
        } else {
            return uu;
        }
    };
    const int li = t - (NT - NODES);
    const bool lrole = li >= 0;
    const int lpx = lrole ? li % PX : 0, lpy = lrole ? li / PX : 0;
    const bool ldn = lrole && X0 - 1 + lpx >= 0 && X0 - 1 + lpx < NX1 && Y0 - 1 + lpy >= 0 && Y0 - 1 + lpy < NY1;
    const int64_t ldoff = ldn ? 3 * ((X0 - 1 + lpx) + NX1 * (Y0 - 1 + lpy)) : 0;

    bool has_src = false, has_rec = false;
    if (MODE == MODE_STEP) {
        for (int k = 0; k < p.nsrc; ++k) {
            const int64_t n = p.src_dof[k] / 3;
            const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
            has_src |= (ix >= X0 && ix < X0 + TX && iy >= Y0 && iy < Y0 + C::TY);
        }
        if (p.it < p.rec_nt)
            for (int k = 0; k < p.nrec; ++k) {
                const int64_t n = p.rec_node[k];
                const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
                has_rec |= (ix >= X0 && ix < X0 + TX && iy >= Y0 && iy < Y0 + C::TY);
            }
    }

    // ---- one-time setup: B operands (component-permuted), zero K padding, TMEM, mbarriers ----
    for (int idx = t; idx < 48 * 96; idx += NT) {
        const int n = idx / 96, kb = idx - n * 96;
        const int off = (n >> 3) * B1_PITCH + (kb >> 4) * 128 + (n & 7) * 16 + (kb & 15);
        const int rp = n >> 1, r = 3 * (rp & 7) + (rp >> 3);          // output r' = 8c + node
        S.B[off] = ((kb & 1) == (n & 1)) ? (uint8_t)(-(int)c_K8[r * 48 + i8c_kval(kb >> 1)]) : (uint8_t)0;
    }
    for (int idx = t; idx < 2 * 48 * 32; idx += NT) {
        const int s2 = idx / (48 * 32), r2 = idx - s2 * 48 * 32;
        const int n = r2 / 32, kb = r2 - n * 32;
        const int off = (n >> 3) * BI_PITCH + (kb >> 4) * 128 + (n & 7) * 16 + (kb & 15);
        const int k = 16 * s2 + (kb >> 1);          // permuted G index 8c + node <-> output r'
        S.BI[s2][off] = ((kb & 1) == (n & 1) && k == (n >> 1)) ? (uint8_t)0x80 : (uint8_t)0;
    }
    for (int idx = t; idx < C::MT * 4 * 128; idx += NT) {
        const int a = idx >> 7, r = idx & 127;
        *reinterpret_cast<uint4 *>(&S.A[a >> 2][a & 3][(r >> 3) * A1_PITCH + 6 * 128 + (r & 7) * 16]) =
            make_uint4(0, 0, 0, 0);
    }
    if (warp == 0) ptx::tmem_alloc<C::TMEM_COLS>(&S.tmem);
    if (t == 0)
        for (int mm = 0; mm < C::MT; ++mm) ptx::mbar_init(&S.mbar[mm], 1);
    for (int i = t; i < p.nmat + 1; i += NT) {
        const int id = i < p.nmat ? i : kZeroMat;
        S.mc[id] = make_double2(c_mat[id].cG, c_mat[id].c1);
    }
    for (int j = 0; j < 2; ++j) {
        const int iz = Lfirst + j;
        if (lrole) {
            double v3[3] = {0.0, 0.0, 0.0};
            if (ldn && iz <= nz)
#pragma unroll
                for (int c = 0; c < 3; ++c) v3[c] = load_in(3 * PSTRIDE * iz + ldoff + c);
            unsigned long long m = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                S.up[ring5(iz)][3 * li + c] = v3[c];
                const unsigned long long b = abs_bits(v3[c]);
                m = b > m ? b : m;
            }
            S.nmax[ring5(iz)][li] = m;
        }
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();

    uint32_t phase = 0;
    int mcur = (ein && Lfirst < nz) ? (int)__ldg(matp + mstride * Lfirst) : kZeroMat;
    int mnxt = (ein && Lfirst + 1 < nz) ? (int)__ldg(matp + mstride * (Lfirst + 1)) : kZeroMat;
    double upv = 0.0, wn = 0.0, uv = 0.0;        // update operands (component cc) of the post plane
    uint8_t dm = 0;
    double plo_b = 0.0, plo_t = 0.0;             // x-pairs P(iy) of the bottom / top face, last epilogue
    double tprev = 0.0;                          // top-face sum T of the layer below the post plane
    double es = 0.0;
    bool edeg = false, edbg = false;
    int em = kZeroMat;
    int64_t edj = -1;

    // ---- post-phase of layer / plane Lp: f_n = T + B for component cc, update ----
    auto post_phase = [&](int Lp, int s3, int s5) {
        if (!tnode) return;
        double B = 0.0, Tn = 0.0;
        if (layer_ok(Lp)) {
            B = __dadd_rn(plo_b, S.ysum[s3][0][ly - 1][lx][cc]);    // P(iy) + P(iy-1), bottom face
            Tn = __dadd_rn(plo_t, S.ysum[s3][1][ly - 1][lx][cc]);   // top face -> plane Lp+1
        }
        const bool plane_done = (Lp >= Z0 && Lp <= nz && Lp < Z1);
        if (own && plane_done) {
            const bool bot_iface = (p.slab_flags & 1) && Lp == 0;
            const bool top_iface = (p.slab_flags & 2) && Lp == nz;
            const int64_t un_id = ucol + PSTRIDE * Lp;
            const int64_t dof = 3 * un_id + cc;
            if (bot_iface) {
                p.iface_bot_b[3 * ucol + cc] = B;
            } else {
                const double f = __dadd_rn(tprev, B);
                if (top_iface) {
                    p.iface_top_A[3 * ucol + cc] = f;
                } else if (MODE == MODE_STEP) {
                    double F = 0.0;
                    if (has_src)
                        for (int k = 0; k < p.nsrc; ++k)
                            if (p.src_dof[k] == dof) F = __dadd_rn(F, p.src_val[k]);
                    const double uc = DAMP ? uv : S.up[s5][(ly * PX + lx) * 3 + cc];
                    double b = __dsub_rn(__dmul_rn(2.0, uc), upv);
                    if constexpr (DAMP) b = __dsub_rn(b, __dmul_rn(p.ca, __dsub_rn(uc, upv)));
                    double un = __fma_rn(wn, __dsub_rn(F, f), b);
                    if ((dm >> cc) & 1) un = 0.0;
                    (DAMP ? p.un : p.uo)[dof] = un;
                    if (has_rec)
                        for (int k = 0; k < p.nrec; ++k)
                            if (p.rec_node[k] == un_id) p.traces[(3 * k + cc) * p.rec_nt + p.it] = un;
                } else {
                    p.fout[dof] = f;
                }
            }
        }
        tprev = Tn;
    };

    // ---- epilogue of layer Le: the 8 outputs of component cc ----
    auto epilogue = [&](int Le, int s3) {
        ptx::mbar_wait(&S.mbar[mt], phase);
        phase ^= 1;
        ptx::tc_fence_after();
        const double alpha = edeg ? 0.0 : -__dmul_rn(S.mc[em].y, __dmul_rn(es, ISCALE));
        const uint32_t tb = S.tmem + ((uint32_t)(qd * 32) << 16) + mt * 256 + 16 * cc;
        double fc[8];                                // node a of component cc
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {             // 4 outputs per round (8 columns per array)
            uint32_t R0[8], R1[8], R2[8] = {}, R3[8] = {};
            ptx::tmem_ld8(tb + 0 + rr * 8, R0);
            ptx::tmem_ld8(tb + 64 + rr * 8, R1);
            if (NA > 2) ptx::tmem_ld8(tb + 128 + rr * 8, R2);
            if (NA > 3) ptx::tmem_ld8(tb + 192 + rr * 8, R3);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int a = 4 * rr + q;
                const int32_t c0 = (int32_t)R0[2 * q], c1_ = (int32_t)R0[2 * q + 1];
                const int32_t c2_ = (int32_t)R1[2 * q], c3 = (int32_t)R1[2 * q + 1];
                const int32_t c4 = (int32_t)R2[2 * q], c5 = (int32_t)R2[2 * q + 1];
                const int32_t c6 = (int32_t)R3[2 * q], c7 = (int32_t)R3[2 * q + 1];
                const double dlo = limb_exact(c0, c1_, c2_, c3);
                const double dhi = NA > 2 ? limb_exact(c4, c5, c6, c7) : 0.0;
                const double Y = NA > 2 ? __fma_rn(dhi, 0x1p32, dlo) : dlo;    // RN(−y)
                const double f = __dmul_rn(alpha, Y);            // = RN(c1s·RN(y))
                if (MODE == MODE_DEBUG && edbg) {
                    const int i = 3 * a + cc;
                    const int32_t Cj[8] = {c0, c1_, c2_, c3, c4, c5, c6, c7};
                    __int128 y = 0;
#pragma unroll
                    for (int jj = 7; jj >= 0; --jj) y = y * 256 - (__int128)Cj[jj];
                    if (p.dbg_C)
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) p.dbg_C[edj * 192 + jj * 24 + i] = -Cj[jj];
                    if (p.dbg_yhi) p.dbg_yhi[edj * 24 + i] = (long long)(y >> 64);
                    if (p.dbg_ylo) p.dbg_ylo[edj * 24 + i] = (long long)(unsigned long long)y;
                    if (p.dbg_fe) p.dbg_fe[edj * 24 + i] = f;
                }
                fc[a] = f;
            }
        }
        ptx::tc_fence_before();
        // local nodes: (-x,-y) 0/4, (+x,-y) 1/5, (+x,+y) 2/6, (-x,+y) 3/7 (bottom/top)
        const double pbm = __shfl_up_sync(0xffffffffu, fc[1], 1), pbp = __shfl_up_sync(0xffffffffu, fc[2], 1);
        const double ptm = __shfl_up_sync(0xffffffffu, fc[5], 1), ptp = __shfl_up_sync(0xffffffffu, fc[6], 1);
        plo_b = __dadd_rn(fc[0], pbm);
        plo_t = __dadd_rn(fc[4], ptm);
        S.ysum[s3][0][ly][lx][cc] = __dadd_rn(fc[3], pbp);
        S.ysum[s3][1][ly][lx][cc] = __dadd_rn(fc[7], ptp);
    };

    // ---- conversion of layer L (component cc: chunks cc and 3+cc) and the MMA hand-off ----
    auto convert = [&](int L, int sL, int sL1) {
        const int64_t eid = ex + p.nx * (ey + p.ny * (int64_t)L);
        const int64_t dj = eid - p.dbg_e0;
        const bool dbg = (MODE == MODE_DEBUG) && ein && lx < TX && ly < C::TY && (L + 1 >= Z0) && (L + 1 < Z1) &&
                         dj >= 0 && dj < p.dbg_ne;
        const unsigned long long *m0 = S.nmax[sL], *m1 = S.nmax[sL1];
        const int n0 = ly * PX + lx;
        unsigned long long ab = m0[n0];
        ab = max(ab, m0[n0 + 1]);
        ab = max(ab, m0[n0 + PX]);
        ab = max(ab, m0[n0 + PX + 1]);
        ab = max(ab, m1[n0]);
        ab = max(ab, m1[n0 + 1]);
        ab = max(ab, m1[n0 + PX]);
        ab = max(ab, m1[n0 + PX + 1]);
        const double amax = __longlong_as_double((long long)ab);
        const double cG = S.mc[mcur].x;
        const double s = fmax(amax, __dmul_rn(cG, amax));
        const bool deg = !ein || !(s >= 0x1p-1022) || !(s <= 0x1.fffffffffffffp1023);
        const bool vzero = !ein || !(s >= 0x1p-1022);
        const bool fast = (s <= 0x1.fffffffffffffp1023) && (vzero || s >= 0x1p-960);
        // the 8 corner values of component cc (local node order of reading Q1)
        double ue[8];
        {
            const double *lo = S.up[sL], *hi = S.up[sL1];
            const int cx[4] = {0, 1, 1, 0}, cy[4] = {0, 0, 1, 1};
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const double *pl = a < 4 ? lo : hi;
                ue[a] = pl[((ly + cy[a & 3]) * PX + (lx + cx[a & 3])) * 3 + cc];
            }
        }
        uint8_t *Ab = &S.A[mt][0][0];
        const uint32_t rowoff = (uint32_t)((row >> 3) * A1_PITCH + (row & 7) * 16);
        const double r = 1.0 / s;                                  // RN(1/s_e), reading Q7
        const double R = vzero ? 0.0 : __dmul_rn(r, SCALE);
        if (__all_sync(0xffffffffu, fast))
            i8c_chunks<MODE, M, true>(p, ue, cc, cG, r, R, deg, Ab, rowoff, dbg, dj);
        else
            i8c_chunks<MODE, M, false>(p, ue, cc, cG, r, R, deg, Ab, rowoff, dbg, dj);
        if (MODE == MODE_DEBUG && dbg && cc == 0 && p.dbg_s) p.dbg_s[dj] = s;
        es = s;
        edeg = deg;
        em = mcur;
        edbg = dbg;
        edj = dj;
        ptx::fence_proxy_async_smem();
        asm volatile("bar.sync %0, 384;" ::"r"(1 + mt) : "memory");   // the 12 warps of this M-tile
        if (wu % 12 == 0) {     // first warp of the M-tile; one elected lane issues
            const int mtu = wu / 12;
            if (ptx::elect_one()) {
                ptx::tc_fence_after();
                const uint32_t b0 = ptx::smem_u32(&S.B[0]);
                const uint32_t bi0 = ptx::smem_u32(&S.BI[0][0]), bi1 = ptx::smem_u32(&S.BI[1][0]);
                const uint32_t a0 = ptx::smem_u32(&S.A[mtu][0][0]);
#pragma unroll
                for (int pa = 0; pa < NA; ++pa) {
                    const uint32_t abase = a0 + pa * A1_BYTES;
                    const uint32_t d = S.tmem + mtu * 256 + pa * 64;
#pragma unroll
                    for (int ks = 0; ks < 3; ++ks)
                        ptx::mma_i8(d, ptx::smem_desc(abase + ks * 256, 128, A1_PITCH),
                                    ptx::smem_desc(b0 + ks * 256, 128, B1_PITCH), IDESC, ks > 0 ? 1u : 0u);
                    ptx::mma_i8(d, ptx::smem_desc(abase + 3 * 128, 128, A1_PITCH),
                                ptx::smem_desc(bi0, 128, BI_PITCH), IDESC, 1u);
                    ptx::mma_i8(d, ptx::smem_desc(abase + 5 * 128, 128, A1_PITCH),
                                ptx::smem_desc(bi1, 128, BI_PITCH), IDESC, 1u);
                }
                ptx::mma_commit(&S.mbar[mtu]);
            }
            __syncwarp();
        }
    };

    int q5_0 = ring5(Z0 - 3), q5_1 = ring5(Z0 - 2), q5_2 = ring5(Z0 - 1), q5_3 = ring5(Z0), q5_4 = ring5(Z0 + 1);
    int q3_0 = ring3(Z0 - 3), q3_1 = ring3(Z0 - 2), q3_2 = ring3(Z0 - 1);
    int64_t ro_plane = 3 * PSTRIDE * (int64_t)(Z0 + 1);
    const uint8_t *ro_mat = matp + mstride * (int64_t)(Z0 + 1);
    int64_t ro_node = ucol + PSTRIDE * (int64_t)(Z0 - 1 - mt);
    double pfv[3] = {0.0, 0.0, 0.0};
    bool pf = false;
    int mfar = kZeroMat;
    double upv_n = 0.0, wn_n = 0.0, uv_n = 0.0;
    uint8_t dm_n = 0;
    for (int h = 2 * (Z0 - 1); h <= 2 * (Z1 + 1) + 1; ++h) {
        const int L = h >> 1;
        const bool odd = h & 1;
        if (!odd) {
            const int pz = L + 2;
            pf = (pz > Lfirst + 1) && (L + 1 < Z1) && (L + 1 < nz);
            if (pf && ldn) {
#pragma unroll
                for (int c = 0; c < 3; ++c) pfv[c] = load_in(ro_plane + ldoff + c);
            }
            mfar = (ein && L + 2 < nz && L >= Lfirst) ? (int)__ldg(ro_mat) : kZeroMat;
            const int Pn = L - mt;
            if (MODE == MODE_STEP && own && Pn >= Z0 && Pn <= nz && Pn < Z1) {
                const int64_t un_next = ro_node;
                upv_n = p.uo[3 * un_next + cc];
                if constexpr (DAMP) uv_n = __ldg(p.u + 3 * un_next + cc);
                wn_n = __ldg(p.w + un_next);
                dm_n = p.dmask ? __ldg(p.dmask + un_next) : (uint8_t)0;
            }
        }
        if (odd == (mt == 1)) {
            if (layer_ok(L)) convert(L, q5_2, q5_3);
        } else {
            post_phase(L - 1 - mt, mt ? q3_0 : q3_1, mt ? q5_0 : q5_1);
            if (layer_ok(L - mt)) epilogue(L - mt, mt ? q3_1 : q3_2);
        }
        if (odd) {
            if (pf && lrole) {
                unsigned long long m = 0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    S.up[q5_4][3 * li + c] = pfv[c];
                    const unsigned long long b = abs_bits(pfv[c]);
                    m = b > m ? b : m;
                }
                S.nmax[q5_4][li] = m;
            }
            if (L >= Lfirst) {
                mcur = mnxt;
                mnxt = mfar;
            }
            upv = upv_n;
            uv = uv_n;
            wn = wn_n;
            dm = dm_n;
            upv_n = 0.0;
            ro_plane += 3 * PSTRIDE;
            ro_mat += mstride;
            ro_node += PSTRIDE;
            {
                const int t5 = q5_0;
                q5_0 = q5_1; q5_1 = q5_2; q5_2 = q5_3; q5_3 = q5_4; q5_4 = t5;
                const int t3 = q3_0;
                q3_0 = q3_1; q3_1 = q3_2; q3_2 = t3;
            }
            __syncthreads();
        }
    }
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc<C::TMEM_COLS>(S.tmem);
}
