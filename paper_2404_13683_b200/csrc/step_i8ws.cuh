// step_i8ws.cuh — warp-specialised INT8 time step (OVX_INT8, the default kernel); included by
// kernels.cu after step_i8w.cuh (whose B-operand image, TMEM layout and limb it shares).
//
// Same arithmetic, tile, TMEM layout and node-sum order as step_i8w (bit-identical results), with
// every warp in ONE role for the whole kernel instead of alternating roles each half-iteration:
//   warps 0-3  converters of M-tile 0 (element rows 0-3; one thread per element: s_e, the 48 scaled
//              F2I conversions, byte packing, the A operand to TMEM) and loaders of the node planes
//              (cp.async, with warps 4-7), warp 0 issues the M-tile's MMAs;
//   warps 4-7  converters of M-tile 1 (rows 4-7), warp 4 issues;
//   warps 8-11 / 12-15  epilogues of M-tiles 0 / 1 (one thread per element: all 24 outputs from
//              TMEM, exact limbs, the face sums in the order of reading U2, the update of the
//              element's (−x,−y) node).
// Hand-offs are mbarriers (plane ready, MMAs complete — one commit per M-tile and layer, waited for
// once by the other M-tile's converters before their first store into the shared A operand and by
// the epilogues —, D free, the row-3 → row-4 face-sum exchange across M-tiles) and one named barrier
// per role group; the element scale α travels with the A operand through TMEM (spare columns
// 496-503: per M-tile, by layer parity), so it is ordered like D.  The converters run up to two
// layers ahead of the epilogues.  The two M-tiles share the TMEM A operand (their MMAs alternate), as
// in step_i8w.  Time steps (DAMP: Rayleigh damping), products, M = 4 / 6 / 8 stages; the debug
// records and the direct N-stage path use step_i8w.  DESIGN.md §6 / §6.1 has the measurements.

#ifdef OVX_TRACE   // per-warp clock64 stamps of one CTA (tools/trace_ws.py): layers TRK0 .. TRK0+TRH-1
#define TRK0 20
#define TRW(pt) do { if (blockIdx.x == OVX_TRACE && lane == 0 && k >= TRK0 && k < TRK0 + TRH) \
                         g_tr[((k - TRK0) * 16 + wu) * TRN + (pt)] = clock64(); } while (0)
#define TRI(pt) do { if (blockIdx.x == OVX_TRACE && k >= TRK0 && k < TRK0 + TRH) \
                         g_tr[((k - TRK0) * 16 + wu) * TRN + (pt)] = clock64(); } while (0)
#else
#define TRW(pt) do { } while (0)
#define TRI(pt) do { } while (0)
#endif

namespace ws {
constexpr int NP = 8;                          // plane ring (the converters load 3-4 planes ahead; a power of two)
constexpr int NYS = 4;                         // face-sum exchange ring (layers)
}  // namespace ws

// node plane held in shared memory: component-major (cp.async loads, the default) or, with BULK
// (OVX_I8_PLANES=bulk), the global node-major rows as the bulk-copy engine delivers them: row r of the
// tile at byte 816·r + 8·s_r (s_r = the row's 16-byte phase in global memory, which alternates with the
// plane parity when (nx+1)(ny+1) is odd), node x at +24·x, component c at +8·c
template <bool BULK>
struct PlaneT {
    double up[3][I8W::NODES];                  // node values, component-major
    unsigned long long nmax[I8W::NODES];       // max_c |u_c| per node (bit patterns)
    uint8_t mid[I8W::NE];                      // material id of each tile element (layer of this plane)
};
template <>
struct PlaneT<true> {
    alignas(16) double raw[I8W::PY][102];      // 9 rows × 816 B
    unsigned long long nmax[I8W::NODES];
    uint8_t mid[I8W::NE];
};
using PlaneWS = PlaneT<false>;
template <bool BULK = false>
struct SmemWST {
    alignas(128) uint8_t B[6 * B1_PITCH];
    alignas(128) uint8_t BI[2][6 * BI_PITCH];
    PlaneT<BULK> pl[ws::NP];
    double ys[ws::NYS][2][3][I8W::EY][I8W::EX];   // [layer slot][face b/t][c][row][lx]: x-pair P' of the +y corners
    double2 mc[kMaxMat];
    uint64_t plane_full[ws::NP];               // the 256 converter threads arrive
    uint64_t mma_done[2];                      // tcgen05.commit after the M-tile's 20 MMAs of a layer
    uint64_t d_free[2];                        // the 128 epilogue threads of the M-tile arrive
    uint64_t ys_ready[ws::NYS];                // the 32 threads of warp 11 (row 3) arrive
    uint64_t plane_tx[ws::NP];                 // BULK: the 9 row copies of the plane landed (9 arrivals + bytes)
    double upst[2][3][I8W::NODES];             // DAMP: u_prev of the planes in flight (by plane parity)
    uint32_t tmem;
};
using SmemWS = SmemWST<false>;

// DAMP (MODE_STEP, cp.async planes): Rayleigh damping, reading R1 — the planes hold the EBE input
// ũ = u + cb·(u − u_prev) (u_prev staged next to the plane and folded in when the plane completes),
// the update reads u and u_prev of its node from global memory and writes u^{it+1} to p.un.
// M (NEXT-4): INT8 stages, a = 2^{7M}; the byte slices of v + 2^{7M} fill NA = 2 (M = 4), 3 (M = 6) or
// 4 (M = 8) half-word arrays (fewer MMAs and limbs for fewer stages).
template <int MODE, bool SLAB, bool BULK = false, bool DAMP = false, int M = 8>
__global__ void __launch_bounds__(512, 1) step_i8ws(const StepParams p) {
    constexpr int NA = ((7 * M + 1 + 7) / 8 + 1) / 2;
    static_assert(!DAMP || (MODE == MODE_STEP && !BULK), "damped: time steps with cp.async planes");
    using C = I8W;
    constexpr int EX = C::EX, PX = C::PX, PY = C::PY, NODES = C::NODES, NE = C::NE;
    constexpr double ISCALE = 1.0 / (double)(1ull << (7 * M));   // exact powers of two
    constexpr double SCALE = (double)(1ull << (7 * M));
    constexpr unsigned long long AOFF = 1ull << (7 * M);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SmemWST<BULK> &S = *reinterpret_cast<SmemWST<BULK> *>(smem_raw);
    using Plane = PlaneT<BULK>;
    const int t = threadIdx.x, lane = t & 31;
    const int wu = __shfl_sync(0xffffffffu, t >> 5, 0);
    const bool is_conv = wu < 8;
    const int m = (wu >> 2) & 1;                 // M-tile
    const int q = wu & 3;                        // TMEM lane quadrant = element row within the M-tile
    const int lx = lane, ly = 4 * m + q;
    const int elem = lx + EX * ly;

    int bid = blockIdx.x;
    const int tx = bid % p.tiles_x;
    bid /= p.tiles_x;
    const int ty = bid % p.tiles_y;
    const int tz = p.tz0 + bid / p.tiles_y;
    const int64_t X0 = (int64_t)tx * C::TX, Y0 = (int64_t)ty * C::TY;
    const int Z0 = tz * p.zchunk;
    const int nz = (int)p.nz;
    const int Z1 = min(Z0 + p.zchunk, nz + 1);
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;
    const int64_t PSTRIDE = NX1 * NY1;
    const int Lfirst = max(Z0 - 1, 0);
    const int Lend = min(nz, Z1);                // element layers [Lfirst, Lend) are computed
    const int Plast = min(Z1 - 1, nz);           // node planes completed by this CTA: [Z0, Plast]
    const int64_t ex = X0 - 1 + lx, ey = Y0 - 1 + ly;
    const bool ein = (ex >= 0 && ex < p.nx && ey >= 0 && ey < p.ny);
    const int64_t mstride = p.nx * p.ny;
    const bool tnode = lx >= 1 && ly >= 1;
    const bool own = tnode && ex < NX1 && ey < NY1;
    const int64_t ucol = own ? ex + NX1 * ey : 0;
    auto slot = [](int z) { return z & (ws::NP - 1); };   // z >= 0
    // BULK: the row phase s = parity of the global node index of the row's x = -1 node in plane z
    const int gx0 = (int)(X0 - 1);
    auto rowpar = [&](int r) { return (int)((gx0 + NX1 * (Y0 - 1 + r)) & 1); };
    const int pspar = (int)(PSTRIDE & 1);
    auto rowp = [&](const Plane &P, int r, int par_r, int z) -> const double * {   // node 0 of row r of plane z
        if constexpr (BULK)
            return reinterpret_cast<const double *>(reinterpret_cast<const char *>(P.raw) + 816 * r +
                                                    8 * ((par_r ^ (pspar & z)) & 1));
        else
            return nullptr;
    };

    // ---- one-time setup ----
    for (int i = t; i < kBImgVec; i += 512) reinterpret_cast<uint4 *>(S.B)[i] = g_bimg[i];
    if (wu == 0) ptx::tmem_alloc<512>(&S.tmem);
    if (t == 0) {
        for (int i = 0; i < ws::NP; ++i) {
            ptx::mbar_init(&S.plane_full[i], 256);
            ptx::mbar_init(&S.plane_tx[i], PY);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&S.mma_done[i], 1);
            ptx::mbar_init(&S.d_free[i], 128);
        }
        for (int i = 0; i < ws::NYS; ++i) ptx::mbar_init(&S.ys_ready[i], 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = t; i < p.nmat + 1; i += 512) {
        const int id = i < p.nmat ? i : kZeroMat;
        S.mc[id] = make_double2(p.mc[id].cG, p.mc[id].c1);
    }
    // planes Lfirst .. Lfirst+2 and their materials, synchronously (every thread helps)
    for (int j = 0; j < 3; ++j) {
        const int iz = Lfirst + j;
        Plane &P = S.pl[slot(iz)];
        for (int li = t; li < NODES; li += 512) {
            const int lpx = li % PX, lpy = li / PX;
            const int64_t gx = X0 - 1 + lpx, gy = Y0 - 1 + lpy;
            const bool ok = gx >= 0 && gx < NX1 && gy >= 0 && gy < NY1 && iz <= nz;
            unsigned long long mx = 0;
            for (int c = 0; c < 3; ++c) {
                double v = ok ? __ldg(p.u + 3 * (PSTRIDE * iz + gx + NX1 * gy) + c) : 0.0;
                if constexpr (DAMP) {   // ũ = u + cb·(u − u_prev), reading R1
                    const double pp = ok ? __ldg(p.uo + 3 * (PSTRIDE * iz + gx + NX1 * gy) + c) : 0.0;
                    v = __dadd_rn(v, __dmul_rn(p.cb, __dsub_rn(v, pp)));
                }
                if constexpr (BULK)
                    const_cast<double *>(rowp(P, lpy, rowpar(lpy), iz))[3 * lpx + c] = v;
                else
                    P.up[c][li] = v;
                const unsigned long long b = abs_bits(v);
                mx = b > mx ? b : mx;
            }
            P.nmax[li] = mx;
        }
        if (t < NE) {
            const int elx = t % EX, ely = t / EX;
            const int64_t gex = X0 - 1 + elx, gey = Y0 - 1 + ely;
            const bool ok = gex >= 0 && gex < p.nx && gey >= 0 && gey < p.ny && iz < nz;
            P.mid[t] = (uint8_t)(ok ? (int)__ldg(p.mat + gex + p.nx * (gey + p.ny * (int64_t)iz)) : kZeroMat);
        }
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (wu < 4) {   // K-padding chunk 6 of the TMEM A arrays: 255 bytes (bias source), written once
#pragma unroll
        for (int pa = 0; pa < 4; ++pa)
            ptx::tmem_st4(S.tmem + ((uint32_t)(q * 32) << 16) + TA_A0 + pa * TA_A_ARR + 24, ~0u, ~0u, ~0u, ~0u);
        ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = S.tmem;

    if (is_conv) {
        // ================================ converters ================================
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + TA_A0;
        const int n0 = ly * PX + lx;
        const int rp_ly = rowpar(ly), rp_ly1 = rowpar(ly + 1);
        const int ld = t;                            // loader index 0..255
        // loader duties (converters; they run ahead of the epilogues): nodes ld, ld+256 of the 297 and
        // element ld of each plane; plane z+3 is completed and z+4 issued after layer z's MMAs
        const int nl = ld < NODES - 256 ? 2 : 1;
        int64_t goff[2];
        bool gok[2];
        for (int j = 0; j < 2; ++j) {
            const int li = ld + 256 * j;
            const int lpx = li % PX, lpy = li / PX;
            const int64_t gx = X0 - 1 + lpx, gy = Y0 - 1 + lpy;
            gok[j] = j < nl && gx >= 0 && gx < NX1 && gy >= 0 && gy < NY1;
            goff[j] = gok[j] ? 3 * (gx + NX1 * gy) : 0;
        }
        const int elx = ld % EX, ely = ld / EX;
        const int64_t gex = X0 - 1 + elx, gey = Y0 - 1 + ely;
        const bool mok = gex >= 0 && gex < p.nx && gey >= 0 && gey < p.ny;
        const uint8_t *mptr = p.mat + (mok ? gex + p.nx * gey : 0);
        const uint8_t *mrow = mptr + mstride * (int64_t)(Lfirst + 3);   // element ld in layer z+1 (running)
        int mid_next = (mok && Lfirst + 3 < nz) ? (int)__ldg(mrow) : kZeroMat;
        // BULK: node coordinates of this thread's nodes and the tile's valid node columns [lox, hix)
        int lpx_[2], lpy_[2], par_[2];
        for (int j = 0; j < 2; ++j) {
            const int li = ld + 256 * j;
            lpy_[j] = li / PX;
            lpx_[j] = li - lpy_[j] * PX;
            par_[j] = rowpar(lpy_[j]);
        }
        const int lox = gx0 < 0 ? -gx0 : 0;
        const int hix = (int)min((int64_t)PX, NX1 - gx0);
        // issue the loads of plane z into its slot (zero-filled outside the grid or beyond nz)
        int64_t zoff = PSTRIDE * 3 * (int64_t)(Lfirst + 3);   // 3·PSTRIDE·z of the next plane to issue
        auto issue_plane = [&](int z) {
            Plane &P = S.pl[slot(z)];
            if constexpr (BULK) {
                // warp 1, lanes 0..8: one node row each — an 8-byte head and tail by plain loads where
                // the row's first / last valid node is not 16-byte aligned, the rest by one bulk copy
                if (wu == 1 && lane < PY) {
                    const int r = lane;
                    const int64_t gy = Y0 - 1 + r;
                    uint32_t bytes = 0;
                    char *dst = nullptr;
                    const char *src = nullptr;
                    if (gy >= 0 && gy < NY1 && z <= nz && hix > lox) {
                        const int64_t nfirst = PSTRIDE * (int64_t)z + NX1 * gy + gx0 + lox;
                        src = reinterpret_cast<const char *>(p.u + 3 * nfirst);
                        dst = const_cast<char *>(reinterpret_cast<const char *>(rowp(P, r, rowpar(r), z) + 3 * lox));
                        const uint32_t len = 24u * (uint32_t)(hix - lox);
                        const uint32_t head = (reinterpret_cast<uintptr_t>(src) & 15) ? 8u : 0u;
                        bytes = (len - head) & ~15u;
                        const uint32_t tail = len - head - bytes;
                        if (head) *reinterpret_cast<double *>(dst) = __ldg(reinterpret_cast<const double *>(src));
                        if (tail)
                            *reinterpret_cast<double *>(dst + head + bytes) =
                                __ldg(reinterpret_cast<const double *>(src + head + bytes));
                        src += head;
                        dst += head;
                    }
                    ptx::fence_proxy_async_smem();   // the slot's earlier generic reads before the async writes
                    ptx::mbar_arrive_expect_tx(&S.plane_tx[slot(z)], bytes);
                    if (bytes) ptx::bulk_g2s(dst, src, bytes, &S.plane_tx[slot(z)]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (j >= nl) break;
                    const int li = ld + 256 * j;
                    const bool ok = gok[j] && z <= nz;
                    const double *src = p.u + (ok ? zoff + goff[j] : 0);
#pragma unroll
                    for (int c = 0; c < 3; ++c) ptx::cp_async8(&P.up[c][li], src + c, ok);
                    if constexpr (DAMP) {
                        const double *srp = p.uo + (ok ? zoff + goff[j] : 0);
#pragma unroll
                        for (int c = 0; c < 3; ++c) ptx::cp_async8(&S.upst[z & 1][c][li], srp + c, ok);
                    }
                }
                ptx::cp_async_commit();
            }
            zoff += 3 * PSTRIDE;
        };
        // finish plane z (its cp.async group is the oldest outstanding one): node maxima, materials of
        // layer z, arrival on the plane's mbarrier
        auto finish_plane = [&](int z) {
            Plane &P = S.pl[slot(z)];
            if constexpr (BULK) {
                ptx::mbar_wait(&S.plane_tx[slot(z)], (uint32_t)(((z - (Lfirst + 3)) / ws::NP) & 1));
                for (int j = 0; j < nl; ++j) {
                    const int li = ld + 256 * j;
                    double *q = const_cast<double *>(rowp(P, lpy_[j], par_[j], z)) + 3 * lpx_[j];
                    unsigned long long mx = 0;
                    if (gok[j] && z <= nz) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const unsigned long long b = abs_bits(q[c]);
                            mx = b > mx ? b : mx;
                        }
                    } else {   // outside the grid: the copies left this node's slot untouched
                        q[0] = q[1] = q[2] = 0.0;
                    }
                    P.nmax[li] = mx;
                }
            } else {
                ptx::cp_async_wait<0>();
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (j >= nl) break;
                    const int li = ld + 256 * j;
                    unsigned long long mx = 0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double v = P.up[c][li];
                        if constexpr (DAMP) {   // ũ = u + cb·(u − u_prev), reading R1
                            v = __dadd_rn(v, __dmul_rn(p.cb, __dsub_rn(v, S.upst[z & 1][c][li])));
                            P.up[c][li] = v;
                        }
                        const unsigned long long b = abs_bits(v);
                        mx = b > mx ? b : mx;
                    }
                    P.nmax[li] = mx;
                }
            }
            P.mid[ld] = (uint8_t)mid_next;                           // layer z, loaded one iteration ago
            mrow += mstride;
            mid_next = (mok && z + 1 < nz) ? (int)__ldg(mrow) : kZeroMat;
            ptx::mbar_arrive(&S.plane_full[slot(z)]);
        };
        if (Lfirst + 3 <= Lend) issue_plane(Lfirst + 3);
        for (int L = Lfirst; L < Lend; ++L) {
            const int k = L - Lfirst;
            TRW(0);
            const int sL = slot(L), sL1 = slot(L + 1);
            if (L + 1 >= Lfirst + 3)   // plane L+1 arrived asynchronously (its k-th use of the slot)
                ptx::mbar_wait(&S.plane_full[sL1], (uint32_t)(((L + 1 - (Lfirst + 3)) / ws::NP) & 1));
            TRW(1);
            const Plane &P0 = S.pl[sL], &P1 = S.pl[sL1];
            const unsigned long long *m0 = P0.nmax, *m1 = P1.nmax;
            auto dv = [](unsigned long long b) { return __longlong_as_double((long long)b); };
            // max of the magnitude bit patterns (monotone for non-negative doubles; a NaN sorts above +inf
            // and makes the element degenerate, as in step_i8w)
            auto umax = [](unsigned long long x, unsigned long long y) { return x > y ? x : y; };
            const double amax = dv(umax(umax(umax(m0[n0], m0[n0 + 1]), umax(m0[n0 + PX], m0[n0 + PX + 1])),
                                        umax(umax(m1[n0], m1[n0 + 1]), umax(m1[n0 + PX], m1[n0 + PX + 1]))));
            const int mcur = P0.mid[elem];
            const double2 mcv = S.mc[mcur];
            const double cG = mcv.x;
            const double s = fmax(amax, __dmul_rn(cG, amax));   // max_i |RN(cG u_i)| = RN(cG max_i |u_i|)
            const bool deg = !ein || !(s >= 0x1p-1022) || !(s <= 0x1.fffffffffffffp1023);
            const bool vzero = !ein || !(s >= 0x1p-1022);
            const bool fast = (s <= 0x1.fffffffffffffp1023) && (vzero || s >= 0x1p-960);
            const double alpha = deg ? 0.0 : -__dmul_rn(mcv.y, __dmul_rn(s, ISCALE));   // −RN(c1·RN(s·2^-7M))
            const double r = 1.0 / s;                                  // RN(1/s_e), reading Q7
            const double R = vzero ? 0.0 : __dmul_rn(r, SCALE);
            TRW(11);
            // the element's 24 node values (local node order of reading Q1; nodes 4-7 in plane L+1)
            double ue[24];
            {
                constexpr int off[4] = {0, 1, PX + 1, PX};
                if constexpr (BULK) {
                    const double *r00 = rowp(P0, ly, rp_ly, L) + 3 * lx, *r01 = rowp(P0, ly + 1, rp_ly1, L) + 3 * lx;
                    const double *r10 = rowp(P1, ly, rp_ly, L + 1) + 3 * lx, *r11 = rowp(P1, ly + 1, rp_ly1, L + 1) + 3 * lx;
                    const double *rb[8] = {r00, r00 + 3, r01 + 3, r01, r10, r10 + 3, r11 + 3, r11};
#pragma unroll
                    for (int a = 0; a < 8; ++a)
#pragma unroll
                        for (int c = 0; c < 3; ++c) ue[3 * a + c] = rb[a][c];
                } else {
#pragma unroll
                    for (int a = 0; a < 8; ++a)
#pragma unroll
                        for (int c = 0; c < 3; ++c) ue[3 * a + c] = (a < 4 ? P0 : P1).up[c][n0 + off[a & 3]];
                }
            }
            // the other M-tile's MMAs must have read the shared A operand (m 0: layer L-1 of tile 1;
            // m 1: layer L of tile 0)
            const bool need_free = (m == 1) || (k > 0);
            const uint32_t fpar = (uint32_t)((m == 1 ? k : k - 1) & 1);
            auto chunks = [&](auto fastc) {
                constexpr bool FAST = decltype(fastc)::value;
#pragma unroll
                for (int ch = 0; ch < 6; ++ch) {            // chunk ch: values 8ch .. 8ch+7 (3-5: the G half)
                    const bool gpart = ch >= 3;
                    const int j0 = 8 * (gpart ? ch - 3 : ch);
                    uint32_t lo[8], hi[8];
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq) {
                        const double ub = gpart ? __dmul_rn(cG, ue[j0 + qq]) : ue[j0 + qq];
                        long long v;
                        if constexpr (FAST) v = __double2ll_rz(__dmul_rn(ub, R));
                        else v = deg ? 0ll : __double2ll_rz(__dmul_rn(__dmul_rn(ub, r), SCALE));
                        if constexpr (7 * M >= 32) {   // v + 2^{7M}: the offset only touches the high word
                            lo[qq] = (uint32_t)(unsigned long long)v;
                            hi[qq] = (uint32_t)((unsigned long long)v >> 32) + (uint32_t)(AOFF >> 32);
                        } else {                       // v + 2^{7M} < 2^32
                            lo[qq] = (uint32_t)(unsigned long long)v + (uint32_t)AOFF;
                            hi[qq] = 0;
                        }
                    }
                    // the other M-tile's MMAs must have read the shared A: one wait for all of them before
                    // the first store (measured: one wait beats chunk-granular release)
                    if (need_free && ch == 0) {
                        ptx::mbar_wait(&S.mma_done[1 - m], fpar);
                        ptx::tc_fence_after();
                    }
                    if (ch == 0) {
                        // α of this layer with the A operand: TMEM columns 496 + 4m + 2·(L&1) of this row
                        // (the epilogue of layer L-2, the previous user, finished before these stores
                        // could start: they wait for MMAs that waited for its D-free arrival)
                        ptx::tmem_st2(ta - TA_A0 + 496 + 4 * m + 2 * (L & 1), (uint32_t)__double2loint(alpha),
                                      (uint32_t)__double2hiint(alpha));
                    }
#pragma unroll
                    for (int pa = 0; pa < NA; ++pa) {
                        const uint32_t *src = pa < 2 ? lo : hi;
                        const uint32_t sel = (pa & 1) ? 0x7632u : 0x5410u;
                        ptx::tmem_st4(ta + pa * TA_A_ARR + 4 * ch, __byte_perm(src[0], src[1], sel),
                                      __byte_perm(src[2], src[3], sel), __byte_perm(src[4], src[5], sel),
                                      __byte_perm(src[6], src[7], sel));
                    }
                }
            };
            TRW(2);
            if (__all_sync(0xffffffffu, fast)) chunks(std::true_type{});
            else chunks(std::false_type{});
            ptx::tmem_st_wait();
            TRW(3);
            ptx::tc_fence_before();
            asm volatile("bar.sync %0, 128;" ::"r"(1 + m) : "memory");   // the 4 converter warps of this M-tile
            TRW(4);
            if (q == 0) {
                if (ptx::elect_one()) {
                    if (k > 0) ptx::mbar_wait(&S.d_free[m], (uint32_t)((k - 1) & 1));   // layer L-1's D read
                    TRI(5);
                    ptx::tc_fence_after();
                    const uint32_t b0 = ptx::smem_u32(&S.B[0]);
                    const uint32_t bi0 = ptx::smem_u32(&S.BI[0][0]), bi1 = ptx::smem_u32(&S.BI[1][0]);
                    // K-step groups (ks0 = chunks 0-1, ks1 = 2-3, fold a = 3-4, ks2 = 4-5, fold b = 5-6),
                    // all arrays each
                    const uint32_t aoff[5] = {0, 8, 12, 16, 20};
                    const uint64_t bdesc[5] = {ptx::smem_desc(b0, 128, B1_PITCH), ptx::smem_desc(b0 + 256, 128, B1_PITCH),
                                               ptx::smem_desc(bi0, 128, BI_PITCH), ptx::smem_desc(b0 + 512, 128, B1_PITCH),
                                               ptx::smem_desc(bi1, 128, BI_PITCH)};
#pragma unroll
                    for (int g = 0; g < 5; ++g) {
#pragma unroll
                        for (int pa = 0; pa < NA; ++pa)
                            ptx::mma_i8_ts(tmem + m * TA_D_TILE + pa * TA_D_ARR, tmem + TA_A0 + pa * TA_A_ARR + aoff[g],
                                           bdesc[g], IDESC, g > 0 ? 1u : 0u);
                    }
                    ptx::mma_commit(&S.mma_done[m]);   // one commit for the layer's 20 MMAs
                    TRI(6);
                }
                __syncwarp();
            }
            // ---- loader duties: plane L+3 completed, plane L+4 issued (its slot, that of plane L-3, is
            // no longer read: these threads' A stores waited for MMAs issued after the epilogues of
            // layer L-2 read D, so both epilogues finished layer L-3) ----
            if (L + 3 <= Lend) {
                finish_plane(L + 3);
                TRW(10);
                if (L + 4 <= Lend) issue_plane(L + 4);
            }
            TRW(9);
        }
    } else {
        // ================================ epilogues ================================
        const uint32_t td = tmem + ((uint32_t)(q * 32) << 16) + m * TA_D_TILE;
        const int rp_ly = rowpar(ly);
        const int n0 = ly * PX + lx;
        bool has_src = false, has_rec = false;
        if (MODE == MODE_STEP) {
            for (int kk = 0; kk < p.nsrc; ++kk) {
                const int64_t n = p.src_dof[kk] / 3;
                const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
                has_src |= (ix >= X0 && ix < X0 + C::TX && iy >= Y0 && iy < Y0 + C::TY);
            }
            if (p.it >= 0 && p.it < p.rec_nt)
                for (int kk = 0; kk < p.nrec; ++kk) {
                    const int64_t n = p.rec_node[kk];
                    const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
                    has_rec |= (ix >= X0 && ix < X0 + C::TX && iy >= Y0 && iy < Y0 + C::TY);
                }
        }

        double T[3] = {0.0, 0.0, 0.0};               // top-face sum of the previous layer at this node
        double upv[3] = {0.0, 0.0, 0.0}, wn = 0.0;
        double uv[3] = {0.0, 0.0, 0.0};              // DAMP: u of the owned node (the plane holds ũ)
        uint8_t dm = 0;
        int64_t nd_next = ucol + PSTRIDE * (int64_t)Lfirst;   // node of plane P of prefetch_update (running)
        auto prefetch_update = [&](int P) {
            if (MODE == MODE_STEP && own && P >= Z0 && P <= Plast) {
                const int64_t nd = nd_next;
                upv[0] = p.uo[3 * nd];
                upv[1] = p.uo[3 * nd + 1];
                upv[2] = p.uo[3 * nd + 2];
                if constexpr (DAMP) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) uv[c] = __ldg(p.u + 3 * nd + c);
                }
                wn = __ldg(p.w + nd);
                dm = p.dmask ? __ldg(p.dmask + nd) : (uint8_t)0;
            }
            nd_next += PSTRIDE;
        };
        int64_t un_cur = ucol + PSTRIDE * (int64_t)Lfirst;   // node of plane L (running)

        prefetch_update(Lfirst);
        for (int L = Lfirst; L <= Plast; ++L) {
            const int k = L - Lfirst;
            TRW(0);
            // ---- element forces of layer L (24 outputs) ----
            double fb[12], ft[12];                   // bottom corners (local nodes 0-3), top (4-7): [corner][c]
            const bool has_layer = L < Lend;
            if (has_layer) {
                ptx::mbar_wait_sleep(&S.mma_done[m], (uint32_t)(k & 1));   // all MMAs of layer L
                TRW(1);
                ptx::tc_fence_after();
                uint32_t alo, ahi;
                ptx::tmem_ld2(td - m * TA_D_TILE + 496 + 4 * m + 2 * (L & 1), alo, ahi);
                ptx::tmem_ld_wait();
                const double alpha = __hiloint2double((int)ahi, (int)alo);
#pragma unroll
                for (int rr = 0; rr < 6; ++rr) {     // outputs 4rr .. 4rr+3
                    uint32_t R0[8], R1[8], R2[8], R3[8];
                    ptx::tmem_ld8(td + 0 * TA_D_ARR + rr * 8, R0);
                    ptx::tmem_ld8(td + 1 * TA_D_ARR + rr * 8, R1);
                    if (NA > 2) ptx::tmem_ld8(td + 2 * TA_D_ARR + rr * 8, R2);
                    if (NA > 3) ptx::tmem_ld8(td + 3 * TA_D_ARR + rr * 8, R3);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        const double dlo = limb_biased((int32_t)R0[2 * qq], (int32_t)R0[2 * qq + 1], (int32_t)R1[2 * qq],
                                                       (int32_t)R1[2 * qq + 1]);
                        double y = dlo;
                        if constexpr (NA > 2) {   // stages beyond NA arrays are absent: the bias value (C_j = 0)
                            const double dhi =
                                limb_biased((int32_t)R2[2 * qq], (int32_t)R2[2 * qq + 1],
                                            NA > 3 ? (int32_t)R3[2 * qq] : I8_BIAS, NA > 3 ? (int32_t)R3[2 * qq + 1] : I8_BIAS);
                            y = __fma_rn(dhi, 0x1p32, dlo);
                        }
                        const double f = __dmul_rn(alpha, y);   // RN(c1s·RN(y))
                        const int j = 4 * rr + qq;
                        if (j < 12) fb[j] = f;
                        else ft[j - 12] = f;
                    }
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&S.d_free[m]);
                TRW(2);
            } else {
#pragma unroll
                for (int j = 0; j < 12; ++j) fb[j] = ft[j] = 0.0;
            }
            // ---- node sums in the order of reading U2 ----
            // x-pairs: P(iy) = own (-x,-y) corner + lane lx-1's (+x,-y) corner; P'(iy) of the +y corners
            // goes to row ly+1 through shared memory
            const int ysl = k % ws::NYS;
            double Pb[3], Pt[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double pmb = __shfl_up_sync(0xffffffffu, fb[3 * 1 + c], 1);
                const double ppb = __shfl_up_sync(0xffffffffu, fb[3 * 2 + c], 1);
                const double pmt = __shfl_up_sync(0xffffffffu, ft[3 * 1 + c], 1);
                const double ppt = __shfl_up_sync(0xffffffffu, ft[3 * 2 + c], 1);
                Pb[c] = __dadd_rn(fb[3 * 0 + c], pmb);
                Pt[c] = __dadd_rn(ft[3 * 0 + c], pmt);
                S.ys[ysl][0][c][ly][lx] = __dadd_rn(fb[3 * 3 + c], ppb);
                S.ys[ysl][1][c][ly][lx] = __dadd_rn(ft[3 * 3 + c], ppt);
            }
            if (m == 0 && q == 3) ptx::mbar_arrive(&S.ys_ready[ysl]);   // row 3 feeds row 4 of the other M-tile
            asm volatile("bar.sync %0, 128;" ::"r"(3 + m) : "memory");   // the 4 epilogue warps of this M-tile
            if (m == 1 && q == 0) ptx::mbar_wait(&S.ys_ready[ysl], (uint32_t)((k / ws::NYS) & 1));
            TRW(6);
            if (tnode) {
                double fbot[3], ftop[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    fbot[c] = has_layer ? __dadd_rn(Pb[c], S.ys[ysl][0][c][ly - 1][lx]) : 0.0;   // B of plane L
                    ftop[c] = has_layer ? __dadd_rn(Pt[c], S.ys[ysl][1][c][ly - 1][lx]) : 0.0;   // T of plane L+1
                }
                const bool plane_done = L >= Z0;     // L <= Plast by the loop bound
                if (own && plane_done) {
                    const int64_t un_id = un_cur;
                    if (SLAB && (p.slab_flags & 1) && L == 0) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) p.iface_bot_b[3 * ucol + c] = fbot[c];
                    } else {
                        double f[3];
#pragma unroll
                        for (int c = 0; c < 3; ++c) f[c] = __dadd_rn(T[c], fbot[c]);
                        if (SLAB && (p.slab_flags & 2) && L == nz) {
#pragma unroll
                            for (int c = 0; c < 3; ++c) p.iface_top_A[3 * ucol + c] = f[c];
                        } else if (MODE == MODE_STEP) {
                            const Plane &P = S.pl[slot(L)];
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
                                double F = 0.0;
                                if (has_src)
                                    for (int kk = 0; kk < p.nsrc; ++kk)
                                        if (p.src_dof[kk] == 3 * un_id + c) F = __dadd_rn(F, p.src_val[kk]);
                                double uc;
                                if constexpr (BULK) uc = rowp(P, ly, rp_ly, L)[3 * lx + c];
                                else uc = P.up[c][n0];
                                if constexpr (DAMP) uc = uv[c];
                                double b = __dsub_rn(__dmul_rn(2.0, uc), upv[c]);
                                if constexpr (DAMP) b = __dsub_rn(b, __dmul_rn(p.ca, __dsub_rn(uc, upv[c])));
                                double un = __fma_rn(wn, __dsub_rn(F, f[c]), b);
                                if ((dm >> c) & 1) un = 0.0;
                                (DAMP ? p.un : p.uo)[3 * un_id + c] = un;
                                if (has_rec)
                                    for (int kk = 0; kk < p.nrec; ++kk)
                                        if (p.rec_node[kk] == un_id) p.traces[(3 * kk + c) * p.rec_nt + p.it] = un;
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < 3; ++c) p.fout[3 * un_id + c] = f[c];
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) T[c] = ftop[c];
            }
            TRW(7);
            un_cur += PSTRIDE;
            prefetch_update(L + 1);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (wu == 0) ptx::tmem_dealloc<512>(S.tmem);
}
