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
// INT8 path: 512 threads, two per element (u-half / G-half of ū_e, bottom / top output nodes),
// two M=128 tcgen05.mma.kind::i8 tiles per layer into TMEM (2 × 4 arrays × N48, 64-col pitch).
// The Eq. 9 diagonal term is folded into the integer product (DESIGN.md variant D): per array
// 3 K-steps against B = −K_e^INT8 ⊗ I_2 plus 2 K-steps of the G bytes against −128·I ⊗ I_2, so
// D = −(K_e^INT8 v + 128 v_G) byte-stage by byte-stage, and f_e = RN(c1 s_e 2^-56)·RN(y).

constexpr int EY_I8V = 4;   // INT8 tile: 32×4 elements = one M=128 MMA tile; 2 CTAs per SM
template <int PATH>
struct V1 {
    static constexpr int EY = PATH == OVX_INT8 ? EY_I8V : 8;
    static constexpr int NE = EX * EY;                 // 256 elements per layer
    static constexpr int TPE = PATH == OVX_INT8 ? 2 : 1;
    static constexpr int NT = NE * TPE;                // threads
    static constexpr int TY = EY - 1;                  // 7 owned node rows
    static constexpr int PY = EY + 1;                  // 9 node rows per smem plane
    static constexpr int NOWN = TX * TY;               // 217 owned nodes per plane
    static constexpr int PLANE = PX * PY * 3;          // 891 doubles per plane
    static constexpr int PF = (PLANE + NT - 1) / NT;   // prefetched doubles per thread
    static constexpr int MT = NE / 128;                // INT8: M=128 MMA tiles per layer
    static constexpr int MINB = PATH == OVX_INT8 ? (MT == 1 ? 2 : 1) : 2;
    static constexpr int TMEM_COLS = MT * 256;
};

struct SmemV1F64 {
    double up[3][V1<OVX_FP64>::PLANE];
    double fe[24][256];
    double facc[2][V1<OVX_FP64>::NOWN * 3];
};

// A operand row (one element, one half-word array): 7 chunks of 16 B — chunks 0-2 the u bytes,
// 3-5 the G bytes, 6 zero (K padding of the identity block's second K-step).
constexpr int A1_CHUNKS = 7;
constexpr int A1_PITCH = A1_CHUNKS * 128 + 16;   // bytes per 8-row core-matrix group (+16: bank spread)
constexpr int A1_BYTES = 16 * A1_PITCH;          // one half-word array of 128 rows
constexpr int B1_PITCH = 6 * 128;                // main B: 48 rows × 96 K-bytes
constexpr int BI_PITCH = 2 * 128;                // identity blocks: 48 rows × 32 K-bytes

struct SmemV1I8 {
    struct {
        uint8_t A[V1<OVX_INT8>::MT][4][A1_BYTES];   // [M-tile][half-word array], K-major layout
    } u;
    double fe[24][V1<OVX_INT8>::NE];  // separate from A: one M-tile's epilogue may run while
                                      // another M-tile's MMAs still read their A arrays
    alignas(128) uint8_t B[6 * B1_PITCH];
    alignas(128) uint8_t BI[2][6 * BI_PITCH];
    double up[3][V1<OVX_INT8>::PLANE];
    double facc[2][V1<OVX_INT8>::NOWN * 3];
    double amax[2][V1<OVX_INT8>::NE];
    uint64_t mbar[V1<OVX_INT8>::MT];
    uint32_t tmem;
};

template <int PATH>
using SmemV1 = typename std::conditional<PATH == OVX_INT8, SmemV1I8, SmemV1F64>::type;

__device__ __forceinline__ auto fe_of(SmemV1I8 &S) { return S.fe; }
__device__ __forceinline__ auto fe_of(SmemV1F64 &S) { return S.fe; }

template <int PATH>
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
        if (iz <= p.nz && ix >= 0 && ix < NX1 && iy >= 0 && iy < NY1) v = __ldg(p.u + 3 * (ix + NX1 * (iy + NY1 * iz)) + c);
        dst[idx] = v;
    }
}

template <int PATH, int MODE>
__global__ void __launch_bounds__(V1<PATH>::NT, V1<PATH>::MINB) step_v1(const StepParams p) {
    using C = V1<PATH>;
    constexpr int NT = C::NT, TY = C::TY, NOWN = C::NOWN, PLANE = C::PLANE, PF = C::PF;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SmemV1<PATH> &S = *reinterpret_cast<SmemV1<PATH> *>(smem_raw);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;

    int bid = blockIdx.x;
    const int tx = bid % p.tiles_x;
    bid /= p.tiles_x;
    const int ty = bid % p.tiles_y;
    const int tz = bid / p.tiles_y;
    const int64_t X0 = (int64_t)tx * TX, Y0 = (int64_t)ty * TY;
    const int64_t Z0 = (int64_t)tz * p.zchunk;
    const int64_t Z1 = min(Z0 + (int64_t)p.zchunk, p.nz + 1);
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;
    const int64_t PSTRIDE = NX1 * NY1;        // nodes per plane

    // element (and half) handled by this thread
    int el, half = 0, mt = 0, row = 0;
    if constexpr (PATH == OVX_INT8) {
        const int g = warp >> 2;          // 0..3: (M-tile, half)
        row = (warp & 3) * 32 + lane;     // TMEM lane = MMA row
        mt = g >> 1;
        half = g & 1;                     // 0: u-part of ū_e, outputs of nodes 0-3; 1: G-part, nodes 4-7
        el = mt * 128 + row;
    } else {
        el = t;
    }
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

    uint32_t phase = 0;
    if constexpr (PATH == OVX_INT8) {
        // resident B operands: B[n = 2i+b'][kb = 2k+b] = −K_e^INT8[i][k]·δ(b,b');
        // BI[s][n][kb] = −128·δ(k, i − 16 s)·δ(b,b') on the G bytes (k = G index within the K-step)
        for (int idx = t; idx < 48 * 96; idx += NT) {
            const int n = idx / 96, kb = idx - n * 96;
            const int off = (n >> 3) * B1_PITCH + (kb >> 4) * 128 + (n & 7) * 16 + (kb & 15);
            S.B[off] = ((kb & 1) == (n & 1)) ? (uint8_t)(-(int)c_K8[(n >> 1) * 48 + (kb >> 1)]) : (uint8_t)0;
        }
        for (int idx = t; idx < 2 * 48 * 32; idx += NT) {
            const int s2 = idx / (48 * 32), r2 = idx - s2 * 48 * 32;
            const int n = r2 / 32, kb = r2 - n * 32;
            const int off = (n >> 3) * BI_PITCH + (kb >> 4) * 128 + (n & 7) * 16 + (kb & 15);
            const int k = 16 * s2 + (kb >> 1);
            S.BI[s2][off] = ((kb & 1) == (n & 1) && k == (n >> 1)) ? (uint8_t)0x80 : (uint8_t)0;
        }
        // zero the K-padding chunk of every A row (never written afterwards)
        for (int idx = t; idx < C::MT * 4 * 128; idx += NT) {
            const int a = idx >> 7, r = idx & 127;
            *reinterpret_cast<uint4 *>(&S.u.A[a >> 2][a & 3][(r >> 3) * A1_PITCH + 6 * 128 + (r & 7) * 16]) =
                make_uint4(0, 0, 0, 0);
        }
        if (warp == 0) ptx::tmem_alloc<C::TMEM_COLS>(&S.tmem);
        if (t == 0) {
            for (int mm = 0; mm < C::MT; ++mm) ptx::mbar_init(&S.mbar[mm], 1);
        }
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
    }
    for (int i = t; i < 2 * NOWN * 3; i += NT) (&S.facc[0][0])[i] = 0.0;
    const int64_t Lfirst = max(Z0 - 1, (int64_t)0);
    v1_load_plane_sync<PATH>(S.up[Lfirst % 3], p, X0, Y0, Lfirst);
    v1_load_plane_sync<PATH>(S.up[(Lfirst + 1) % 3], p, X0, Y0, Lfirst + 1);
    __syncthreads();
    if constexpr (PATH == OVX_INT8) ptx::tc_fence_after();

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
        const double *uplane = p.u + 3 * PSTRIDE * pz;
#pragma unroll
        for (int j = 0; j < PF; ++j) pfv[j] = (pf && pfok[j]) ? __ldg(uplane + pfoff[j]) : 0.0;
        const bool upd = plane_done && own;
        const int64_t un_id = ucol + PSTRIDE * L;
        double upv[3] = {0.0, 0.0, 0.0}, wn = 0.0;
        uint8_t dm = 0;
        if (MODE == MODE_STEP && upd) {
            upv[0] = p.uo[3 * un_id];
            upv[1] = p.uo[3 * un_id + 1];
            upv[2] = p.uo[3 * un_id + 2];
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
            if constexpr (PATH == OVX_FP64) {
                double fe[24];
                element_force_wht(ue, c_mat[m], fe);   // zero material -> fe = 0 exactly
#pragma unroll
                for (int r = 0; r < 24; ++r) {
                    S.fe[r][el] = fe[r];
                    if (MODE == MODE_DEBUG && dbg && p.dbg_fe) p.dbg_fe[dj * 24 + r] = fe[r];
                }
            } else if constexpr (PATH == OVX_FP64_DENSE) {
                const double ck = c_mat[m].ck, cg = c_mat[m].cg;
#pragma unroll 1
                for (int r = 0; r < 24; ++r) {
                    double a = 0.0, b = 0.0;
#pragma unroll
                    for (int c = 0; c < 24; ++c) {
                        a = __dadd_rn(a, __dmul_rn(c_Kk[r * 24 + c], ue[c]));
                        b = __dadd_rn(b, __dmul_rn(c_Kg[r * 24 + c], ue[c]));
                    }
                    const double f = __dadd_rn(__dmul_rn(ck, a), __dmul_rn(cg, b));
                    S.fe[r][el] = ein ? f : 0.0;
                    if (MODE == MODE_DEBUG && dbg && p.dbg_fe) p.dbg_fe[dj * 24 + r] = f;
                }
            } else {
                // ---- Eqs. 10-16: s_e, INT64 image, byte slices -> A operand (this thread: 24 of 48) ----
                const double cG = c_mat[m].cG;
                double hm = 0.0;
                if (half) {
#pragma unroll
                    for (int i = 12; i < 24; ++i) hm = fmax(hm, fabs(ue[i]));
                } else {
#pragma unroll
                    for (int i = 0; i < 12; ++i) hm = fmax(hm, fabs(ue[i]));
                }
                S.amax[half][el] = hm;
                asm volatile("bar.sync %0, 256;" ::"r"(1 + mt) : "memory");   // the 8 warps of this M-tile
                const double amax = fmax(S.amax[0][el], S.amax[1][el]);
                // max_i |RN(cG u_i)| = RN(cG max_i |u_i|)  (RN is monotone, cG > 0)
                const double s = fmax(amax, __dmul_rn(cG, amax));
                const bool deg = !ein || !(s >= 0x1p-1022) || isinf(s);
                uint8_t *Ab = &S.u.A[mt][0][0];
                const uint32_t rowoff = (uint32_t)((row >> 3) * A1_PITCH + (row & 7) * 16) + (uint32_t)(3 * half) * 128;
                // ū_e for this half: u_e (half 0) or RN(cG·u_e) (half 1); half is warp-uniform
                if (half) {
#pragma unroll
                    for (int i = 0; i < 24; ++i) ue[i] = __dmul_rn(cG, ue[i]);
                }
                const bool straight = !deg && s >= 0x1p-960;
                const double r = 1.0 / s;                          // RN(1/s_e), reading Q7
                const double R = __dmul_rn(r, 0x1p56);             // exact power-of-two scaling
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {                   // 8 values at a time: convert, pack, store
                    long long v[8];
                    if (straight) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) v[q] = __double2ll_rz(__dmul_rn(ue[ch * 8 + q], R));  // trunc (Q8)
                    } else {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            v[q] = deg ? 0ll : __double2ll_rz(__dmul_rn(__dmul_rn(ue[ch * 8 + q], r), 0x1p56));
                    }
                    uint32_t lo[8], hi[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const unsigned long long vp = (unsigned long long)v[q] + (1ull << 56);
                        lo[q] = (uint32_t)vp;
                        hi[q] = (uint32_t)(vp >> 32);
                        if (MODE == MODE_DEBUG && dbg) {
                            const int k = 24 * half + ch * 8 + q;
                            if (p.dbg_v) p.dbg_v[dj * 48 + k] = v[q];
                            if (p.dbg_d)
#pragma unroll
                                for (int j = 0; j < 8; ++j) p.dbg_d[dj * 384 + j * 48 + k] = (uint8_t)(vp >> (8 * j));
                        }
                    }
                    const uint32_t off = rowoff + (uint32_t)ch * 128;
#pragma unroll
                    for (int pa = 0; pa < 4; ++pa) {
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
                if (MODE == MODE_DEBUG && dbg && half == 0 && p.dbg_s) p.dbg_s[dj] = s;

                // ---- Eq. 17 (+ folded diagonal): this M-tile, 4 arrays × (3 + 2) K-steps, M128 N48 K32 ----
                // Each M-tile (8 warps) hands off to the tensor core on its own named barrier, so one
                // M-tile's MMAs overlap the other M-tile's digit or epilogue work.
                ptx::fence_proxy_async_smem();
                asm volatile("bar.sync %0, 256;" ::"r"(1 + mt) : "memory");
                if (t == 256 * mt) {
                    ptx::tc_fence_after();
                    const uint32_t b0 = ptx::smem_u32(&S.B[0]);
                    const uint32_t bi0 = ptx::smem_u32(&S.BI[0][0]), bi1 = ptx::smem_u32(&S.BI[1][0]);
                    {
                        const int mm = mt;
                        const uint32_t a0 = ptx::smem_u32(&S.u.A[mm][0][0]);
#pragma unroll
                        for (int pa = 0; pa < 4; ++pa) {
                            const uint32_t ab = a0 + pa * A1_BYTES;
                            const uint32_t d = S.tmem + mm * 256 + pa * 64;
#pragma unroll
                            for (int ks = 0; ks < 3; ++ks)
                                ptx::mma_i8(d, ptx::smem_desc(ab + ks * 256, 128, A1_PITCH),
                                            ptx::smem_desc(b0 + ks * 256, 128, B1_PITCH), IDESC, ks > 0 ? 1u : 0u);
                            ptx::mma_i8(d, ptx::smem_desc(ab + 3 * 128, 128, A1_PITCH),
                                        ptx::smem_desc(bi0, 128, BI_PITCH), IDESC, 1u);
                            ptx::mma_i8(d, ptx::smem_desc(ab + 5 * 128, 128, A1_PITCH),
                                        ptx::smem_desc(bi1, 128, BI_PITCH), IDESC, 1u);
                        }
                        ptx::mma_commit(&S.mbar[mm]);
                    }
                }
                // one warp of the M-tile polls the MMA-completion mbarrier; the other seven block in
                // hardware on the named barrier (no issue slots spent spinning)
                if (warp == 8 * mt) ptx::mbar_wait(&S.mbar[mt], phase);
                asm volatile("bar.sync %0, 256;" ::"r"(1 + mt) : "memory");
                phase ^= 1;
                ptx::tc_fence_after();

                // ---- epilogue: 12 outputs (nodes 4·half .. 4·half+3) ----
                // D_p holds −C_j with C_j = K_D·b_j (K_D·1 = 0, so y = Σ_j 256^j C_j exactly).
                // Two 64-bit limbs (< 2^44) through the 1.5·2^52 magic, one rounding in the fma.
                const double alpha = -__dmul_rn(c_mat[m].c1, __dmul_rn(s, 0x1p-56));   // −RN(c1·s·2^-56)
                const uint32_t tb = S.tmem + ((uint32_t)((warp & 3) * 32) << 16) + mt * 256 + half * 24;
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {           // 4 outputs per round (8 columns per array)
                    uint32_t R0[8], R1[8], R2[8], R3[8];
                    ptx::tmem_ld8(tb + 0 + cc * 8, R0);
                    ptx::tmem_ld8(tb + 64 + cc * 8, R1);
                    ptx::tmem_ld8(tb + 128 + cc * 8, R2);
                    ptx::tmem_ld8(tb + 192 + cc * 8, R3);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int i = 12 * half + cc * 4 + q;
                        const int32_t c0 = (int32_t)R0[2 * q], c1_ = (int32_t)R0[2 * q + 1];
                        const int32_t c2_ = (int32_t)R1[2 * q], c3 = (int32_t)R1[2 * q + 1];
                        const int32_t c4 = (int32_t)R2[2 * q], c5 = (int32_t)R2[2 * q + 1];
                        const int32_t c6 = (int32_t)R3[2 * q], c7 = (int32_t)R3[2 * q + 1];
                        const double dlo = ptx::limb_magic(c0, c1_, c2_, c3) - (0x1.8p52 + 0x1p31);
                        const double dhi = ptx::limb_magic(c4, c5, c6, c7) - (0x1.8p52 + 0x1p31);
                        const double Y = __fma_rn(dhi, 0x1p32, dlo);    // RN(−y)
                        const double f = __dmul_rn(alpha, Y);            // = RN(c1s·RN(y))
                        if (MODE == MODE_DEBUG && dbg) {
                            const int32_t Cj[8] = {c0, c1_, c2_, c3, c4, c5, c6, c7};
                            __int128 y = 0;
#pragma unroll
                            for (int j = 7; j >= 0; --j) y = y * 256 - (__int128)Cj[j];
                            if (p.dbg_C)
#pragma unroll
                                for (int j = 0; j < 8; ++j) p.dbg_C[dj * 192 + j * 24 + i] = -Cj[j];
                            if (p.dbg_yhi) p.dbg_yhi[dj * 24 + i] = (long long)(y >> 64);
                            if (p.dbg_ylo) p.dbg_ylo[dj * 24 + i] = (long long)(unsigned long long)y;
                            if (p.dbg_fe) p.dbg_fe[dj * 24 + i] = f;
                        }
                        S.fe[i][el] = f;
                    }
                }
                ptx::tc_fence_before();
            }
        }
        __syncthreads();

        // ---- (3) scatter (U2 tree order) + update of the completed plane L ----
        if (t < NOWN) {
            auto fe = fe_of(S);
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
                        const double b = __dsub_rn(__dmul_rn(2.0, up[c]), upv[c]);
                        double un = __fma_rn(wn, __dsub_rn(F, fl[c]), b);
                        if ((dm >> c) & 1) un = 0.0;
                        p.uo[dof] = un;
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
    if constexpr (PATH == OVX_INT8) {
        ptx::tc_fence_after();
        if (warp == 0) ptx::tmem_dealloc<C::TMEM_COLS>(S.tmem);
    }
}
