// kernels.cu — sm_100a kernels of the OVFEM / TCOVFEM explicit time step.
//
// One fused kernel per time step:
//   CTA  = a tile of TX×TY owned node columns marching in z over a chunk of node planes.
//   Per element layer L it computes the 128 = (TX+1)(TY+1) elements touching its owned
//   nodes (one halo element ring recomputed by the neighbour tile, so no cross-CTA
//   reduction is needed), accumulates their forces into two shared-memory node planes
//   in global element order (bit-identical to the oracle's scatter order), and applies
//   the central-difference update (Eq. 3, L263-L266 with the sign of Eq. 3)
//   to each completed plane.
//
// Element force, two paths:
//   OVX_FP64: f_e = (κ ds/256)·(K^κ u_e) + (G ds/384)·((K̄^G+128I) u_e), integer matrices
//             applied first with sequential FP64 sums (DESIGN.md oracle (i) step 3).
//   OVX_INT8: PAPER.md Eq. 9 via Eqs. 10-17: s_e = max|ū_e|, v = trunc(2^56 ū_e/s_e),
//             byte slices of v + 2^56 (variant B) as the u8 A operand of
//             tcgen05.mma.kind::i8 (M=128 elements, N=48, K=96, 4 half-word arrays),
//             K_e^INT8 ⊗ I_2 as the resident s8 B operand, s32 accumulators in TMEM,
//             exact two-limb recombination y = K_e^INT8 v and f_e = c1·(RN(y)·s_e 2^-56 + c2 u_e).
#include "ovx_internal.h"
#include "ptx.cuh"

#include "../../include/ovx.h"

namespace ovx {

__constant__ MatConst c_mat[kMaxMat];
__constant__ double c_Kk[576];
__constant__ double c_Kg[576];
__constant__ int8_t c_K8[1152];

namespace {

constexpr int EX = 32;                    // element columns per layer (x)
constexpr int TX = EX - 1;                // owned node columns (x)
constexpr int PX = TX + 2;                // node columns of a u plane held in smem (x)
template <int EY> struct Tile {
    static constexpr int TY = EY - 1;          // owned node rows (y)
    static constexpr int NE = EX * EY;         // elements per layer = threads per CTA
    static constexpr int PY = TY + 2;          // node rows of a u plane in smem
    static constexpr int PLANE_D = PX * PY * 3;
    static constexpr int NOWN = TX * TY;
    static constexpr int FPL = NOWN * 3;
};
constexpr int EY_I8 = 4;                  // INT8 path: 128 elements = MMA M
constexpr int EY_F64 = 8;                 // FP64 paths: 256 elements per layer
constexpr int KB = 96;                    // K bytes per A row / B row (48 values × 2 bytes)
constexpr int ROWGRP = 8 * KB;            // bytes per 8-row core-matrix group (6 chunks × 128)
constexpr int A_BYTES = 128 * KB;         // one half-word array (M = 128 rows)
constexpr int B_ROWS = 48;                // N = 24 outputs × 2 byte positions
constexpr int B_BYTES = B_ROWS * KB;
constexpr int TMEM_COLS = 256;            // 4 accumulators of 48 columns at 64-column pitch
constexpr uint32_t IDESC = ptx::idesc_i8(128, 48);

template <int EY>
struct SmemF64 {
    using T = Tile<EY>;
    double up[2][T::PLANE_D];
    double fe[24][T::NE];
    double facc[2][T::FPL];
};

struct SmemI8 {
    using T = Tile<EY_I8>;
    alignas(1024) uint8_t A[4][A_BYTES];
    alignas(128) uint8_t B[B_BYTES];
    double up[2][T::PLANE_D];
    double fe[24][T::NE];
    double facc[2][T::FPL];
    double sig[T::NE];
    int deg[T::NE];
    uint64_t mbar;
    uint32_t tmem;
};

template <int PATH>
struct PathCfg {
    static constexpr int EY = PATH == OVX_INT8 ? EY_I8 : EY_F64;
    using T = Tile<EY>;
    using Smem = typename std::conditional<PATH == OVX_INT8, SmemI8, SmemF64<EY>>::type;
};

// Load node plane iz of u (tile-local columns [X0-1, X0+TX] × [Y0-1, Y0+TY]) into smem.
template <int EY>
__device__ __forceinline__ void load_plane(double *dst, const double *__restrict__ u, const StepParams &p,
                                           int64_t X0, int64_t Y0, int64_t iz) {
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;
    for (int idx = threadIdx.x; idx < Tile<EY>::PLANE_D; idx += Tile<EY>::NE) {
        int py = idx / (PX * 3);
        int rem = idx - py * (PX * 3);
        int px = rem / 3, c = rem - px * 3;
        int64_t ix = X0 - 1 + px, iy = Y0 - 1 + py;
        double v = 0.0;
        if (ix >= 0 && ix < NX1 && iy >= 0 && iy < NY1) v = __ldg(u + 3 * (ix + NX1 * (iy + NY1 * iz)) + c);
        dst[idx] = v;
    }
}

// Gather u_e (local node order of reading Q1) of tile-local element (lx, ly) from the two planes.
template <int PY>
__device__ __forceinline__ void gather(double (&ue)[24], const double *lo, const double *hi, int lx, int ly) {
    const int cx[4] = {0, 1, 1, 0}, cy[4] = {0, 0, 1, 1};
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const double *pl = a < 4 ? lo : hi;
        int o = ((ly + cy[a & 3]) * PX + (lx + cx[a & 3])) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) ue[3 * a + c] = pl[o + c];
    }
}

// ---- factored FP64 element force (OVX_FP64) -----------------------------------
// K_e^o u_e = Σ_β B_βᵀ c B_β u_e / g_β (Eq. 5) evaluated through the 3-D Walsh-Hadamard
// transform of the corner values: with h_c[S] = Σ_α Π_{j∈S} r̄_j^α u_c^α, the mode-β strain is
// (ds²/4)2^{-|β|} h_c[{i}∪β] (reading Q3), and f_c^α = Σ_S Π_{j∈S} r̄_j^α F_c[S] with
// F_c[S] = (ds/16) Σ (3/4)^{|β|} τ_β[c][i].  ≈180 FP64 operations instead of 1152 FMAs;
// equal to K_e^o u_e in exact arithmetic (rounding differs from the dense order).
__device__ __forceinline__ void wht8(double (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int st = 1 << j;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (!(b & st)) {
                const double a = v[b], c = v[b | st];
                v[b] = a + c;
                v[b | st] = c - a;
            }
    }
}
__device__ __forceinline__ void iwht8(double (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int st = 1 << j;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (!(b & st)) {
                const double a = v[b], c = v[b | st];
                v[b] = a - c;
                v[b | st] = a + c;
            }
    }
}
__device__ __forceinline__ void element_force_wht(const double (&ue)[24], const MatConst &m, double (&fe)[24]) {
    constexpr int BORD[8] = {0, 1, 3, 2, 4, 5, 7, 6};  // local node -> bit index x | y<<1 | z<<2
    double h[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int a = 0; a < 8; ++a) h[c][BORD[a]] = ue[3 * a + c];
        wht8(h[c]);
    }
    double F[3][8];
    F[0][0] = F[1][0] = F[2][0] = 0.0;
    // β = ∅ : full gradient h_c[{i}]
    const double lt0 = m.L0 * (h[0][1] + h[1][2] + h[2][4]);
    F[0][1] = fma(m.M0x2, h[0][1], lt0);
    F[1][2] = fma(m.M0x2, h[1][2], lt0);
    F[2][4] = fma(m.M0x2, h[2][4], lt0);
    const double sxy = m.M0 * (h[0][2] + h[1][1]);
    const double syz = m.M0 * (h[1][4] + h[2][2]);
    const double szx = m.M0 * (h[2][1] + h[0][4]);
    F[0][2] = sxy; F[1][1] = sxy;
    F[1][4] = syz; F[2][2] = syz;
    F[2][1] = szx; F[0][4] = szx;
    // |β| = 1
    const double ltx = m.L1 * (h[1][3] + h[2][5]);
    const double lty = m.L1 * (h[0][3] + h[2][6]);
    const double ltz = m.L1 * (h[0][5] + h[1][6]);
    F[0][3] = fma(m.M1x3, h[0][3], lty);
    F[1][3] = fma(m.M1x3, h[1][3], ltx);
    F[0][5] = fma(m.M1x3, h[0][5], ltz);
    F[2][5] = fma(m.M1x3, h[2][5], ltx);
    F[1][6] = fma(m.M1x3, h[1][6], ltz);
    F[2][6] = fma(m.M1x3, h[2][6], lty);
    const double pp = h[2][3], qq = h[1][5], rr = h[0][6], tt = pp + qq + rr;
    F[2][3] = m.M1 * (tt + pp);
    F[1][5] = m.M1 * (tt + qq);
    F[0][6] = m.M1 * (tt + rr);
    // |β| = 2
    F[0][7] = m.C2 * h[0][7];
    F[1][7] = m.C2 * h[1][7];
    F[2][7] = m.C2 * h[2][7];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        iwht8(F[c]);
#pragma unroll
        for (int a = 0; a < 8; ++a) fe[3 * a + c] = F[c][BORD[a]];
    }
}

template <int PATH, int MODE>
__global__ void __launch_bounds__(PathCfg<PATH>::T::NE) step_kernel(const StepParams p) {
    using Cfg = PathCfg<PATH>;
    using T = typename Cfg::T;
    constexpr int EY = Cfg::EY;
    constexpr int NT = T::NE, TY = T::TY, PY = T::PY, NOWN = T::NOWN, FPL = T::FPL;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    typename Cfg::Smem &S = *reinterpret_cast<typename Cfg::Smem *>(smem_raw);
    const int t = threadIdx.x;
    const int warp = t >> 5;

    int bid = blockIdx.x;
    const int tx = bid % p.tiles_x;
    bid /= p.tiles_x;
    const int ty = bid % p.tiles_y;
    const int tz = bid / p.tiles_y;
    const int64_t X0 = (int64_t)tx * TX, Y0 = (int64_t)ty * TY;
    const int64_t Z0 = (int64_t)tz * p.zchunk;
    const int64_t Z1 = min(Z0 + (int64_t)p.zchunk, p.nz + 1);
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;

    const int lx = t % EX, ly = t / EX;
    const int64_t ex = X0 - 1 + lx, ey = Y0 - 1 + ly;
    const bool ein = (ex >= 0 && ex < p.nx && ey >= 0 && ey < p.ny);

    uint32_t phase = 0;
    if constexpr (PATH == OVX_INT8) {
        // Resident B operand: B[n = 2i+b'][kb = 2k+b] = K_e^INT8[i][k]·δ(b,b'), K-major core matrices.
        for (int idx = t; idx < B_BYTES; idx += NT) {
            int grp = idx / ROWGRP, rem = idx - grp * ROWGRP;
            int chunk = rem >> 7;
            rem &= 127;
            int n = grp * 8 + (rem >> 4), kb = chunk * 16 + (rem & 15);
            S.B[idx] = ((kb & 1) == (n & 1)) ? (uint8_t)c_K8[(n >> 1) * 48 + (kb >> 1)] : (uint8_t)0;
        }
        if (warp == 0) ptx::tmem_alloc<TMEM_COLS>(&S.tmem);
        if (t == 0) ptx::mbar_init(&S.mbar, 1);
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
    }
    for (int i = t; i < 2 * FPL; i += NT) (&S.facc[0][0])[i] = 0.0;
    __syncthreads();
    if constexpr (PATH == OVX_INT8) ptx::tc_fence_after();

    const int64_t Lfirst = max(Z0 - 1, (int64_t)0);
    for (int64_t L = Z0 - 1; L < Z1; ++L) {
        const bool layer_ok = (L >= 0 && L < p.nz);
        if (layer_ok) {
            if (L == Lfirst) load_plane<EY>(S.up[L & 1], p.u, p, X0, Y0, L);
            load_plane<EY>(S.up[(L + 1) & 1], p.u, p, X0, Y0, L + 1);
            __syncthreads();
            const double *plo = S.up[L & 1], *phi = S.up[(L + 1) & 1];
            const int m = ein ? (int)__ldg(p.mat + ex + p.nx * (ey + p.ny * L)) : 0;
            const bool dbg_w = (MODE == MODE_DEBUG) && ein && lx < TX && ly < TY && (L + 1 >= Z0) && (L + 1 < Z1);
            const int64_t eid = ex + p.nx * (ey + p.ny * L);
            const int64_t dj = eid - p.dbg_e0;
            const bool dbg = dbg_w && dj >= 0 && dj < p.dbg_ne;

            if constexpr (PATH == OVX_FP64) {
                double ue[24], fe[24];
                gather<PY>(ue, plo, phi, lx, ly);
                element_force_wht(ue, c_mat[m], fe);
#pragma unroll
                for (int r = 0; r < 24; ++r) {
                    S.fe[r][t] = ein ? fe[r] : 0.0;
                    if (MODE == MODE_DEBUG && dbg && p.dbg_fe) p.dbg_fe[dj * 24 + r] = fe[r];
                }
            } else if constexpr (PATH == OVX_FP64_DENSE) {
                double ue[24];
                gather<PY>(ue, plo, phi, lx, ly);
                const double ck = c_mat[m].ck, cg = c_mat[m].cg;
#pragma unroll 1
                for (int r = 0; r < 24; ++r) {
                    double a = 0.0, b = 0.0;
#pragma unroll
                    for (int c = 0; c < 24; ++c) {
                        a = __dadd_rn(a, __dmul_rn(c_Kk[r * 24 + c], ue[c]));
                        b = __dadd_rn(b, __dmul_rn(c_Kg[r * 24 + c], ue[c]));
                    }
                    double f = __dadd_rn(__dmul_rn(ck, a), __dmul_rn(cg, b));
                    S.fe[r][t] = ein ? f : 0.0;
                    if (MODE == MODE_DEBUG && dbg && p.dbg_fe) p.dbg_fe[dj * 24 + r] = f;
                }
            } else {
                // ---- Eqs. 10-16 on CUDA cores: scale, INT64 image, byte slices -> A operand ----
                double ue[24];
                gather<PY>(ue, plo, phi, lx, ly);
                const double cG = c_mat[m].cG;
                double amax = 0.0;
#pragma unroll
                for (int i = 0; i < 24; ++i) amax = fmax(amax, fabs(ue[i]));
                // max_i |RN(cG u_i)| = RN(cG max_i |u_i|)  (RN is monotone, cG > 0)
                const double s = fmax(amax, __dmul_rn(cG, amax));
                const bool deg = !ein || !(s >= 0x1p-1022) || isinf(s);
                const bool fast = s >= 0x1p-960;
                const double r = 1.0 / s;                          // RN(1/s_e), reading Q7
                const double R = fast ? __dmul_rn(r, 0x1p56) : r;  // exact power-of-two scaling
#pragma unroll
                for (int ch = 0; ch < 6; ++ch) {
                    uint32_t lo[8], hi[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int k = ch * 8 + q;
                        const double ub = k < 24 ? ue[k] : __dmul_rn(cG, ue[k - 24]);
                        const double tt = fast ? __dmul_rn(ub, R) : __dmul_rn(__dmul_rn(ub, r), 0x1p56);
                        const long long v = deg ? 0ll : __double2ll_rz(tt);  // truncation toward 0 (Q8)
                        const unsigned long long vp = (unsigned long long)v + (1ull << 56);
                        lo[q] = (uint32_t)vp;
                        hi[q] = (uint32_t)(vp >> 32);
                        if (MODE == MODE_DEBUG && dbg) {
                            if (p.dbg_v) p.dbg_v[dj * 48 + k] = v;
                            if (p.dbg_d)
#pragma unroll
                                for (int j = 0; j < 8; ++j) p.dbg_d[dj * 384 + j * 48 + k] = (uint8_t)(vp >> (8 * j));
                        }
                    }
                    // half-word arrays: array pa holds bytes (2pa, 2pa+1) of v' for every k
                    const uint32_t off = (uint32_t)((t >> 3) * ROWGRP + ch * 128 + (t & 7) * 16);
#pragma unroll
                    for (int pa = 0; pa < 4; ++pa) {
                        const uint32_t *src = pa < 2 ? lo : hi;
                        const uint32_t sel = (pa & 1) ? 0x7632u : 0x5410u;
                        uint4 wv;
                        wv.x = __byte_perm(src[0], src[1], sel);
                        wv.y = __byte_perm(src[2], src[3], sel);
                        wv.z = __byte_perm(src[4], src[5], sel);
                        wv.w = __byte_perm(src[6], src[7], sel);
                        *reinterpret_cast<uint4 *>(&S.A[pa][off]) = wv;
                    }
                }
                S.sig[t] = __dmul_rn(s, 0x1p-56);
                S.deg[t] = deg;
#pragma unroll
                for (int i = 0; i < 24; ++i) S.fe[i][t] = ue[i];  // parked for the epilogue (c2·u_e)
                if (MODE == MODE_DEBUG && dbg && p.dbg_s) p.dbg_s[dj] = s;

                // ---- Eq. 17 on tensor cores: 4 arrays × 3 K-steps of M128 N48 K32 ----
                ptx::fence_proxy_async_smem();
                __syncthreads();
                if (t == 0) {
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(&S.A[0][0]), b0 = ptx::smem_u32(&S.B[0]);
#pragma unroll
                    for (int pa = 0; pa < 4; ++pa)
#pragma unroll
                        for (int ks = 0; ks < 3; ++ks) {
                            uint64_t ad = ptx::smem_desc(a0 + pa * A_BYTES + ks * 256, 128, ROWGRP);
                            uint64_t bd = ptx::smem_desc(b0 + ks * 256, 128, ROWGRP);
                            ptx::mma_i8(S.tmem + pa * 64, ad, bd, IDESC, ks > 0 ? 1u : 0u);
                        }
                    ptx::mma_commit(&S.mbar);
                }
                ptx::mbar_wait(&S.mbar, phase);
                phase ^= 1;
                ptx::tc_fence_after();

                // ---- epilogue: exact recombination + Eq. 9 scalars ----
                const double c1 = c_mat[m].c1, c2 = c_mat[m].c2;
                const double sig = S.sig[t];
                const uint32_t tbase = S.tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
                for (int cc = 0; cc < 3; ++cc) {
                    uint32_t R0[16], R1[16], R2[16], R3[16];
                    ptx::tmem_ld16(tbase + 0 + cc * 16, R0);
                    ptx::tmem_ld16(tbase + 64 + cc * 16, R1);
                    ptx::tmem_ld16(tbase + 128 + cc * 16, R2);
                    ptx::tmem_ld16(tbase + 192 + cc * 16, R3);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int i = cc * 8 + q;
                        const int32_t C[8] = {(int32_t)R0[2 * q], (int32_t)R0[2 * q + 1], (int32_t)R1[2 * q],
                                              (int32_t)R1[2 * q + 1], (int32_t)R2[2 * q], (int32_t)R2[2 * q + 1],
                                              (int32_t)R3[2 * q], (int32_t)R3[2 * q + 1]};
                        const int32_t L0 = C[0] + 256 * C[1], L1 = C[2] + 256 * C[3];
                        const int32_t L2 = C[4] + 256 * C[5], L3 = C[6] + 256 * C[7];
                        // y = Σ_j 256^j C'_j + 2^63 = lo + 2^32 hi  (K_e^INT8·1 = −128 per row)
                        const long long lo = (long long)L0 + (long long)L1 * 65536ll;
                        const long long hi = (long long)L2 + (long long)L3 * 65536ll + (1ll << 31);
                        const double Y = __fma_rn(__ll2double_rn(hi), 0x1p32, __ll2double_rn(lo));  // RN(y)
                        const double f = __dmul_rn(c1, __dadd_rn(__dmul_rn(Y, sig), __dmul_rn(c2, S.fe[i][t])));
                        const bool dg = S.deg[t];
                        S.fe[i][t] = dg ? 0.0 : f;
                        if (MODE == MODE_DEBUG && dbg) {
                            if (p.dbg_C)
#pragma unroll
                                for (int j = 0; j < 8; ++j) p.dbg_C[dj * 192 + j * 24 + i] = C[j];
                            __int128 y = (__int128)hi * ((__int128)1 << 32) + (__int128)lo;
                            if (p.dbg_yhi) p.dbg_yhi[dj * 24 + i] = (long long)(y >> 64);
                            if (p.dbg_ylo) p.dbg_ylo[dj * 24 + i] = (long long)(unsigned long long)y;
                            if (p.dbg_fe) p.dbg_fe[dj * 24 + i] = dg ? 0.0 : f;
                        }
                    }
                }
                ptx::tc_fence_before();
            }
            __syncthreads();

            // ---- scatter in global element order into the two force planes ----
            if (t < NOWN) {
                const int nxl = t % TX, nyl = t / TX;
                const int e00 = nxl + EX * nyl, e10 = e00 + 1, e01 = e00 + EX, e11 = e01 + 1;
                if (L >= Z0) {  // bottom corners of layer L -> plane L
                    double *fa = &S.facc[L & 1][t * 3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double f = fa[c];
                        f = __dadd_rn(f, S.fe[3 * 2 + c][e00]);
                        f = __dadd_rn(f, S.fe[3 * 3 + c][e10]);
                        f = __dadd_rn(f, S.fe[3 * 1 + c][e01]);
                        f = __dadd_rn(f, S.fe[3 * 0 + c][e11]);
                        fa[c] = f;
                    }
                }
                if (L + 1 < Z1) {  // top corners of layer L -> plane L+1
                    double *fa = &S.facc[(L + 1) & 1][t * 3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double f = fa[c];
                        f = __dadd_rn(f, S.fe[3 * 6 + c][e00]);
                        f = __dadd_rn(f, S.fe[3 * 7 + c][e10]);
                        f = __dadd_rn(f, S.fe[3 * 5 + c][e01]);
                        f = __dadd_rn(f, S.fe[3 * 4 + c][e11]);
                        fa[c] = f;
                    }
                }
            }
            __syncthreads();
        }
        // ---- plane L is complete: update (or emit f) ----
        if (L >= Z0 && L <= p.nz) {
            if (t < NOWN) {
                const int nxl = t % TX, nyl = t / TX;
                const int64_t ix = X0 + nxl, iy = Y0 + nyl;
                double *fa = &S.facc[L & 1][t * 3];
                if (ix < NX1 && iy < NY1) {
                    const int64_t n = ix + NX1 * (iy + NY1 * L);
                    const double *up = &S.up[L & 1][((nyl + 1) * PX + (nxl + 1)) * 3];
                    if (MODE == MODE_STEP) {
                        const double wn = __ldg(p.w + n);
                        const uint8_t dm = p.dmask ? __ldg(p.dmask + n) : (uint8_t)0;
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const int64_t dof = 3 * n + c;
                            double F = 0.0;
                            for (int k = 0; k < p.nsrc; ++k)
                                if (p.src_dof[k] == dof) F = __dadd_rn(F, p.src_val[k]);
                            const double b = __dsub_rn(__dmul_rn(2.0, up[c]), p.uo[dof]);
                            double un = __fma_rn(wn, __dsub_rn(F, fa[c]), b);
                            if ((dm >> c) & 1) un = 0.0;
                            p.uo[dof] = un;
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 3; ++c) p.fout[3 * n + c] = fa[c];
                    }
                }
                fa[0] = fa[1] = fa[2] = 0.0;
            }
            __syncthreads();
        }
    }
    if constexpr (PATH == OVX_INT8) {
        ptx::tc_fence_after();
        if (warp == 0) ptx::tmem_dealloc<TMEM_COLS>(S.tmem);
    }
}

template <int PATH, int MODE>
cudaError_t launch_t(const StepParams &p, int64_t ctas, cudaStream_t st) {
    static bool attr = false;
    const int smem = (int)sizeof(typename PathCfg<PATH>::Smem);
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(step_kernel<PATH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    step_kernel<PATH, MODE><<<(unsigned)ctas, PathCfg<PATH>::T::NE, smem, st>>>(p);
    return cudaGetLastError();
}

template <int PATH>
cudaError_t launch_mode(int mode, const StepParams &p, int64_t ctas, cudaStream_t st) {
    if (mode == MODE_STEP) return launch_t<PATH, MODE_STEP>(p, ctas, st);
    if (mode == MODE_APPLY) return launch_t<PATH, MODE_APPLY>(p, ctas, st);
    return launch_t<PATH, MODE_DEBUG>(p, ctas, st);
}

__global__ void node_w_kernel(int64_t nx, int64_t ny, int64_t nz, const uint8_t *__restrict__ mat, double dt,
                              double *__restrict__ w) {
    const int64_t NX1 = nx + 1, NY1 = ny + 1, nn = NX1 * NY1 * (nz + 1);
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nn; n += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ix = n % NX1, iy = (n / NX1) % NY1, iz = n / (NX1 * NY1);
        double m = 0.0;
        // elements around the node in increasing element id: (ez, ey, ex) lexicographic
        for (int dz = -1; dz <= 0; ++dz)
            for (int dy = -1; dy <= 0; ++dy)
                for (int dx = -1; dx <= 0; ++dx) {
                    const int64_t ex = ix + dx, ey = iy + dy, ez = iz + dz;
                    if (ex < 0 || ex >= nx || ey < 0 || ey >= ny || ez < 0 || ez >= nz) continue;
                    m = __dadd_rn(m, c_mat[mat[ex + nx * (ey + ny * ez)]].rho_vol8);
                }
        w[n] = __ddiv_rn(__dmul_rn(dt, dt), m);
    }
}

__global__ void finite_kernel(const double *__restrict__ u, int64_t n, int *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(u[i])) *flag = 1;
}

constexpr int kZChunk = 64;

template <int PATH>
LaunchInfo info_t(int64_t nx, int64_t ny, int64_t nz) {
    using T = typename PathCfg<PATH>::T;
    LaunchInfo li;
    const int64_t tx = (nx + 1 + TX - 1) / TX, ty = (ny + 1 + T::TY - 1) / T::TY;
    const int64_t tz = (nz + 1 + kZChunk - 1) / kZChunk;
    li.ctas = tx * ty * tz;
    li.threads = T::NE;
    li.smem = (int)sizeof(typename PathCfg<PATH>::Smem);
    return li;
}

}  // namespace

cudaError_t upload_constants(const MatConst *mats, int nmat, const int8_t *k8, const double *kk, const double *kg,
                             cudaStream_t st) {
    cudaError_t e;
    if ((e = cudaMemcpyToSymbolAsync(c_mat, mats, sizeof(MatConst) * nmat, 0, cudaMemcpyHostToDevice, st))) return e;
    if ((e = cudaMemcpyToSymbolAsync(c_K8, k8, 1152, 0, cudaMemcpyHostToDevice, st))) return e;
    if ((e = cudaMemcpyToSymbolAsync(c_Kk, kk, 576 * 8, 0, cudaMemcpyHostToDevice, st))) return e;
    if ((e = cudaMemcpyToSymbolAsync(c_Kg, kg, 576 * 8, 0, cudaMemcpyHostToDevice, st))) return e;
    return cudaStreamSynchronize(st);
}

LaunchInfo step_launch_info(int path, int64_t nx, int64_t ny, int64_t nz) {
    if (path == OVX_INT8) return info_t<OVX_INT8>(nx, ny, nz);
    if (path == OVX_FP64) return info_t<OVX_FP64>(nx, ny, nz);
    return info_t<OVX_FP64_DENSE>(nx, ny, nz);
}

cudaError_t launch_step(int path, int mode, StepParams p, cudaStream_t st) {
    const int ty = path == OVX_INT8 ? Tile<EY_I8>::TY : Tile<EY_F64>::TY;
    p.tiles_x = (int)((p.nx + 1 + TX - 1) / TX);
    p.tiles_y = (int)((p.ny + 1 + ty - 1) / ty);
    p.zchunk = kZChunk;
    const int64_t tz = (p.nz + 1 + p.zchunk - 1) / p.zchunk;
    const int64_t ctas = (int64_t)p.tiles_x * p.tiles_y * tz;
    if (path == OVX_INT8) return launch_mode<OVX_INT8>(mode, p, ctas, st);
    if (path == OVX_FP64) return launch_mode<OVX_FP64>(mode, p, ctas, st);
    return launch_mode<OVX_FP64_DENSE>(mode, p, ctas, st);
}

cudaError_t launch_node_w(int64_t nx, int64_t ny, int64_t nz, const uint8_t *mat, double dt, double *w,
                          cudaStream_t st) {
    node_w_kernel<<<1184, 256, 0, st>>>(nx, ny, nz, mat, dt, w);
    return cudaGetLastError();
}

cudaError_t launch_finite_check(const double *u, int64_t n, int *flag, cudaStream_t st) {
    finite_kernel<<<1184, 256, 0, st>>>(u, n, flag);
    return cudaGetLastError();
}

}  // namespace ovx
