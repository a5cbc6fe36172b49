// step_i8x.cuh — fused time step of the INT8 tensor-core path (OVX_INT8), round-2 kernel; included
// by kernels.cu after step_i8w.cuh (whose tile geometry and conversion conventions it shares).
//
// Same arithmetic as step_i8w — the same exact integer y = K_D v per element output and the same
// node-sum order (reading U2), so bit-identical results — with fewer CUDA-core
// instructions per element:
//   * WORD layout of the A operand: the 64-bit image v' = v + 2^{7M} of each value goes to TMEM as
//     its two 32-bit words (array 0 = bytes 0-3, array 1 = bytes 4-7), K index = 4·value + byte, and
//     the resident B operand is −K_D ⊗ I_4 (N = 96 = 24 outputs × 4 byte positions), so the tensor
//     core separates the byte stages: D[4o + j] of array a is the stage-(4a + j) product of output o.
//     No byte permutes (step_i8w packs half-words with PRMT: ≈100 instructions per element), at
//     twice the (idle) tensor-pipe work.  The Eq. 9 diagonal fold (variant D) is 3 K-steps of the G
//     words against −128·I ⊗ I_4, the accumulator bias one K-step of 0xFF bytes against 127.
//   * s_e (Eq. 10) from per-ELEMENT quad maxima of each plane, formed once per element by M-tile 1 one
//     iteration before use (6-plane ring, planes prefetched three layers ahead).
//   * every shared-memory access at a per-thread 32-bit address computed once (rotating slot
//     addresses), the two-limb recombination with one wide multiply-add per limb.
// CTA = 32 × 8 elements per layer (one halo ring recomputed by the neighbour tiles) marching in z,
// 512 threads, two per element (warp w: M-tile mt = w/8, face half hf = (w/4)&1, TMEM lane quadrant
// w&3); the two M-tiles are skewed by half an iteration and share one TMEM A operand.  MODE_DEBUG is
// not compiled here (the debug records come from step_i8w).

#include <type_traits>

namespace x8 {
constexpr int NOUT = 96;                       // MMA N: 24 outputs × 4 byte positions
constexpr int KW = 48;                         // K words (4 bytes) per array: one per value
constexpr int BM_PITCH = (4 * KW / 16) * 128;  // main B: bytes per 8-row group (12 K-chunks of 16 B)
constexpr int BF_PITCH = (4 * 24 / 16) * 128;  // fold B: 96 K-bytes (the 24 G values)
constexpr int BB_PITCH = 2 * 128;              // bias B: 32 K-bytes
constexpr int BM_BYTES = 12 * BM_PITCH;        // 96 rows
constexpr int BF_BYTES = 12 * BF_PITCH;
constexpr int BB_BYTES = 12 * BB_PITCH;
constexpr int B_BYTES = BM_BYTES + BF_BYTES + BB_BYTES;
constexpr int A_ARR = 56;                      // TMEM columns per A array: 48 value words + 8 bias words
constexpr uint32_t A0 = 384;                   // A columns (both arrays, shared by the M-tiles)
constexpr uint32_t D_TILE = 192;               // D columns per M-tile: 2 arrays × 96
constexpr int32_t BIAS = 32 * 255 * 127;       // every D = −C + BIAS > 0 (max |C| = 255·1258)
constexpr uint32_t IDESC = ptx::idesc_i8(128, NOUT);
constexpr uint32_t IDESC_H = ptx::idesc_i8(128, 48);    // half-word layout (LAY 0)
}  // namespace x8

// The B operands in the canonical K-major core-matrix layout (8 rows × 16 B per core matrix), built
// once per constant upload from c_K8:
//   main (96 rows × 192 K-bytes): row n = 4o + j, K-byte kb = 4k + j' → −K_e^INT8[o][k] if j == j';
//   fold (96 × 96):  G value g = kb/4 (value 24 + g): −128 if g == o and j == j' (Eq. 9 diagonal, D);
//   bias (96 × 32):  127 everywhere (against the A bias words 0xFFFFFFFF).
__device__ uint4 g_bimgx[x8::B_BYTES / 16];
__global__ void i8x_bimg_kernel() {
    using namespace x8;
    uint8_t *Bm = reinterpret_cast<uint8_t *>(g_bimgx), *Bf = Bm + BM_BYTES, *Bb = Bf + BF_BYTES;
    auto off = [](int n, int kb, int pitch) { return (n >> 3) * pitch + (kb >> 4) * 128 + (n & 7) * 16 + (kb & 15); };
    for (int idx = threadIdx.x; idx < 96 * 192; idx += blockDim.x) {
        const int n = idx / 192, kb = idx - n * 192;
        Bm[off(n, kb, BM_PITCH)] = ((kb & 3) == (n & 3)) ? (uint8_t)(-(int)c_K8[(n >> 2) * 48 + (kb >> 2)]) : (uint8_t)0;
    }
    for (int idx = threadIdx.x; idx < 96 * 96; idx += blockDim.x) {
        const int n = idx / 96, kb = idx - n * 96;
        Bf[off(n, kb, BF_PITCH)] = ((kb & 3) == (n & 3) && (kb >> 2) == (n >> 2)) ? (uint8_t)0x80 : (uint8_t)0;
    }
    for (int idx = threadIdx.x; idx < 96 * 32; idx += blockDim.x) {
        const int n = idx / 32, kb = idx - n * 32;
        Bb[off(n, kb, BB_PITCH)] = (uint8_t)127;
    }
}

namespace sm {   // shared-memory access at 32-bit shared-window addresses
__device__ __forceinline__ double ld_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned long long ld_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void st_f64(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ void st_u64(uint32_t a, unsigned long long v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v));
}
__device__ __forceinline__ void st_u8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ uint32_t ld_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
}  // namespace sm

// registers -> TMEM, 8 consecutive columns of this warp's lane quadrant
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// −(Σ_{j<4} 256^j C_j) from the four biased stage accumulators D_j = −C_j + BIAS of one limb: the
// limb L = p0 + 2^16·p1 < 2^45 (p0 = D0 + 256·D1, p1 = D2 + 256·D3 < 2^29) is assembled under the
// 1.5·2^52 magic exponent as two words (low word with carry-out, high word = p1 >> 16 + carry +
// 0x43380000: two shifted adds, no 64-bit multiply), and one subtraction removes the magic and the
// bias exactly.
template <int32_t BIASV>
__device__ __forceinline__ double limb_x(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3) {
    constexpr double MAGIC = 0x1.8p52 + (double)BIASV * 16843009.0;
    const uint32_t p0 = d0 + 256u * d1, p1 = d2 + 256u * d3;
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0x43380000;" : "=r"(lo), "=r"(hi) : "r"(p0), "r"(p1 << 16),
        "r"(p1 >> 16));
    return __hiloint2double((int)hi, (int)lo) - MAGIC;
}

// One slot of the 6-plane ring: everything the kernel keeps per node plane / element layer, so one
// rotating byte offset addresses all of it.
struct PlaneSlotX {
    double up[3][I8W::NODES];                          // node values, component-major
    unsigned long long nmax[I8W::NODES];               // max_c |u_c| per node (bit patterns)
    unsigned long long qmax[I8W::NE];                  // max over the 4 nodes of each tile element
    uint8_t mid[I8W::NE];                              // material id of each tile element (this layer)
};
struct SmemI8X {
    alignas(128) uint8_t B[x8::B_BYTES];               // LAY 0 uses the first kBImgVec·16 bytes
    PlaneSlotX pl[6];
    double ysum[3][2][3][I8W::EY][I8W::EX];            // [layer slot][face][c] x-pair P of the +y corners
    double tf[2][3][I8W::NE];                          // [layer parity][c][tile node] top-face sums T
    double2 mc[kMaxMat];                               // (cG, c1) per material
    uint64_t mbar[2];                                  // MMAs of M-tile mt complete (all arrays)
    uint64_t mbar_lo[2];                               // LAY 1: array 0 (the low limb) complete
    uint32_t tmem;
};

// LAY 1: the word layout above; LAY 0: the half-word layout of step_i8w (4 arrays of byte pairs,
// B = −K_e^INT8 ⊗ I_2, N = 48; PRMT packing) — kept to measure the two against each other.
template <int MODE, int M, bool DAMP, bool SLAB, int LAY>
__global__ void __launch_bounds__(512, 1) step_i8x(const StepParams p) {
    using namespace x8;
    using C = I8W;
    constexpr int EX = C::EX, PX = C::PX, NODES = C::NODES, NE = C::NE, NT = C::NT;
    constexpr int NAW = (7 * M + 1 + 31) / 32;           // word arrays of v' = v + 2^{7M}: 2 (M = 8, 6), 1 (M = 4)
    constexpr double SCALE = (double)(1ull << (7 * M));
    constexpr double ISCALE = 1.0 / SCALE;
    constexpr unsigned long long AOFF = 1ull << (7 * M);
    // plane / ring strides in bytes
    constexpr uint32_t PLANE_B = (uint32_t)sizeof(PlaneSlotX), COMP_B = NODES * 8;
    constexpr uint32_t YS_SLOT_B = 2 * 3 * C::EY * EX * 8, YS_FACE_B = 3 * C::EY * EX * 8, YS_C_B = C::EY * EX * 8;
    constexpr uint32_t TF_PAR_B = 3 * NE * 8, TF_C_B = NE * 8;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SmemI8X &S = *reinterpret_cast<SmemI8X *>(smem_raw);
    const int t = threadIdx.x;
    const int lane = t & 31;
    const int wu = __shfl_sync(0xffffffffu, t >> 5, 0);
    const int mt = wu >> 3, hf = (wu >> 2) & 1, qd = wu & 3;

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
    const int Lend = min(nz, Z1);                        // layers [Lfirst, Lend) are computed

    const int lx = lane, ly = 4 * mt + qd;              // this thread's tile element
    const int64_t ex = X0 - 1 + lx, ey = Y0 - 1 + ly;
    const bool ein = (ex >= 0 && ex < p.nx && ey >= 0 && ey < p.ny);
    const int elem = lx + EX * ly;
    const int64_t mstride = p.nx * p.ny;
    const bool tnode = lx >= 1 && ly >= 1;               // node (lx, ly) is in the tile's owned range
    const bool own = tnode && ex < NX1 && ey < NY1;
    const int64_t ucol = own ? ex + NX1 * ey : 0;
    const bool upd_role = own && hf == 0;

    auto load_in = [&](int64_t o) {
        const double uu = __ldg(p.u + o);
        if constexpr (DAMP) {
            const double pp = __ldg(p.uo + o);
            return __dadd_rn(uu, __dmul_rn(p.cb, __dsub_rn(uu, pp)));
        } else {
            return uu;
        }
    };
    // plane loader role: node li of the smem plane (the last NODES threads)
    const int li = t - (NT - NODES);
    const bool lrole = li >= 0;
    const int lpx = lrole ? li % PX : 0, lpy = lrole ? li / PX : 0;
    const bool ldn = lrole && X0 - 1 + lpx >= 0 && X0 - 1 + lpx < NX1 && Y0 - 1 + lpy >= 0 && Y0 - 1 + lpy < NY1;
    const int64_t ldoff = ldn ? 3 * ((X0 - 1 + lpx) + NX1 * (Y0 - 1 + lpy)) : 0;
    // quad-max role (M-tile 1 threads): tile element qe = t - 256
    const int qe = t - 256;
    const int qn = (qe >= 0) ? (qe % EX) + PX * (qe / EX) : 0;

    bool has_src = false, has_rec = false;
    if (MODE == MODE_STEP && hf == 0) {
        for (int k = 0; k < p.nsrc; ++k) {
            const int64_t n = p.src_dof[k] / 3;
            const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
            has_src |= (ix >= X0 && ix < X0 + C::TX && iy >= Y0 && iy < Y0 + C::TY);
        }
        if (p.it >= 0 && p.it < p.rec_nt)
            for (int k = 0; k < p.nrec; ++k) {
                const int64_t n = p.rec_node[k];
                const int64_t ix = n % NX1, iy = (n / NX1) % NY1;
                has_rec |= (ix >= X0 && ix < X0 + C::TX && iy >= Y0 && iy < Y0 + C::TY);
            }
    }

    // ---- one-time setup ----
    if constexpr (LAY == 1)
        for (int i = t; i < x8::B_BYTES / 16; i += NT) reinterpret_cast<uint4 *>(S.B)[i] = g_bimgx[i];
    else
        for (int i = t; i < kBImgVec; i += NT) reinterpret_cast<uint4 *>(S.B)[i] = g_bimg[i];
    if (wu == 0) ptx::tmem_alloc<512>(&S.tmem);
    if (t == 0) {
        ptx::mbar_init(&S.mbar[0], 1);
        ptx::mbar_init(&S.mbar[1], 1);
        ptx::mbar_init(&S.mbar_lo[0], 1);
        ptx::mbar_init(&S.mbar_lo[1], 1);
    }
    for (int i = t; i < 2 * 3 * NE; i += NT) (&S.tf[0][0][0])[i] = 0.0;
    for (int i = t; i < p.nmat + 1; i += NT) {
        const int id = i < p.nmat ? i : kZeroMat;
        S.mc[id] = make_double2(p.mc[id].cG, p.mc[id].c1);
    }
    const uint8_t *matp = p.mat + (ein ? ex + p.nx * ey : 0);
    if (hf == 0)
        for (int j = 0; j < 2; ++j) {   // material ids of layers Lfirst, Lfirst + 1
            const int iz = Lfirst + j;
            S.pl[(iz + 12) % 6].mid[elem] = (uint8_t)((ein && iz < nz) ? (int)__ldg(matp + mstride * iz) : kZeroMat);
        }
    for (int j = 0; j < 3; ++j) {   // planes Lfirst .. Lfirst + 2
        const int iz = Lfirst + j;
        if (lrole) {
            double v3[3] = {0.0, 0.0, 0.0};
            if (ldn && iz <= nz)
#pragma unroll
                for (int c = 0; c < 3; ++c) v3[c] = load_in(3 * PSTRIDE * iz + ldoff + c);
            unsigned long long m = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                S.pl[(iz + 12) % 6].up[c][li] = v3[c];
                const unsigned long long b = abs_bits(v3[c]);
                m = b > m ? b : m;
            }
            S.pl[(iz + 12) % 6].nmax[li] = m;
        }
    }
    ptx::fence_proxy_async_smem();   // B (generic-proxy stores) is read by the tensor core
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (qe >= 0)   // quad maxima of planes Lfirst, Lfirst + 1
        for (int j = 0; j < 2; ++j) {
            PlaneSlotX &P = S.pl[(Lfirst + j + 12) % 6];
            P.qmax[qe] = max(max(P.nmax[qn], P.nmax[qn + 1]), max(P.nmax[qn + PX], P.nmax[qn + PX + 1]));
        }
    if (wu < 4) {   // the bias words of both A arrays (columns 48..55): 0xFFFFFFFF, written once
        const uint32_t ones[8] = {~0u, ~0u, ~0u, ~0u, ~0u, ~0u, ~0u, ~0u};
        const uint32_t tb = S.tmem + ((uint32_t)(qd * 32) << 16) + A0;
        if constexpr (LAY == 1) {
            tmem_st8(tb + 48, ones);
            if (NAW > 1) tmem_st8(tb + A_ARR + 48, ones);
        } else {   // chunk 6 (16 bytes) of each half-word array
#pragma unroll
            for (int pa = 0; pa < 4; ++pa) ptx::tmem_st4(tb + pa * TA_A_ARR + 24, ~0u, ~0u, ~0u, ~0u);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
    }
    __syncthreads();
    ptx::tc_fence_after();

    // ---- per-thread constants of the layer loop ----
    const uint32_t tmem = S.tmem;
    const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + A0;                      // this row's A words
    const uint32_t tdl = tmem + ((uint32_t)(qd * 32) << 16) + mt * D_TILE + (LAY == 1 ? 48 : 24) * hf;  // D, this face
    uint64_t *const mybar = &S.mbar[mt];
    uint64_t *const mybar_lo = &S.mbar_lo[mt];
    uint64_t *const xbar = &S.mbar[1 - mt];
    const int n0 = ly * PX + lx;                         // node (lx, ly) in a smem plane
    // per-thread addresses in ring slot 0 (+ the slot's byte offset, a multiple of PLANE_B)
    const uint32_t a_up = ptx::smem_u32(&S.pl[0].up[0][n0]);
    const uint32_t a_qmax = ptx::smem_u32(&S.pl[0].qmax[elem]);
    const uint32_t a_mid = ptx::smem_u32(&S.pl[0].mid[elem]);
    const uint32_t a_ys_w = ptx::smem_u32(&S.ysum[0][0][0][0][0]) + hf * YS_FACE_B + 8u * elem;   // + slot
    const uint32_t a_ys_r = a_ys_w - 8u * EX;                             // row ly - 1
    const uint32_t a_tf = ptx::smem_u32(&S.tf[0][0][0]) + 8u * elem;      // + parity·TF_PAR_B
    const uint32_t a_mc = ptx::smem_u32(&S.mc[0]);
    const uint32_t a_ld = ptx::smem_u32(&S.pl[0].up[0][lrole ? li : 0]);
    const uint32_t a_nm = ptx::smem_u32(&S.pl[0].nmax[lrole ? li : 0]);
    const uint32_t a_qn = ptx::smem_u32(&S.pl[0].nmax[qn]);
    const uint32_t a_qw = ptx::smem_u32(&S.pl[0].qmax[qe >= 0 ? qe : 0]);
    uint32_t phase = 0;
    uint32_t xpar = mt == 0 ? 1u : 0u;
    double upv[3] = {0.0, 0.0, 0.0}, wn = 0.0, uv[3] = {0.0, 0.0, 0.0};
    uint8_t dm = 0;
    double plo[3] = {0.0, 0.0, 0.0};
    double es = 0.0;
    bool edeg = false;
    uint32_t emc = a_mc;                                 // (cG, c1) of the converted element

    // one chunk of 8 values: scaled F2I (Eqs. 10-12), v' = v + 2^{7M}, the two words to TMEM columns
    // 8·ch (array 0) and A_ARR + 8·ch (array 1)
    auto chunk = [&](auto fastc, const double (&ue)[16], int j0, bool gpart, int ch, double cG, double R, double r,
                     bool deg, bool first) {
        constexpr bool FAST = decltype(fastc)::value;
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double ub = gpart ? __dmul_rn(cG, ue[j0 + q]) : ue[j0 + q];
            long long v;
            if constexpr (FAST)   // one DMUL + one F2I per value (R = RN(1/s)·2^{7M}, or 0 for a zero image)
                v = __double2ll_rz(__dmul_rn(ub, R));
            else                  // tiny-normal or non-finite s: the two roundings of Eq. 10 as written
                v = deg ? 0ll : __double2ll_rz(__dmul_rn(__dmul_rn(ub, r), SCALE));
            if constexpr (7 * M >= 32) {
                lo[q] = (uint32_t)(unsigned long long)v;
                hi[q] = (uint32_t)((unsigned long long)v >> 32) + (uint32_t)(AOFF >> 32);
            } else {
                lo[q] = (uint32_t)(unsigned long long)v + (uint32_t)AOFF;
                hi[q] = 0;
            }
        }
        if (first) {   // the shared TMEM A: the other M-tile's MMAs must have read it
            ptx::mbar_wait(xbar, xpar);
            ptx::tc_fence_after();
        }
        if constexpr (LAY == 1) {
            tmem_st8(ta + 8 * ch, lo);
            if (NAW > 1) tmem_st8(ta + A_ARR + 8 * ch, hi);
        } else {   // half-word arrays pa: bytes (2pa, 2pa+1) of values q, q+1 per 32-bit word
            constexpr int NB = (7 * M + 1 + 7) / 8, NA = (NB + 1) / 2;
#pragma unroll
            for (int pa = 0; pa < NA; ++pa) {
                const uint32_t *src = pa < 2 ? lo : hi;
                const uint32_t sel = (pa & 1) ? 0x7632u : 0x5410u;
                ptx::tmem_st4(ta + pa * TA_A_ARR + 4 * ch, __byte_perm(src[0], src[1], sel), __byte_perm(src[2], src[3], sel),
                              __byte_perm(src[4], src[5], sel), __byte_perm(src[6], src[7], sel));
            }
        }
    };

    // ---- conversion of layer L (this thread's 24 of the 48 values) and the MMA hand-off ----
    auto convert = [&](uint32_t oL, uint32_t oL1) {   // slot byte offsets of planes L, L+1
        const double amax = __longlong_as_double((long long)max(sm::ld_u64(a_qmax + oL), sm::ld_u64(a_qmax + oL1)));
        const uint32_t mcur = sm::ld_u8(a_mid + oL);
        emc = a_mc + 16u * mcur;
        const double cG = sm::ld_f64(emc);
        const double s = fmax(amax, __dmul_rn(cG, amax));   // max_i |RN(cG u_i)| = RN(cG max_i |u_i|)
        const bool deg = !ein || !(s >= 0x1p-1022) || !(s <= 0x1.fffffffffffffp1023);
        const bool vzero = !ein || !(s >= 0x1p-1022);
        const bool fast = (s <= 0x1.fffffffffffffp1023) && (vzero || s >= 0x1p-960);
        const double r = 1.0 / s;                                  // RN(1/s_e), reading Q7
        const double R = vzero ? 0.0 : __dmul_rn(r, SCALE);        // exact power-of-two scaling
        // ū values 8hf .. 8hf+15 (local node order of reading Q1; nodes 4-7 in plane L+1)
        double ue[16];
        {
            constexpr int off[4] = {0, 1, PX + 1, PX};
            const uint32_t lo = a_up + oL, hi = a_up + oL1;
            if (hf == 0) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int k = j, a = k / 3, c = k - 3 * a;
                    ue[j] = sm::ld_f64((a < 4 ? lo : hi) + c * COMP_B + 8 * off[a & 3]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int k = 8 + j, a = k / 3, c = k - 3 * a;
                    ue[j] = sm::ld_f64((a < 4 ? lo : hi) + c * COMP_B + 8 * off[a & 3]);
                }
            }
        }
        // half 0: chunks 0, 1 (ū 0-15) and 3 (G 0-7); half 1: chunk 2 (ū 16-23), 4, 5 (G 8-23)
        auto chunks = [&](auto fc) {
            if (hf == 0) {
                chunk(fc, ue, 0, false, 0, cG, R, r, deg, true);
                chunk(fc, ue, 8, false, 1, cG, R, r, deg, false);
                chunk(fc, ue, 0, true, 3, cG, R, r, deg, false);
            } else {
                chunk(fc, ue, 8, false, 2, cG, R, r, deg, true);
                chunk(fc, ue, 0, true, 4, cG, R, r, deg, false);
                chunk(fc, ue, 8, true, 5, cG, R, r, deg, false);
            }
        };
        if (__all_sync(0xffffffffu, fast)) chunks(std::true_type{});
        else chunks(std::false_type{});
        xpar ^= 1u;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        es = s;
        edeg = deg;
        asm volatile("bar.sync %0, 256;" ::"r"(1 + mt) : "memory");   // the 8 warps of this M-tile
        if ((wu & 7) == 0) {
            if (ptx::elect_one()) {
                ptx::tc_fence_after();
                const uint32_t bm = ptx::smem_u32(&S.B[0]), bf = bm + BM_BYTES, bb = bf + BF_BYTES;
                if constexpr (LAY == 1) {
#pragma unroll
                    for (int a = 0; a < NAW; ++a) {
                        const uint32_t at = tmem + A0 + a * A_ARR;
                        const uint32_t d = tmem + mt * D_TILE + a * NOUT;
#pragma unroll
                        for (int ks = 0; ks < 6; ++ks)
                            ptx::mma_i8_ts(d, at + 8 * ks, ptx::smem_desc(bm + ks * 256, 128, BM_PITCH), x8::IDESC,
                                           ks > 0 ? 1u : 0u);
#ifndef OVX_ABL_NOFOLD   // (timing ablation only: results wrong without the fold)
#pragma unroll
                        for (int ks = 0; ks < 3; ++ks)   // G words (values 24-47) against −128·I ⊗ I_4
                            ptx::mma_i8_ts(d, at + 24 + 8 * ks, ptx::smem_desc(bf + ks * 256, 128, BF_PITCH), x8::IDESC, 1u);
#endif
                        ptx::mma_i8_ts(d, at + 48, ptx::smem_desc(bb, 128, BB_PITCH), x8::IDESC, 1u);   // bias
                        if (a == 0 && NAW > 1) ptx::mma_commit(mybar_lo);   // the low limb can start
                    }
                } else {
                    constexpr int NB = (7 * M + 1 + 7) / 8, NA = (NB + 1) / 2;
                    const uint32_t b0 = bm, bi0 = bm + 6 * B1_PITCH, bi1 = bi0 + 6 * BI_PITCH;
#pragma unroll
                    for (int pa = 0; pa < NA; ++pa) {
                        const uint32_t at = tmem + TA_A0 + pa * TA_A_ARR;
                        const uint32_t d = tmem + mt * TA_D_TILE + pa * TA_D_ARR;
#pragma unroll
                        for (int ks = 0; ks < 3; ++ks)
                            ptx::mma_i8_ts(d, at + 8 * ks, ptx::smem_desc(b0 + ks * 256, 128, B1_PITCH), x8::IDESC_H,
                                           ks > 0 ? 1u : 0u);
                        ptx::mma_i8_ts(d, at + 12, ptx::smem_desc(bi0, 128, BI_PITCH), x8::IDESC_H, 1u);
                        ptx::mma_i8_ts(d, at + 20, ptx::smem_desc(bi1, 128, BI_PITCH), x8::IDESC_H, 1u);
                    }
                }
                ptx::mma_commit(mybar);
            }
            __syncwarp();
        }
    };

    // ---- epilogue of the layer whose MMAs were issued last: the 4 corner nodes of this face ----
    auto epilogue = [&](uint32_t oys) {                 // ysum slot byte offset
        const double c1 = sm::ld_f64(emc + 8);
        ptx::mbar_wait_sleep((LAY == 1 && NAW > 1) ? mybar_lo : mybar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
        const double alpha = edeg ? 0.0 : -__dmul_rn(c1, __dmul_rn(es, ISCALE));
        double fc[12];
        if constexpr (LAY == 1) {
            // low limbs (array 0) as soon as its MMAs complete, then the high limbs
            double dl[12];
#pragma unroll
            for (int rr = 0; rr < 3; ++rr) {            // outputs 4rr .. 4rr+3 of this face
                uint32_t R0[16];
                tmem_ld16(tdl + 16 * rr, R0);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 4; ++q) dl[4 * rr + q] = limb_x<BIAS>(R0[4 * q], R0[4 * q + 1], R0[4 * q + 2], R0[4 * q + 3]);
            }
            if constexpr (NAW > 1) {
                ptx::mbar_wait_sleep(mybar, phase ^ 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int rr = 0; rr < 3; ++rr) {
                    uint32_t R1[16];
                    tmem_ld16(tdl + NOUT + 16 * rr, R1);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double dhi = limb_x<BIAS>(R1[4 * q], R1[4 * q + 1], R1[4 * q + 2], R1[4 * q + 3]);
                        fc[4 * rr + q] = __dmul_rn(alpha, __fma_rn(dhi, 0x1p32, dl[4 * rr + q]));   // RN(c1s·RN(y))
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 12; ++j) fc[j] = __dmul_rn(alpha, dl[j]);
            }
        } else {
            constexpr int NB = (7 * M + 1 + 7) / 8, NA = (NB + 1) / 2;
#pragma unroll
            for (int rr = 0; rr < 3; ++rr) {
                uint32_t R0[8], R1[8], R2[8] = {}, R3[8] = {};
                ptx::tmem_ld8(tdl + 0 + rr * 8, R0);
                ptx::tmem_ld8(tdl + TA_D_ARR + rr * 8, R1);
                if (NA > 2) ptx::tmem_ld8(tdl + 2 * TA_D_ARR + rr * 8, R2);
                if (NA > 3) ptx::tmem_ld8(tdl + 3 * TA_D_ARR + rr * 8, R3);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t c4 = NA > 2 ? R2[2 * q] : (uint32_t)I8_BIAS, c5 = NA > 2 ? R2[2 * q + 1] : (uint32_t)I8_BIAS;
                    const uint32_t c6 = NA > 3 ? R3[2 * q] : (uint32_t)I8_BIAS, c7 = NA > 3 ? R3[2 * q + 1] : (uint32_t)I8_BIAS;
                    const double dlo = limb_x<I8_BIAS>(R0[2 * q], R0[2 * q + 1], R1[2 * q], R1[2 * q + 1]);
                    const double dhi = NA > 2 ? limb_x<I8_BIAS>(c4, c5, c6, c7) : 0.0;
                    const double Y = NA > 2 ? __fma_rn(dhi, 0x1p32, dlo) : dlo;
                    fc[4 * rr + q] = __dmul_rn(alpha, Y);
                }
            }
        }
        ptx::tc_fence_before();
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double pm = __shfl_up_sync(0xffffffffu, fc[3 * 1 + c], 1);   // (+x,-y) of lx-1
            const double pp = __shfl_up_sync(0xffffffffu, fc[3 * 2 + c], 1);   // (+x,+y) of lx-1
            plo[c] = __dadd_rn(fc[3 * 0 + c], pm);      // lane 0 (lx = 0) is no tile node: unused
            sm::st_f64(a_ys_w + oys + c * YS_C_B, __dadd_rn(fc[3 * 3 + c], pp));
        }
    };

    // ---- post-phase of plane Lp (face sums of layer Lp, f_n = T + B, update) ----
    auto post_phase = [&](int Lp, uint32_t oys, uint32_t oup, bool faces_ok, bool plane_done) {
        if (!tnode) return;
        const uint32_t tfr = a_tf + ((Lp - 1) & 1) * TF_PAR_B, tfw = a_tf + (Lp & 1) * TF_PAR_B;
        double ysv[3], tfv[3], ucv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            ysv[c] = sm::ld_f64(a_ys_r + oys + c * YS_C_B);
            tfv[c] = sm::ld_f64(tfr + c * TF_C_B);
            ucv[c] = sm::ld_f64(a_up + oup + c * COMP_B);
        }
        double face[3] = {0.0, 0.0, 0.0};
        if (faces_ok) {
#pragma unroll
            for (int c = 0; c < 3; ++c) face[c] = __dadd_rn(plo[c], ysv[c]);
        }
        if (hf == 1) {
#pragma unroll
            for (int c = 0; c < 3; ++c) sm::st_f64(tfw + c * TF_C_B, face[c]);
        } else if (own && plane_done) {
            const int64_t un_id = ucol + PSTRIDE * Lp;
            if (SLAB && (p.slab_flags & 1) && Lp == 0) {
#pragma unroll
                for (int c = 0; c < 3; ++c) p.iface_bot_b[3 * ucol + c] = face[c];
            } else {
                double f[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) f[c] = __dadd_rn(tfv[c], face[c]);
                if (SLAB && (p.slab_flags & 2) && Lp == nz) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) p.iface_top_A[3 * ucol + c] = f[c];
                } else if (MODE == MODE_STEP) {
                    double *dst = (DAMP ? p.un : p.uo) + 3 * un_id;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double F = 0.0;
                        if (has_src)
                            for (int k = 0; k < p.nsrc; ++k)
                                if (p.src_dof[k] == 3 * un_id + c) F = __dadd_rn(F, p.src_val[k]);
                        const double uc = DAMP ? uv[c] : ucv[c];
                        double b = __dsub_rn(__dmul_rn(2.0, uc), upv[c]);
                        if constexpr (DAMP) b = __dsub_rn(b, __dmul_rn(p.ca, __dsub_rn(uc, upv[c])));
                        double un = __fma_rn(wn, __dsub_rn(F, f[c]), b);
                        if ((dm >> c) & 1) un = 0.0;
                        dst[c] = un;
                        if (has_rec)
                            for (int k = 0; k < p.nrec; ++k)
                                if (p.rec_node[k] == un_id) p.traces[(3 * k + c) * p.rec_nt + p.it] = un;
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 3; ++c) p.fout[3 * un_id + c] = f[c];
                }
            }
        }
    };

    // ring slots of planes L-2 .. L+3 as byte offsets into the plane ring (slot·PLANE_B), and of
    // layers L-2 .. L in the face-sum ring (slot·YS_SLOT_B)
    auto pslot = [&](int z) { return (uint32_t)((z + 12) % 6); };
    uint32_t o0 = pslot(Z0 - 3) * PLANE_B, o1 = pslot(Z0 - 2) * PLANE_B, o2 = pslot(Z0 - 1) * PLANE_B,
             o3 = pslot(Z0) * PLANE_B, o4 = pslot(Z0 + 1) * PLANE_B, o5 = pslot(Z0 + 2) * PLANE_B;
    uint32_t y0 = (uint32_t)((Z0 - 3 + 12) % 3) * YS_SLOT_B, y1 = (uint32_t)((Z0 - 2 + 12) % 3) * YS_SLOT_B,
             y2 = (uint32_t)((Z0 - 1 + 12) % 3) * YS_SLOT_B;
    // running offsets: plane L+3 of u, material of layer L+2, the node updated next (plane L - mt)
    int64_t ro_plane = 3 * PSTRIDE * (int64_t)(Z0 + 2) + ldoff;
    const uint8_t *ro_mat = matp + mstride * (int64_t)(Z0 + 1);
    int64_t ro_node = ucol + PSTRIDE * (int64_t)(Z0 - 1 - mt);

    // half-iterations h = 2L (even: prefetch; M-tile 0 converts layer L, M-tile 1 finishes layer L-1)
    // and 2L+1 (odd: M-tile 0 finishes layer L, M-tile 1 converts layer L; park; one CTA barrier).
    // One copy of each phase body, selected per warp (keeps the instruction footprint small).
    double pfv[3] = {0.0, 0.0, 0.0};
    bool pf = false, mf = false;
    int mfar = kZeroMat;
    double upv_n[3] = {0.0, 0.0, 0.0}, uv_n[3] = {0.0, 0.0, 0.0}, wn_n = 0.0;
    uint8_t dm_n = 0;
    for (int h = 2 * (Z0 - 1); h <= 2 * (Z1 + 1) + 1; ++h) {
        const int L = h >> 1;
        const bool odd = h & 1;
        // byte offsets: planes L-2 = o0, L-1 = o1, L = o2, L+1 = o3, L+2 = o4, L+3 = o5
        if (!odd) {
            pf = (L + 3 > Lfirst + 2) && (L + 3 <= Z1) && (L + 3 <= nz);   // plane L+3 needed
            if (pf && ldn) {
#pragma unroll
                for (int c = 0; c < 3; ++c) pfv[c] = load_in(ro_plane + c);
            }
            mf = (L + 2 < Lend) && (L >= Lfirst);                           // layer L+2 computed
            mfar = (mf && ein) ? (int)__ldg(ro_mat) : kZeroMat;
            const int Pn = L - mt;                    // plane this thread updates in the next iteration
            if (MODE == MODE_STEP && upd_role && Pn >= Z0 && Pn <= nz && Pn < Z1) {
                upv_n[0] = p.uo[3 * ro_node];
                upv_n[1] = p.uo[3 * ro_node + 1];
                upv_n[2] = p.uo[3 * ro_node + 2];
                if constexpr (DAMP) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) uv_n[c] = __ldg(p.u + 3 * ro_node + c);
                }
                wn_n = __ldg(p.w + ro_node);
                dm_n = p.dmask ? __ldg(p.dmask + ro_node) : (uint8_t)0;
            }
        }
        if (odd == (mt == 1)) {
            if (L >= Lfirst && L < Lend) convert(o2, o3);
        } else {
            const int Lp = L - 1 - mt;                // M-tile 1 lags by half an iteration
            post_phase(Lp, mt ? y0 : y1, mt ? o0 : o1, Lp >= Lfirst && Lp < Lend, Lp >= Z0 && Lp <= nz && Lp < Z1);
            if (Lp + 1 >= Lfirst && Lp + 1 < Lend) epilogue(mt ? y1 : y2);
        }
        if (odd) {
            // quad maxima of plane L+2 (its node maxima were parked at the end of the previous iteration)
            if (qe >= 0 && L + 2 <= Z1 && L + 2 <= nz) {
                const uint32_t nb = a_qn + o4;
                const unsigned long long m0 = sm::ld_u64(nb), m1 = sm::ld_u64(nb + 8), m2 = sm::ld_u64(nb + 8 * PX),
                                         m3 = sm::ld_u64(nb + 8 * PX + 8);
                sm::st_u64(a_qw + o4, max(max(m0, m1), max(m2, m3)));
            }
            // park plane L+3 into its slot (that of plane L-3, no longer read)
            if (pf && lrole) {
                unsigned long long m = 0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    sm::st_f64(a_ld + o5 + c * COMP_B, pfv[c]);
                    const unsigned long long b = abs_bits(pfv[c]);
                    m = b > m ? b : m;
                }
                sm::st_u64(a_nm + o5, m);
            }
            if (hf == 0 && mf) sm::st_u8(a_mid + o4, (uint32_t)mfar);
            upv[0] = upv_n[0]; upv[1] = upv_n[1]; upv[2] = upv_n[2];
            uv[0] = uv_n[0]; uv[1] = uv_n[1]; uv[2] = uv_n[2];
            wn = wn_n;
            dm = dm_n;
            upv_n[0] = upv_n[1] = upv_n[2] = 0.0;
            wn_n = 0.0;
            dm_n = 0;
            ro_plane += 3 * PSTRIDE;
            ro_mat += mstride;
            ro_node += PSTRIDE;
            {
                const uint32_t tt = o0;
                o0 = o1; o1 = o2; o2 = o3; o3 = o4; o4 = o5; o5 = tt;
                const uint32_t t3 = y0;
                y0 = y1; y1 = y2; y2 = t3;
            }
            __syncthreads();
        }
    }
    ptx::tc_fence_after();
    if (wu == 0) ptx::tmem_dealloc<512>(S.tmem);
}
