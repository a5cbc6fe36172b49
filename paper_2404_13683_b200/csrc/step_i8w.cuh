// step_i8w.cuh — fused time step of the INT8 tensor-core path (OVX_INT8); included by kernels.cu.
//
// CTA = 32 × 8 elements per layer (one halo ring recomputed by the neighbour tiles), marching in
// z over a chunk of node planes; 512 threads, two per element.  The TMEM budget (D of both M-tiles,
// 2 × 192 columns, plus the shared A operand, 112: all 512 allocated) and the register file allow
// one CTA per SM, so each element's work is split across two threads to double the resident warps:
//   * warp w: M-tile mt = w/8, half hf = (w/4)&1, TMEM lane quadrant q = w&3; element row
//     32q + lane of M-tile mt = tile element (lx = lane, ly = 4mt + q);
//   * conversion (Eqs. 10-16): s_e = max|ū_e| from per-node maxima |u| kept with each
//     smem u plane; half 0 writes A chunks {0,1,3} (ū values 0-15 and the G copy of 0-7), half 1
//     chunks {2,4,5}, with tcgen05.st into the TMEM A operand (TA; OVX_I8_KERNEL=smem: shared
//     memory); one elected lane per M-tile issues the tcgen05.mma.kind::i8 chain
//     (4 arrays × [3 K-steps against −K_e^INT8 ⊗ I_2 + 2 K-steps of the G bytes against
//     −128·I ⊗ I_2] = Eq. 17 with the Eq. 9 diagonal folded in, variant D);
//   * epilogue: half hf reads the accumulators of outputs 12hf..12hf+11 = the 4 corner nodes of
//     its face (hf 0 bottom, hf 1 top), exact two-limb recombination, f = RN(c1 s 2^-7M)·RN(y);
//   * node sums in the order of reading U2 without staging element forces: the x-pair
//     P = f(ix,iy)[(-x,-y)] + f(ix-1,iy)[(+x,-y)] by one warp shuffle, the y-pair P(iy) + P(iy-1)
//     through a small smem exchange, f_n = T_n (top face of layer L-1, from half 1) + B_n (bottom
//     face of layer L, half 0), then the central-difference update (Eq. 3 / L263-L266
//     with the sign of Eq. 3).  This post-phase of layer L-1 runs while the MMAs of layer L are
//     in flight.  Results are bit-identical to the test oracle's.

// Per-warp phase timeline (profiling builds only: -DOVX_TRACE, tools/trace_i8.py): clock64 stamps
// of one CTA (block OVX_TRACE) over TRH half-iterations, TRN points each.
#ifdef OVX_TRACE
#define TRN 16
#define TRH 16
__device__ unsigned long long g_tr[TRH * 16 * TRN];
#define TR(pt) do { if (blockIdx.x == OVX_TRACE && lane == 1 && trh >= 0 && trh < TRH) \
                        g_tr[(trh * 16 + warp) * TRN + (pt)] = clock64(); } while (0)
#else
#define TR(pt) do { } while (0)
#endif

// A operand row (one element, one half-word array): 7 chunks of 16 B — chunks 0-2 the u bytes,
// 3-5 the G bytes, 6 zero (K padding of the identity block's second K-step).
constexpr int A1_CHUNKS = 7;
constexpr int A1_PITCH = A1_CHUNKS * 128 + 16;   // bytes per 8-row core-matrix group (+16: bank spread)
constexpr int A1_BYTES = 16 * A1_PITCH;          // one half-word array of 128 rows
constexpr int B1_PITCH = 6 * 128;                // main B: 48 rows × 96 K-bytes
constexpr int BI_PITCH = 2 * 128;                // identity blocks: 48 rows × 32 K-bytes

// The shared-memory image of the resident B operands (K-major canonical core-matrix layout):
//   B  (48 rows × 96 K-bytes): row n = 2·output + byte parity, K-byte kb = 2·value + parity,
//      entry −K_e^INT8[n/2][kb/2] where the parities agree (⊗ I_2), 0 elsewhere;
//   BI (2 × 48 rows × 32 K-bytes): the Eq. 9 diagonal fold (−128 on the G bytes, variant D) and, in the
//      second block against the A padding chunk, 127 (the accumulator bias).
// Built once per constant upload from c_K8; every CTA copies it with 16-byte loads.
constexpr int kBImgVec = (6 * B1_PITCH + 2 * 6 * BI_PITCH) / 16;
__device__ uint4 g_bimg[kBImgVec];
__global__ void i8_bimg_kernel() {
    uint8_t *B = reinterpret_cast<uint8_t *>(g_bimg), *BI = B + 6 * B1_PITCH;
    for (int idx = threadIdx.x; idx < 48 * 96; idx += blockDim.x) {
        const int n = idx / 96, kb = idx - n * 96;
        const int off = (n >> 3) * B1_PITCH + (kb >> 4) * 128 + (n & 7) * 16 + (kb & 15);
        B[off] = ((kb & 1) == (n & 1)) ? (uint8_t)(-(int)c_K8[(n >> 1) * 48 + (kb >> 1)]) : (uint8_t)0;
    }
    for (int idx = threadIdx.x; idx < 2 * 48 * 32; idx += blockDim.x) {
        const int s2 = idx / (48 * 32), r2 = idx - s2 * 48 * 32;
        const int n = r2 / 32, kb = r2 - n * 32;
        const int off = s2 * 6 * BI_PITCH + (n >> 3) * BI_PITCH + (kb >> 4) * 128 + (n & 7) * 16 + (kb & 15);
        const int k = 16 * s2 + (kb >> 1);
        BI[off] = (s2 == 1 && kb >= 16) ? (uint8_t)127
                  : ((kb & 1) == (n & 1) && k == (n >> 1)) ? (uint8_t)0x80 : (uint8_t)0;
    }
}

// Tile geometry: EXv element columns × 8 rows per layer, MTv = EXv·8/128 M-tiles per CTA; the kernel
// runs I8G<32>: 512 threads, one CTA per SM, the two M-tiles skewed by half an iteration.  (A 16 × 8
// tile, two CTAs per SM with the A operand in shared memory, measured 2.34 vs 2.27 ms per C2 step:
// profiles/r1_int8_v24_tile16.md.)
template <int EXv>
struct I8G {
    static constexpr int EX = EXv;                     // element columns per layer (x)
    static constexpr int TX = EX - 1;                  // owned node columns (x)
    static constexpr int PX = TX + 2;                  // node columns of a u plane held in smem
    static constexpr int EY = 8;
    static constexpr int NE = EX * EY;                 // elements per layer
    static constexpr int NT = 2 * NE;                  // threads
    static constexpr int MT = NE / 128;                // M=128 MMA tiles per layer
    static constexpr int TY = EY - 1;
    static constexpr int PY = EY + 1;
    static constexpr int NOWN = TX * TY;
    static constexpr int NODES = PX * PY;              // nodes of one u plane held in smem
    static constexpr int PLANE = NODES * 3;
    static constexpr int TMEM_COLS = MT * 256;
    static constexpr int NS3 = MT == 2 ? 3 : 2;        // face-sum slots (the skew needs a third)
    static constexpr int CPS = MT == 2 ? 1 : 2;        // resident CTAs per SM
};
using I8W = I8G<32>;

template <class G, bool TA>
struct SmemI8 {
    uint8_t A[G::MT][4][TA ? 16 : A1_BYTES];   // [M-tile][half-word array], K-major canonical layout (TA: in TMEM)
    alignas(128) uint8_t B[6 * B1_PITCH];
    alignas(128) uint8_t BI[2][6 * BI_PITCH];
    double up[5][3][G::NODES];                      // ring: L-2, L-1 (updates), L, L+1 (gather), L+2;
                                                    // component-major: a warp's loads are contiguous
    unsigned long long nmax[5][G::NODES];           // max_c |u_c| of each node (bit patterns)
    double ysum[G::NS3][2][3][G::EY][G::EX];        // [layer slot][face][c] x-pair P of the +y corners
    double tf[2][3][G::NE];                         // [layer parity][c][tile node] top-face sums T
    double2 mc[kMaxMat];                            // (cG, c1) per material, staged from c_mat
    uint8_t mid[5][G::NE];                          // material id of each tile element, ring like up
    uint64_t mbar[G::MT];
    uint32_t tmem;
};

// ū values 8hf .. 8hf+15 of tile element (lx, ly) (local node order of reading Q1)
template <int HF, int PX, int NODES>
__device__ __forceinline__ void gather16(double (&ue)[16], const double *lo, const double *hi, int lx, int ly) {
    const int cx[4] = {0, 1, 1, 0}, cy[4] = {0, 0, 1, 1};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int k = 8 * HF + j, a = k / 3, c = k - 3 * a;
        const double *pl = a < 4 ? lo : hi;
        ue[j] = pl[c * NODES + (ly + cy[a & 3]) * PX + (lx + cx[a & 3])];
    }
}

// TMEM layout of the TA (A operand in TMEM) kernel, 512 columns: D of M-tile mt, array pa at
// mt·192 + pa·48 (48 columns = N); A (shared by the two skewed M-tiles) at 384 + pa·28 + 4·chunk.
constexpr uint32_t TA_D_TILE = 192, TA_D_ARR = 48, TA_A0 = 384, TA_A_ARR = 28;

// DIR (OVX_INT8_DIRECT, NEXT-4; Fig. 2 left, Eqs. 11-14 with a = 2^7, N = M): the
// direct method — every one of the M stages converts the FP64 remainder to an INT8 digit,
// d_i = INT(a·r_{i-1}) clamped to ±127, r_i = a·r_{i-1} − d_i (exact) — i.e. 2M conversions per value
// (F2I and back) instead of one; the digits (signed, lowest weight first) take the byte slots of
// the hierarchical path's v + 2^{7M}, the MMA reads A as s8, the stages recombine in base 2^7.
template <int MODE, int M, int HF, bool FAST, bool TA, bool DIR = false>
__device__ __forceinline__ void i8w_chunks(const StepParams &p, const double (&ue)[16], double cG, double r, double R,
                                           bool deg, uint8_t *Ab, uint32_t rowoff, bool dbg, int64_t dj,
                                           uint32_t ta, uint64_t *xbar, uint32_t xpar) {
    constexpr int NB = (7 * M + 1 + 7) / 8;
    constexpr int NA = (NB + 1) / 2;
    constexpr double SCALE = (double)(1ull << (7 * M));
    constexpr unsigned long long AOFF = 1ull << (7 * M);
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const int ch = HF == 0 ? (cc == 2 ? 3 : cc) : (cc == 0 ? 2 : cc + 3);
        const bool gpart = ch >= 3;
        const int j0 = 8 * (gpart ? ch - 3 : ch) - 8 * HF;     // index into ue of value 0 of the chunk
        long long v[8];
        uint32_t lo[8], hi[8];
        if constexpr (DIR) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double ub = gpart ? __dmul_rn(cG, ue[j0 + q]) : ue[j0 + q];
                double rr = deg ? 0.0 : __dmul_rn(ub, r);          // ū_es (Eq. 10)
                unsigned long long w = 0;
                long long V = 0;
#pragma unroll
                for (int st = 0; st < M; ++st) {                    // stage i = st + 1 (Eqs. 12-14)
                    const double t = __dmul_rn(128.0, rr);          // a·r_{i-1}, exact
                    const int d = max(-127, min(127, __double2int_rz(t)));
                    rr = __dsub_rn(t, (double)d);                   // r_i, exact
                    w |= (unsigned long long)(uint8_t)d << (8 * (M - 1 - st));
                    V = V * 128 + d;
                }
                lo[q] = (uint32_t)w;
                hi[q] = (uint32_t)(w >> 32);
                v[q] = V;
            }
        } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double ub = gpart ? __dmul_rn(cG, ue[j0 + q]) : ue[j0 + q];
            if (FAST)   // one DMUL + one F2I per value (R = RN(1/s)·2^{7M}, or 0 for a zero image)
                v[q] = __double2ll_rz(__dmul_rn(ub, R));
            else        // tiny-normal or non-finite s: the two roundings of Eq. 10 as written
                v[q] = deg ? 0ll : __double2ll_rz(__dmul_rn(__dmul_rn(ub, r), SCALE));
        }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if constexpr (DIR) {
            } else if constexpr (7 * M >= 32) {   // v + 2^{7M}: the offset only touches the high word
                lo[q] = (uint32_t)(unsigned long long)v[q];
                hi[q] = (uint32_t)((unsigned long long)v[q] >> 32) + (uint32_t)(AOFF >> 32);
            } else {                        // v + 2^{7M} < 2^32
                lo[q] = (uint32_t)(unsigned long long)v[q] + (uint32_t)AOFF;
                hi[q] = 0;
            }
            if (MODE == MODE_DEBUG && dbg) {
                const unsigned long long vp = ((unsigned long long)hi[q] << 32) | lo[q];
                const int k = ch * 8 + q;
                if (p.dbg_v) p.dbg_v[dj * 48 + k] = v[q];
                if (p.dbg_d)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        p.dbg_d[dj * 384 + j * 48 + k] = (DIR ? j < M : j < NB) ? (uint8_t)(vp >> (8 * j)) : 0;
            }
        }
        const uint32_t off = rowoff + (uint32_t)ch * 128;
        if (TA && cc == 0) {   // the shared TMEM A: the other M-tile's MMAs must have read it
            ptx::mbar_wait(xbar, xpar);
            ptx::tc_fence_after();
        }
#pragma unroll
        for (int pa = 0; pa < NA; ++pa) {
            const uint32_t *src = pa < 2 ? lo : hi;
            const uint32_t sel = (pa & 1) ? 0x7632u : 0x5410u;
            uint4 wv;
            wv.x = __byte_perm(src[0], src[1], sel);
            wv.y = __byte_perm(src[2], src[3], sel);
            wv.z = __byte_perm(src[4], src[5], sel);
            wv.w = __byte_perm(src[6], src[7], sel);
            if constexpr (TA)
                ptx::tmem_st4(ta + pa * TA_A_ARR + 4 * ch, wv.x, wv.y, wv.z, wv.w);
            else
                *reinterpret_cast<uint4 *>(Ab + pa * A1_BYTES + off) = wv;
        }
    }
}

template <int MODE, int M, int HF, bool TA, bool DIR = false>
__device__ __forceinline__ void i8w_convert(const StepParams &p, const double (&ue)[16], double cG, double s,
                                            bool deg, bool vzero, bool fast, uint8_t *Ab, uint32_t rowoff,
                                            bool dbg, int64_t dj, uint32_t ta, uint64_t *xbar, uint32_t xpar) {
    constexpr double SCALE = (double)(1ull << (7 * M));
    const double r = 1.0 / s;                                  // RN(1/s_e), reading Q7
    const double R = vzero ? 0.0 : __dmul_rn(r, SCALE);        // exact power-of-two scaling
    if constexpr (DIR)
        i8w_chunks<MODE, M, HF, false, TA, true>(p, ue, cG, r, R, deg, Ab, rowoff, dbg, dj, ta, xbar, xpar);
    else if (__all_sync(0xffffffffu, fast))
        i8w_chunks<MODE, M, HF, true, TA>(p, ue, cG, r, R, deg, Ab, rowoff, dbg, dj, ta, xbar, xpar);
    else
        i8w_chunks<MODE, M, HF, false, TA>(p, ue, cG, r, R, deg, Ab, rowoff, dbg, dj, ta, xbar, xpar);
}

__device__ __forceinline__ int ring5(int x) { return (x + 10) % 5; }   // x >= -10
template <int NS3>
__device__ __forceinline__ int ring3(int x) { return (x + 12) % NS3; }  // x >= -12

// Skewed M-tiles: iteration L = half-iterations 2L, 2L+1 (one CTA barrier at its end)
//   M-tile 0: [convert(L) -> MMA(L)] | [post-phase(L-1), epilogue(L)]
//   M-tile 1: [post-phase(L-2), epilogue(L-1)] | [convert(L) -> MMA(L)]   (its MMAs run across the barrier)
// so one M-tile's conversion (F2I / FP64 heavy) overlaps the other's epilogue (integer heavy) and the
// tensor core work of the two M-tiles is spread over the iteration.  Node row 4 (M-tile 1) reads the
// x-pairs of element row 3 (M-tile 0) one iteration after they were written.
// DAMP (MODE_STEP only): Rayleigh damping, reading R1 — the smem planes hold the EBE input
// ũ = u + cb·(u − u_prev) (node maxima of ũ), the update reads u and u_prev from global memory and
// writes u^{it+1} to p.un.
template <int MODE, int M, bool DAMP, class G, bool TA, bool DIR = false>
__global__ void __launch_bounds__(G::NT, G::CPS) step_i8w(const StepParams p) {
    static_assert(!TA || G::MT == 2, "the TMEM A operand is shared by two skewed M-tiles");
    // accumulator bias source: 16 padding bytes per row against B = 127: 255 (u8 A) or 127 (s8 A, DIR)
    constexpr uint32_t PADW = DIR ? 0x7F7F7F7Fu : 0xFFFFFFFFu;
    constexpr int32_t BIASV = DIR ? 16 * 127 * 127 : I8_BIAS;
    constexpr uint32_t IDS = DIR ? (IDESC | (1u << 7)) : IDESC;   // a_format: signed 8-bit for DIR
    using C = G;
    constexpr int EX = C::EX, TX = C::TX, PX = C::PX;
    constexpr int NB = (7 * M + 1 + 7) / 8;
    constexpr int NA = (NB + 1) / 2;
    constexpr double ISCALE = 1.0 / (double)(1ull << (7 * M));    // exact power of two
    constexpr int NT = C::NT, NODES = C::NODES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SmemI8<C, TA> &S = *reinterpret_cast<SmemI8<C, TA> *>(smem_raw);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int wu = __shfl_sync(0xffffffffu, warp, 0);   // the warp index as a uniform value
    const int mt = wu >> 3, hf = (wu >> 2) & 1, qd = wu & 3;   // warp-uniform roles (uniform registers)
    const int row = 32 * qd + lane;                      // MMA row = TMEM lane

    int trh = -1000;   // trace: half-iteration index (OVX_TRACE builds)
    (void)trh;
    int bid = blockIdx.x;
    const int tx = bid % p.tiles_x;
    bid /= p.tiles_x;
    const int ty = bid % p.tiles_y;
    const int tz = p.tz0 + bid / p.tiles_y;            // z-chunk (a launch may cover a subrange)
    const int64_t X0 = (int64_t)tx * TX, Y0 = (int64_t)ty * C::TY;
    const int Z0 = tz * p.zchunk;
    const int Z1 = (int)min((int64_t)Z0 + p.zchunk, p.nz + 1);
    const int nz = (int)p.nz;
    const int64_t NX1 = p.nx + 1, NY1 = p.ny + 1;
    const int64_t PSTRIDE = NX1 * NY1;
    const int Lfirst = max(Z0 - 1, 0);
    const int Lend = min(nz, Z1);                       // layers [Lfirst, Lend) are computed
    auto layer_ok = [&](int x) { return x >= Lfirst && x < Lend; };

    // element (lx, ly) of the tile; its (-x,-y) corner is tile node (lx, ly)
    const int lx = (128 * mt + row) % EX, ly = (128 * mt + row) / EX;
    const int64_t ex = X0 - 1 + lx, ey = Y0 - 1 + ly;
    const bool ein = (ex >= 0 && ex < p.nx && ey >= 0 && ey < p.ny);
    const int elem = lx + EX * ly;                   // tile element of this thread
    const uint8_t *matp = p.mat + (ein ? ex + p.nx * ey : 0);
    const int64_t mstride = p.nx * p.ny;
    // node (lx, ly): owned by this tile (lx, ly >= 1) if inside the grid; half 0 updates it
    const bool tnode = lx >= 1 && ly >= 1;
    const bool own = tnode && ex < NX1 && ey < NY1;
    const int64_t ucol = own ? ex + NX1 * ey : 0;
    const bool upd_role = own && hf == 0;

    // u (undamped) or ũ = u + cb·(u − u_prev) (damped) of one node component (global offset o)
    auto load_in = [&](int64_t o) {
        const double uu = __ldg(p.u + o);
        if constexpr (DAMP) {
            const double pp = __ldg(p.uo + o);    // u_prev is read-only in a damped step
            return __dadd_rn(uu, __dmul_rn(p.cb, __dsub_rn(uu, pp)));
        } else {
            return uu;
        }
    };
    // plane loader role: node li of the smem plane, taken by the last NODES threads
    const int li = t - (NT - NODES);
    const bool lrole = li >= 0;
    const int lpx = lrole ? li % PX : 0, lpy = lrole ? li / PX : 0;
    const bool ldn = lrole && X0 - 1 + lpx >= 0 && X0 - 1 + lpx < NX1 && Y0 - 1 + lpy >= 0 && Y0 - 1 + lpy < NY1;
    const int64_t ldoff = ldn ? 3 * ((X0 - 1 + lpx) + NX1 * (Y0 - 1 + lpy)) : 0;

    bool has_src = false, has_rec = false;
    if (MODE == MODE_STEP && hf == 0) {
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

    // ---- one-time setup: B operands, zero K-padding chunks, TMEM, mbarriers ----
    // B operands (−K_e^INT8 ⊗ I_2, the identity fold and the bias rows): one 16-byte copy per thread
    // of the image built once per constant upload (i8_bimg_kernel), B and BI being contiguous
    static_assert(sizeof(S.B) + sizeof(S.BI) == 16 * kBImgVec, "B image size");
    for (int i = t; i < kBImgVec; i += NT) reinterpret_cast<uint4 *>(S.B)[i] = g_bimg[i];
    if (!TA)
    for (int idx = t; idx < C::MT * 4 * 128; idx += NT) {   // K-padding bytes: 255 (bias source)
        const int a = idx >> 7, r = idx & 127;
        *reinterpret_cast<uint4 *>(&S.A[a >> 2][a & 3][(r >> 3) * A1_PITCH + 6 * 128 + (r & 7) * 16]) =
            make_uint4(PADW, PADW, PADW, PADW);
    }
    if (warp == 0) ptx::tmem_alloc<C::TMEM_COLS>(&S.tmem);
    if (t == 0)
        for (int mm = 0; mm < C::MT; ++mm) ptx::mbar_init(&S.mbar[mm], 1);
    for (int i = t; i < 2 * 3 * C::NE; i += NT) (&S.tf[0][0][0])[i] = 0.0;
    for (int i = t; i < p.nmat + 1; i += NT) {      // a per-lane indexed constant-bank load serialises
        const int id = i < p.nmat ? i : kZeroMat;
        S.mc[id] = make_double2(p.mc[id].cG, p.mc[id].c1);
    }
    if (hf == 0)
        for (int j = 0; j < 2; ++j) {   // material ids of layers Lfirst, Lfirst + 1
            const int iz = Lfirst + j;
            S.mid[ring5(iz)][elem] = (uint8_t)((ein && iz < nz) ? (int)__ldg(matp + mstride * iz) : kZeroMat);
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
                S.up[ring5(iz)][c][li] = v3[c];
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
    if (TA && wu < 4) {   // K-padding chunk 6 of the TMEM A arrays: 255 bytes (bias source), written once
#pragma unroll
        for (int pa = 0; pa < 4; ++pa)
            ptx::tmem_st4(S.tmem + ((uint32_t)(qd * 32) << 16) + TA_A0 + pa * TA_A_ARR + 24, PADW, PADW, PADW, PADW);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();   // ordered before the first MMA by the M-tile barrier of convert()
    }

    uint32_t phase = 0;
    uint32_t xpar = mt == 0 ? 1u : 0u;   // TA: parity of the other M-tile's MMA completion to wait for
    double upv[3] = {0.0, 0.0, 0.0}, wn = 0.0;   // update operands of this M-tile's post-phase plane
    double uv[3] = {0.0, 0.0, 0.0};              // DAMP: u of the owned node (the plane holds ũ)
    uint8_t dm = 0;
    double plo[3] = {0.0, 0.0, 0.0};             // x-pair P(iy) of this thread's face, last epilogue layer
    // conversion -> epilogue hand-over (the same iteration for M-tile 0, the next one for M-tile 1)
    double es = 0.0;
    bool edeg = false, edbg = false;
    int em = kZeroMat;
    int64_t edj = -1;

    // ---- post-phase of layer / plane Lp: face sums, f_n = T + B, update ----
    auto post_phase = [&](int Lp, int s3, int s5) {   // s3, s5: ring slots of Lp
        if (!tnode) return;
        const bool plane_done = (Lp >= Z0 && Lp <= nz && Lp < Z1);
        const bool bot_iface = (p.slab_flags & 1) && Lp == 0;
        const bool top_iface = (p.slab_flags & 2) && Lp == nz;
        // all shared-memory operands first (one round trip instead of three dependent ones): the
        // y-pair P(iy-1), T of plane Lp (half 0) and u of the node (indices in range for every thread)
        double ysv[3], tfv[3], ucv[3];
        {
#pragma unroll
            for (int c = 0; c < 3; ++c) {   // component-major: a warp's loads are contiguous
                ysv[c] = S.ysum[s3][hf][c][ly - 1][lx];
                tfv[c] = S.tf[(Lp - 1) & 1][c][lx + EX * ly];
                ucv[c] = S.up[s5][c][ly * PX + lx];
            }
        }
        double face[3] = {0.0, 0.0, 0.0};
        if (layer_ok(Lp)) {
#pragma unroll
            for (int c = 0; c < 3; ++c) face[c] = __dadd_rn(plo[c], ysv[c]);   // P(iy) + P(iy-1)
        }
        TR(9);
        if (hf == 1) {        // top face of layer Lp: T of plane Lp+1
#pragma unroll
            for (int c = 0; c < 3; ++c) S.tf[Lp & 1][c][lx + EX * ly] = face[c];
        } else if (own && plane_done) {
            const int64_t un_id = ucol + PSTRIDE * Lp;
            if (bot_iface) {  // interface plane: B waits for T from the rank below
#pragma unroll
                for (int c = 0; c < 3; ++c) p.iface_bot_b[3 * ucol + c] = face[c];
            } else {
                double f[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) f[c] = __dadd_rn(tfv[c], face[c]);
                if (top_iface) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) p.iface_top_A[3 * ucol + c] = f[c];
                } else if (MODE == MODE_STEP) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int64_t dof = 3 * un_id + c;
                        double F = 0.0;
                        if (has_src)
                            for (int k = 0; k < p.nsrc; ++k)
                                if (p.src_dof[k] == dof) F = __dadd_rn(F, p.src_val[k]);
                        if (c == 0) TR(10);
                        const double uc = DAMP ? uv[c] : ucv[c];
                        double b = __dsub_rn(__dmul_rn(2.0, uc), upv[c]);
                        if constexpr (DAMP) b = __dsub_rn(b, __dmul_rn(p.ca, __dsub_rn(uc, upv[c])));
                        double un = __fma_rn(wn, __dsub_rn(F, f[c]), b);
                        if ((dm >> c) & 1) un = 0.0;
                        (DAMP ? p.un : p.uo)[dof] = un;
                        if (c == 2) TR(11);
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

    // ---- epilogue of layer Le: the 4 corner nodes of this thread's face ----
    auto epilogue = [&](int Le, int s3) {              // s3: ysum slot of Le
        ptx::mbar_wait_sleep(&S.mbar[mt], phase);
        TR(5);
        phase ^= 1;
        ptx::tc_fence_after();
        // −RN(c1·s·2^{-7M}); a degenerate element contributes 0 (oracle: fe = 0)
        const double alpha = edeg ? 0.0 : -__dmul_rn(S.mc[em].y, __dmul_rn(es, ISCALE));
        constexpr uint32_t DARR = TA ? TA_D_ARR : 64;
        const uint32_t tb = S.tmem + ((uint32_t)(qd * 32) << 16) + mt * (TA ? TA_D_TILE : 256) + 24 * hf;
        double fc[12];                               // [corner][c] of the face
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {             // 4 outputs per round (8 columns per array)
            uint32_t R0[8], R1[8], R2[8] = {}, R3[8] = {};
            ptx::tmem_ld8(tb + 0 + rr * 8, R0);
            ptx::tmem_ld8(tb + DARR + rr * 8, R1);
            if (NA > 2) ptx::tmem_ld8(tb + 2 * DARR + rr * 8, R2);
            if (NA > 3) ptx::tmem_ld8(tb + 3 * DARR + rr * 8, R3);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 4 * rr + q;
                const int32_t c0 = (int32_t)R0[2 * q], c1_ = (int32_t)R0[2 * q + 1];
                const int32_t c2_ = (int32_t)R1[2 * q], c3 = (int32_t)R1[2 * q + 1];
                // stages beyond NA arrays are absent: give them the bias value (C_j = 0 after removal)
                const int32_t c4 = NA > 2 ? (int32_t)R2[2 * q] : BIASV, c5 = NA > 2 ? (int32_t)R2[2 * q + 1] : BIASV;
                const int32_t c6 = NA > 3 ? (int32_t)R3[2 * q] : BIASV, c7 = NA > 3 ? (int32_t)R3[2 * q + 1] : BIASV;
                // D_j = −C_j + BIAS, C_j = K_D·b_j (K_D·1 = 0): y = Σ_j 256^j C_j (DIR: 128^j), two limbs
                const double dlo = DIR ? limb_biased128<BIASV>(c0, c1_, c2_, c3) : limb_biased(c0, c1_, c2_, c3);
                const double dhi = NA > 2 ? (DIR ? limb_biased128<BIASV>(c4, c5, c6, c7) : limb_biased(c4, c5, c6, c7)) : 0.0;
                const double Y = NA > 2 ? __fma_rn(dhi, DIR ? 0x1p28 : 0x1p32, dlo) : dlo;    // RN(−y)
                const double f = __dmul_rn(alpha, Y);            // = RN(c1s·RN(y))
                if (MODE == MODE_DEBUG && edbg) {
                    const int i = 12 * hf + j;
                    const int32_t Cj[8] = {c0 - BIASV, c1_ - BIASV, c2_ - BIASV, c3 - BIASV,
                                           c4 - BIASV, c5 - BIASV, c6 - BIASV, c7 - BIASV};
                    __int128 y = 0;
#pragma unroll
                    for (int jj = 7; jj >= 0; --jj) y = y * (DIR ? 128 : 256) - (__int128)Cj[jj];
                    if (p.dbg_C)
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) p.dbg_C[edj * 192 + jj * 24 + i] = -Cj[jj];
                    if (p.dbg_yhi) p.dbg_yhi[edj * 24 + i] = (long long)(y >> 64);
                    if (p.dbg_ylo) p.dbg_ylo[edj * 24 + i] = (long long)(unsigned long long)y;
                    if (p.dbg_fe) p.dbg_fe[edj * 24 + i] = f;
                }
                fc[j] = f;
            }
        }
        ptx::tc_fence_before();
        // x-pairs: P(iy) of node (lx, ly) = own (-x,-y) corner + lane lx-1's (+x,-y) corner;
        // the +y corners give P(iy-1) of node (lx, ly+1), exchanged through smem
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double pm = __shfl_up_sync(0xffffffffu, fc[3 * 1 + c], 1, EX);   // (+x,-y) of lx-1
            const double pp = __shfl_up_sync(0xffffffffu, fc[3 * 2 + c], 1, EX);   // (+x,+y) of lx-1
            plo[c] = __dadd_rn(fc[3 * 0 + c], pm);
            S.ysum[s3][hf][c][ly][lx] = __dadd_rn(fc[3 * 3 + c], pp);
        }
    };

    // ---- conversion of layer L (this thread's three chunks) and the MMA hand-off ----
    auto convert = [&](int L, int sL, int sL1) {       // ring slots of planes L, L+1
        const int64_t eid = ex + p.nx * (ey + p.ny * (int64_t)L);
        const int64_t dj = eid - p.dbg_e0;
        const bool dbg = (MODE == MODE_DEBUG) && ein && lx < TX && ly < C::TY && (L + 1 >= Z0) && (L + 1 < Z1) &&
                         dj >= 0 && dj < p.dbg_ne;
        // s_e from the per-node maxima of the two planes
        const unsigned long long *m0 = S.nmax[sL], *m1 = S.nmax[sL1];
        const int n0 = ly * PX + lx;
        // the node maxima are |u| bit patterns of finite values: as doubles, one DMNMX per pair (a
        // balanced tree) instead of a 64-bit integer compare-and-select
        auto dv = [](unsigned long long b) { return __longlong_as_double((long long)b); };
        const double amax = fmax(fmax(fmax(dv(m0[n0]), dv(m0[n0 + 1])), fmax(dv(m0[n0 + PX]), dv(m0[n0 + PX + 1]))),
                                 fmax(fmax(dv(m1[n0]), dv(m1[n0 + 1])), fmax(dv(m1[n0 + PX]), dv(m1[n0 + PX + 1]))));
        const int mcur = S.mid[sL][elem];
        const double cG = S.mc[mcur].x;
        const double s = fmax(amax, __dmul_rn(cG, amax));   // max_i |RN(cG u_i)| = RN(cG max_i |u_i|)
        const bool deg = !ein || !(s >= 0x1p-1022) || !(s <= 0x1.fffffffffffffp1023);
        const bool vzero = !ein || !(s >= 0x1p-1022);
        const bool fast = (s <= 0x1.fffffffffffffp1023) && (vzero || s >= 0x1p-960);
        uint8_t *Ab = &S.A[mt][0][0];
        const uint32_t rowoff = (uint32_t)((row >> 3) * A1_PITCH + (row & 7) * 16);
        double ue[16];
        const uint32_t ta = S.tmem + ((uint32_t)(qd * 32) << 16) + TA_A0;
        uint64_t *xbar = &S.mbar[C::MT - 1 - mt];
        if (hf == 0) {
            gather16<0, PX, C::NODES>(ue, &S.up[sL][0][0], &S.up[sL1][0][0], lx, ly);
            i8w_convert<MODE, M, 0, TA, DIR>(p, ue, cG, s, deg, vzero, fast, Ab, rowoff, dbg, dj, ta, xbar, xpar);
            if (MODE == MODE_DEBUG && dbg && p.dbg_s) p.dbg_s[dj] = s;
        } else {
            gather16<1, PX, C::NODES>(ue, &S.up[sL][0][0], &S.up[sL1][0][0], lx, ly);
            i8w_convert<MODE, M, 1, TA, DIR>(p, ue, cG, s, deg, vzero, fast, Ab, rowoff, dbg, dj, ta, xbar, xpar);
        }
        xpar ^= 1u;
        if (TA) {
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
        }
        es = s;
        edeg = deg;
        em = mcur;
        edbg = dbg;
        edj = dj;
        ptx::fence_proxy_async_smem();
        TR(1);
        asm volatile("bar.sync %0, 256;" ::"r"(1 + mt) : "memory");   // the 8 warps of this M-tile
        TR(2);
        if ((wu & 7) == 0) {     // first warp of the M-tile; one elected lane issues
            const int mtu = wu >> 3;
            if (ptx::elect_one()) {
                ptx::tc_fence_after();
                const uint32_t b0 = ptx::smem_u32(&S.B[0]);
                const uint32_t bi0 = ptx::smem_u32(&S.BI[0][0]), bi1 = ptx::smem_u32(&S.BI[1][0]);
                const uint32_t a0 = ptx::smem_u32(&S.A[mtu][0][0]);
#pragma unroll
                for (int pa = 0; pa < NA; ++pa) {
                    if constexpr (TA) {   // A from TMEM: column 8·ks = chunks 2ks, 2ks+1; identity: chunks 3-4, 5-6
                        const uint32_t at = S.tmem + TA_A0 + pa * TA_A_ARR;
                        const uint32_t d = S.tmem + mtu * TA_D_TILE + pa * TA_D_ARR;
#pragma unroll
                        for (int ks = 0; ks < 3; ++ks)
                            ptx::mma_i8_ts(d, at + 8 * ks, ptx::smem_desc(b0 + ks * 256, 128, B1_PITCH), IDS,
                                           ks > 0 ? 1u : 0u);
                        ptx::mma_i8_ts(d, at + 12, ptx::smem_desc(bi0, 128, BI_PITCH), IDS, 1u);
                        ptx::mma_i8_ts(d, at + 20, ptx::smem_desc(bi1, 128, BI_PITCH), IDS, 1u);
                    } else {
                    const uint32_t abase = a0 + pa * A1_BYTES;
                    const uint32_t d = S.tmem + mtu * 256 + pa * 64;
#pragma unroll
                    for (int ks = 0; ks < 3; ++ks)
                        ptx::mma_i8(d, ptx::smem_desc(abase + ks * 256, 128, A1_PITCH),
                                    ptx::smem_desc(b0 + ks * 256, 128, B1_PITCH), IDS, ks > 0 ? 1u : 0u);
                    ptx::mma_i8(d, ptx::smem_desc(abase + 3 * 128, 128, A1_PITCH),
                                ptx::smem_desc(bi0, 128, BI_PITCH), IDS, 1u);
                    ptx::mma_i8(d, ptx::smem_desc(abase + 5 * 128, 128, A1_PITCH),
                                ptx::smem_desc(bi1, 128, BI_PITCH), IDS, 1u);
                    }
                }
                ptx::mma_commit(&S.mbar[mtu]);
            }
            __syncwarp();
        }
        TR(3);
    };

    // ring slots of planes / layers L-2 .. L+2 (q5_k = (L-2+k) mod 5) and L-2 .. L (q3_k = (L-2+k) mod 3)
    int q5_0 = ring5(Z0 - 3), q5_1 = ring5(Z0 - 2), q5_2 = ring5(Z0 - 1), q5_3 = ring5(Z0), q5_4 = ring5(Z0 + 1);
    int q3_0 = ring3<C::NS3>(Z0 - 3), q3_1 = ring3<C::NS3>(Z0 - 2), q3_2 = ring3<C::NS3>(Z0 - 1);
    // running offsets of the prefetch (advanced once per iteration): plane L+2 of u, the material of
    // layer L+2, the owned node of plane L - mt
    int64_t ro_plane = 3 * PSTRIDE * (int64_t)(Z0 + 1);
    const uint8_t *ro_mat = matp + mstride * (int64_t)(Z0 + 1);
    int64_t ro_node = ucol + PSTRIDE * (int64_t)(Z0 - 1 - mt);
    // half-iterations: h = 2L (even) and 2L+1 (odd); one copy of each phase body, selected per M-tile
    double pfv[3] = {0.0, 0.0, 0.0};
    bool pf = false;
    int mfar = kZeroMat;
    double upv_n[3] = {0.0, 0.0, 0.0}, wn_n = 0.0, uv_n[3] = {0.0, 0.0, 0.0};
    uint8_t dm_n = 0;
    for (int h = 2 * (Z0 - 1); h <= 2 * (Z1 + 1) + 1; ++h) {
        const int L = h >> 1;
        const bool odd = h & 1;
#ifdef OVX_TRACE
        trh = h - 2 * (Z0 - 1) - 20;
#endif
        TR(0);
        if (!odd) {
            // ---- prefetch: plane L+2, material of layer L+2, update operands of the next post plane ----
            const int pz = L + 2;
            pf = (pz > Lfirst + 1) && (L + 1 < Z1) && (L + 1 < nz);
            if (pf && ldn) {
#pragma unroll
                for (int c = 0; c < 3; ++c) pfv[c] = load_in(ro_plane + ldoff + c);
            }
            mfar = (ein && L + 2 < nz && L >= Lfirst) ? (int)__ldg(ro_mat) : kZeroMat;
            const int Pn = L - mt;                    // plane this thread updates in the next iteration
            if (MODE == MODE_STEP && upd_role && Pn >= Z0 && Pn <= nz && Pn < Z1) {
                const int64_t un_next = ro_node;
                upv_n[0] = p.uo[3 * un_next];
                upv_n[1] = p.uo[3 * un_next + 1];
                upv_n[2] = p.uo[3 * un_next + 2];
                if constexpr (DAMP) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) uv_n[c] = __ldg(p.u + 3 * un_next + c);
                }
                wn_n = __ldg(p.w + un_next);
                dm_n = p.dmask ? __ldg(p.dmask + un_next) : (uint8_t)0;
            }
        }
        // M-tile 0: convert at even h, post-phase + epilogue at odd h; M-tile 1 the other way round
        if (odd == (mt == 1)) {
            if (layer_ok(L)) convert(L, q5_2, q5_3);
        } else {
            post_phase(L - 1 - mt, mt ? q3_0 : q3_1, mt ? q5_0 : q5_1);
            TR(4);
            if (layer_ok(L - mt)) epilogue(L - mt, mt ? q3_1 : q3_2);
            TR(6);
        }
        if (odd) {
            // ---- park plane L+2 (slot of plane L-3, no longer read) with its node maxima ----
            const int pz = L + 2;
            if (pf && lrole) {
                unsigned long long m = 0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    S.up[q5_4][c][li] = pfv[c];
                    const unsigned long long b = abs_bits(pfv[c]);
                    m = b > m ? b : m;
                }
                S.nmax[q5_4][li] = m;
            }
            if (hf == 0 && pf) S.mid[q5_4][elem] = (uint8_t)mfar;   // material of layer L+2
            upv[0] = upv_n[0];
            upv[1] = upv_n[1];
            upv[2] = upv_n[2];
            uv[0] = uv_n[0];
            uv[1] = uv_n[1];
            uv[2] = uv_n[2];
            wn = wn_n;
            dm = dm_n;
            upv_n[0] = upv_n[1] = upv_n[2] = 0.0;
            ro_plane += 3 * PSTRIDE;
            ro_mat += mstride;
            ro_node += PSTRIDE;
            {   // advance the ring slots to L+1 (rotation instead of a modulo per use)
                const int t5 = q5_0;
                q5_0 = q5_1; q5_1 = q5_2; q5_2 = q5_3; q5_3 = q5_4; q5_4 = t5;
                const int t3 = C::NS3 == 3 ? q3_0 : q3_1;   // two slots: (a, b, a) -> (b, a, b)
                q3_0 = q3_1; q3_1 = q3_2; q3_2 = t3;
            }
            wn_n = 0.0;
            dm_n = 0;
            TR(7);
            __syncthreads();
            TR(8);
        }
    }
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc<C::TMEM_COLS>(S.tmem);
}
