// kernels.cu — sm_100a kernels of the OVFEM / TCOVFEM explicit time step.
//
// One fused kernel per time step:
//   CTA  = a tile of 32 × 8 elements per layer (owned node columns 31 × 7; one halo element ring
//   recomputed by the neighbour tiles, so no cross-CTA reduction), marching in z over a chunk of
//   node planes (chunk count from a wave model).  Per element layer it computes the element
//   forces, sums them into node forces in the pairwise order of reading U2 (bit-identical to the
//   oracle) and applies the central-difference update (Eq. 3, L263-L266 with the sign
//   of Eq. 3; Rayleigh damping, reading R1, optional) to each completed plane.
//
// Kernels (paths of include/ovx.h):
//   step_i8w  OVX_INT8: PAPER.md Eq. 9 via Eqs. 10-17 — s_e = max|ū_e|, v = trunc(2^{7M} ū_e/s_e),
//             byte slices of v + 2^{7M} (variant B) as the u8 A operand (in TMEM) of
//             tcgen05.mma.kind::i8 (M=128 elements, N=48, 4 half-word arrays), −K_e^INT8 ⊗ I_2 and the folded Eq. 9
//             diagonal (variant D) as the resident s8 B operand, s32 accumulators in TMEM, exact
//             two-limb recombination, f_e = RN(c1 s_e 2^{-7M})·RN(y).
//   step_f64  OVX_FP64 / OVX_VFEM: factored FP64 element forces (Walsh-Hadamard modes of the
//             corner values; OVFEM or trilinear VFEM weights), shuffle / SMEM node sums.
//   step_v1   OVX_FP64_DENSE / OVX_VFEM_DENSE (and the FP64 / VFEM debug records): the literal
//             dense form with sequential _rn sums, a bit-exact mirror of the test oracle's definition.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ovx_internal.h"
#include "ptx.cuh"

#include "../../include/ovx.h"

namespace ovx {

// Element matrices, identical for every context (upload_device_constants, once per device): the
// dense integer matrices [0] OVFEM K^κ, K̄^G + 128 I and [1] VFEM Vk, Vg (step_v1), and K_e^INT8.
__constant__ double c_Kk[2][576];
__constant__ double c_Kg[2][576];
__constant__ int8_t c_K8[1152];

namespace {

constexpr int EX = 32;                    // element columns per layer (x)
constexpr int TX = EX - 1;                // owned node columns (x)
constexpr int PX = TX + 2;                // node columns of a u plane held in smem (x)
constexpr int KB = 96;                    // K bytes per A row / B row (48 values × 2 bytes)
constexpr int ROWGRP = 8 * KB;            // bytes per 8-row core-matrix group (6 chunks × 128)
constexpr int A_BYTES = 128 * KB;         // one half-word array (M = 128 rows)
constexpr int B_ROWS = 48;                // N = 24 outputs × 2 byte positions
constexpr int B_BYTES = B_ROWS * KB;
constexpr int TMEM_COLS = 256;            // 4 accumulators of 48 columns at 64-column pitch
constexpr uint32_t IDESC = ptx::idesc_i8(128, 48);

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
template <class MC>   // MatConst or a shared-memory copy with the same L0 .. C2 fields
__device__ __forceinline__ void element_force_wht(const double (&ue)[24], const MC &m, double (&fe)[24]) {
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

// ---- factored VFEM element force (OVX_VFEM, NEXT-3) ---------------------------
// The trilinear field of the corner values is u_c(r) = (1/8) Σ_S h_c[S] Π_{j∈S} r_j with the same
// Walsh-Hadamard transform h_c[S] as above, so ∂_i u_c = (1/(4ds)) Σ_{T ∌ i} h_c[T ∪ {i}] m_T(r),
// m_T = Π_{j∈T} r_j.  The monomials are orthogonal on the cube (∫ m_T m_T' dv = δ ds³ 3^{-|T|}),
// hence the strain energy of K_e^V (exact integration = the paper's 2×2×2 Gauss rule) splits per
// monomial T, and  F_c[S] = ∂E/∂h_c[S] = Σ_{i∈S, T = S∖{i}} w_T ·
//     (c = i:  λ Σ_{j∉T} h_j[T ∪ {j}] + 2μ h_i[S];   c ≠ i:  μ (h_c[S] + h_i[T ∪ {c}]·[c ∉ T])),
// w_T = (ds/16) 3^{-|T|}; then f_c^α = Σ_S F_c[S] Π_{j∈S} r̄_j^α (inverse transform).
// Equal to K_e^V u_e in exact arithmetic (≈250 FP64 operations instead of 1152 FMAs).
template <class MC>   // anything with vl[3] = w_T λ, vm[3] = w_T μ for |T| = 0, 1, 2
__device__ __forceinline__ void element_force_vfem_wht(const double (&ue)[24], const MC &m, double (&fe)[24]) {
    constexpr int BORD[8] = {0, 1, 3, 2, 4, 5, 7, 6};  // local node -> bit index x | y<<1 | z<<2
    double h[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int a = 0; a < 8; ++a) h[c][BORD[a]] = ue[3 * a + c];
        wht8(h[c]);
    }
    double F[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int S = 0; S < 8; ++S) F[c][S] = 0.0;
#pragma unroll
    for (int T = 0; T < 8; ++T) {
        const int nT = (T & 1) + ((T >> 1) & 1) + ((T >> 2) & 1);
        if (nT == 3) continue;
        const double lam = m.vl[nT], mu = m.vm[nT];
        double div = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
            if (!((T >> j) & 1)) div += h[j][T | (1 << j)];
        const double ldiv = lam * div;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if ((T >> i) & 1) continue;
            const int S = T | (1 << i);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (c == i) {
                    F[c][S] += fma(2.0 * mu, h[i][S], ldiv);
                } else {
                    const double gic = ((T >> c) & 1) ? 0.0 : h[i][T | (1 << c)];
                    F[c][S] += mu * (h[c][S] + gic);
                }
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        iwht8(F[c]);
#pragma unroll
        for (int a = 0; a < 8; ++a) fe[3 * a + c] = F[c][BORD[a]];
    }
}

// Biased stage products (INT8 kernel): the A operand's K-padding bytes are 255 and the matching B
// entries 127 (16 bytes per row), so every accumulator D_j = −C_j + I8_BIAS with I8_BIAS =
// 16·255·127 = 518160 > max|C_j| = 255·1258 = 320790 (max absolute row sum of K_D): all D_j > 0.
// The limb p0 + 2^16 p1 (p0 = D0 + 256 D1, p1 = D2 + 256 D3, both in [0, 2^28)) then needs no sign
// extension, and the bias comes out exactly with the magic: 1.5·2^52 + I8_BIAS·(1 + 2^8 + 2^16 + 2^24)
// is an integer below 2^53.
constexpr int32_t I8_BIAS = 16 * 255 * 127;
constexpr double I8_LIMB_MAGIC = 0x1.8p52 + (double)I8_BIAS * 16843009.0;
__device__ __forceinline__ double limb_biased(int32_t d0, int32_t d1, int32_t d2, int32_t d3) {
    // L = p0 + 2^16·p1 < 2^44 assembled under the magic exponent as two 32-bit words: the low word
    // with carry-out, the high word (p1 >> 16) + carry + 0x43380000 (no 64-bit multiply-add)
    const uint32_t p0 = (uint32_t)(d0 + 256 * d1), p1 = (uint32_t)(d2 + 256 * d3);
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0x43380000;" : "=r"(lo), "=r"(hi) : "r"(p0), "r"(p1 << 16),
        "r"(p1 >> 16));
    return __hiloint2double((int)hi, (int)lo) - I8_LIMB_MAGIC;
}
// The same for the direct N-stage path (DIR): stages in base 2^7, D_j = −C_j + B (B = 16·127·127,
// s8 digits): L = p0 + 2^14·p1 (p0 = D0 + 128·D1, p1 = D2 + 128·D3 < 2^26), L < 2^41, assembled as
// two words under the magic exponent; the bias B·(1 + 2^7 + 2^14 + 2^21) comes out with the magic.
template <int32_t B>
__device__ __forceinline__ double limb_biased128(int32_t d0, int32_t d1, int32_t d2, int32_t d3) {
    constexpr double MAGIC = 0x1.8p52 + (double)B * 2113665.0;
    const uint32_t p0 = (uint32_t)(d0 + 128 * d1), p1 = (uint32_t)(d2 + 128 * d3);
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0x43380000;" : "=r"(lo), "=r"(hi) : "r"(p0), "r"(p1 << 14),
        "r"(p1 >> 18));
    return __hiloint2double((int)hi, (int)lo) - MAGIC;
}
// max_i |x_i| of finite / infinite doubles as the integer max of their magnitude bit patterns
// (monotone for non-NaN values; a NaN sorts above +inf and makes the element degenerate)
__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}

#include "step_v1.cuh"
#include "step_f64.cuh"

#include "step_i8w.cuh"
#include "step_i8x.cuh"
#include "step_i8ws.cuh"

// cudaFuncSetAttribute state is per device: remember it per device index
inline bool attr_done(unsigned &mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    return (mask >> (dev & 31)) & 1u;
}
inline void attr_set(unsigned &mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    mask |= 1u << (dev & 31);
}

template <int MODE, int M, bool DAMP, class G, bool TA, bool DIR = false>
cudaError_t launch_i8w(const StepParams &p, int64_t ctas, cudaStream_t st) {
    static unsigned attr = 0;
    const int smem = (int)sizeof(SmemI8<G, TA>);
    if (!attr_done(attr)) {
        cudaError_t e = cudaFuncSetAttribute(step_i8w<MODE, M, DAMP, G, TA, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        // all of the unified L1/shared array as shared memory, so G::CPS CTAs fit one SM
        e = cudaFuncSetAttribute(step_i8w<MODE, M, DAMP, G, TA, DIR>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        attr_set(attr);
    }
    step_i8w<MODE, M, DAMP, G, TA, DIR><<<(unsigned)ctas, G::NT, smem, st>>>(p);
    return cudaGetLastError();
}

// INT8 kernel variant (OVX_I8_KERNEL): "ws" (default) step_i8ws, warp-specialised (time steps,
// damped or not, and products; M = 4 / 6 undamped single contexts; the direct path, the debug records
// and M = 4 / 6 damped or on z-slabs use step_i8w); "tmem"
// step_i8w with the A operand in TMEM (the round-1 kernel); "smem" step_i8w with A in shared memory;
// "x" step_i8x (word or half-word operand layout, OVX_I8X_LAYOUT).  All bit-identical; DESIGN.md
// §6.1 has the measurements.
int i8_variant() {
    static const int v = [] {
        const char *e = std::getenv("OVX_I8_KERNEL");
        if (e && std::strcmp(e, "smem") == 0) return 1;
        if (e && std::strcmp(e, "x") == 0) return 2;
        if (e && std::strcmp(e, "tmem") == 0) return 0;
        return 3;
    }();
    return v;
}

// node planes of step_i8ws (OVX_I8_PLANES): "cp" (default) per-thread cp.async, "bulk" the bulk-copy
// (TMA) engine, one copy per node row
bool i8_bulk_planes() {
    static const bool v = [] {
        const char *e = std::getenv("OVX_I8_PLANES");
        return e && std::strcmp(e, "bulk") == 0;
    }();
    return v;
}

template <int MODE, bool SLAB, bool BULK, bool DAMP = false, int M = 8>
cudaError_t launch_i8ws_b(const StepParams &p, int64_t ctas, cudaStream_t st) {
    const int smem = (int)sizeof(SmemWST<BULK>);
    static unsigned attr = 0;
    if (!attr_done(attr)) {
        cudaError_t e =
            cudaFuncSetAttribute(step_i8ws<MODE, SLAB, BULK, DAMP, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(step_i8ws<MODE, SLAB, BULK, DAMP, M>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        attr_set(attr);
    }
    step_i8ws<MODE, SLAB, BULK, DAMP, M><<<(unsigned)ctas, 512, smem, st>>>(p);
    return cudaGetLastError();
}
template <int MODE, bool SLAB>
cudaError_t launch_i8ws(const StepParams &p, int64_t ctas, cudaStream_t st) {
    if constexpr (MODE == MODE_STEP)
        if (p.damped) return launch_i8ws_b<MODE, SLAB, false, true>(p, ctas, st);
    return i8_bulk_planes() ? launch_i8ws_b<MODE, SLAB, true>(p, ctas, st) : launch_i8ws_b<MODE, SLAB, false>(p, ctas, st);
}

// step_i8x operand layout (OVX_I8X_LAYOUT): "word" (default, B = −K_D ⊗ I_4) or "half" (⊗ I_2)
int i8x_layout() {
    static const int v = [] {
        const char *e = std::getenv("OVX_I8X_LAYOUT");
        return (e && std::strcmp(e, "half") == 0) ? 0 : 1;
    }();
    return v;
}

template <int MODE, int M, bool DAMP, bool SLAB, int LAY>
cudaError_t launch_i8x_l(const StepParams &p, int64_t ctas, cudaStream_t st) {
    const int smem = (int)sizeof(SmemI8X);
    static unsigned attr = 0;
    if (!attr_done(attr)) {
        cudaError_t e = cudaFuncSetAttribute(step_i8x<MODE, M, DAMP, SLAB, LAY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(step_i8x<MODE, M, DAMP, SLAB, LAY>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        attr_set(attr);
    }
    step_i8x<MODE, M, DAMP, SLAB, LAY><<<(unsigned)ctas, 512, smem, st>>>(p);
    return cudaGetLastError();
}
template <int MODE, int M, bool DAMP, bool SLAB>
cudaError_t launch_i8x(const StepParams &p, int64_t ctas, cudaStream_t st) {
    return i8x_layout() == 1 ? launch_i8x_l<MODE, M, DAMP, SLAB, 1>(p, ctas, st)
                             : launch_i8x_l<MODE, M, DAMP, SLAB, 0>(p, ctas, st);
}

template <int M, class G, bool TA>
cudaError_t launch_i8_mode_g(int mode, const StepParams &p, int64_t ctas, cudaStream_t st) {
    if (mode == MODE_STEP)
        return p.damped ? launch_i8w<MODE_STEP, M, true, G, TA>(p, ctas, st)
                        : launch_i8w<MODE_STEP, M, false, G, TA>(p, ctas, st);
    if (mode == MODE_APPLY) return launch_i8w<MODE_APPLY, M, false, G, TA>(p, ctas, st);
    return launch_i8w<MODE_DEBUG, M, false, G, TA>(p, ctas, st);
}

template <int M, bool SLAB>
cudaError_t launch_i8x_mode(int mode, const StepParams &p, int64_t ctas, cudaStream_t st) {
    if (mode == MODE_STEP)
        return p.damped ? launch_i8x<MODE_STEP, M, true, SLAB>(p, ctas, st)
                        : launch_i8x<MODE_STEP, M, false, SLAB>(p, ctas, st);
    return launch_i8x<MODE_APPLY, M, false, SLAB>(p, ctas, st);
}

template <int M>
cudaError_t launch_i8_mode(int mode, const StepParams &p, int64_t ctas, cudaStream_t st) {
    if (p.direct) {   // NEXT-4: the direct N-stage conversion (M = 8, undamped; OVX_INT8_DIRECT)
        if constexpr (M == 8) {
            if (mode == MODE_STEP) return launch_i8w<MODE_STEP, 8, false, I8W, true, true>(p, ctas, st);
            if (mode == MODE_APPLY) return launch_i8w<MODE_APPLY, 8, false, I8W, true, true>(p, ctas, st);
            return launch_i8w<MODE_DEBUG, 8, false, I8W, true, true>(p, ctas, st);
        }
        return cudaErrorInvalidValue;
    }
    const int v = i8_variant();
    if constexpr (M == 8) {
        if (v == 3 && mode != MODE_DEBUG && (!p.damped || mode == MODE_STEP)) {   // warp-specialised kernel (M = 8)
            if (mode == MODE_STEP)
                return p.slab_flags ? launch_i8ws<MODE_STEP, true>(p, ctas, st) : launch_i8ws<MODE_STEP, false>(p, ctas, st);
            return p.slab_flags ? launch_i8ws<MODE_APPLY, true>(p, ctas, st) : launch_i8ws<MODE_APPLY, false>(p, ctas, st);
        }
    } else {   // M = 4 / 6 on the warp-specialised kernel: single contexts, undamped
        if (v == 3 && mode != MODE_DEBUG && !p.damped && !p.slab_flags)
            return mode == MODE_STEP ? launch_i8ws_b<MODE_STEP, false, false, false, M>(p, ctas, st)
                                     : launch_i8ws_b<MODE_APPLY, false, false, false, M>(p, ctas, st);
    }
    if (v == 2 && mode != MODE_DEBUG)
        return p.slab_flags ? launch_i8x_mode<M, true>(mode, p, ctas, st) : launch_i8x_mode<M, false>(mode, p, ctas, st);
    return v == 1 ? launch_i8_mode_g<M, I8W, false>(mode, p, ctas, st)
                  : launch_i8_mode_g<M, I8W, true>(mode, p, ctas, st);
}

template <int PATH, int MODE, bool DAMP = false>
cudaError_t launch_t(const StepParams &p, int64_t ctas, cudaStream_t st) {
    static unsigned attr = 0;
    const int smem = (int)sizeof(SmemV1<PATH>);
    if (!attr_done(attr)) {
        cudaError_t e = cudaFuncSetAttribute(step_v1<PATH, MODE, DAMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set(attr);
    }
    step_v1<PATH, MODE, DAMP><<<(unsigned)ctas, V1<PATH>::NT, smem, st>>>(p);
    return cudaGetLastError();
}

template <int MODE, bool DAMP, bool VF>
cudaError_t launch_f64(const StepParams &p, int64_t ctas, cudaStream_t st) {
    static unsigned attr = 0;
    const int smem = (int)sizeof(SmemF2);
    if (!attr_done(attr)) {
        cudaError_t e = cudaFuncSetAttribute(step_f64<MODE, DAMP, VF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set(attr);
    }
    step_f64<MODE, DAMP, VF><<<(unsigned)ctas, F2::NT, smem, st>>>(p);
    return cudaGetLastError();
}

template <int PATH>
cudaError_t launch_mode(int mode, const StepParams &p, int64_t ctas, cudaStream_t st) {
    if constexpr (PATH == OVX_FP64 || PATH == OVX_VFEM) {   // dedicated shuffle/register kernel;
        constexpr bool VF = PATH == OVX_VFEM;                   // debug records via step_v1
        if (mode == MODE_STEP)
            return p.damped ? launch_f64<MODE_STEP, true, VF>(p, ctas, st) : launch_f64<MODE_STEP, false, VF>(p, ctas, st);
        if (mode == MODE_APPLY) return launch_f64<MODE_APPLY, false, VF>(p, ctas, st);
    }
    if (mode == MODE_STEP)
        return p.damped ? launch_t<PATH, MODE_STEP, true>(p, ctas, st) : launch_t<PATH, MODE_STEP, false>(p, ctas, st);
    if (mode == MODE_APPLY) return launch_t<PATH, MODE_APPLY>(p, ctas, st);
    return launch_t<PATH, MODE_DEBUG>(p, ctas, st);
}

__global__ void node_w_kernel(int64_t nx, int64_t ny, int64_t nz, const uint8_t *__restrict__ mat,
                              const uint8_t *__restrict__ mat_below, const MatConst *__restrict__ mc, double dt,
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
                    if (ex < 0 || ex >= nx || ey < 0 || ey >= ny || ez >= nz) continue;
                    if (ez < 0) {   // element layer below the slab (z-slab halo), if any
                        if (mat_below) m = __dadd_rn(m, mc[mat_below[ex + nx * ey]].rho_vol8);
                        continue;
                    }
                    m = __dadd_rn(m, mc[mat[ex + nx * (ey + ny * ez)]].rho_vol8);
                }
        w[n] = __ddiv_rn(__dmul_rn(dt, dt), m);
    }
}

__global__ void finite_kernel(const double *__restrict__ u, int64_t n, int *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(u[i])) *flag = 1;
}

// z-chunk length (node planes per CTA).  Each CTA recomputes one halo layer below its chunk, and
// the grid runs in waves of (SMs × resident CTAs per SM); pick the chunk count n minimising
//   waves(n) × layers per CTA = ceil(tiles_xy·n / (SMs·cps)) × (ceil(planes/n) + 1)
// (fewest chunks on ties), with chunks of at least 8 planes.
int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return n;
}

int choose_zchunk(int64_t planes, int64_t tiles_xy, int ctas_per_sm) {
    static const int forced = [] {   // tuning knob (tools): OVX_ZCHUNKS=n forces n z-chunks
        const char *e = std::getenv("OVX_ZCHUNKS");
        return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) return (int)((planes + forced - 1) / forced);
    const int64_t slots = (int64_t)num_sms() * ctas_per_sm;
    const int64_t nmax = std::max<int64_t>(1, planes / 8);
    int64_t best_n = 1, best_cost = -1;
    for (int64_t n = 1; n <= nmax; ++n) {
        const int64_t len = (planes + n - 1) / n;
        const int64_t cost = ((tiles_xy * n + slots - 1) / slots) * (len + 1);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best_n = n;
        }
    }
    return (int)((planes + best_n - 1) / best_n);
}

template <int PATH>
LaunchInfo info_t(int64_t nx, int64_t ny, int64_t nz) {
    using C = V1<PATH>;
    LaunchInfo li;
    const int64_t tx = (nx + 1 + TX - 1) / TX, ty = (ny + 1 + C::TY - 1) / C::TY;
    const int zc = choose_zchunk(nz + 1, tx * ty, 2);
    li.ctas = tx * ty * ((nz + 1 + zc - 1) / zc);
    li.threads = C::NT;
    li.smem = (PATH == OVX_FP64 || PATH == OVX_VFEM) ? (int)sizeof(SmemF2) : (int)sizeof(SmemV1<PATH>);
    return li;
}

}  // namespace

cudaError_t upload_device_constants(const int8_t *k8, const double *kk2, const double *kg2) {
    cudaError_t e;
    if ((e = cudaMemcpyToSymbol(c_K8, k8, 1152))) return e;
    if ((e = cudaMemcpyToSymbol(c_Kk, kk2, 2 * 576 * 8))) return e;
    if ((e = cudaMemcpyToSymbol(c_Kg, kg2, 2 * 576 * 8))) return e;
    i8_bimg_kernel<<<1, 512>>>();    // the INT8 kernels' B-operand images from c_K8
    i8x_bimg_kernel<<<1, 512>>>();
    if ((e = cudaGetLastError())) return e;
    return cudaDeviceSynchronize();
}

LaunchInfo step_launch_info(int path, int64_t nx, int64_t ny, int64_t nz) {
    if (path == OVX_INT8) {
        LaunchInfo li;
        const int tx_ = I8W::TX, tyy = I8W::TY, cps = I8W::CPS;
        const int64_t tx = (nx + 1 + tx_ - 1) / tx_, ty = (ny + 1 + tyy - 1) / tyy;
        const int zc = choose_zchunk(nz + 1, tx * ty, cps);
        li.ctas = tx * ty * ((nz + 1 + zc - 1) / zc);
        li.threads = I8W::NT;
        li.smem = i8_variant() == 3 ? (i8_bulk_planes() ? (int)sizeof(SmemWST<true>) : (int)sizeof(SmemWS)) : i8_variant() == 2 ? (int)sizeof(SmemI8X)
                  : i8_variant() == 0 ? (int)sizeof(SmemI8<I8W, true>) : (int)sizeof(SmemI8<I8W, false>);
        return li;
    }
    if (path == OVX_FP64) return info_t<OVX_FP64>(nx, ny, nz);
    if (path == OVX_VFEM) return info_t<OVX_VFEM>(nx, ny, nz);
    return info_t<OVX_FP64_DENSE>(nx, ny, nz);
}

static cudaError_t launch_chunks(int path, int mode, StepParams p, cudaStream_t st, int c0, int c1) {
    if (c1 <= c0) return cudaSuccess;
    p.tz0 = c0;
    const int64_t ctas = (int64_t)p.tiles_x * p.tiles_y * (c1 - c0);
    if (path == OVX_INT8) {
        if (p.stages == 4) return launch_i8_mode<4>(mode, p, ctas, st);
        if (p.stages == 6) return launch_i8_mode<6>(mode, p, ctas, st);
        return launch_i8_mode<8>(mode, p, ctas, st);
    }
    if (path == OVX_FP64) return launch_mode<OVX_FP64>(mode, p, ctas, st);
    if (path == OVX_VFEM) return launch_mode<OVX_VFEM>(mode, p, ctas, st);
    return launch_mode<OVX_FP64_DENSE>(mode, p, ctas, st);   // OVX_FP64_DENSE and OVX_VFEM_DENSE (its matrices)
}

cudaError_t launch_step(int path, int mode, StepParams p, cudaStream_t st, int part, int *nlaunch) {
    const int ty = path == OVX_INT8 ? I8W::TY : V1<OVX_FP64>::TY;
    const int tx = path == OVX_INT8 ? I8W::TX : TX;
    const int cps = path == OVX_INT8 ? I8W::CPS : 2;
    p.tiles_x = (int)((p.nx + 1 + tx - 1) / tx);
    p.tiles_y = (int)((p.ny + 1 + ty - 1) / ty);
    p.zchunk = choose_zchunk(p.nz + 1, (int64_t)p.tiles_x * p.tiles_y, cps);
    const int n = (int)((p.nz + 1 + p.zchunk - 1) / p.zchunk);
    int cnt = 0;
    cudaError_t e = cudaSuccess;
    auto go = [&](int c0, int c1) {
        if (e == cudaSuccess && c1 > c0) {
            e = launch_chunks(path, mode, p, st, c0, c1);
            ++cnt;
        }
    };
    if (part < 0) {
        go(0, n);
    } else if (part == 0) {
        go(0, 1);
        if (n > 1) go(n - 1, n);
    } else {
        go(1, n - 1);
    }
    if (nlaunch) *nlaunch = cnt;
    return e;
}

cudaError_t launch_node_w(int64_t nx, int64_t ny, int64_t nz, const uint8_t *mat, const uint8_t *mat_below,
                          const MatConst *mc, double dt, double *w, cudaStream_t st) {
    node_w_kernel<<<1184, 256, 0, st>>>(nx, ny, nz, mat, mat_below, mc, dt, w);
    return cudaGetLastError();
}

// Interface plane (local plane 0) of a z-slab: f_n = T_n (the top-face sum received from the
// rank below) + B_n (this rank's layer-0 bottom-face sum), reading U2; then update.
__global__ void iface_update_kernel(const StepParams p, const double *__restrict__ a_recv, double *__restrict__ u_send) {
    const int64_t nn2 = (p.nx + 1) * (p.ny + 1);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nn2; j += (int64_t)gridDim.x * blockDim.x) {
        const double wn = p.w[j];
        const uint8_t dm = p.dmask ? p.dmask[j] : (uint8_t)0;
        for (int c = 0; c < 3; ++c) {
            const double f = __dadd_rn(a_recv[3 * j + c], p.iface_bot_b[3 * j + c]);
            const int64_t dof = 3 * j + c;
            double F = 0.0;
            for (int k = 0; k < p.nsrc; ++k)
                if (p.src_dof[k] == dof) F = __dadd_rn(F, p.src_val[k]);
            const double uc = p.u[dof], upc = p.uo[dof];
            double b = __dsub_rn(__dmul_rn(2.0, uc), upc);
            if (p.damped) b = __dsub_rn(b, __dmul_rn(p.ca, __dsub_rn(uc, upc)));   // reading R1
            double un = __fma_rn(wn, __dsub_rn(F, f), b);
            if ((dm >> c) & 1) un = 0.0;
            (p.damped ? p.un : p.uo)[dof] = un;
            u_send[dof] = un;
            if (p.it < p.rec_nt)
                for (int k = 0; k < p.nrec; ++k)
                    if (p.rec_node[k] == j) p.traces[(3 * k + c) * p.rec_nt + p.it] = un;
        }
    }
}

cudaError_t launch_iface_update(const StepParams &p, const double *a_recv, double *u_send, cudaStream_t st) {
    iface_update_kernel<<<296, 256, 0, st>>>(p, a_recv, u_send);
    return cudaGetLastError();
}

// Power iteration on M⁻¹K (ovx_critical_dt's dt_power_iter): given y = K x, accumulate the
// Rayleigh-quotient terms xᵀy, xᵀMx (M = dt²/w per node) and form z = M⁻¹y with fixed DOFs zeroed,
// with ‖z‖² for the normalisation.  acc: [xᵀKx, xᵀMx, zᵀz], doubles, zeroed by the caller.
__global__ void power_iter_kernel(int64_t nn, const double *__restrict__ x, const double *__restrict__ y,
                                  const double *__restrict__ w, const uint8_t *__restrict__ dmask, double dt2,
                                  double *__restrict__ z, double *__restrict__ acc) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nn; n += (int64_t)gridDim.x * blockDim.x) {
        const double minv = w[n] / dt2, m = dt2 / w[n];
        const uint8_t dm = dmask ? dmask[n] : 0;
        for (int k = 0; k < 3; ++k) {
            const double xi = x[3 * n + k], yi = y[3 * n + k];
            a += xi * yi;
            b += xi * m * xi;
            const double zi = ((dm >> k) & 1) ? 0.0 : minv * yi;
            z[3 * n + k] = zi;
            c += zi * zi;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, a);
        atomicAdd(acc + 1, b);
        atomicAdd(acc + 2, c);
    }
}
__global__ void scale_kernel(int64_t n, const double *__restrict__ z, const double *__restrict__ acc,
                             double *__restrict__ x) {
    const double s = 1.0 / sqrt(acc[2]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = z[i] * s;
}
cudaError_t launch_power_iter(int64_t nn, const double *x, const double *y, const double *w, const uint8_t *dmask,
                              double dt2, double *z, double *acc, double *xnext, cudaStream_t st) {
    power_iter_kernel<<<592, 256, 0, st>>>(nn, x, y, w, dmask, dt2, z, acc);
    scale_kernel<<<592, 256, 0, st>>>(3 * nn, z, acc, xnext);
    return cudaGetLastError();
}

cudaError_t launch_finite_check(const double *u, int64_t n, int *flag, cudaStream_t st) {
    finite_kernel<<<1184, 256, 0, st>>>(u, n, flag);
    return cudaGetLastError();
}

}  // namespace ovx

#ifdef OVX_TRACE
extern "C" int ovx_trace_read(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, ovx::g_tr, sizeof(unsigned long long) * TRH * 16 * TRN);
}
#endif
