/*
 * ovx_oracle.c — plain, slow, obviously-correct CPU oracle for the OVFEM /
 * TCOVFEM explicit time step (arxiv 2404.13683).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header or constant generator with the product library
 * (paper_2404_13683_b200/csrc); the integer element matrix it multiplies is
 * passed in from oracle/element.py (exact-rational derivation, also oracle).
 *
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math (see oracle/build.py)
 * -ffp-contract=off matters: every a*b+c below is two roundings unless fma()
 * is written explicitly.
 *
 * Numbering (PAPER.md L38 voxel grid; reading D1):
 *   node (ix,iy,iz) -> ix + (nx+1)*(iy + (ny+1)*iz)
 *   element (ex,ey,ez) -> ex + nx*(ey + ny*ez)
 * Local node order (reading Q1): (---),(+--),(++-),(-+-),(--+),(+-+),(+++),(-++).
 * DOF order inside an element vector: 3*local_node + axis.
 * Node arrays: 3 doubles per node, node-major xyz.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const int CX[8] = {0, 1, 1, 0, 0, 1, 1, 0};
static const int CY[8] = {0, 0, 1, 1, 0, 0, 1, 1};
static const int CZ[8] = {0, 0, 0, 0, 1, 1, 1, 1};

int64_t oracle_node_id(int64_t nx, int64_t ny, int64_t ix, int64_t iy, int64_t iz) {
    return ix + (nx + 1) * (iy + (ny + 1) * iz);
}

/* The 8 global node ids of element e in local order (Fig. 1 / reading Q1). */
void oracle_element_nodes(int64_t nx, int64_t ny, int64_t e, int64_t out[8]) {
    int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);
    for (int a = 0; a < 8; ++a)
        out[a] = oracle_node_id(nx, ny, ex + CX[a], ey + CY[a], ez + CZ[a]);
}

/* Per-node  w_n = dt^2 / m_n,  m_n = sum_{e ∋ n} rho_e ds^3 / 8  (Eq. 6;
 * reading Q15).  Masses are scattered in element order. */
void oracle_node_w(int64_t nx, int64_t ny, int64_t nz, double ds, const uint8_t *mat,
                   const double *rho, double dt, double *w) {
    int64_t nn = (nx + 1) * (ny + 1) * (nz + 1), ne = nx * ny * nz;
    double *m = (double *)calloc((size_t)nn, sizeof(double));
    double vol8 = ds * ds * ds / 8.0;
    int64_t nodes[8];
    for (int64_t e = 0; e < ne; ++e) {
        double me = rho[mat[e]] * vol8;
        oracle_element_nodes(nx, ny, e, nodes);
        for (int a = 0; a < 8; ++a) m[nodes[a]] += me;
    }
    for (int64_t n = 0; n < nn; ++n) w[n] = (dt * dt) / m[n];
    free(m);
}

/* ---------------------------------------------------------------------------
 * (i) FP64 path.  f_e = κ ds A_κ u_e + G ds A_G u_e  with A_κ = Kk/256 and
 * A_G = Kg/384, Kk = K^κ and Kg = K̄^G + 128 I  (DESIGN.md
 * oracle (i) step 3): the integer matrices are applied first (sequential
 * sums), then the two scalars.
 * ------------------------------------------------------------------------- */
void oracle_element_fp64(const double *ue, double kappa, double G, double ds,
                         const int32_t *Kk, const int32_t *Kg, double *fe) {
    double ck = kappa * ds / 256.0, cg = G * ds / 384.0;
    for (int r = 0; r < 24; ++r) {
        double a = 0.0, b = 0.0;
        for (int c = 0; c < 24; ++c) {
            a = a + (double)Kk[r * 24 + c] * ue[c];
            b = b + (double)Kg[r * 24 + c] * ue[c];
        }
        fe[r] = ck * a + cg * b;
    }
}

/* ---------------------------------------------------------------------------
 * (iii) VFEM (NEXT-3, the paper's conventional trilinear voxel element
 * with lumped mass): f_e = κ ds A_κ^V u_e + G ds A_G^V u_e with A_κ^V = Vk/72 and
 * A_G^V = Vg/216 (oracle/element.py derives Vk, Vg exactly); same operation order as (i).
 * ------------------------------------------------------------------------- */
void oracle_element_vfem(const double *ue, double kappa, double G, double ds,
                         const int32_t *Vk, const int32_t *Vg, double *fe) {
    double ck = kappa * ds / 72.0, cg = G * ds / 216.0;
    for (int r = 0; r < 24; ++r) {
        double a = 0.0, b = 0.0;
        for (int c = 0; c < 24; ++c) {
            a = a + (double)Vk[r * 24 + c] * ue[c];
            b = b + (double)Vg[r * 24 + c] * ue[c];
        }
        fe[r] = ck * a + cg * b;
    }
}

/* ---------------------------------------------------------------------------
 * (ii) Integer path (Eqs. 10-17), per element.
 *   digits == 0 : the paper's b = 2^7, M stages of signed 7-bit slices with a
 *                 signed top digit; v clamped to ±(2^(7M)-1) (reading Q9).
 *   digits == 1 : B200 byte slices: v' = v + 2^(7M), u8 digits b_j = byte j of v'
 *                 (DESIGN.md variant B).  No clamp is needed: v' < 2^64.
 * a = 2^(7M) (M = 8: a = 2^56, N = 1).
 * Outputs (any may be NULL): s, v[48], d[nd*48], C[nd*24] (nd = M for the 7-bit
 * digits, ceil((7M+1)/8) for bytes), y as two int64 halves of the int128
 * (y = y_hi*2^64 + (uint64)y_lo), fe[24].
 * Returns 0, or 1 if s is subnormal / non-finite (element treated as zero:
 * reading Q6').
 * ------------------------------------------------------------------------- */
/* Digit expansion of one INT64 value (Eq. 16).
 *   digits == 0: d_j = (v >> 7(j-1)) & 127 for j < M, top digit d_M = v >> 7(M-1)
 *                (arithmetic shift), so v = Σ_j 2^{7(j-1)} d_j with d_j ∈ [-128,127]
 *                (two's-complement 7-bit slices, reading Q10).  Requires |v| < 2^{7M}.
 *   digits == 1: bytes of v' = v + 2^{7M}: d_j = (v' >> 8(j-1)) & 255, j = 1..ceil((7M+1)/8);
 *                v = Σ_j 256^{j-1} d_j − 2^{7M} (variant B).  Requires |v| ≤ 2^{7M}+2^6. */
void oracle_digits(int64_t v, int M, int digits, int32_t *d) {
    int nbits = 7 * M;
    if (!digits) {
        for (int j = 0; j < M; ++j)
            d[j] = (j < M - 1) ? (int32_t)((v >> (7 * j)) & 127) : (int32_t)(v >> (7 * j));
    } else {
        int nd = (nbits + 1 + 7) / 8;
        uint64_t vp = (uint64_t)(v + ((int64_t)1 << nbits));
        for (int j = 0; j < nd; ++j) d[j] = (int32_t)((vp >> (8 * j)) & 255u);
    }
}

int oracle_element_int8(const double *ue, double kappa, double G, double ds,
                        const int8_t *K8 /*24x48 row-major*/, int M, int digits,
                        double *s_out, int64_t *v_out, int32_t *d_out, int64_t *C_out,
                        int64_t *y_hi, int64_t *y_lo, double *fe) {
    /* digits bit 1 ("fold", DESIGN.md variant D): the Eq. 9 diagonal term (256/3)(G/κ)u_e =
     * 128·ū_{e,G} is taken in the integer domain, y_D = K_D v with K_D = [K^κ | K̄^G + 128 I]
     * (= [256 A_κ | 384 A_G]), and f_e = RN(c1s·RN(y_D)), c1s = RN(c1·RN(s_e·2^-56)). */
    /* digits bit 2 ("direct", Fig. 2 left; Eqs. 11-14 with a = 2^7, N = M stages): every
     * stage converts the FP64 remainder to an INT8 digit, d_i = INT(a·r_{i-1}), r_i = a·r_{i-1} − d_i
     * (r_0 = ū_es; each step exact in FP64), digits clamped to ±127 (reading Q9 for |x| = 1: the
     * residual then carries 127 into every later stage, i.e. ±(2^{7M}−1) as in the paper-digit
     * hierarchical path).  y = Σ_i a^{N−i} K d_i.  Stored lowest weight first (dall[k][0] = d_N). */
    const int direct = (digits >> 2) & 1;
    const int fold = (digits >> 1) & 1;
    digits &= 1;
    if (direct) digits = 0;
    double cG = (2.0 * G) / (3.0 * kappa);       /* (2/3) G/κ, */
    double c1 = kappa * ds / 256.0;              /* κ ds / 256, Eq. 9          */
    double c2 = (256.0 * G) / (3.0 * kappa);     /* (256/3) G/κ, Eq. 9         */
    int nbits = 7 * M;
    int64_t A = (int64_t)1 << nbits;             /* a = 2^(7M) as an integer   */
    double Ad = ldexp(1.0, nbits);
    int nd = digits ? (nbits + 1 + 7) / 8 : M;

    double ub[48];
    for (int i = 0; i < 24; ++i) { ub[i] = ue[i]; ub[24 + i] = cG * ue[i]; }
    /* Eq. 10: s_e = max_i |ū_ei| */
    double s = 0.0;
    for (int i = 0; i < 48; ++i) { double t = fabs(ub[i]); if (t > s) s = t; }
    if (s_out) *s_out = s;
    int64_t v[48];
    __int128 y[24];
    int degenerate = !(s >= 0x1p-1022) || !isfinite(s);
    if (degenerate) {
        for (int i = 0; i < 48; ++i) v[i] = 0;
    } else {
        double r = 1.0 / s;                      /* reading Q7: one reciprocal  */
        for (int i = 0; i < 48; ++i) {
            double x = ub[i] * r;                /* ū_es, Eq. 10                */
            if (direct) {
                double rr = x;
                int64_t V = 0;
                for (int st = 0; st < M; ++st) {
                    double t = 128.0 * rr;       /* a·r_{i-1}, exact                 */
                    int64_t d = (int64_t)t;      /* INT(·): truncation toward 0 (Q8) */
                    if (d > 127) d = 127;
                    if (d < -127) d = -127;
                    rr = t - (double)d;          /* r_i, exact (Sterbenz)            */
                    V = V * 128 + d;
                }
                v[i] = V;
                continue;
            }
            double t = x * Ad;                   /* exact power-of-two scaling  */
            v[i] = (int64_t)t;                   /* truncation toward 0, Eq. 12 (Q8) */
            if (!digits) {                       /* reading Q9 clamp            */
                if (v[i] > A - 1) v[i] = A - 1;
                if (v[i] < -(A - 1)) v[i] = -(A - 1);
            }
        }
    }
    if (v_out) memcpy(v_out, v, sizeof v);
    for (int r = 0; r < 24; ++r) y[r] = 0;
    int32_t dall[48][8];
    if (direct) {   /* the digits of the direct recursion, recomputed (lowest weight first) */
        double r = degenerate ? 0.0 : 1.0 / s;
        for (int k = 0; k < 48; ++k) {
            double rr = degenerate ? 0.0 : ub[k] * r;
            int32_t tmp[8];
            for (int st = 0; st < M; ++st) {
                double t = 128.0 * rr;
                int64_t d = (int64_t)t;
                if (d > 127) d = 127;
                if (d < -127) d = -127;
                rr = t - (double)d;
                tmp[st] = (int32_t)d;
            }
            for (int st = 0; st < M; ++st) dall[k][st] = tmp[M - 1 - st];
        }
    } else {
        for (int k = 0; k < 48; ++k) oracle_digits(v[k], M, digits, dall[k]);
    }
    for (int j = 0; j < nd; ++j) {
        int32_t d[48];
        for (int k = 0; k < 48; ++k) {
            d[k] = dall[k][j];
            if (d_out) d_out[j * 48 + k] = d[k];
        }
        for (int r = 0; r < 24; ++r) {
            int64_t c = 0;                       /* Eq. 17: K_e^INT8 · digits_j   */
            for (int k = 0; k < 48; ++k) c += (int64_t)K8[r * 48 + k] * d[k];
            if (fold) c += 128 * (int64_t)d[24 + r];   /* + 128 I on the G block */
            if (C_out) C_out[j * 24 + r] = c;
            __int128 w = digits ? ((__int128)1 << (8 * j)) : ((__int128)1 << (7 * j));
            y[r] += w * (__int128)c;
        }
    }
    if (digits) {
        /* K_e^INT8 · (a·1) = a · rowsum; subtract it back:  y = K v' − a K 1 */
        for (int r = 0; r < 24; ++r) {
            int64_t rs = fold ? 128 : 0;
            for (int k = 0; k < 48; ++k) rs += K8[r * 48 + k];
            y[r] -= (__int128)A * (__int128)rs;
        }
    }
    double sig = s * ldexp(1.0, -nbits);         /* s_e / a (Eq. 15)              */
    for (int r = 0; r < 24; ++r) {
        if (y_hi) y_hi[r] = (int64_t)(y[r] >> 64);
        if (y_lo) y_lo[r] = (int64_t)(uint64_t)y[r];
        if (fe) {
            double Y = degenerate ? 0.0 : (double)y[r];  /* RN(y), one rounding (Q13) */
            if (fold) {
                fe[r] = degenerate ? 0.0 : (c1 * sig) * Y;
            } else {
                double a = Y * sig;
                double b = c2 * ue[r];
                fe[r] = degenerate ? 0.0 : c1 * (a + b);    /* Eq. 9, literal order */
            }
        }
    }
    return degenerate;
}

/* f = Σ_e scatter(K_e u_e) (Eq. 2 assembled element by element; SURVEY
 * §8(c)(i) step 4).  The paper adds element results straight into the global vector (atomics, order
 * unspecified); the DEFINITION used here is the plain one:
 *
 *   order == ORDER_ELEMENT (0):  f = +0.0;  for e = 0 .. E-1 (element id order),
 *                                for local node a = 0 .. 7, for axis c = 0 .. 2:
 *                                    f[3·node_a(e) + c] += fe_e[3a + c].
 *
 * order == ORDER_ABS (2) is not a product: Σ_e |f_e[n]| (element order), the scale of the rounding
 * bound  |Σ in one order − Σ in another| ≤ 2·γ_7·Σ_e |f_e[n]|  that tests use across orders.
 * order == ORDER_U2 (1) is a MIRROR VARIANT, not the definition: the per-node pairwise tree the
 * B200 kernels sum in (reading U2), kept so that tests can also compare the kernels bit
 * for bit.  Any two orders differ only by the rounding of an 8-term sum (≤ 2·γ_7·Σ|terms|):
 *   f_n = T_n + B_n,  T_n = face(iz-1, top corners),  B_n = face(iz, bottom corners),
 *   face(ez, z) = P(iy) + P(iy-1),
 *   P(iy)   = f(ix, iy,   ez)[(-x,-y,z)] + f(ix-1, iy,   ez)[(+x,-y,z)],
 *   P(iy-1) = f(ix, iy-1, ez)[(-x,+y,z)] + f(ix-1, iy-1, ez)[(+x,+y,z)],
 * where a missing element (outside the grid) contributes 0.0.
 * path 0: FP64 (Kk, Kg);  path 1: integer path (K8, M, digits);  path 2: VFEM (Kk, Kg hold
 * the VFEM integer matrices Vk, Vg). */
static double face_sum(const double *fe_all, int64_t nx, int64_t ny, int64_t nz, int64_t ix, int64_t iy,
                       int64_t ez, int top, int c) {
    /* corner (local node) of element (ix - dx, iy - dy) that is node (ix, iy): Q1 order */
    static const int CORNER[2][2] = {{0, 1}, {3, 2}};   /* [dy][dx] */
    double v[2][2];
    for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
            int64_t ex = ix - dx, ey = iy - dy;
            v[dy][dx] = 0.0;
            if (ex >= 0 && ex < nx && ey >= 0 && ey < ny && ez >= 0 && ez < nz) {
                int64_t e = ex + nx * (ey + ny * ez);
                v[dy][dx] = fe_all[24 * e + 3 * (CORNER[dy][dx] + 4 * top) + c];
            }
        }
    double p0 = v[0][0] + v[0][1];   /* P(iy)   */
    double p1 = v[1][0] + v[1][1];   /* P(iy-1) */
    return p0 + p1;
}

/* Element forces of every element (f_e of the chosen path), 24 per element in element id order. */
static double *element_forces_all(int64_t nx, int64_t ny, int64_t nz, double ds, const uint8_t *mat,
                                  const double *kappa, const double *G, int path,
                                  const int32_t *Kk, const int32_t *Kg, const int8_t *K8, int M, int digits,
                                  const double *u) {
    int64_t ne = nx * ny * nz;
    double *fe_all = (double *)malloc(sizeof(double) * 24 * (size_t)(ne > 0 ? ne : 1));
    /* The element forces are independent of each other (each depends only on u_e); OpenMP may
     * compute them on several host threads (OMP_NUM_THREADS; 1 = the plain serial loop) — the
     * arithmetic of every element and the summations are unchanged, so the result is the same
     * bits for any thread count. */
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; ++e) {
        int64_t en[8];
        double ue[24];
        oracle_element_nodes(nx, ny, e, en);
        for (int a = 0; a < 8; ++a)
            for (int c = 0; c < 3; ++c) ue[3 * a + c] = u[3 * en[a] + c];
        int m = mat[e];
        if (path == 0) oracle_element_fp64(ue, kappa[m], G[m], ds, Kk, Kg, fe_all + 24 * e);
        else if (path == 2) oracle_element_vfem(ue, kappa[m], G[m], ds, Kk, Kg, fe_all + 24 * e);
        else oracle_element_int8(ue, kappa[m], G[m], ds, K8, M, digits,
                                 NULL, NULL, NULL, NULL, NULL, NULL, fe_all + 24 * e);
    }
    return fe_all;
}

/* Scatter of the element forces into node forces in one order (0 element, 1 U2 mirror, 2 |·| bound). */
static void scatter(int64_t nx, int64_t ny, int64_t nz, const double *fe_all, int order, double *f) {
    int64_t ne = nx * ny * nz, nn = (nx + 1) * (ny + 1) * (nz + 1);
    int64_t nodes[8];
    if (order == 0 || order == 2) {       /* the definition: element order (2: magnitudes) */
        for (int64_t i = 0; i < 3 * nn; ++i) f[i] = 0.0;
        for (int64_t e = 0; e < ne; ++e) {
            oracle_element_nodes(nx, ny, e, nodes);
            for (int a = 0; a < 8; ++a)
                for (int c = 0; c < 3; ++c) {
                    double t = fe_all[24 * e + 3 * a + c];
                    f[3 * nodes[a] + c] += order == 2 ? fabs(t) : t;
                }
        }
    } else {                              /* mirror variant U2 */
        for (int64_t iz = 0; iz <= nz; ++iz)
            for (int64_t iy = 0; iy <= ny; ++iy)
                for (int64_t ix = 0; ix <= nx; ++ix) {
                    int64_t n = oracle_node_id(nx, ny, ix, iy, iz);
                    for (int c = 0; c < 3; ++c) {
                        double T = face_sum(fe_all, nx, ny, nz, ix, iy, iz - 1, 1, c);
                        double B = face_sum(fe_all, nx, ny, nz, ix, iy, iz, 0, c);
                        f[3 * n + c] = T + B;
                    }
                }
    }
}

void oracle_apply_K(int64_t nx, int64_t ny, int64_t nz, double ds, const uint8_t *mat,
                    const double *kappa, const double *G, int path,
                    const int32_t *Kk, const int32_t *Kg, const int8_t *K8, int M, int digits,
                    int order, const double *u, double *f) {
    double *fe_all = element_forces_all(nx, ny, nz, ds, mat, kappa, G, path, Kk, Kg, K8, M, digits, u);
    scatter(nx, ny, nz, fe_all, order, f);
    free(fe_all);
}

/* The three scatters of one set of element forces (any output may be NULL): the definition
 * (element order), the U2 mirror, and the |·| bound scale — one element pass for all three. */
void oracle_apply_K3(int64_t nx, int64_t ny, int64_t nz, double ds, const uint8_t *mat,
                     const double *kappa, const double *G, int path,
                     const int32_t *Kk, const int32_t *Kg, const int8_t *K8, int M, int digits,
                     const double *u, double *f_elem, double *f_u2, double *f_abs) {
    double *fe_all = element_forces_all(nx, ny, nz, ds, mat, kappa, G, path, Kk, Kg, K8, M, digits, u);
    if (f_elem) scatter(nx, ny, nz, fe_all, 0, f_elem);
    if (f_u2) scatter(nx, ny, nz, fe_all, 1, f_u2);
    if (f_abs) scatter(nx, ny, nz, fe_all, 2, f_abs);
    free(fe_all);
}

/* Central-difference time stepping (Eq. 3, update L263-L266 with the
 * sign of Eq. 3: F − K u, reading Q14):
 *   u^{it+1} = fma(w, F^{it} − f, 2 u^{it} − u^{it−1}),  f = K u^{it},  w = dt²/m
 * Rayleigh damping ("Rayleigh damping (100–125 kHz) is used"; reading R1,
 * the SPEC's backward-difference velocity v = (u − u_prev)/dt so the update stays explicit),
 * one (alpha, beta) for the model, C = alpha M + beta K:
 *   u^{it+1} = 2u − u_prev + dt² M⁻¹ (F − K u − C v)
 *            = fma(w, F − K ũ, (2u − u_prev) − ca·d),  d = u − u_prev,
 *   ũ = u + cb·d,  ca = alpha·dt,  cb = beta/dt   (each operation rounded once, in this order).
 * alpha = beta = 0 takes the undamped branch (identical results).
 * Dirichlet: bit a of dmask[n] set -> component a forced to 0 after the update.
 * Sources: src_node[k], src_axis[k], amplitude amp[k*n_t + it] (0 beyond n_t).
 * u and u_prev are advanced in place; *it is incremented per step.
 * Returns 0, or 3 if a non-finite value appeared (the step index is in *it). */
int oracle_run(int64_t nx, int64_t ny, int64_t nz, double ds, const uint8_t *mat,
               const double *kappa, const double *G, const double *w, const uint8_t *dmask,
               int path, const int32_t *Kk, const int32_t *Kg, const int8_t *K8, int M, int digits,
               int order, int nsrc, const int64_t *src_node, const int32_t *src_axis, int64_t n_t,
               const double *amp, double dt, double alpha, double beta,
               double *u, double *u_prev, int64_t *it, int64_t nsteps) {
    int64_t nn = (nx + 1) * (ny + 1) * (nz + 1);
    double *f = (double *)malloc(sizeof(double) * 3 * (size_t)nn);
    double *F = (double *)calloc(3 * (size_t)nn, sizeof(double));
    int damped = (alpha != 0.0 || beta != 0.0);
    double ca = alpha * dt, cb = beta / dt;
    double *ut = damped ? (double *)malloc(sizeof(double) * 3 * (size_t)nn) : NULL;
    int status = 0;
    for (int64_t step = 0; step < nsteps; ++step) {
        if (damped) {
            for (int64_t i = 0; i < 3 * nn; ++i) {
                double d = u[i] - u_prev[i];
                ut[i] = u[i] + cb * d;
            }
            oracle_apply_K(nx, ny, nz, ds, mat, kappa, G, path, Kk, Kg, K8, M, digits, order, ut, f);
        } else {
            oracle_apply_K(nx, ny, nz, ds, mat, kappa, G, path, Kk, Kg, K8, M, digits, order, u, f);
        }
        for (int k = 0; k < nsrc; ++k)
            F[3 * src_node[k] + src_axis[k]] += (*it < n_t) ? amp[(int64_t)k * n_t + *it] : 0.0;
        for (int64_t n = 0; n < nn; ++n) {
            for (int c = 0; c < 3; ++c) {
                int64_t i = 3 * n + c;
                double b = 2.0 * u[i] - u_prev[i];
                if (damped) {
                    double d = u[i] - u_prev[i];
                    b = b - ca * d;
                }
                double un = fma(w[n], F[i] - f[i], b);
                if (dmask && (dmask[n] >> c) & 1) un = 0.0;
                if (!isfinite(un)) status = 3;
                u_prev[i] = u[i];
                u[i] = un;
            }
        }
        for (int k = 0; k < nsrc; ++k) F[3 * src_node[k] + src_axis[k]] = 0.0;
        *it += 1;
        if (status) break;
    }
    free(f);
    free(F);
    free(ut);
    return status;
}

/* Central-difference update of n DOFs (Eq. 3): up[i] <- fma(w[i], F[i] - f[i], 2u[i] - up[i]).
 * Used by the z-slab protocol emulation in the tests. */
void oracle_update_dofs(int64_t n, const double *w, const double *F, const double *f, const double *u,
                        double *up) {
    for (int64_t i = 0; i < n; ++i) {
        double b = 2.0 * u[i] - up[i];
        up[i] = fma(w[i], F[i] - f[i], b);
    }
}
