// element_setup.cpp — host-side (L1) derivation of the constant OVFEM element data.
//
// K_e^INT8 = (K_e^κ, K̄_e^G) is derived here in exact rational
// arithmetic from Eqs. 5, 7, 8 (L66-L89) under DESIGN.md reading Q3 (∂φ/∂r_i is a
// Dirac delta on the mid-plane r_i = 0), then checked to be an integer matrix with
// entries in [-128, 127] (L110).  This is the product's own derivation; the oracle
// derives the same matrix independently (oracle/element.py) and the tests compare
// both against tests/golden/k_int8.csv.
#include <cstdint>
#include <cstdlib>
#include <cmath>

namespace ovx {

namespace {

struct Q {  // exact rational num/den, den > 0, reduced
    int64_t n, d;
};

int64_t gcd64(int64_t a, int64_t b) {
    a = a < 0 ? -a : a;
    b = b < 0 ? -b : b;
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a ? a : 1;
}
Q mk(int64_t n, int64_t d = 1) {
    if (d < 0) { n = -n; d = -d; }
    int64_t g = gcd64(n, d);
    return Q{n / g, d / g};
}
Q add(Q a, Q b) { return mk(a.n * b.d + b.n * a.d, a.d * b.d); }
Q mul(Q a, Q b) { return mk(a.n * b.n, a.d * b.d); }
Q dvd(Q a, Q b) { return mk(a.n * b.d, a.d * b.n); }

// corner signs r̄ of local nodes (reading Q1)
const int SG[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                      {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
// ψ modes as exponents of (r1, r2, r3) (Eq. 8)
const int PE[7][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {0, 1, 1}, {1, 0, 1}};
// Voigt pairs xx,yy,zz,xy,yz,zx
const int VP[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {1, 2}, {2, 0}};

// (ψ^β ∂_{x_i} φ^α)_e for ds = 1:  (1/2)^3 (2) r̄_i ∫∫_quadrant ψ(r_i = 0)
Q psi_dphi(int b, int i, int a) {
    if (PE[b][i]) return mk(0);
    Q q = mk(1);
    for (int j = 0; j < 3; ++j) {
        if (j == i) continue;
        // ∫ r^e over the half interval of sign r̄_j: e = 0 -> 1, e = 1 -> r̄_j / 2
        q = mul(q, PE[b][j] ? mk(SG[a][j], 2) : mk(1));
    }
    return mul(mk(SG[a][i], 4), q);
}

}  // namespace

// Returns 0 on success, -1 if an entry is not an INT8 integer (PAPER.md L110 violated).
// Ak, Ag (24x24, may be null): A_κ, A_G with K_e^o = κ ds A_κ + G ds A_G.
int derive_element_matrices(int8_t *k8 /*24x48*/, double *Ak, double *Ag) {
    Q B[7][6][24];
    for (int b = 0; b < 7; ++b)
        for (int s = 0; s < 6; ++s)
            for (int c = 0; c < 24; ++c) B[b][s][c] = mk(0);
    for (int b = 0; b < 7; ++b)
        for (int s = 0; s < 6; ++s) {
            int p = VP[s][0], q = VP[s][1];
            for (int a = 0; a < 8; ++a) {
                if (p == q) {
                    B[b][s][3 * a + p] = add(B[b][s][3 * a + p], psi_dphi(b, p, a));
                } else {  // engineering shear γ_pq = ∂_q u_p + ∂_p u_q
                    B[b][s][3 * a + p] = add(B[b][s][3 * a + p], psi_dphi(b, q, a));
                    B[b][s][3 * a + q] = add(B[b][s][3 * a + q], psi_dphi(b, p, a));
                }
            }
        }
    // Gram diagonal (ψψ')_e for ds = 1
    const Q gram[7] = {mk(1), mk(1, 3), mk(1, 3), mk(1, 3), mk(1, 9), mk(1, 9), mk(1, 9)};
    // c = κ Cκ + G CG (Voigt, engineering shear)
    Q Ck[6][6], Cg[6][6];
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
            Ck[i][j] = mk((i < 3 && j < 3) ? 1 : 0);
            if (i < 3 && j < 3) Cg[i][j] = (i == j) ? mk(4, 3) : mk(-2, 3);
            else Cg[i][j] = mk(i == j ? 1 : 0);
        }
    int bad = 0;
    for (int r = 0; r < 24; ++r)
        for (int c = 0; c < 24; ++c) {
            Q ak = mk(0), ag = mk(0);
            for (int b = 0; b < 7; ++b) {
                Q sk = mk(0), sg = mk(0);
                for (int s = 0; s < 6; ++s)
                    for (int t = 0; t < 6; ++t) {
                        if (B[b][s][r].n == 0 || B[b][t][c].n == 0) continue;
                        Q bb = mul(B[b][s][r], B[b][t][c]);
                        sk = add(sk, mul(bb, Ck[s][t]));
                        sg = add(sg, mul(bb, Cg[s][t]));
                    }
                ak = add(ak, dvd(sk, gram[b]));
                ag = add(ag, dvd(sg, gram[b]));
            }
            Q kk = mul(ak, mk(256));
            Q kg = add(mul(ag, mk(384)), mk(r == c ? -128 : 0));
            if (kk.d != 1 || kg.d != 1 || kk.n < -128 || kk.n > 127 || kg.n < -128 || kg.n > 127) bad = 1;
            if (k8) {
                k8[r * 48 + c] = (int8_t)kk.n;
                k8[r * 48 + 24 + c] = (int8_t)kg.n;
            }
            if (Ak) Ak[r * 24 + c] = (double)ak.n / (double)ak.d;
            if (Ag) Ag[r * 24 + c] = (double)ag.n / (double)ag.d;
        }
    return bad ? -1 : 0;
}

// Largest eigenvalue of a symmetric 24x24 matrix by power iteration with a shift-free
// Rayleigh quotient (the matrix is PSD).  Used for the element-bound stability limit.
double sym_lambda_max(const double *A) {
    double x[24], y[24];
    for (int i = 0; i < 24; ++i) x[i] = 1.0 + 0.01 * i * ((i % 3) - 1);
    double lam = 0.0;
    for (int it = 0; it < 2000; ++it) {
        double nrm = 0.0;
        for (int i = 0; i < 24; ++i) {
            double s = 0.0;
            for (int j = 0; j < 24; ++j) s += A[i * 24 + j] * x[j];
            y[i] = s;
            nrm += s * s;
        }
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) return 0.0;
        double num = 0.0, den = 0.0;
        for (int i = 0; i < 24; ++i) { num += x[i] * y[i]; den += x[i] * x[i]; }
        lam = num / den;
        for (int i = 0; i < 24; ++i) x[i] = y[i] / nrm;
    }
    return lam;
}

// VFEM (NEXT-3): the conventional trilinear voxel element.  φ^a = Π_j (1 + r̄_j^a r_j)/2
// on r ∈ [-1,1]³; K_e^V = ∫ Bᵀ c B dv, integrated exactly here (the paper's 2×2×2 Gauss rule is
// exact for this integrand): with λ = κ − 2G/3, μ = G and g_ab[i][k] = ∫ ∂_i φ^a ∂_k φ^b dv,
//   K[3a+p][3b+q] = λ g[p][q] + μ (g[q][p] + δ_pq Σ_r g[r][r]).
// Written as K_e^V = κ ds Vk/72 + G ds Vg/216 with integer Vk, Vg (checked).  Lumped mass ρ ds³/8 per
// node, the same as OVFEM.  Returns 0, or -1 if an entry is not an integer.
int derive_vfem_matrices(double *Vk /*24x24*/, double *Vg /*24x24*/) {
    Q g[8][8][3][3];
    for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b)
            for (int i = 0; i < 3; ++i)
                for (int k = 0; k < 3; ++k) {
                    // ds = 1: ∂_i φ^a = r̄_i^a Π_{j≠i} (1 + r̄_j^a r_j)/2, dv = dr/8
                    Q v = mul(mk(SG[a][i] * SG[b][k]), mk(1, 8));
                    for (int j = 0; j < 3; ++j) {
                        const bool fa = j != i, fb = j != k;
                        if (fa && fb)      // ∫ (1 + s r)(1 + t r)/4 dr = (1 + st/3)/2
                            v = mul(v, mul(add(mk(1), mk(SG[a][j] * SG[b][j], 3)), mk(1, 2)));
                        else if (!fa && !fb)
                            v = mul(v, mk(2));   // ∫ dr
                        // exactly one factor present: ∫ (1 + s r)/2 dr = 1
                    }
                    g[a][b][i][k] = v;
                }
    for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b) {
            const Q tr = add(add(g[a][b][0][0], g[a][b][1][1]), g[a][b][2][2]);
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) {
                    const Q lam = g[a][b][p][q];
                    Q mu = g[a][b][q][p];
                    if (p == q) mu = add(mu, tr);
                    const Q kk = mul(lam, mk(72));                                  // κ part × 72
                    const Q gg = mul(add(mu, mul(mk(-2, 3), lam)), mk(216));        // G part × 216
                    if (kk.d != 1 || gg.d != 1) return -1;
                    Vk[(3 * a + p) * 24 + 3 * b + q] = (double)kk.n;
                    Vg[(3 * a + p) * 24 + 3 * b + q] = (double)gg.n;
                }
        }
    return 0;
}

}  // namespace ovx
