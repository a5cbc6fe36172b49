"""OVFEM element data derived in exact rational arithmetic.

TEST INFRASTRUCTURE — part of the oracle. Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` legs may import this
module. The product path (paper_2404_13683_b200/) never imports it and shares no
code with it.

Everything here follows PAPER.md (arxiv 2404.13683) step by step, in exact
rationals (`fractions.Fraction`), so a reader can check it against the paper:

* Local frame, local node numbering and corner signs  r̄^α   — PAPER.md L42, L53-L58
  (Fig. 1 is missing; reading Q1 in DESIGN.md fixes the order).
* Displacement basis  φ^β = H(r̄1 r1) H(r̄2 r2) H(r̄3 r3)      — PAPER.md L76-L79 (Eq. 7)
* Stress basis  ψ = {1, r1, r2, r3, r1 r2, r2 r3, r1 r3}       — PAPER.md L80-L89 (Eq. 8)
* K_e^o = (ψ∇φ)ᵀ_e (ψψ')⁻¹_e c (ψ∇φ)_e                        — PAPER.md L66-L69 (Eq. 5)
* M_e^o = ρ (φ^β φ^β')_e  (diagonal)                            — PAPER.md L70-L74 (Eq. 6)
* κ/G split, K_e^INT8 = (K_e^κ, K̄_e^G) with K̄^G = ... − 128 I   — PAPER.md L94-L103
* Eq. 9:  K_e^o u_e = (κ ds/256)(K_e^INT8 ū_e + (256/3)(G/κ) u_e) — PAPER.md L104-L108

Reading Q3: ∂φ/∂r_i of the Heaviside basis is the Dirac delta on the
element mid-plane r_i = 0 (element faces carry no jump because the global field
is piecewise constant on node dual cells).  Under this reading

    (ψ^β ∂_i φ^α)_e = (ds/2)^3 (2/ds) r̄_i^α  ∫∫_{quadrant α} ψ^β(r_i = 0) dr_j dr_k ,

which the tests pin against an independent integration-by-parts evaluation.
"""
from __future__ import annotations

from fractions import Fraction as Fr
from itertools import product

# Local node α -> corner signs (r̄1, r̄2, r̄3).  Reading Q1: counter-clockwise on
# the bottom face r3 = -1, then the same on the top face r3 = +1.
CORNERS = [(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1),
           (-1, -1, 1), (1, -1, 1), (1, 1, 1), (-1, 1, 1)]

# Stress modes ψ^β as exponent tuples (e1, e2, e3) of r1^e1 r2^e2 r3^e3 (Eq. 8).
PSI = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 1, 1), (1, 0, 1)]

# Voigt order of stress/strain components (reading Q5), engineering shear.
VOIGT = [(0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (2, 0)]


def _int_monomial_half(e: int, sign: int) -> Fr:
    """∫ r^e dr over the half interval [0,1] (sign=+1) or [-1,0] (sign=-1)."""
    # ∫_0^1 r^e = 1/(e+1);  ∫_{-1}^0 r^e = (-1)^e/(e+1)
    return Fr(sign ** e, e + 1)


def _int_monomial_full(e: int) -> Fr:
    """∫_{-1}^{1} r^e dr."""
    return Fr(0) if e % 2 else Fr(2, e + 1)


def psi_grad_phi(ds: Fr = Fr(1)) -> list[list[list[Fr]]]:
    """P[β][i][α] = (ψ^β ∂_{x_i} φ^α)_e  (Eq. 5 factor, reading Q3).

    ∂_{x_i} = (2/ds) ∂_{r_i};  dv = (ds/2)^3 dr1 dr2 dr3;
    ∂_{r_i} H(r̄_i r_i) = r̄_i δ(r_i).
    """
    ds = Fr(ds)
    P = [[[Fr(0)] * 8 for _ in range(3)] for _ in range(len(PSI))]
    for b, ex in enumerate(PSI):
        for i in range(3):
            for a, rb in enumerate(CORNERS):
                if ex[i] != 0:          # ψ vanishes on the plane r_i = 0
                    continue
                q = Fr(1)
                for j in range(3):
                    if j != i:
                        q *= _int_monomial_half(ex[j], rb[j])
                P[b][i][a] = (ds / 2) ** 3 * (2 / ds) * rb[i] * q
    return P


def psi_gram(ds: Fr = Fr(1)) -> list[Fr]:
    """Diagonal of the Gram matrix (ψ^β ψ^β')_e (Eq. 5); off-diagonals vanish by parity."""
    ds = Fr(ds)
    g = []
    for ex in PSI:
        v = Fr(1)
        for j in range(3):
            v *= _int_monomial_full(2 * ex[j])
        g.append((ds / 2) ** 3 * v)
    return g


def psi_gram_full(ds: Fr = Fr(1)) -> list[list[Fr]]:
    """Full 7×7 Gram matrix, to check the off-diagonal zeros."""
    ds = Fr(ds)
    n = len(PSI)
    Gm = [[Fr(0)] * n for _ in range(n)]
    for b1 in range(n):
        for b2 in range(n):
            v = Fr(1)
            for j in range(3):
                v *= _int_monomial_full(PSI[b1][j] + PSI[b2][j])
            Gm[b1][b2] = (ds / 2) ** 3 * v
    return Gm


def strain_matrix(ds: Fr = Fr(1)) -> list[list[list[Fr]]]:
    """B[β] (6×24): Voigt strain (engineering shear) of mode β from u_e.

    DOF order: 3·α + c (node-major, xyz within node) — reading Q5.
    """
    P = psi_grad_phi(ds)
    B = []
    for b in range(len(PSI)):
        Bb = [[Fr(0)] * 24 for _ in range(6)]
        for s, (p, q) in enumerate(VOIGT):
            for a in range(8):
                if p == q:          # ε_pp = ∂_p u_p
                    Bb[s][3 * a + p] += P[b][p][a]
                else:               # γ_pq = ∂_q u_p + ∂_p u_q
                    Bb[s][3 * a + p] += P[b][q][a]
                    Bb[s][3 * a + q] += P[b][p][a]
        B.append(Bb)
    return B


def c_kappa() -> list[list[Fr]]:
    """∂c/∂κ in Voigt form: ones(3×3) ⊕ 0   (isotropic c = κ C_κ + G C_G)."""
    C = [[Fr(0)] * 6 for _ in range(6)]
    for i in range(3):
        for j in range(3):
            C[i][j] = Fr(1)
    return C


def c_shear() -> list[list[Fr]]:
    """∂c/∂G in Voigt form: deviatoric block [[4/3,-2/3,-2/3],...] ⊕ I3."""
    C = [[Fr(0)] * 6 for _ in range(6)]
    for i in range(3):
        for j in range(3):
            C[i][j] = Fr(4, 3) if i == j else Fr(-2, 3)
    for i in range(3, 6):
        C[i][i] = Fr(1)
    return C


def _btcb(B, C, g) -> list[list[Fr]]:
    """Σ_β B_βᵀ C B_β / g_β  (Eq. 5 with diagonal Gram)."""
    K = [[Fr(0)] * 24 for _ in range(24)]
    for b in range(len(B)):
        Bb = B[b]
        CB = [[sum(C[s][t] * Bb[t][col] for t in range(6)) for col in range(24)] for s in range(6)]
        for r in range(24):
            for col in range(24):
                acc = Fr(0)
                for s in range(6):
                    acc += Bb[s][r] * CB[s][col]
                K[r][col] += acc / g[b]
    return K


def stiffness_parts(ds: Fr = Fr(1)) -> tuple[list[list[Fr]], list[list[Fr]]]:
    """(Kκ_part, KG_part) with K_e^o = κ·Kκ_part + G·KG_part   (Eq. 5, κ/G split L94)."""
    B = strain_matrix(ds)
    g = psi_gram(ds)
    return _btcb(B, c_kappa(), g), _btcb(B, c_shear(), g)


def k_int8() -> list[list[int]]:
    """K_e^INT8 = (K_e^κ, K̄_e^G), 24×48.

    With ds = 1:  K_e^κ = 256·A_κ  and  K̄_e^G = 384·A_G − 128·I, where
    K_e^o = κ ds A_κ + G ds A_G.  (These are the paper's 256/3 B̄ᵀD̄^κB̄ ds⁴ and
    128 B̄ᵀD̄^GB̄ ds⁴ − 128 I, with D̄ = 3 ∂((ψψ')⁻¹c)/∂(κ|G) ds³; reading Q4.)
    Raises if any entry is not an integer in [-128, 127].
    """
    Ak, Ag = stiffness_parts(Fr(1))
    K = [[0] * 48 for _ in range(24)]
    for r in range(24):
        for col in range(24):
            vk = 256 * Ak[r][col]
            vg = 384 * Ag[r][col] - (128 if r == col else 0)
            for v in (vk, vg):
                if v.denominator != 1 or not (-128 <= v.numerator <= 127):
                    raise ValueError(f"K_e^INT8 entry ({r},{col}) = {v} is not an INT8 integer")
            K[r][col] = vk.numerator
            K[r][24 + col] = vg.numerator
    return K


def k_int8_split() -> tuple[list[list[int]], list[list[int]]]:
    """(K^κ, K̄^G + 128 I): the two integer 24×24 matrices the FP64 oracle multiplies
    first (A_κ = K^κ/256, A_G = (K̄^G + 128 I)/384; DESIGN.md oracle (i) step 3)."""
    K = k_int8()
    Kk = [row[:24] for row in K]
    Kg = [[K[r][24 + c] + (128 if r == c else 0) for c in range(24)] for r in range(24)]
    return Kk, Kg


def element_stiffness(kappa: Fr, G: Fr, ds: Fr) -> list[list[Fr]]:
    """K_e^o exactly, from Eq. 5 with c = κ C_κ + G C_G."""
    Ak, Ag = stiffness_parts(Fr(ds))
    return [[Fr(kappa) * Ak[r][c] + Fr(G) * Ag[r][c] for c in range(24)] for r in range(24)]


def element_mass_diag(rho: Fr, ds: Fr) -> list[Fr]:
    """Diagonal of M_e^o = ρ(φ^β φ^β')_e (Eq. 6): each octant indicator has volume ds³/8."""
    return [Fr(rho) * Fr(ds) ** 3 / 8] * 24


def element_mass_full(rho: Fr, ds: Fr) -> list[list[Fr]]:
    """Full 8×8 (per displacement component) ∫ φ^β φ^β' dv from the octant supports."""
    M = [[Fr(0)] * 8 for _ in range(8)]
    for a, b in product(range(8), range(8)):
        # ∫ H(..)H(..) over [-1,1]^3: overlap of octant a and octant b
        v = Fr(1)
        for j in range(3):
            v *= Fr(1) if CORNERS[a][j] == CORNERS[b][j] else Fr(0)
        M[a][b] = Fr(rho) * (Fr(ds) / 2) ** 3 * v
    return M


# ---------------------------------------------------------------------------
# VFEM: the paper's conventional voxel element (NEXT-3).
# Trilinear basis φ^β = Π_j (1 + r̄_j^β r_j)/2 on the reference cube r ∈ [-1, 1]³ (the printed
# "−1/8(r1+r̄1)(r2+r̄2)(r3+r̄3)" is sign-garbled, reading Q2; this is the standard form it
# names), the same isotropic c, K_e^V = ∫ Bᵀ c B dv integrated exactly (the paper's 2×2×2 Gauss
# rule is exact for this degree-2-per-variable integrand), lumped mass ρ ds³/8 per node
# ("diagonal terms are approximated as ρ/8(1)_e"), the same as OVFEM.
# ---------------------------------------------------------------------------

def _lin_pair_integral(s: int, t: int) -> Fr:
    """∫_{-1}^{1} (1 + s r)/2 · (1 + t r)/2 dr = (1 + s t/3)/2."""
    return (1 + Fr(s * t, 3)) / 2


def vfem_grad_gram(ds: Fr = Fr(1)) -> list[list[list[list[Fr]]]]:
    """G[a][b][i][k] = ∫_e ∂_i φ^a ∂_k φ^b dv for the trilinear basis on a cube of side ds."""
    ds = Fr(ds)
    G = [[[[Fr(0)] * 3 for _ in range(3)] for _ in range(8)] for _ in range(8)]
    for a, b in product(range(8), range(8)):
        sa, sb = CORNERS[a], CORNERS[b]
        for i, k in product(range(3), range(3)):
            # ∂_i φ^a = (2/ds)(r̄_i^a/2) Π_{j≠i} (1 + r̄_j^a r_j)/2 ;  dv = (ds/2)³ dr
            v = (2 / ds) * Fr(sa[i], 2) * (2 / ds) * Fr(sb[k], 2) * (ds / 2) ** 3
            for j in range(3):
                fa, fb = j != i, j != k
                if fa and fb:
                    v *= _lin_pair_integral(sa[j], sb[j])
                elif fa or fb:
                    v *= 1          # ∫ (1 + s r)/2 dr = 1
                else:
                    v *= 2          # ∫ dr
            G[a][b][i][k] = v
    return G


def vfem_stiffness_parts(ds: Fr = Fr(1)) -> tuple[list[list[Fr]], list[list[Fr]]]:
    """(A_κ^V, A_G^V) with K_e^V = κ A_κ^V + G A_G^V.  With λ = κ − 2G/3, μ = G:
    K[ap][bq] = λ G_ab[p][q] + μ (G_ab[q][p] + δ_pq Σ_r G_ab[r][r])."""
    G = vfem_grad_gram(ds)
    Ak = [[Fr(0)] * 24 for _ in range(24)]
    Ag = [[Fr(0)] * 24 for _ in range(24)]
    for a, b in product(range(8), range(8)):
        tr = sum(G[a][b][r][r] for r in range(3))
        for p, q in product(range(3), range(3)):
            lam_part = G[a][b][p][q]
            mu_part = G[a][b][q][p] + (tr if p == q else 0)
            Ak[3 * a + p][3 * b + q] = lam_part                        # κ multiplies λ's matrix
            Ag[3 * a + p][3 * b + q] = mu_part - Fr(2, 3) * lam_part   # G: μ part − (2/3) λ part
    return Ak, Ag


VFEM_DK, VFEM_DG = 72, 216    # common denominators of A_κ^V, A_G^V at ds = 1


def vfem_int_matrices() -> tuple[list[list[int]], list[list[int]]]:
    """Integer (Vk, Vg) with A_κ^V = ds·Vk/72, A_G^V = ds·Vg/216 (checked exact)."""
    Ak, Ag = vfem_stiffness_parts(Fr(1))
    Vk = [[Ak[r][c] * VFEM_DK for c in range(24)] for r in range(24)]
    Vg = [[Ag[r][c] * VFEM_DG for c in range(24)] for r in range(24)]
    for M in (Vk, Vg):
        for row in M:
            for x in row:
                if x.denominator != 1:
                    raise ValueError("VFEM matrix not integral at the stated denominator")
    return [[int(x) for x in row] for row in Vk], [[int(x) for x in row] for row in Vg]


def vfem_element_stiffness(kappa: Fr, G: Fr, ds: Fr) -> list[list[Fr]]:
    Ak, Ag = vfem_stiffness_parts(Fr(ds))
    return [[Fr(kappa) * Ak[r][c] + Fr(G) * Ag[r][c] for c in range(24)] for r in range(24)]
