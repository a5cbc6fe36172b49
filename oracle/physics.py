"""Closed forms and metrics used to pin the oracle (TEST INFRASTRUCTURE).

* err_metric: PAPER.md L232-L235 (the §3 Err definition).
* Central-difference recurrence for one eigenmode (Eq. 3): with
  K φ = λ M φ and u^n = a_n φ,  a_{n+1} = (2 − λ dt²) a_n − a_{n−1}.
* 1-D lattice dispersion for axis-aligned plane waves on a homogeneous voxel
  mesh (textbook two-node bar + diagonal mass):  λ = (4 V²/ds²) sin²(k ds/2).
* Leapfrog energy invariant for Eq. 3 (textbook):
  E_{n+½} = ½ v_{n+½}ᵀ M v_{n+½} + ½ u_nᵀ K u_{n+1},  v_{n+½} = (u_{n+1} − u_n)/dt.
"""
from __future__ import annotations

import math

import numpy as np


def err_metric(obs: np.ndarray, ref: np.ndarray) -> float:
    """Err = (1/n_c) Σ_i Σ_j (u_obs − u_ref)² / Σ_j u_ref²   (channels × steps)."""
    obs = np.asarray(obs, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if obs.shape != ref.shape:
        raise ValueError("channel/step mismatch")
    den = np.sum(ref * ref, axis=1)
    if np.any(den == 0):
        raise ValueError("zero-energy reference channel")
    return float(np.mean(np.sum((obs - ref) ** 2, axis=1) / den))


def lattice_lambda_axis(V: float, k: float, ds: float) -> float:
    """M⁻¹K eigenvalue of an axis-aligned plane wave with speed V (P: Vp, S: Vs)."""
    return 4.0 * V * V / (ds * ds) * math.sin(k * ds / 2.0) ** 2


def mode_amplitude(lam: float, dt: float, n: int, a0: float = 1.0, am1: float | None = None) -> float:
    """Closed-form a_n of a_{n+1} = (2 − λdt²) a_n − a_{n−1} (default a_{−1} = a_0)."""
    if am1 is None:
        am1 = a0
    c = 1.0 - lam * dt * dt / 2.0
    th = math.acos(c)
    # a_n = A cos nθ + B sin nθ;  A = a0,  a_{-1} = A cos θ − B sin θ
    B = (a0 * math.cos(th) - am1) / math.sin(th)
    return a0 * math.cos(n * th) + B * math.sin(n * th)


def mode_amplitude_damped(lam: float, dt: float, alpha: float, beta: float, n: int) -> float:
    """Closed-form a_n of the Rayleigh-damped modal recurrence (reading R1, backward-difference
    velocity): a_{n+1} = p a_n − q a_{n−1}, p = 2 − α dt − λ dt² − β λ dt, q = 1 − α dt − β λ dt,
    a_0 = a_{−1} = 1; a_n = A r1^n + B r2^n with r1, r2 the roots of r² − p r + q = 0."""
    p = 2.0 - alpha * dt - lam * dt * dt - beta * lam * dt
    q = 1.0 - alpha * dt - beta * lam * dt
    disc = complex(p * p - 4.0 * q) ** 0.5
    r1, r2 = (p + disc) / 2.0, (p - disc) / 2.0
    # A + B = 1,  A/r1 + B/r2 = 1
    B = (1.0 - 1.0 / r1) / (1.0 / r2 - 1.0 / r1)
    A = 1.0 - B
    return (A * r1 ** n + B * r2 ** n).real


def rayleigh_zeta(alpha: float, beta: float, w: float) -> float:
    """Modal damping ratio of C = αM + βK at angular frequency w (continuous time)."""
    return alpha / (2.0 * w) + beta * w / 2.0


def leapfrog_energy(K, m_diag, u_n, u_np1, dt) -> float:
    v = (u_np1 - u_n) / dt
    return 0.5 * float(v @ (m_diag * v)) + 0.5 * float(u_n @ (K @ u_np1))


def ricker(t: np.ndarray, f0: float, t0: float) -> np.ndarray:
    a = (math.pi * f0 * (t - t0)) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


def bloch_symbol(kappa: float, G: float, ds: float, k) -> np.ndarray:
    """OVFEM Bloch symbol Ŝ(k) (3×3, real symmetric) of the assembled K on a homogeneous voxel
    lattice (derived from PAPER.md Eqs. 5-8 with the seven ψ modes, L80-L89):
    s_i = sin(k_i ds/2), c_i = cos(k_i ds/2), λ = κ − 2G/3, μ = G,
        Ŝ = ds Σ_β w_β [(λ+μ) conj(g_β) g_βᵀ + μ |g_β|² I],
    with the mode weights w_β = 1/(Gram of ψ_β)·(ds³ normalisation) = 1, 3, 3, 3, 9, 9, 9 and
        g_1 = 2i(s_x c_y c_z, c_x s_y c_z, c_x c_y s_z),
        g_2 = −(0, s_x s_y c_z, s_x c_y s_z),  g_3 = −(s_x s_y c_z, 0, c_x s_y s_z),
        g_4 = −(s_x c_y s_z, c_x s_y s_z, 0),
        g_5 = −(i/2)(0, 0, s_x s_y s_z),  g_6 = −(i/2)(s_x s_y s_z, 0, 0),  g_7 = −(i/2)(0, s_x s_y s_z, 0).
    Plane-wave eigenvalues of M⁻¹K: eig(Ŝ)/(ρ ds³)."""
    sx, sy, sz = (math.sin(kk * ds / 2) for kk in k)
    cx, cy, cz = (math.cos(kk * ds / 2) for kk in k)
    sss = sx * sy * sz
    g = [(1, 2j * np.array([sx * cy * cz, cx * sy * cz, cx * cy * sz])),
         (3, -np.array([0.0, sx * sy * cz, sx * cy * sz])),
         (3, -np.array([sx * sy * cz, 0.0, cx * sy * sz])),
         (3, -np.array([sx * cy * sz, cx * sy * sz, 0.0])),
         (9, -0.5j * np.array([0.0, 0.0, sss])),
         (9, -0.5j * np.array([sss, 0.0, 0.0])),
         (9, -0.5j * np.array([0.0, sss, 0.0]))]
    lam, mu = kappa - 2.0 * G / 3.0, G
    S = np.zeros((3, 3), dtype=complex)
    for w, gb in g:
        gb = gb.astype(complex)
        S += w * ((lam + mu) * np.outer(np.conj(gb), gb) + mu * np.vdot(gb, gb) * np.eye(3))
    assert np.abs(S.imag).max() <= 1e-15 * max(1.0, np.abs(S.real).max())
    return ds * S.real


def bloch_modes(kappa: float, G: float, rho: float, ds: float, k):
    """(λ_i, U_i): eigenvalues of M⁻¹K (ascending) and unit eigenvectors of Ŝ(k) for a plane wave k."""
    ev, U = np.linalg.eigh(bloch_symbol(kappa, G, ds, k))
    return ev / (rho * ds ** 3), U
