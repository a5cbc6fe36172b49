"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no element matrices, no
integer expansion, no time stepping, no dispersion relation).  It only builds
the inputs the paper's problem statement takes (PAPER.md L38 voxel grid, L187
materials / source / fixed corners): grid sizes, per-element material ids,
per-material (ρ, κ, G), a Dirichlet mask, point sources with a Ricker
amplitude series, and initial fields.  Recipes follow SURVEY.md §8(d) and are
restated in DESIGN.md §Inputs.  Seed 13683 wherever randomness is used.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED = 13683


def moduli(rho: float, vp: float, vs: float) -> tuple[float, float, float]:
    """(ρ, κ, G) from density and wave speeds: G = ρ Vs², κ = ρ Vp² − 4G/3."""
    G = rho * vs * vs
    return rho, rho * vp * vp - 4.0 * G / 3.0, G


CONCRETE = (2400.0, 4000.0, 2400.0)   # S:L90 defaults (the paper does not state them, L187)
STEEL = (7850.0, 5900.0, 3200.0)
SOIL = (1800.0, 1000.0, 300.0)
ROCK = (2500.0, 4000.0, 2000.0)


def ricker(t: np.ndarray, f0: float, t0: float) -> np.ndarray:
    a = (math.pi * f0 * (t - t0)) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


@dataclass
class Model:
    name: str
    nx: int
    ny: int
    nz: int
    ds: float
    rho: np.ndarray
    kappa: np.ndarray
    G: np.ndarray
    mat: np.ndarray                  # uint8 per element, id ex + nx(ey + ny ez)
    dt: float
    dirichlet: np.ndarray | None     # uint8 per node, bit a = axis a fixed
    src_node: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    src_axis: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    amp: np.ndarray = field(default_factory=lambda: np.zeros((0, 1)))
    steps: int = 0
    alpha: float = 0.0       # Rayleigh damping C = alpha M + beta K (reading R1); 0 = undamped
    beta: float = 0.0

    @property
    def n_nodes(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def n_elems(self) -> int:
        return self.nx * self.ny * self.nz

    def node(self, ix, iy, iz) -> int:
        return ix + (self.nx + 1) * (iy + (self.ny + 1) * iz)

    def as_dict(self) -> dict:
        return dict(nx=self.nx, ny=self.ny, nz=self.nz, ds=self.ds, rho=self.rho, kappa=self.kappa,
                    G=self.G, mat=self.mat, dt=self.dt, dirichlet=self.dirichlet,
                    src_node=self.src_node, src_axis=self.src_axis, amp=self.amp,
                    alpha=self.alpha, beta=self.beta)


def rayleigh_coeffs(f1: float, f2: float, zeta: float) -> tuple[float, float]:
    """Two-point Rayleigh fit (SPEC rayleigh_coeffs; "Rayleigh damping (100--125 kHz)"):
    modal damping ratio zeta(w) = alpha/(2w) + beta w/2 equal to zeta at w1 = 2 pi f1, w2 = 2 pi f2."""
    if not 0 < f1 < f2 or zeta < 0:
        raise ValueError("need 0 < f1 < f2 and zeta >= 0")
    w1, w2 = 2 * math.pi * f1, 2 * math.pi * f2
    return 2 * zeta * w1 * w2 / (w1 + w2), 2 * zeta / (w1 + w2)


def _materials(*specs):
    r = np.array([moduli(*s) for s in specs], dtype=np.float64)
    return r[:, 0].copy(), r[:, 1].copy(), r[:, 2].copy()


def corner_mask(nx, ny, nz) -> np.ndarray:
    """The four bottom (z = 0) corner nodes fixed in x, y, z."""
    m = np.zeros((nz + 1, ny + 1, nx + 1), dtype=np.uint8)
    for iy in (0, ny):
        for ix in (0, nx):
            m[0, iy, ix] = 7
    return m.reshape(-1)


def roller_mask(nx, ny, nz) -> np.ndarray:
    """Rollers on all six faces: the normal component is fixed on each face (reading Q16)."""
    m = np.zeros((nz + 1, ny + 1, nx + 1), dtype=np.uint8)
    m[:, :, 0] |= 1
    m[:, :, nx] |= 1
    m[:, 0, :] |= 2
    m[:, ny, :] |= 2
    m[0, :, :] |= 4
    m[nz, :, :] |= 4
    return m.reshape(-1)


def point_source(model: Model, ix, iy, iz, axis, f0, t0, n_t, scale=1.0) -> None:
    t = np.arange(n_t) * model.dt
    model.src_node = np.array([model.node(ix, iy, iz)], dtype=np.int64)
    model.src_axis = np.array([axis], dtype=np.int32)
    model.amp = (scale * ricker(t, f0, t0)).reshape(1, -1)


# --- configs (BASELINE.json "configs") ---------------------

def c1_cube(n: int = 8, steps: int = 100) -> Model:
    """C1: n³ homogeneous concrete, ds = 2 mm, dt = 5e-8 s,
    z-force Ricker f0 = 112.5 kHz (L187) at the top-centre node, 4 bottom corners fixed."""
    rho, kappa, G = _materials(CONCRETE)
    m = Model("c1_cube", n, n, n, 2e-3, rho, kappa, G, np.zeros(n ** 3, np.uint8), 5e-8,
              corner_mask(n, n, n), steps=steps)
    f0 = 112.5e3
    point_source(m, n // 2, n // 2, n, 2, f0, 1.2 / f0, steps, scale=1.0e3)
    return m


def c2_block(n: int = 256, nu: str = "0.25", steps: int = 1000) -> Model:
    """C2: n³ homogeneous block, ds = 1, ρ = 1; ν = 0.25 (κ = 5/3, G = 1, dt = 0.5·0.4472)
    or ν = 0.35 (κ = 3, G = 1); rollers on all faces; IC = a plane standing wave."""
    kappa, G = (5.0 / 3.0, 1.0) if nu == "0.25" else (3.0, 1.0)
    dt = 0.5 * (0.4472135954999579 if nu == "0.25" else 2.0 / math.sqrt(8.0 * 3.0))
    m = Model(f"c2_block{n}", n, n, n, 1.0, np.array([1.0]), np.array([kappa]), np.array([G]),
              np.zeros(n ** 3, np.uint8), dt, roller_mask(n, n, n), steps=steps)
    return m


def standing_wave(model: Model, mvec=(16, 0, 0), U=(1.0, 0.0, 0.0)) -> np.ndarray:
    """u_a = U_a sin(k_a x_a) Π_{b≠a} cos(k_b x_b), k = π m / L (roller-box mode shape)."""
    nx, ny, nz, ds = model.nx, model.ny, model.nz, model.ds
    k = [math.pi * mvec[0] / (nx * ds), math.pi * mvec[1] / (ny * ds), math.pi * mvec[2] / (nz * ds)]
    x = np.arange(nx + 1) * ds
    y = np.arange(ny + 1) * ds
    z = np.arange(nz + 1) * ds
    s = [np.sin(k[0] * x), np.sin(k[1] * y), np.sin(k[2] * z)]
    c = [np.cos(k[0] * x), np.cos(k[1] * y), np.cos(k[2] * z)]
    u = np.zeros((nz + 1, ny + 1, nx + 1, 3))
    u[..., 0] = U[0] * (c[2][:, None, None] * c[1][None, :, None] * s[0][None, None, :])
    u[..., 1] = U[1] * (c[2][:, None, None] * s[1][None, :, None] * c[0][None, None, :])
    u[..., 2] = U[2] * (s[2][:, None, None] * c[1][None, :, None] * c[0][None, None, :])
    return u.reshape(-1)


def c3_two_layer(n: int = 512, steps: int = 1000, soil_layers: int | None = None) -> Model:
    """C3: n³, ds = 1 m, top n/4 element layers soil over bedrock; Ricker f0 = 25 Hz z-force at
    the top-surface centre; 4 bottom corners fixed; dt = 1e-4 s."""
    rho, kappa, G = _materials(SOIL, ROCK)
    soil = n // 4 if soil_layers is None else soil_layers
    ez = np.arange(n)
    lay = np.where(ez >= n - soil, 0, 1).astype(np.uint8)
    mat = np.broadcast_to(lay[:, None, None], (n, n, n)).reshape(-1).copy()
    m = Model(f"c3_two_layer{n}", n, n, n, 1.0, rho, kappa, G, mat, 1e-4, corner_mask(n, n, n),
              steps=steps)
    point_source(m, n // 2, n // 2, n, 2, 25.0, 1.2 / 25.0, steps, scale=1.0e6)
    return m


def c4_ground(nx: int = 891, ny: int = 352, nz: int = 1056, steps: int = 200) -> Model:
    """C4: multi-layer ground + stiff cylinder ∥ y (analogue of the paper's rebar model, L187)."""
    rho, kappa, G = _materials((1700.0, 800.0, 200.0), (1900.0, 1800.0, 500.0),
                               (2200.0, 3000.0, 1400.0), (2600.0, 5000.0, 2800.0),
                               (7850.0, 5900.0, 3200.0))
    ez = np.arange(nz)
    depth = (nz - 1 - ez) / nz                   # 0 at the top layer
    lay = np.select([depth < 0.05, depth < 0.20, depth < 0.45], [0, 1, 2], 3).astype(np.uint8)
    mat = np.empty((nz, ny, nx), dtype=np.uint8)
    mat[:] = lay[:, None, None]
    cx, cz, r = 160.0 / 324.0 * nx, 100.0 / 384.0 * nz, 41.0
    xc = np.arange(nx) + 0.5
    zc = np.arange(nz) + 0.5
    inside = ((xc[None, :] - cx) ** 2 + (zc[:, None] - cz) ** 2) <= r * r
    mat[:, :, :][np.broadcast_to(inside[:, None, :], mat.shape)] = 4
    m = Model("c4_ground", nx, ny, nz, 1.0, rho, kappa, G, mat.reshape(-1), 6.3e-5,
              corner_mask(nx, ny, nz), steps=steps)
    point_source(m, int(round(156 / 324 * nx)), int(round(72 / 128 * ny)), nz, 2, 10.0, 0.12, steps,
                 scale=1.0e6)
    return m


def bandlimited_impulse(t_c: float, f_lo: float, f_hi: float, dt: float, n: int) -> np.ndarray:
    """SPEC bandlimited_impulse for the paper's "impulse force with a center time of
    4.096e-4 s and a center frequency of 112.5 kHz with a bandpass of 100--125 kHz":
    h(t) = 2 f_hi sinc(2 f_hi τ) − 2 f_lo sinc(2 f_lo τ), τ = t − t_c, Hann window of half-width
    4/f_lo, normalised to unit peak."""
    tau = np.arange(n) * dt - t_c
    h = 2 * f_hi * np.sinc(2 * f_hi * tau) - 2 * f_lo * np.sinc(2 * f_lo * tau)
    hw = 4.0 / f_lo
    win = np.where(np.abs(tau) < hw, 0.5 * (1.0 + np.cos(np.pi * tau / hw)), 0.0)
    h = h * win
    peak = np.abs(h).max()
    return h / peak if peak > 0 else h


# PAPER.md Table 1: source and observation points (mm)
E1_SOURCE_MM = (156.0, 72.0, 384.0)
E1_OBS_MM = [(26.0, 60.0, 384.0), (60.0, 60.0, 384.0), (108.0, 60.0, 384.0), (144.0, 60.0, 384.0),
             (180.0, 60.0, 384.0), (216.0, 60.0, 384.0), (264.0, 60.0, 384.0), (300.0, 60.0, 384.0)]


def e1_rebar(ds_mm: float = 2.0, steps: int = 16384, zeta: float = 0.01, dt: float = 5e-8,
             amp: float = 1.0e3) -> Model:
    """E1 (NEXT-2): the paper's ultrasonic model (Fig. 5, Table 1).  324 × 128 × 384 mm
    concrete block, steel rebar of radius 15 mm ∥ y centred at x = 160, z = 100 mm; the four bottom
    corners fixed in x, y, z; z-direction band-limited impulse (t_c = 4.096e-4 s, 100-125 kHz) at the
    Table 1 input point; Rayleigh damping fitted to ζ at 100 and 125 kHz (ζ is not stated by the
    paper — an input here); dt = 5e-8 s at ds = 2 mm (Table 2 pairing), 8.192e-4 s = 16,384 steps.
    Materials: the SPEC's non-authoritative concrete / steel defaults (P:L187 states none).
    Points off the grid (coarser ds) snap to the nearest node.  model.receivers: the 8 Table 1
    observation nodes."""
    ds = ds_mm * 1e-3
    nx, ny, nz = int(round(324 / ds_mm)), int(round(128 / ds_mm)), int(round(384 / ds_mm))
    rho, kappa, G = _materials(CONCRETE, STEEL)
    xc = (np.arange(nx) + 0.5) * ds_mm
    zc = (np.arange(nz) + 0.5) * ds_mm
    inside = ((xc[None, :] - 160.0) ** 2 + (zc[:, None] - 100.0) ** 2) <= 15.0 ** 2   # [z, x]
    mat = np.zeros((nz, ny, nx), dtype=np.uint8)
    mat[np.broadcast_to(inside[:, None, :], mat.shape)] = 1
    m = Model(f"e1_rebar_ds{ds_mm:g}mm", nx, ny, nz, ds, rho, kappa, G, mat.reshape(-1), dt,
              corner_mask(nx, ny, nz), steps=steps)
    snap = lambda p: tuple(int(round(c / ds_mm)) for c in p)   # noqa: E731
    sx, sy, sz = snap(E1_SOURCE_MM)
    m.src_node = np.array([m.node(sx, sy, sz)], dtype=np.int64)
    m.src_axis = np.array([2], dtype=np.int32)
    m.amp = (amp * bandlimited_impulse(4.096e-4, 100e3, 125e3, dt, steps)).reshape(1, -1)
    m.receivers = np.array([m.node(*snap(p)) for p in E1_OBS_MM], dtype=np.int64)
    if zeta > 0:
        m.alpha, m.beta = rayleigh_coeffs(100e3, 125e3, zeta)
    return m


def c5_layered(g: int = 1, n: int = 256, steps: int = 200) -> Model:
    """C5: n × n × (n·g), soil/rock alternating every 64 element layers (weak-scaling grid)."""
    rho, kappa, G = _materials(SOIL, ROCK)
    nz = n * g
    lay = ((np.arange(nz) // 64) % 2).astype(np.uint8)
    mat = np.broadcast_to(lay[:, None, None], (nz, n, n)).reshape(-1).copy()
    m = Model(f"c5_layered{n}x{g}", n, n, nz, 1.0, rho, kappa, G, mat, 1e-4, corner_mask(n, n, nz),
              steps=steps)
    point_source(m, n // 2, n // 2, nz, 2, 25.0, 1.2 / 25.0, steps, scale=1.0e6)
    return m


def random_field(model: Model, seed: int = SEED, scale: float = 1.0) -> np.ndarray:
    """u ~ N(0, scale²) i.i.d. per DOF (reading Q21: the Table 3 random vector)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal(3 * model.n_nodes) * scale


def random_materials(model: Model, nmat: int = 3, seed: int = SEED) -> None:
    """Random per-element material ids over nmat random (ρ, Vp, Vs) triples."""
    rng = np.random.default_rng(seed + 1)
    specs = []
    for _ in range(nmat):
        vs = rng.uniform(300.0, 3000.0)
        vp = vs * rng.uniform(1.6, 2.2)
        specs.append((rng.uniform(1500.0, 8000.0), vp, vs))
    model.rho, model.kappa, model.G = _materials(*specs)
    model.mat = rng.integers(0, nmat, size=model.n_elems, dtype=np.uint8)


def small_random(nx=5, ny=4, nz=3, seed: int = SEED, ds: float = 0.5, dt: float = 1e-5) -> Model:
    """Ragged small heterogeneous model for parity tests (several tiles + ragged tails)."""
    m = Model(f"rand{nx}x{ny}x{nz}", nx, ny, nz, ds, np.zeros(1), np.zeros(1), np.zeros(1),
              np.zeros(nx * ny * nz, np.uint8), dt, corner_mask(nx, ny, nz))
    random_materials(m, 3, seed)
    return m
