"""Pins for the oracle's integer-path emulation (Eqs. 10-17).

Pinned against: hand-derived digit values of Eq. 16; the round-trip identity;
linearity (Σ_j b^j K d_j = K v, checked with Python big integers); the exact
rational value of Eq. 9 (a-priori truncation bound, the paper's "56 fraction
bits" claim, L245); the paper's Table 3 accuracy ordering; exact oddness.
"""
from fractions import Fraction as Fr
import math

import numpy as np
import pytest

import oracle
from oracle import element as el

K8 = el.k_int8()


def test_paper_digit_examples_eq16():
    D = oracle.DIGITS_PAPER
    assert oracle.digits(2 ** 56 - 1, 8, D) == [127] * 8
    assert oracle.digits(-(2 ** 56 - 1), 8, D) == [1, 0, 0, 0, 0, 0, 0, -128]
    assert oracle.digits(-1, 8, D) == [127] * 7 + [-1]
    assert oracle.digits(128, 8, D) == [0, 1, 0, 0, 0, 0, 0, 0]
    assert oracle.digits(0, 8, D) == [0] * 8


def test_byte_digit_examples():
    B = oracle.DIGITS_BYTES
    assert oracle.digits(0, 8, B) == [0] * 7 + [1]             # v' = 2^56
    assert oracle.digits(-1, 8, B) == [255] * 7 + [0]          # v' = 2^56 − 1
    assert oracle.digits(2 ** 56, 8, B) == [0] * 7 + [2]       # unclamped +1.0
    assert oracle.digits(-(2 ** 56), 8, B) == [0] * 8


@pytest.mark.parametrize("scheme", [oracle.DIGITS_PAPER, oracle.DIGITS_BYTES])
@pytest.mark.parametrize("M", [8, 6, 4])
def test_digit_round_trip(scheme, M):
    rng = np.random.default_rng(13683 + M)
    lim = 2 ** (7 * M) - 1
    vals = [int(x) for x in rng.integers(-lim, lim, size=20000, endpoint=True)] + [lim, -lim, 0, 1, -1]
    for v in vals:
        d = oracle.digits(v, M, scheme)
        if scheme == oracle.DIGITS_PAPER:
            assert sum(dj << (7 * j) for j, dj in enumerate(d)) == v
            assert all(-128 <= x <= 127 for x in d)
            assert all(0 <= x <= 127 for x in d[:-1])
        else:
            assert sum(dj << (8 * j) for j, dj in enumerate(d)) - (1 << (7 * M)) == v
            assert all(0 <= x <= 255 for x in d)


def _elem_inputs(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        u = rng.standard_normal(24) * 10.0 ** rng.uniform(-12, 3)
        if i % 7 == 0:   # Nyquist-like sign pattern, the adversarial case of SURVEY H3
            u = np.sign(rng.standard_normal(24)) * 3.0
        kappa = 10 ** rng.uniform(8, 11)
        G = kappa * rng.uniform(0.05, 1.4)
        out.append((u, kappa, G, 10 ** rng.uniform(-3, 0)))
    return out


@pytest.mark.parametrize("scheme", [oracle.DIGITS_PAPER, oracle.DIGITS_BYTES])
def test_staged_accumulation_equals_integer_product(scheme):
    """Σ_j b^{j-1} K d_j  ==  K v  (Eq. 17 vs the plain product, big-int arithmetic)."""
    for (u, kappa, G, ds) in _elem_inputs(1, 60):
        r = oracle.element_int8(u, kappa, G, ds, 8, scheme)
        v = [int(x) for x in r["v"]]
        for i in range(24):
            assert r["y"][i] == sum(K8[i][k] * v[k] for k in range(48))
        # per-stage products are K·d_j exactly and fit INT32 (SURVEY H3 bound)
        for j in range(r["d"].shape[0]):
            for i in range(24):
                c = sum(K8[i][k] * int(r["d"][j][k]) for k in range(48))
                assert r["C"][j][i] == c and abs(c) < 2 ** 31


def test_digit_schemes_agree_when_no_clamp():
    for (u, kappa, G, ds) in _elem_inputs(2, 60):
        a = oracle.element_int8(u, kappa, G, ds, 8, oracle.DIGITS_PAPER)
        b = oracle.element_int8(u, kappa, G, ds, 8, oracle.DIGITS_BYTES)
        if np.all(np.abs(b["v"]) < 2 ** 56):
            assert a["y"] == b["y"]
            assert np.array_equal(a["fe"], b["fe"])
        else:  # only the ±1.0 components differ, by at most 2^56 + 16 − (2^56 − 1) = 17 units
            assert np.all(np.abs(a["v"] - b["v"]) <= 17)


def _exact_eq9(u, kappa, G, ds):
    ku = [Fr(x) for x in u]
    fk, fg, fd = Fr(kappa), Fr(G), Fr(ds)
    ub = ku + [Fr(2, 3) * fg / fk * x for x in ku]
    return [fk * fd / 256 * (sum(K8[r][k] * ub[k] for k in range(48)) + Fr(256, 3) * fg / fk * ku[r])
            for r in range(24)]


def test_a_priori_truncation_bound():
    """|f_int − f_exact| ≤ c1·s·2^-56·(2·1130+Δ) + a few ulps — the "56 fraction bits" of L245.

    Δ covers the rounding of ū_G = RN(cG·u), x = RN(ū·RN(1/s)) (each ≤ 1 ulp of a ≤ 1 number,
    i.e. ≤ 2^4 units of 2^-56 per component): bound = c1·s·2^-56·1130·(2 + 2·16) + 8 ulp.
    """
    for (u, kappa, G, ds) in _elem_inputs(3, 40):
        r = oracle.element_int8(u, kappa, G, ds, 8, oracle.DIGITS_BYTES)
        ex = _exact_eq9(u, kappa, G, ds)
        c1 = kappa * ds / 256
        s = r["s"]
        for i in range(24):
            err = abs(Fr(r["fe"][i]) - ex[i])
            bound = Fr(c1 * s) * Fr(2) ** -56 * 1130 * 34 + 8 * Fr(math.ulp(abs(float(ex[i])) + c1 * s))
            assert err <= bound, (i, float(err), float(bound))


def test_table3_accuracy_hierarchy():
    """PAPER.md Table 3 / L245: M=4 ~ FP32 (28 bits), M=8 ≥ FP64 (56 bits)."""
    errs = {8: [], 4: [], "fp64": [], "fp32": []}
    rng = np.random.default_rng(13683)
    Kk = np.array([r[:24] for r in K8], dtype=np.float64)
    Kg = np.array([[K8[r][24 + c] + (128 if r == c else 0) for c in range(24)] for r in range(24)],
                  dtype=np.float64)
    for _ in range(60):
        u = rng.standard_normal(24)
        kappa, G, ds = 2.0e10, 1.4e10, 2e-3
        ex = np.array([float(x) for x in _exact_eq9(u, kappa, G, ds)])
        sc = np.linalg.norm(ex)
        for M in (8, 4):
            errs[M].append(np.linalg.norm(oracle.element_int8(u, kappa, G, ds, M)["fe"] - ex) / sc)
        errs["fp64"].append(np.linalg.norm(oracle.element_fp64(u, kappa, G, ds) - ex) / sc)
        u32 = u.astype(np.float32)
        f32 = (np.float32(kappa * ds / 256) * (Kk.astype(np.float32) @ u32)
               + np.float32(G * ds / 384) * (Kg.astype(np.float32) @ u32))
        errs["fp32"].append(np.linalg.norm(f32.astype(np.float64) - ex) / sc)
    med = {k: float(np.median(v)) for k, v in errs.items()}
    assert med[8] <= 2 * med["fp64"] and med[8] < 1e-15
    assert med["fp64"] < med["fp32"]
    assert med[4] < 4 * med["fp32"] and med[4] > med[8] * 1e4
    assert 1e-10 < med[4] < 1e-6


def test_integer_path_is_exactly_odd():
    for (u, kappa, G, ds) in _elem_inputs(4, 30):
        a = oracle.element_int8(u, kappa, G, ds)
        b = oracle.element_int8(-u, kappa, G, ds)
        assert np.array_equal(a["fe"], -b["fe"])
        assert a["y"] == [-y for y in b["y"]]


def test_zero_and_subnormal_elements_give_zero_force():
    z = oracle.element_int8(np.zeros(24), 2.0, 1.0, 1.0)
    assert z["s"] == 0.0 and np.all(z["fe"] == 0.0) and all(y == 0 for y in z["y"])
    t = oracle.element_int8(np.full(24, 5e-324), 2.0, 1.0, 1.0)
    assert t["degenerate"] and np.all(t["fe"] == 0.0)


def test_rn_of_y_is_correctly_rounded():
    """fe = c1·(RN(y)·s·2^-56 + c2 u): recompute with Python's correctly rounded int→float."""
    for (u, kappa, G, ds) in _elem_inputs(5, 30):
        r = oracle.element_int8(u, kappa, G, ds, 8, oracle.DIGITS_BYTES)
        c1 = kappa * ds / 256.0
        c2 = (256.0 * G) / (3.0 * kappa)
        sig = r["s"] * 2.0 ** -56
        for i in range(24):
            assert r["fe"][i] == c1 * (float(r["y"][i]) * sig + c2 * u[i])


# ---- variant D (Eq. 9 diagonal term folded into the integer product) -----------------

def test_fold_variant_integer_identity_and_bound():
    """y_D = K_D v with K_D = [K^κ | K̄^G + 128 I] (big integers), and f within the truncation
    bound of the exact Eq. 9 value (one extra 128·s·2^-56 term from truncating ū_G)."""
    KD = [row[:24] + [row[24 + c] + (128 if c == r else 0) for c in range(24)] for r, row in enumerate(K8)]
    for (u, kappa, G, ds) in _elem_inputs(6, 40):
        r = oracle.element_int8(u, kappa, G, ds, 8, oracle.DIGITS_BYTES_FOLD)
        v = [int(x) for x in r["v"]]
        for i in range(24):
            assert r["y"][i] == sum(KD[i][k] * v[k] for k in range(48))
        ex = _exact_eq9(u, kappa, G, ds)
        c1, s = kappa * ds / 256, r["s"]
        for i in range(24):
            err = abs(Fr(r["fe"][i]) - ex[i])
            bound = Fr(c1 * s) * Fr(2) ** -56 * (1130 + 128) * 34 + 8 * Fr(math.ulp(abs(float(ex[i])) + c1 * s))
            assert err <= bound


def test_fold_variant_matches_literal_to_fp64_precision_and_is_odd():
    for (u, kappa, G, ds) in _elem_inputs(8, 40):
        a = oracle.element_int8(u, kappa, G, ds, 8, oracle.DIGITS_BYTES_FOLD)
        b = oracle.element_int8(u, kappa, G, ds, 8, oracle.DIGITS_BYTES)
        sc = kappa * ds / 256 * a["s"] * 1300
        assert np.abs(a["fe"] - b["fe"]).max() <= 2.0 ** -48 * sc
        n = oracle.element_int8(-u, kappa, G, ds, 8, oracle.DIGITS_BYTES_FOLD)
        assert np.array_equal(a["fe"], -n["fe"])


def _elem_with_max(xmax_component):
    """An element vector whose scaled image has a chosen first component (the max is 1)."""
    ue = np.zeros(24)
    ue[0] = 1.0
    ue[1] = xmax_component
    return ue


@pytest.mark.parametrize("M", [4, 6, 8])
def test_direct_n_stage_conversion_equals_hierarchical(M):
    """NEXT-4, Fig. 2 left (Eqs. 11-14, a = 2^7, N = M): converting the FP64 remainder to INT8
    at every stage gives the same integer image v = Σ_i a^{N-i} d_i as the hierarchical FP64→INT64→INT8
    path (one conversion, then 7-bit slices), hence the same y and element force — the paper's
    "the total computation accuracy is the same when N = M" (L146).  Random and adversarial inputs."""
    rng = np.random.default_rng(40 + M)
    for trial in range(300):
        ue = rng.standard_normal(24) * 10.0 ** rng.uniform(-8, 8)
        if trial % 5 == 0:
            ue = np.sign(ue) * 3.0                       # every component at ±max: the clamp is active
        if trial % 11 == 0:
            ue[rng.integers(0, 24)] = 0.0
        for fold in (0, 2):
            a = oracle.element_int8(ue, 1.7, 1.1, 0.01, M, oracle.DIGITS_DIRECT | fold)
            b = oracle.element_int8(ue, 1.7, 1.1, 0.01, M, oracle.DIGITS_PAPER | fold)
            assert np.array_equal(a["v"], b["v"]), trial
            assert a["y"] == b["y"] and np.array_equal(a["fe"], b["fe"]), trial
            d = a["d"]
            assert d.shape == (M, 48) and np.abs(d).max() <= 127
            recon = sum((128 ** j) * d[j].astype(object) for j in range(M))   # lowest weight first
            assert list(recon) == [int(x) for x in a["v"]]


def test_direct_digits_worked_examples():
    """Hand-derived digit sequences of the direct recursion d_i = INT(a r_{i-1}), r_i = a r_{i-1} − d_i:
    x = 0.75 → (96, 0, …); x = −0.75 → (−96, 0, …); x = 1 (the max component) → 127 at every stage
    (= 2^56 − 1, reading Q9); x = fl(1/3) → the base-128 digits of ⌊2^56·fl(1/3)⌋ (exact rationals):
    42, 85, 42, 85, … ending in 84 because fl(1/3) < 1/3."""
    K = dict(kappa=1.7, G=1.1, ds=0.01)
    r = oracle.element_int8(_elem_with_max(0.75), K["kappa"], K["G"], K["ds"], 8, oracle.DIGITS_DIRECT)
    d = r["d"][::-1]                                  # highest weight first: d_1 .. d_8
    assert list(d[:, 1]) == [96, 0, 0, 0, 0, 0, 0, 0]
    assert list(d[:, 0]) == [127] * 8 and int(r["v"][0]) == 2 ** 56 - 1
    r = oracle.element_int8(_elem_with_max(1.0 / 3.0), K["kappa"], K["G"], K["ds"], 8, oracle.DIGITS_DIRECT)
    d = r["d"][::-1]
    from fractions import Fraction
    V = int(Fraction(1.0 / 3.0) * 2 ** 56)        # the FP64 value of 1/3 is slightly below 1/3
    assert list(d[:, 1]) == [(V >> (7 * (7 - i))) & 127 for i in range(8)] == [42, 85, 42, 85, 42, 85, 42, 84]
    r = oracle.element_int8(-_elem_with_max(0.75), K["kappa"], K["G"], K["ds"], 8, oracle.DIGITS_DIRECT)
    d = r["d"][::-1]
    assert list(d[:, 1]) == [-96, 0, 0, 0, 0, 0, 0, 0] and list(d[:, 0]) == [-127] * 8
