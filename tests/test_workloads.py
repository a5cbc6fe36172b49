"""Workload generators: the E1 rebar model of the paper's experiment (Table 1) and the
SPEC's band-limited impulse."""
import math

import numpy as np

import workloads as wl


def test_bandlimited_impulse_band_and_peak():
    dt, n = 5e-8, 16384
    h = wl.bandlimited_impulse(4.096e-4, 100e3, 125e3, dt, n)
    assert abs(np.abs(h).max() - 1.0) < 1e-15
    assert np.argmax(np.abs(h)) == int(round(4.096e-4 / dt))      # centred at t_c
    F = np.abs(np.fft.rfft(h))
    f = np.fft.rfftfreq(n, dt)
    assert 100e3 <= f[np.argmax(F)] <= 125e3                        # peak within the band
    band = (f >= 75e3) & (f <= 150e3)
    assert np.sum(F[band] ** 2) >= 0.95 * np.sum(F ** 2)            # energy concentrated


def test_e1_geometry_and_table1_points():
    m = wl.e1_rebar(2.0, steps=16)
    assert (m.nx, m.ny, m.nz) == (162, 64, 192) and m.ds == 2e-3 and m.dt == 5e-8
    steel = np.bincount(m.mat, minlength=2)[1]
    assert abs(steel - math.pi * 15.0 ** 2 / 4.0 * 64) < 0.03 * steel     # r = 15 mm cylinder ∥ y
    mat = m.mat.reshape(m.nz, m.ny, m.nx)
    assert mat[50, 10, 80] == 1 and mat[50, 10, 100] == 0 and np.all(mat[:, 0, :] == mat[:, 63, :])
    assert m.src_node[0] == m.node(78, 36, 192) and m.src_axis[0] == 2
    assert [int(n) for n in m.receivers] == [m.node(x, 30, 192) for x in (13, 30, 54, 72, 90, 108, 132, 150)]
    a, b = wl.rayleigh_coeffs(100e3, 125e3, 0.01)
    assert (m.alpha, m.beta) == (a, b)
    assert int(np.count_nonzero(m.dirichlet)) == 4
