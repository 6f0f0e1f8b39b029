"""Pins for the oracle's force/moment quadrature (Sec. 2.4-III, PAPER.md:173-175;
reading R-A14): closed-form integrals of special pressure fields, symmetry and
linearity."""
import math

import numpy as np


def _still(gi, e=(0, 0, 0, 0), U_theta=0.0, U_y=0.0, p_in=0.0, p_out=0.0):
    c = gi.condition(e, (0, 0, 0, 0))
    c[9], c[10], c[11], c[12] = U_theta, U_y, p_in, p_out
    return c


def test_uniform_pressure_no_lateral_load(orc, gi):
    """Uniform p, e = 0 -> lateral F and M vanish by symmetry."""
    g = gi.grid(64, 32)
    P = 4e6
    c = _still(gi, p_in=P, p_out=P)
    w = orc.wrench(g, c, np.full((32, 64), P))
    scale = P * 2 * math.pi * gi.R_K * c[8]
    assert np.all(np.abs(w[[0, 1, 3, 4, 5]]) <= 1e-12 * scale * max(1.0, c[8]))
    # Fp_z == 0 exactly; Mp_z = R cos * Fy - R sin * Fx cancels to rounding only
    assert w[2] == 0.0 and abs(w[5]) <= 1e-15 * scale * gi.R_K


def test_cosine_pressure_closed_form(orc, gi):
    """p = P1 cos(theta) on every interior row, 0 on the ghost rows:
    Fp_x = -P1 pi R_k cos(dtheta/2) * (effective length) and the matching Mp_y
    (midpoint rule on cells, the two boundary cell rows at half weight)."""
    nt, ny = 48, 20
    g = gi.grid(nt, ny)
    P1 = 1e6
    # interior rows carry P1 cos(theta); the Dirichlet ghost rows carry p_in = p_out = 0
    th = 2 * np.pi * np.arange(nt) / nt
    p = np.tile(P1 * np.cos(th), (ny, 1))
    c = _still(gi)
    w = orc.wrench(g, c, p)
    L = c[8]
    dy = L / (ny + 1)
    # cells j=0..ny-2 have all four corners at P1 cos; the two boundary cell rows
    # (j=-1 and j=ny-1) have two corners at P1 cos and two at 0 -> half weight.
    rows = (ny - 1) + 0.5 + 0.5
    fx = -P1 * math.pi * gi.R_K * math.cos(np.pi / nt) * rows * dy
    assert abs(w[0] - fx) <= 1e-13 * abs(fx)
    assert abs(w[1]) <= 1e-12 * abs(fx)
    yc = np.array([(j + 1.5) * dy for j in range(-1, ny)])
    wt = np.array([0.5] + [1.0] * (ny - 1) + [0.5])
    my = -P1 * math.pi * gi.R_K * math.cos(np.pi / nt) * float(np.sum(wt * yc)) * dy
    assert abs(w[4] - my) <= 1e-12 * abs(my)


def test_couette_shear_closed_form(orc, gi):
    """p = 0, constant film h: Fs_z = -(mu U_y / h) 2 pi R_k L_F and
    Ms_z = -(mu U_theta / h) R_k 2 pi R_k L_F; lateral shear ~ 0."""
    g = gi.grid(128, 64)
    c = _still(gi, U_theta=0.7, U_y=0.45)
    w = orc.wrench(g, c, np.zeros((64, 128)))
    h = gi.R_C - gi.R_K
    L = c[8]
    area = 2 * math.pi * gi.R_K * L
    fz = -(g["mu"] * 0.45 / h) * area
    mz = -(g["mu"] * 0.7 / h) * gi.R_K * area
    assert abs(w[8] - fz) <= 1e-12 * abs(fz)
    assert abs(w[11] - mz) <= 1e-12 * abs(mz)
    assert abs(w[6]) <= 1e-12 * abs(mz / gi.R_K) and abs(w[7]) <= 1e-12 * abs(mz / gi.R_K)


def test_poiseuille_shear_closed_form(orc, gi, ):
    """Uniform film, linear p in y from p_in to p_out:
    Fs_z = -pi R_k h (p_out - p_in); lateral Fp, Mp ~ 0."""
    nt, ny = 64, 40
    g = gi.grid(nt, ny)
    pin, pout = 10e6, 0.5e6
    c = _still(gi, p_in=pin, p_out=pout)
    j = np.arange(ny)
    p = np.tile((pin + (pout - pin) * (j + 1) / (ny + 1))[:, None], (1, nt))
    w = orc.wrench(g, c, p)
    h = gi.R_C - gi.R_K
    fz = -math.pi * gi.R_K * h * (pout - pin)
    assert abs(w[8] - fz) <= 1e-12 * abs(fz)
    scale = pin * 2 * math.pi * gi.R_K * c[8]
    assert abs(w[0]) <= 1e-12 * scale and abs(w[1]) <= 1e-12 * scale


def test_pressure_part_linear_in_p(orc, gi):
    """The pressure part is linear in p; shear is affine with U = 0 linear."""
    g = gi.grid(40, 20, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8)
    rng = np.random.default_rng(0)
    c = _still(gi, e=(1e-6, -1e-6, 0.5e-6, 0.2e-6))
    p1 = rng.uniform(0, 1e7, (20, 40))
    p2 = rng.uniform(0, 1e7, (20, 40))
    w1, w2 = orc.wrench(g, c, p1), orc.wrench(g, c, p2)
    w12 = orc.wrench(g, c, p1 + 2 * p2)
    assert np.allclose(w12, w1 + 2 * w2, rtol=1e-12, atol=1e-12 * np.abs(w12).max())


def test_quadrature_second_order(orc, gi):
    """Midpoint quadrature of a smooth field converges O(h^2)."""
    vals = []
    for nt, ny in [(32, 15), (64, 31), (128, 63)]:
        g = gi.grid(nt, ny)
        c = _still(gi, e=(1e-6, -0.5e-6, 2e-6, 0.3e-6), U_theta=0.3, U_y=0.4, p_in=2e6, p_out=1e6)
        L = c[8]
        th = 2 * np.pi * np.arange(nt) / nt
        y = (np.arange(ny) + 1) * L / (ny + 1)
        p = 2e6 - 1e6 * y[:, None] / L + 1.5e6 * np.sin(np.pi * y[:, None] / L) * np.cos(th)[None]
        vals.append(orc.wrench(g, c, p))
    d1 = np.abs(vals[0] - vals[1])
    d2 = np.abs(vals[1] - vals[2])
    for q in (0, 4, 8):        # Fp_x, Mp_y, Fs_z are O(1) components
        assert 3.5 <= d1[q] / d2[q] <= 4.5, (q, d1[q] / d2[q])
