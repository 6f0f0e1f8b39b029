"""Pins for the oracle's thickness (Eq. 2.3) and rate (Eq. 2.2).

Each test checks the oracle against something other than itself: closed forms,
invariants, a finite-difference derivative, or a first-order expansion.
"""
import math

import numpy as np
import pytest


def _cond(gi, e=(0, 0, 0, 0), ed=(0, 0, 0, 0), **kw):
    c = gi.condition(e, ed)
    for k, v in kw.items():
        c[{"L_F": 8, "U_theta": 9, "U_y": 10, "p_in": 11, "p_out": 12}[k]] = v
    return c


def test_centred_film_is_clearance(orc, gi):
    """e = 0, smooth -> h == R_c - R_k everywhere."""
    g = gi.grid(64, 32)
    h, hd = orc.thickness(g, _cond(gi))
    assert np.allclose(h, 6e-6, rtol=1e-12, atol=0)
    assert np.all(hd == 0.0)


def test_texture_adds_depth_only_on_mask(orc, gi):
    """Texture raises h by h_Text at masked nodes and changes no other node."""
    gs = gi.grid(240, 80)
    gt = gi.grid(240, 80, "short")
    c = gi.condition()
    hs, _ = orc.thickness(gs, c)
    ht, _ = orc.thickness(gt, c)
    T = orc.texture_mask(gt).astype(bool)
    assert T.sum() > 0
    assert np.array_equal(hs[~T], ht[~T])
    d = ht[T] - hs[T]
    assert np.all(np.abs(d - 20e-6) <= 4 * np.spacing(ht[T]))
    # ghost rows are never textured, only the bottom band is
    assert not T[0].any() and not T[-1].any()
    assert not T[1 + gt["tex_band_rows"]:].any()


def test_texture_fill_fraction(orc, gi):
    """50% x 50% fill of the dimple pitch inside the band -> ~25% of band nodes (R-A7)."""
    g = gi.grid(1200, 400, "short")
    T = orc.texture_mask(g)
    band = T[1:1 + g["tex_band_rows"]]
    assert abs(band.mean() - 0.25) < 0.01
    # 60 dimples around theta: count rising edges in row 0 of the band
    row = band[0].astype(int)
    assert int(np.sum((np.roll(row, 1) == 0) & (row == 1))) == 60


def test_mesh_too_coarse(orc, gi):
    assert orc.check_grid(gi.grid(100, 80, "short")) == orc.E_MESH_TOO_COARSE   # 100 < 2*60
    assert orc.check_grid(gi.grid(120, 79, "short")) == orc.E_MESH_TOO_COARSE   # band 19 < 20
    assert orc.check_grid(gi.grid(120, 80, "short")) == orc.OK
    assert orc.check_grid(gi.grid(3, 80)) == orc.E_INVALID_MESH


def test_contact_is_rejected(orc, gi):
    """e = (6um, 0, 6um, 0), theta = 0 -> h = 0 -> NonPositiveThickness."""
    with pytest.raises(orc.OracleError) as ei:
        orc.thickness(gi.grid(64, 32), _cond(gi, e=(6e-6, 0, 6e-6, 0)))
    assert ei.value.code == orc.E_NONPOSITIVE_THICKNESS


def test_pure_shift_at_theta0_exact(orc, gi):
    """e = (eps,0,eps,0): at theta=0 the radicand is (R_c - eps)^2 -> h = R_c - eps - R_k."""
    eps = 1.5e-6
    h, _ = orc.thickness(gi.grid(64, 32), _cond(gi, e=(eps, 0, eps, 0)))
    assert np.allclose(h[:, 0], (gi.R_C - eps) - gi.R_K, rtol=1e-10, atol=0)


def test_first_order_expansion(orc, gi):
    """h = (R_c-R_k) - (e1 + s y) cos(th) - (e2 + t y) sin(th) + O(|off|^2 / R_c).

    A sign, index or slope error in Eq. 2.3 (e.g. e3 <-> e4 swapped) changes h by
    ~1e-6 m; the quadratic remainder is < 1e-9 m."""
    rng = np.random.default_rng(3)
    g = gi.grid(48, 20)
    for _ in range(5):
        e = rng.uniform(-3e-6, 3e-6, 4)
        c = _cond(gi, e=e)
        h, _ = orc.thickness(g, c)
        LF = c[8]
        th = 2 * np.pi * np.arange(48) / 48
        y = (np.arange(-1, 21) + 1) * (LF / 21)
        ox = e[0] + (e[2] - e[0]) / LF * y
        oy = e[1] + (e[3] - e[1]) / LF * y
        lin = (gi.R_C - gi.R_K) - ox[:, None] * np.cos(th)[None] - oy[:, None] * np.sin(th)[None]
        assert np.max(np.abs(h - lin)) < 1.2e-9


def test_rate_closed_form(orc, gi):
    """e = 0, edot = (v,0,0,0), theta = 0, y = 0 -> dh/dt = -v."""
    v = 2.5e-5
    _, hd = orc.thickness(gi.grid(64, 32), _cond(gi, ed=(v, 0, 0, 0)))
    assert abs(hd[0, 0] - (-v)) <= 1e-15 * v
    _, hd = orc.thickness(gi.grid(64, 32), _cond(gi))
    assert np.all(hd == 0.0)


def test_rate_matches_time_difference(orc, gi):
    """dh/dt agrees with (h(e + dt edot) - h(e - dt edot)) / 2dt, dt = 1e-6 s."""
    rng = np.random.default_rng(11)
    g = gi.grid(32, 16, "smooth")
    dt = 1e-6
    for _ in range(4):
        e = rng.uniform(-2.1e-6, 2.1e-6, 4)
        ed = rng.uniform(-8e-5, 8e-5, 4)
        _, hd = orc.thickness(g, _cond(gi, e=e, ed=ed))
        hp, _ = orc.thickness(g, _cond(gi, e=e + dt * ed, ed=ed))
        hm, _ = orc.thickness(g, _cond(gi, e=e - dt * ed, ed=ed))
        fd = (hp - hm) / (2 * dt)
        scale = np.max(np.abs(hd))
        assert np.max(np.abs(fd - hd)) <= 1e-6 * scale


def test_theta_refinement_bitwise(orc, gi):
    """Doubling n_theta reproduces h bit for bit at the even nodes (uniform theta
    mesh: theta_i = i * 2pi/n_theta, P:45 'R_c cos theta')."""
    c = gi.condition(e=(1e-6, -0.5e-6, 2e-6, 0.3e-6))
    h1, _ = orc.thickness(gi.grid(40, 16), c)
    h2, _ = orc.thickness(gi.grid(80, 16), c)
    assert np.array_equal(h1, h2[:, ::2])
