"""Pins for the oracle's FVM assembly (Eqs. 2.4-2.7).

Pinned by: exact symmetry, row-sum conservation, SPD (textbook Cholesky),
the structural fact that Eq. 2.3 has no e-dot (A_5..8 == A_0), closed-form
solutions of the discrete Reynolds problem (linear Poiseuille profile, constant
pressure), and an O(h^2) manufactured-solution convergence study against the
symbolically differentiated PDE (reading R-A1) -- none of which re-types the
oracle's own formulas.
"""
import math

import numpy as np
import pytest


def _zero_motion(gi, c, e=None):
    c = c.copy()
    if e is not None:
        c[0:4] = e
    c[4:8] = 0.0        # no squeeze
    c[9] = 0.0          # U_theta
    c[10] = 0.0         # U_y
    return c


def test_symmetric_bitwise(orc, gi):
    g = gi.grid(48, 24, "smooth")
    c = gi.random_conditions(5, 1)[0]
    AP, AE, AN, S = orc.assemble(g, c)
    A = orc.expand_dense(AP, AE, AN)
    assert np.array_equal(A, A.T)


def test_row_sums_are_dirichlet_faces(orc, gi):
    """Interior rows: A_P + sum(off-diagonals) = 0 (discrete conservation);
    boundary rows: the residual is the folded Dirichlet face (positive)."""
    g = gi.grid(40, 20, "smooth")
    AP, AE, AN, S = orc.assemble(g, gi.random_conditions(9, 1)[0])
    A = orc.expand_dense(AP, AE, AN)
    rs = A.sum(axis=1).reshape(20, 40)
    scale = AP.max()
    assert np.max(np.abs(rs[1:-1])) <= 8 * np.spacing(scale)
    assert np.all(rs[0] > 1e-3 * scale) and np.all(rs[-1] > 1e-3 * scale)
    assert np.all(AE < 0) and np.all(AN[:-1] < 0) and np.all(AN[-1] == 0)


def test_spd_cholesky(orc, gi):
    g = gi.grid(32, 16, "smooth")
    AP, AE, AN, S = orc.assemble(g, gi.random_conditions(2, 1)[0])
    A = orc.expand_dense(AP, AE, AN)
    orc.cholesky_solve(A, S.ravel())          # raises on a non-positive pivot
    assert np.linalg.eigvalsh(A).min() > 0


def test_edot_conditions_share_matrix(orc, gi):
    """Eq. 2.3 depends on e only, so A_5..A_8 == A_0 bitwise while
    A_1..A_4 differ; every S differs (Eqs. 2.18-2.19)."""
    g = gi.grid(64, 32, "smooth")
    conds = gi.fd_conditions(gi.condition())
    AP, AE, AN, S = orc.assemble_joint(g, conds)
    for k in range(5, 9):
        assert np.array_equal(AP[k], AP[0]) and np.array_equal(AE[k], AE[0]) and np.array_equal(AN[k], AN[0])
        assert not np.array_equal(S[k], S[0])
    for k in range(1, 5):
        assert not np.array_equal(AP[k], AP[0])
        assert not np.array_equal(S[k], S[0])


def test_linear_poiseuille_profile(orc, gi):
    """Uniform film, no motion, p_in != p_out -> p_j = p_in + (p_out-p_in)(j+1)/(n_y+1)
    (the 5-point stencil is exact on linear fields)."""
    g = gi.grid(40, 24, "smooth")
    c = _zero_motion(gi, gi.condition(), e=(0, 0, 0, 0))
    AP, AE, AN, S = orc.assemble(g, c)
    A = orc.expand_dense(AP, AE, AN)
    p = orc.cholesky_solve(A, S.ravel()).reshape(24, 40)
    j = np.arange(24)
    exact = c[11] + (c[12] - c[11]) * (j + 1) / 25.0
    assert np.max(np.abs(p - exact[:, None])) <= 1e-12 * c[11]


def test_constant_pressure(orc, gi):
    """p_in = p_out = P with no wedge or squeeze -> p == P, any film shape."""
    g = gi.grid(40, 24, "short", tex_n_theta=6, tex_n_y=3, tex_band_rows=12)
    c = _zero_motion(gi, gi.condition(), e=(1e-6, -2e-6, 0.5e-6, 1e-6))
    c[11] = c[12] = 3.3e6
    AP, AE, AN, S = orc.assemble(g, c)
    p = orc.cholesky_solve(orc.expand_dense(AP, AE, AN), S.ravel())
    assert np.max(np.abs(p - 3.3e6)) <= 1e-12 * 3.3e6


def test_mu_scaling(orc, gi):
    """Bands scale as 1/mu exactly when mu -> 2 mu (power-of-two); S's
    motion terms do not depend on mu."""
    g1 = gi.grid(32, 16, "smooth")
    g2 = dict(g1, mu=2 * g1["mu"])
    c = gi.random_conditions(4, 1)[0]
    a1 = orc.assemble(g1, c)
    a2 = orc.assemble(g2, c)
    for q in range(3):
        assert np.array_equal(a1[q], 2 * a2[q])


def _mms_problem(gi, orc, nt, ny):
    """Manufactured solution of div(g grad p) = f with g = h^3/(12 mu), h from Eq. 2.3
    (x = R_k theta), p* = p_in + (p_out-p_in) y/L + P1 sin(pi y/L) cos(theta)."""
    import sympy as sp
    th, y = sp.symbols("theta y", real=True)
    e = (1e-6, -0.5e-6, 2e-6, 0.3e-6)
    g = gi.grid(nt, ny, "smooth")
    c = _zero_motion(gi, gi.condition(), e=e)
    L, pin, pout, P1 = c[8], c[11], c[12], 2e6
    Rk, Rc, mu = g["R_k"], g["R_c"], g["mu"]
    a = Rc * sp.cos(th) - (e[2] - e[0]) / L * y - e[0]
    b = Rc * sp.sin(th) - (e[3] - e[1]) / L * y - e[1]
    h = sp.sqrt(a ** 2 + b ** 2) - Rk
    gg = h ** 3 / (12 * mu)
    p = pin + (pout - pin) * y / L + P1 * sp.sin(sp.pi * y / L) * sp.cos(th)
    f = sp.diff(gg * sp.diff(p, th) / Rk, th) / Rk + sp.diff(gg * sp.diff(p, y), y)
    ff = sp.lambdify((th, y), f, "numpy")
    pf = sp.lambdify((th, y), p, "numpy")
    AP, AE, AN, _ = orc.assemble(g, c)
    dth = 2 * math.pi / nt
    dy = L / (ny + 1)
    TH, Y = np.meshgrid(np.arange(nt) * dth, (np.arange(ny) + 1) * dy)
    # A = -(discrete div), so S = -f * cell area, plus the Dirichlet faces
    S = -ff(TH, Y) * (Rk * dth) * dy
    A = orc.expand_dense(AP, AE, AN) if nt * ny <= 4096 else None
    # boundary face conductances from the row sums (conservation, see test above)
    rowsum = (AP + AE + np.roll(AE, 1, axis=1))
    rowsum[1:] += AN[:-1]
    rowsum[:-1] += AN[:-1]
    S[0] += rowsum[0] * pin
    S[-1] += rowsum[-1] * pout
    return (AP, AE, AN), S, pf(TH, Y)


def test_manufactured_solution_second_order(orc, gi):
    """Max nodal error of the discrete solution vs p* decreases ~4x per halving of
    both spacings (n_theta -> 2 n_theta, n_y -> 2 n_y + 1): a consistent 2nd-order
    FVM discretisation of the Reynolds operator (reading R-A1, R-A3, R-A4)."""
    errs = []
    for nt, ny in [(32, 15), (64, 31), (128, 63)]:
        (AP, AE, AN), S, pex = _mms_problem(gi, orc, nt, ny)
        res = orc.pcg_joint(AP, AE, AN, S, tol=1e-14, precond="assor2", omega=1.5, max_iter=50000)
        errs.append(np.max(np.abs(res.p - pex)))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.5 <= r1 <= 4.5 and 3.5 <= r2 <= 4.5, (errs, r1, r2)


def test_discrete_manufactured_solution(orc, gi):
    """S := A p*, solve -> p* (<= 1e-8 at rtol 1e-12)."""
    g = gi.grid(64, 32, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8)
    AP, AE, AN, _ = orc.assemble(g, gi.condition())
    rng = np.random.default_rng(0)
    pstar = rng.uniform(1e5, 1e7, (32, 64))
    S = orc.spmv(AP, AE, AN, pstar)
    res = orc.pcg_joint(AP, AE, AN, S, tol=1e-12, precond="assor2", omega=1.6)
    assert res.converged
    assert np.linalg.norm(res.p - pstar) <= 1e-8 * np.linalg.norm(pstar)


# ------------------------------------------------------ the source's motion terms
def _source_mms(gi, orc, nt, ny):
    """S of orc_assemble with ALL motion terms live (e, e-dot, U_theta, U_y non-zero) and
    p_in = p_out = 0 (no Dirichlet folds), against the right-hand side of the Reynolds equation
    (reading R-A1): S / (dx dy) = -[(U_theta/2) dh/dx + (U_y/2) dh/dy + dh/dt] with x = R_k theta,
    h from Eq. 2.3 with e(t) = e + t e-dot, differentiated symbolically by sympy."""
    import sympy as sp
    th, y, t = sp.symbols("theta y t", real=True)
    e0 = (1.2e-6, -0.7e-6, 0.9e-6, 1.5e-6)
    ed = (3e-5, -2e-5, -4e-5, 1e-5)
    g = gi.grid(nt, ny)
    c = gi.condition().copy()
    c[0:4], c[4:8] = e0, ed
    c[9], c[10] = 0.37, 0.45          # U_theta, U_y
    c[11] = c[12] = 0.0               # p_in = p_out = 0
    L, Rk, Rc = c[8], g["R_k"], g["R_c"]
    e = [e0[i] + ed[i] * t for i in range(4)]
    a = Rc * sp.cos(th) - (e[2] - e[0]) / L * y - e[0]
    b = Rc * sp.sin(th) - (e[3] - e[1]) / L * y - e[1]
    h = sp.sqrt(a ** 2 + b ** 2) - Rk
    rhs = (c[9] / 2) * sp.diff(h, th) / Rk + (c[10] / 2) * sp.diff(h, y) + sp.diff(h, t)
    f = sp.lambdify((th, y), rhs.subs(t, 0), "numpy")
    _, _, _, S = orc.assemble(g, c)
    dth, dy = 2 * math.pi / nt, L / (ny + 1)
    TH, Y = np.meshgrid(np.arange(nt) * dth, (np.arange(ny) + 1) * dy)
    exact = -f(TH, Y)
    return np.max(np.abs(S / ((Rk * dth) * dy) - exact)), np.max(np.abs(exact))


def test_source_motion_terms_converge_to_the_reynolds_rhs(orc, gi):
    """The wedge terms (central differences, R-A5) converge at O(h^2) to the symbolic
    right-hand side and the squeeze term is exact: error ratio in [3.5, 4.5] over three
    refinements, and small against the right-hand side.  A dropped term, a sign error or a
    wrong factor in any of t1, t2, t3 (gmaf_oracle.c orc_assemble) leaves an O(1) error."""
    errs = [_source_mms(gi, orc, nt, ny) for nt, ny in [(32, 15), (64, 31), (128, 63), (256, 127)]]
    ratios = [errs[i][0] / errs[i + 1][0] for i in range(3)]
    assert all(3.5 <= q <= 4.5 for q in ratios), (errs, ratios)
    assert errs[-1][0] <= 2e-4 * errs[-1][1]


def test_squeeze_film_sign_and_damping(orc, gi):
    """Pure lateral translation e = 0, e-dot = (v, 0, v, 0), no sliding, p_in = p_out = 0:
    h-dot = -v cos(theta) (a closing gap at theta = 0).  The squeeze film must push back: by the
    maximum principle p = f(y) cos(theta) with f > 0, so sign(p) = sign(-h-dot) everywhere, and the
    pressure force opposes the motion (F_x < 0, negative power)."""
    g = gi.grid(64, 32)
    v = 1e-4
    c = gi.condition().copy()
    c[0:4], c[4:8] = 0.0, (v, 0.0, v, 0.0)
    c[9] = c[10] = 0.0
    c[11] = c[12] = 0.0
    AP, AE, AN, S = orc.assemble(g, c)
    _, hd = orc.thickness(g, c)
    p = orc.cholesky_solve(orc.expand_dense(AP, AE, AN), S.ravel()).reshape(32, 64)
    hdi = hd[1:-1]
    live = np.abs(hdi) > 0.05 * v
    assert np.all(np.sign(p[live]) == np.sign(-hdi[live]))
    assert p[16, 0] > 0 and p[16, 32] < 0
    w = orc.wrench(g, c, p)
    assert w[0] < 0 and abs(w[1]) <= 1e-9 * abs(w[0])


def test_squeeze_damping_matrix_is_symmetric_negative_definite(orc, gi):
    """J_e-dot (Eq. 2.14) from the 9-condition joint solve (Eq. 2.19): the
    e-dot-perturbed conditions differ from the base ONLY through the squeeze term of S, so
    J_e-dot = dF/d(e-dot) is the squeeze-film damping matrix.  The Reynolds operator is self-
    adjoint and F is the virtual work conjugate to e (R-A28), so it must be symmetric
    (reciprocity) and negative definite (dissipation) -- a sign or factor slip in the squeeze term
    or in the generalized-force mapping breaks one of the two; and dF1/d(e-dot 1) < 0."""
    import oracle.picard as OP
    g = gi.grid(64, 32)
    st = gi.condition()
    res, W = orc.joint_step(g, gi.fd_conditions(st), tol=1e-12, omega=1.8)
    assert res.converged
    Fo = np.stack([OP.oil_force(W[k], st[8]) for k in range(9)])
    _, Jv = OP.fd_jacobians(Fo, gi.DE, gi.DEDOT)
    assert Jv[0, 0] < 0
    assert np.max(np.abs(Jv - Jv.T)) <= 1e-8 * np.max(np.abs(Jv))
    assert np.linalg.eigvalsh(0.5 * (Jv + Jv.T)).max() < 0
