"""Pins of the Picard-driver oracle (oracle/picard.py; Sec. 2.3, Eqs. 2.10-2.22) and CPU parity
of the library's host-only generalized-force call (gmaf_general_forces, no GPU needed)."""
import math

import numpy as np
import pytest

import gmaf_inputs as gi
from oracle import picard as OP


def _wrench_of_points(forces, zs):
    """(F, M about the bottom centre) of lateral point forces on the axis at heights zs."""
    F = np.zeros(3)
    M = np.zeros(3)
    for f, z in zip(forces, zs):
        F += f
        M += np.cross([0.0, 0.0, z], f)
    return F, M


def test_generalized_force_equals_two_point_shape_functions():
    # virtual work of point forces = sum f (1 - z/L) at the bottom node + f z/L at the top node
    rng = np.random.default_rng(3)
    L = 0.037
    fs = [np.array([*rng.normal(size=2) * 100, 0.0]) for _ in range(7)]
    zs = rng.uniform(0, L, 7)
    F, M = _wrench_of_points(fs, zs)
    Q = OP.generalized(F, M, L)
    bottom = sum(f[:2] * (1 - z / L) for f, z in zip(fs, zs))
    top = sum(f[:2] * z / L for f, z in zip(fs, zs))
    np.testing.assert_allclose(Q, [bottom[0], bottom[1], top[0], top[1]], rtol=1e-12, atol=1e-10)


def test_mid_length_force_splits_in_half_and_wrench_round_trips():
    L = 0.04
    Q = OP.point_load(np.array([10.0, -4.0, 0.0]), L / 2, L)
    np.testing.assert_allclose(Q, [5.0, -2.0, 5.0, -2.0], rtol=1e-14)
    # (F1..F4) -> (F_X, F_Y, M_X, M_Y) reconstruction: F_X = F1 + F3, M_Y = L F3, F_Y = F2 + F4, M_X = -L F4
    rng = np.random.default_rng(5)
    w = rng.normal(size=12) * 50
    Q = OP.oil_force(w, L)
    np.testing.assert_allclose([Q[0] + Q[2], Q[1] + Q[3], -L * Q[3], L * Q[2]],
                               [w[0] + w[6], w[1] + w[7], w[3] + w[9], w[4] + w[10]], rtol=1e-12)
    assert np.all(OP.oil_force(np.zeros(12), L) == 0.0)


def test_loads_special_cases():
    pump = gi.pump()
    c = gi.condition(p_in=10e6)
    ext = OP.external_force(pump, c, 0.7)
    # p_in pi R_k^2 tan(beta) = 553.9 N, all at the top node
    assert abs(np.hypot(ext[2], ext[3]) - 10e6 * math.pi * 1e-4 * math.tan(math.radians(10))) < 1e-9
    assert abs(np.hypot(ext[2], ext[3]) - 553.9) < 0.1 and ext[0] == 0.0 and ext[1] == 0.0
    assert np.allclose(OP.external_force(dict(pump, beta=0.0), c, 0.7), 0.0)
    ine = OP.inertial_force(pump, c, 0.7)
    assert abs(ine.sum() - (pump["m_k"] + pump["m_G"]) * pump["omega_s"] ** 2 * pump["R_b"]) < 1e-12
    assert np.allclose(OP.inertial_force(dict(pump, omega_s=0.0), c, 0.7), 0.0)


def _linear_model(seed=0):
    rng = np.random.default_rng(seed)
    Ke = rng.normal(size=(4, 4)) * 1e8 + np.eye(4) * 5e8       # N/m
    Kv = rng.normal(size=(4, 4)) * 1e6 + np.eye(4) * 4e7       # N s/m
    F0 = rng.normal(size=4) * 100
    return Ke, Kv, F0


def test_fd_jacobians_of_a_linear_model_are_exact():
    Ke, Kv, F0 = _linear_model()
    base = gi.condition()
    conds = gi.fd_conditions(base)
    F9 = np.stack([F0 + Ke @ c[0:4] + Kv @ c[4:8] for c in conds])
    Je, Jv = OP.fd_jacobians(F9, gi.DE, gi.DEDOT)
    np.testing.assert_allclose(Je, Ke, rtol=1e-6)
    np.testing.assert_allclose(Jv, Kv, rtol=1e-6)


def test_general_update_reaches_the_linear_equilibrium():
    Ke, Kv, F0 = _linear_model(1)
    e, v, dt = np.full(4, 1e-7), np.full(4, 2e-6), 1e-4
    F = F0 + Ke @ e + Kv @ v
    e1, v1 = OP.update(F, Ke, Kv, e, v, dt, "general")
    np.testing.assert_allclose(e1 - e, dt * (v1 - v), rtol=1e-12, atol=1e-22)   # backward difference
    assert np.linalg.norm(F0 + Ke @ e1 + Kv @ v1) < 1e-8 * np.linalg.norm(F)
    # F = 0 -> unchanged (both schemes); J_e = 0 -> general == simplified
    for sch in ("general", "simplified"):
        e2, v2 = OP.update(np.zeros(4), Ke, Kv, e, v, dt, sch)
        assert np.array_equal(e2, e) and np.array_equal(v2, v)
    ga = OP.update(F, np.zeros((4, 4)), Kv, e, v, dt, "general")
    si = OP.update(F, Ke, Kv, e, v, dt, "simplified")
    np.testing.assert_allclose(ga[0], si[0], rtol=1e-14)
    np.testing.assert_allclose(ga[1], si[1], rtol=1e-14)
    # simplified scheme with no e-dependence is exact too (Eqs. 2.21-2.22)
    e3, v3 = OP.update(F0 + Kv @ v, np.zeros((4, 4)), Kv, e, v, dt, "simplified")
    assert np.linalg.norm(F0 + Kv @ v3) < 1e-8 * np.linalg.norm(F0 + Kv @ v)


def test_picard_iterations_on_the_reynolds_model_converge():
    # small mesh, base state of Table 8 at phi = 90 deg: the Newton-like general scheme drives
    # ||F|| down by orders of magnitude in a few iterations (P:345 reports 4-6 per step)
    g = gi.grid(32, 16)
    pump = gi.pump()
    phi, dt = math.pi / 2, 2 * math.pi / gi.OMEGA_S / 360.0
    state = gi.condition()
    norms = []
    for _ in range(4):
        it = OP.picard_iteration(g, pump, state, phi, dt, "general", tol=1e-12, omega=1.8)
        norms.append(np.linalg.norm(it["F"]))
        assert np.all(np.isfinite(it["J_e"])) and np.all(np.isfinite(it["J_edot"]))
        state = state.copy()
        state[0:4], state[4:8] = it["e_next"], it["edot_next"]
    assert norms[-1] < 1e-3 * norms[0], norms


def test_library_general_forces_match_the_oracle_on_cpu():
    import paper_2511_06824_b200 as P
    pump = gi.pump()
    rng = np.random.default_rng(9)
    for phi in (0.0, 1.1, 4.0):
        c = gi.condition(phi_deg=math.degrees(phi), p_in=gi.p_in_trapezoid(phi))
        w = rng.normal(size=12) * 300
        fo, fe, fi = P.general_forces(pump, c, phi, w)
        np.testing.assert_allclose(fo, OP.oil_force(w, c[8]), rtol=1e-13, atol=1e-12)
        np.testing.assert_allclose(fe, OP.external_force(pump, c, phi), rtol=1e-13, atol=1e-10)
        np.testing.assert_allclose(fi, OP.inertial_force(pump, c, phi), rtol=1e-13, atol=1e-12)


# ----------------------------------------------------------- the orbit drift
def test_pure_translation_has_no_static_film_force():
    """A translated, untilted piston (e1 = e3, e2 = e4) at rest with no sliding: h depends on theta
    only, every theta-column is a constant-coefficient 1-D problem, so p is the linear profile
    between p_in and p_out EXACTLY (Eq. 2.3 + Eqs. 2.4-2.7) and the lateral film force vanishes
    (pressure and shear); only the axial Poiseuille shear, larger where the gap is wider, leaves a
    small moment about the lateral axes (Sec. 2.4-III)."""
    import oracle as orc
    g = gi.grid(64, 32)
    c = gi.condition().copy()
    c[0:4] = (2e-6, -1e-6, 2e-6, -1e-6)
    c[4:8] = 0.0
    c[9] = c[10] = 0.0
    AP, AE, AN, S = orc.assemble(g, c)
    p = orc.cholesky_solve(orc.expand_dense(AP, AE, AN), S.ravel()).reshape(32, 64)
    j = np.arange(32)
    lin = c[11] + (c[12] - c[11]) * (j + 1) / 33.0
    assert np.max(np.abs(p - lin[:, None])) <= 1e-9 * c[11]
    w = orc.wrench(g, c, p)
    lateral = w[[0, 1, 3, 4, 6, 7]]          # Fp_x, Fp_y, Mp_x, Mp_y, Fs_x, Fs_y
    assert np.max(np.abs(lateral)) <= 1e-9 * np.max(np.abs(w))
    assert abs(w[9]) > 0 and abs(w[10]) > 0  # the axial-shear moment of the eccentric film


def test_static_film_stiffness_is_circulatory():
    """The film's static response to e under the p_in -> p_out pressure drop (no motion): a
    translation gives no force (above) while a TILT gives a lateral force (the tapered-gap
    'hydraulic lock' effect), so J_e = dF/de has the circulatory form [[a, -b], [b, -a]] per
    direction with a ~ b and no restoring stiffness for a translation (eigenvalues +-i*sqrt(b^2-a^2)).
    This is why the C4 orbit's mean position is not held by the film's static response: it drifts
    under the non-zero mean of the R-A29/A30 loads."""
    import oracle as orc
    g = gi.grid(64, 32)

    def F(e):
        c = gi.condition().copy()
        c[0:4], c[4:8], c[9], c[10] = e, 0.0, 0.0, 0.0
        res, W = orc.joint_step(g, c[None], tol=1e-12, omega=1.8)
        return OP.oil_force(W[0], c[8])

    h = 1e-8
    F0 = F(np.zeros(4))
    J = np.stack([(F(h * np.eye(4)[j]) - F0) / h for j in range(4)], axis=1)
    scale = np.abs(J).max()
    trans_x, tilt_x = np.array([1.0, 0, 1, 0]), np.array([1.0, 0, -1, 0])
    assert np.linalg.norm(J @ trans_x) <= 2e-3 * scale
    ft = J @ tilt_x
    assert ft[0] > 0 and ft[2] > 0 and abs(ft[0] - ft[2]) <= 2e-3 * scale   # a translating force
    assert np.all(np.abs(np.linalg.eigvals(J).real) <= 1e-3 * scale)


def _load_case(constant_p_in):
    def lc(phi):
        p_in = gi.P_IN if constant_p_in else gi.p_in_trapezoid(phi)
        return [gi.coupling_length(phi), 0.0, gi.stroke_speed(phi), p_in, gi.P_OUT]
    return lc


def test_orbit_bounded_under_a_zero_mean_load():
    """Under a load periodic by construction with ZERO mean -- constant p_in (the swashplate
    reaction (-cos phi, sin phi) * const, R-A29) and no centrifugal load (masses 0, R-A30) -- the
    Picard march settles into a bounded orbit: after the transient the per-revolution max |e|
    stops growing.  Under the R-A29/A30 loads themselves (trapezoid p_in: a non-zero mean lateral
    load) the same march drifts until the film is pinched (h < h_min), as the GPU's C4 trajectory
    drifted (profiles/round1_picard_3rev_c4.json): the drift is the load model, not the solver."""
    import oracle
    g = gi.grid(32, 16)
    pump0 = dict(gi.pump(), m_k=0.0, m_G=0.0)
    state0 = gi.condition(phi_deg=0.0, p_in=gi.P_IN)
    e = OP.march(g, pump0, state0, 8 * 36, 10.0, _load_case(True), omega=1.8) * 1e6
    per_rev = [np.abs(e[r * 36:(r + 1) * 36]).max() for r in range(8)]
    assert max(per_rev) < 6.0                                   # clearance R_c - R_k = 6 um
    # the transient (the mean position settling, ~4 revolutions) is over: no further growth
    assert all(per_rev[r + 1] <= 1.01 * per_rev[r] for r in (4, 5, 6)), per_rev
    # the R-A29/A30 loads: the mean position runs away (contact within a few revolutions)
    with pytest.raises((RuntimeError, oracle.OracleError)):
        OP.march(g, gi.pump(), gi.condition(phi_deg=0.0, p_in=gi.p_in_trapezoid(0.0)), 8 * 36, 10.0,
                 _load_case(False), omega=1.8)
