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
