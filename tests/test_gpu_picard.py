"""GPU parity of the Picard driver (gmaf_picard_iteration / gmaf_picard_step, Sec. 2.3) against
the oracle (oracle/picard.py) on the same seeded states, through the C ABI."""
import math

import numpy as np
import pytest

import gmaf_inputs as gi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    from paper_2511_06824_b200 import build as B
    B.build()
    import paper_2511_06824_b200 as P
    return P


def relnorm(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("scheme,texture", [("general", "smooth"), ("simplified", "smooth"), ("general", "short")])
def test_picard_iteration_matches_oracle(P, scheme, texture):
    from oracle import picard as OP
    g = gi.grid(64, 32) if texture == "smooth" else gi.grid(120, 80, "short")
    pump = gi.pump()
    phi = 1.2
    state = gi.condition(phi_deg=math.degrees(phi), p_in=gi.p_in_trapezoid(phi))
    dt = 2 * math.pi / gi.OMEGA_S / 360.0
    omega = 1.8 if texture == "smooth" else 1.6
    S = P.JointSolver(g, 9)
    got = S.picard_iteration(pump, state, phi, dt, scheme, tol=1e-11, omega=omega)
    ref = OP.picard_iteration(g, pump, state, phi, dt, scheme, tol=1e-11, omega=omega)
    S.close()
    # loads are host arithmetic on the same inputs
    np.testing.assert_allclose(got["F_ext"], ref["F_ext"], rtol=1e-13, atol=1e-10)
    np.testing.assert_allclose(got["F_inertial"], ref["F_inertial"], rtol=1e-13, atol=1e-12)
    # oil force: two solves at rtol 1e-11 (R-A23: ~1e-10 agreement)
    assert relnorm(got["F_oil"], ref["F_oil"]) < 1e-8
    assert relnorm(got["F"], ref["F"]) < 1e-8
    # FD Jacobians: differences of forces 1e-9 m / 1e-8 m/s apart amplify the solve error
    assert relnorm(got["J_e"], ref["J_e"]) < 1e-4
    assert relnorm(got["J_edot"], ref["J_edot"]) < 1e-4
    du_g = np.concatenate([got["e_next"] - state[0:4], got["edot_next"] - state[4:8]])
    du_r = np.concatenate([ref["e_next"] - state[0:4], ref["edot_next"] - state[4:8]])
    assert relnorm(du_g, du_r) < 1e-4


def test_picard_step_converges_like_the_oracle(P):
    from oracle import picard as OP
    g = gi.grid(64, 32)
    pump = gi.pump()
    dt = 2 * math.pi / gi.OMEGA_S / 360.0
    phi = 0.5
    prev = gi.condition(phi_deg=math.degrees(phi), p_in=gi.p_in_trapezoid(phi))
    S = P.JointSolver(g, 9)
    new, n_pic, res, pcg, code = S.picard_step(pump, prev, phi, dt, "general", eps_dyn=1e-6, max_picard=12,
                                               tol=1e-11, omega=1.8)
    S.close()
    assert code == 0 and 1 <= n_pic <= 12 and res <= 1e-6 and pcg > 0
    # the oracle's march of the same step (R-A31): start at e_l + dt edot_l, iterate to the test
    cur = prev.copy()
    cur[0:4] = prev[0:4] + dt * prev[4:8]
    scale = max(np.linalg.norm(OP.external_force(pump, cur, phi)), 1.0)
    for k in range(12):
        it = OP.picard_iteration(g, pump, cur, phi, dt, "general", tol=1e-11, omega=1.8)
        if np.linalg.norm(it["F"]) / scale <= 1e-6:
            break
        cur = cur.copy()
        cur[0:4], cur[4:8] = it["e_next"], it["edot_next"]
    assert k + 1 == n_pic
    # same iterates (the Jacobians agree to ~1e-11): the converged states agree closely
    assert relnorm(new[0:4], cur[0:4]) < 1e-8
    assert relnorm(new[4:8], cur[4:8]) < 1e-6
    # backward difference of the time step (R-A31): e_{l+1} = e_l + dt edot_{l+1}
    np.testing.assert_allclose(new[0:4] - prev[0:4], dt * new[4:8], rtol=1e-9, atol=1e-20)


def test_picard_errors(P):
    g = gi.grid(64, 32)
    S = P.JointSolver(g, 3)
    with pytest.raises(P.GmafError) as ei:
        S.picard_iteration(gi.pump(), gi.condition(), 0.0, 1e-4)
    assert ei.value.code == -1
    S.close()
    S = P.JointSolver(g, 9)
    with pytest.raises(P.GmafError) as ei:
        S.picard_iteration(gi.pump(), gi.condition(), 0.0, -1.0)
    assert ei.value.code == -1
    S.close()


def test_march_matches_the_oracle_and_stays_bounded(P):
    """The product's Picard march (gmaf_picard_step) under a zero-mean periodic load (constant
    p_in: the R-A29 swashplate reaction rotates in the piston frame; no centrifugal load) follows
    the oracle's march (oracle.picard.march, R-A31) over a revolution and settles into a bounded
    orbit over 8 (the R-A29/A30 mean load is what made C4's orbit drift)."""
    from oracle import picard as OP
    g = gi.grid(32, 16)
    pump0 = dict(gi.pump(), m_k=0.0, m_G=0.0)
    deg = 10.0
    dt = 2 * math.pi / gi.OMEGA_S / 360.0 * deg

    def lc(phi):
        return [gi.coupling_length(phi), 0.0, gi.stroke_speed(phi), gi.P_IN, gi.P_OUT]

    state0 = gi.condition(phi_deg=0.0, p_in=gi.P_IN)
    S = P.JointSolver(g, 9)
    state = state0.copy()
    E = []
    for s in range(1, 8 * 36 + 1):
        phi = math.radians(s * deg)
        state = state.copy()
        state[8:13] = lc(phi)
        state, n_pic, res, pcg, code = S.picard_step(pump0, state, phi, dt, "general", eps_dyn=1e-3,
                                                     max_picard=20, tol=1e-10, omega=1.8)
        assert code == 0
        E.append(state[0:4].copy())
    S.close()
    E = np.array(E) * 1e6
    ref = OP.march(g, pump0, state0, 36, deg, lc, omega=1.8) * 1e6
    assert relnorm(E[:36], ref) <= 1e-6, relnorm(E[:36], ref)
    per_rev = [np.abs(E[r * 36:(r + 1) * 36]).max() for r in range(8)]
    assert max(per_rev) < 6.0 and all(per_rev[r + 1] <= 1.01 * per_rev[r] for r in (4, 5, 6)), per_rev
