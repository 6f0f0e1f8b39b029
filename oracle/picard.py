"""Oracle of the Picard driver (Sec. 2.3, Eqs. 2.10-2.22) -- TEST
INFRASTRUCTURE ONLY (same import rule as the package: tests, smoke, bench's CPU legs).

Plain numpy, step by step in the paper's order:
  * the 9 working conditions (Eqs. 2.17-2.19) are solved jointly by the C oracle
    (``oracle.joint_step``), which also integrates their wrenches (Sec. 2.4-III);
  * generalized forces F = {F1..F4} (Eq. 2.11) from the RIGID-BODY VIRTUAL WORK of each load
    under the four unit virtual displacements of e (readings R-A28..R-A30) --
    evaluated here from the displacement field, not from a closed form;
  * finite-difference Jacobians (Eqs. 2.13-2.14), forward differences;
  * the update (R-A31): simplified Eqs. 2.21-2.22 or the general Eq. 2.12 with the backward
    difference e' - e = dt (edot' - edot), by ``numpy.linalg.solve``.
"""
from __future__ import annotations

import math

import numpy as np

import gmaf_inputs as gi

from . import joint_step


def _rigid_motion(de: np.ndarray, L: float):
    """Translation t (at the bottom centre) and small rotation psi of the rigid piston whose axis
    points move by (de1, de2) at y = 0 and (de3, de4) at y = L (Eq. 2.3's axis line)."""
    t = np.array([de[0], de[1], 0.0])
    # axis point at height z moves by t + psi x (0, 0, z) = (t_x + psi_y z, t_y - psi_x z, .)
    psi = np.array([-(de[3] - de[1]) / L, (de[2] - de[0]) / L, 0.0])
    return t, psi


def generalized(force: np.ndarray, moment: np.ndarray, L: float) -> np.ndarray:
    """Q_j = virtual work of the load (force, moment about the bottom centre) under unit de_j."""
    Q = np.zeros(4)
    for j in range(4):
        t, psi = _rigid_motion(np.eye(4)[j], L)
        Q[j] = force @ t + moment @ psi
    return Q


def oil_force(wrench12, L: float) -> np.ndarray:
    """R-A28: generalized force of an oil-film wrench (pressure + shear parts, gmaf layout)."""
    w = np.asarray(wrench12, dtype=np.float64)
    return generalized(w[0:3] + w[6:9], w[3:6] + w[9:12], L)


def point_load(f: np.ndarray, z: float, L: float) -> np.ndarray:
    """Generalized force of a lateral point force f = (f_X, f_Y, 0) acting on the axis at height z."""
    f = np.asarray(f, dtype=np.float64)
    return generalized(f, np.cross(np.array([0.0, 0.0, z]), f), L)


def external_force(pump: dict, cond, phi: float) -> np.ndarray:
    """R-A29: lateral swashplate reaction to the pressure thrust on the piston bottom, at y = L_F."""
    c = np.asarray(cond, dtype=np.float64)
    L, p_in = c[8], c[11]
    thrust = p_in * math.pi * pump["R_k"] ** 2
    lateral = thrust * math.tan(pump["beta"])
    return point_load(np.array([-lateral * math.cos(phi), lateral * math.sin(phi), 0.0]), L, L)


def inertial_force(pump: dict, cond, phi: float) -> np.ndarray:
    """R-A30: centrifugal load of the piston (at L_F/2) and the slipper (at L_F), radial (+X)."""
    L = float(np.asarray(cond)[8])
    a = pump["omega_s"] ** 2 * pump["R_b"]
    return (point_load(np.array([pump["m_k"] * a, 0.0, 0.0]), 0.5 * L, L)
            + point_load(np.array([pump["m_G"] * a, 0.0, 0.0]), L, L))


def fd_jacobians(F9: np.ndarray, de: float, dedot: float):
    """Eqs. 2.13-2.14: column j of dF/de from condition 1+j, of dF/d(edot) from 5+j."""
    F9 = np.asarray(F9, dtype=np.float64)
    Je = np.stack([(F9[1 + j] - F9[0]) / de for j in range(4)], axis=1)
    Jv = np.stack([(F9[5 + j] - F9[0]) / dedot for j in range(4)], axis=1)
    return Je, Jv


def update(F, Je, Jv, e, edot, dt: float, scheme: str):
    """R-A31.  simplified: Eqs. 2.21-2.22; general: Eq. 2.12 with e' - e = dt (edot' - edot)."""
    M = Jv if scheme == "simplified" else dt * Je + Jv
    d = np.linalg.solve(M, -np.asarray(F, dtype=np.float64))
    return np.asarray(e) + dt * d, np.asarray(edot) + d


def picard_iteration(g: dict, pump: dict, state, phi: float, dt: float, scheme="general", de=gi.DE,
                     dedot=gi.DEDOT, tol=1e-10, omega=1.6) -> dict:
    """One Picard iteration: 9 joint solves, general forces, Jacobians, update."""
    state = np.asarray(state, dtype=np.float64).reshape(13)
    conds = gi.fd_conditions(state, de, dedot)
    res, W = joint_step(g, conds, tol=tol, omega=omega)
    L = state[8]
    Fo = np.stack([oil_force(W[k], L) for k in range(9)])
    Fe = external_force(pump, state, phi)
    Fi = inertial_force(pump, state, phi)
    F = Fe + Fi + Fo[0]
    Je, Jv = fd_jacobians(Fo, de, dedot)
    e_next, edot_next = update(F, Je, Jv, state[0:4], state[4:8], dt, scheme)
    return dict(F=F, F_oil=Fo[0], F_ext=Fe, F_inertial=Fi, J_e=Je, J_edot=Jv, e_next=e_next,
                edot_next=edot_next, wrench=W[0], pcg_iterations=res.iterations)


def picard_step(g: dict, pump: dict, prev, phi: float, dt: float, scheme="general", eps_dyn=1e-3,
                max_picard=20, tol=1e-10, omega=1.6):
    """One time step t_l -> t_l + dt (Sec. 2.3; R-A31): start from e = e_l + dt edot_l,
    edot = edot_l (prev carries e_l, edot_l and the load case of t_l + dt) and iterate until
    ||F|| <= eps_dyn max(||F_E||, 1 N).  Returns (state, Picard iterations, converged)."""
    cur = np.asarray(prev, dtype=np.float64).reshape(13).copy()
    cur[0:4] = cur[0:4] + dt * cur[4:8]
    scale = max(np.linalg.norm(external_force(pump, cur, phi)), 1.0)
    for k in range(max_picard):
        it = picard_iteration(g, pump, cur, phi, dt, scheme, tol=tol, omega=omega)
        if np.linalg.norm(it["F"]) <= eps_dyn * scale:
            return cur, k + 1, True
        cur = cur.copy()
        cur[0:4], cur[4:8] = it["e_next"], it["edot_next"]
    return cur, max_picard, False


def march(g: dict, pump: dict, state0, n_steps: int, deg: float, load_case, scheme="general", omega=1.6):
    """The Picard time march over n_steps steps of `deg` degrees from shaft angle 0: load_case(phi)
    -> (L_F, U_theta, U_y, p_in, p_out) of each step.  Returns the [n_steps][4] eccentricities."""
    dt = 2 * math.pi / pump["omega_s"] / 360.0 * deg
    state = np.asarray(state0, dtype=np.float64).reshape(13).copy()
    out = []
    for s in range(1, n_steps + 1):
        phi = math.radians(s * deg)
        state[8:13] = load_case(phi)
        state, _, ok = picard_step(g, pump, state, phi, dt, scheme, omega=omega)
        if not ok:
            raise RuntimeError(f"march: step {s} did not converge")
        out.append(state[0:4].copy())
    return np.array(out)
