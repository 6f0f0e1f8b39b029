"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no thickness, assembly,
solve or quadrature).  It only produces the plain inputs both sides consume:
the mesh/texture description (a dict) and the K condition records
``[e1..e4, edot1..edot4, L_F, U_theta, U_y, p_in, p_out]`` (float64, shape
(K, 13)), following

* Table 8 for geometry, base state and FD steps,
* Eqs. 2.17-2.19 for the 9 working conditions of one Picard step
  (k=0 base; k=1..4 e_k += de; k=5..8 edot_{k-4} += dedot) -- SURVEY 8(a) row a1,
* Fig. 10 for the dimple arrays (60x10 short, 60x20 long, 20 um),
* DESIGN.md section 4 (the input recipe) for everything the paper leaves open
  (viscosity, sliding speed, coupling length law, p_in waveform).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Table 8
R_K = 1e-2
R_C = 1e-2 + 6e-6
R_B = 4.05e-2
L_FMIN = 3e-2
BETA = math.radians(10.0)
RPM = 600.0
OMEGA_S = 2.0 * math.pi * RPM / 60.0
E_BASE = (-0.2e-6, 0.2e-6, 0.2e-6, -0.2e-6)
EDOT_BASE = (-3.78e-7, 3.78e-7, 3.78e-7, -3.78e-7)
M_K = 0.128       # piston mass, kg (Table 8)
M_G = 0.0259      # slipper mass, kg (Table 8)
DE = 1e-9
DEDOT = 1e-8
# readings (R-A8/A20)
MU = 0.03
H_MIN = 5e-8
P_OUT = 0.5e6
P_IN = 10e6
TEX_DEPTH = 20e-6

TEXTURES = {
    "smooth": (0, 0, 0),
    "short": (60, 10, 4),   # (n_theta dimples, n_y dimples, band = n_y // divisor)
    "long": (60, 20, 2),
}


def grid(n_theta: int, n_y: int, texture: str = "smooth", **over) -> dict:
    """Mesh + texture description (same field names as both C structs)."""
    mt, my, div = TEXTURES[texture]
    g = dict(n_theta=int(n_theta), n_y=int(n_y), R_k=R_K, R_c=R_C, mu=MU, h_min=H_MIN,
             tex_n_theta=mt, tex_n_y=my, tex_band_rows=(n_y // div if div else 0),
             tex_fill_num=1, tex_fill_den=2, tex_depth=(TEX_DEPTH if div else 0.0))
    g.update(over)
    return g


def pump() -> dict:
    """Table 8 pump constants for the Picard driver (masses, pitch radius, swash angle, speed)."""
    return dict(m_k=M_K, m_G=M_G, R_b=R_B, beta=BETA, omega_s=OMEGA_S, R_k=R_K)


def coupling_length(phi: float) -> float:
    """L_F(phi) = L_Fmin + R_b tan(beta) (1 + cos phi)  (reading R-A20)."""
    return L_FMIN + R_B * math.tan(BETA) * (1.0 + math.cos(phi))


def stroke_speed(phi: float) -> float:
    """Axial sliding speed U_y(phi) = omega_s R_b tan(beta) sin(phi) (R-A20)."""
    return OMEGA_S * R_B * math.tan(BETA) * math.sin(phi)


def p_in_trapezoid(phi: float, lo: float = P_OUT, hi: float = P_IN) -> float:
    """Inlet pressure waveform stand-in for the unpublished Fig. 9: 50% duty,
    5% ramps (R-A8)."""
    x = (phi / (2.0 * math.pi)) % 1.0
    ramp = 0.05
    if x < ramp:
        return lo + (hi - lo) * x / ramp
    if x < 0.5:
        return hi
    if x < 0.5 + ramp:
        return hi - (hi - lo) * (x - 0.5) / ramp
    return lo


def condition(e=E_BASE, edot=EDOT_BASE, phi_deg: float = 90.0, p_in: float | None = None,
              U_theta: float = 0.0) -> np.ndarray:
    phi = math.radians(phi_deg)
    return np.array(list(e) + list(edot) + [coupling_length(phi), U_theta, stroke_speed(phi),
                    P_IN if p_in is None else p_in, P_OUT], dtype=np.float64)


def fd_conditions(base: np.ndarray, de: float = DE, dedot: float = DEDOT) -> np.ndarray:
    """The 9 working conditions of Eqs. 2.17-2.19."""
    base = np.asarray(base, dtype=np.float64).reshape(13)
    out = np.repeat(base[None], 9, axis=0)
    for j in range(4):
        out[1 + j, j] += de          # A_j = A(e_j + de_j), j = 1..4
        out[5 + j, 4 + j] += dedot   # A_{j+4} = A(edot_j + dedot_j)
    return out


def random_conditions(seed: int, K: int, e_max: float = 3e-6, edot_max: float = 1e-4,
                      phi_deg: float | None = None) -> np.ndarray:
    """Randomised states for parity sweeps."""
    rng = np.random.default_rng(seed)
    out = np.empty((K, 13))
    for k in range(K):
        phi = rng.uniform(0.0, 360.0) if phi_deg is None else phi_deg
        e = rng.uniform(-e_max, e_max, 4)
        ed = rng.uniform(-edot_max, edot_max, 4)
        c = condition(e, ed, phi_deg=phi, p_in=float(rng.uniform(P_OUT, P_IN)),
                      U_theta=float(rng.uniform(-0.5, 0.5)))
        out[k] = c
    return out


@dataclass
class Config:
    name: str
    grid: dict
    conds: np.ndarray
    omega: float
    tol: float
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def K(self) -> int:
        return int(self.conds.shape[0])

    @property
    def dof(self) -> int:
        return self.K * self.grid["n_theta"] * self.grid["n_y"]


def c5_conditions() -> np.ndarray:
    """72 = 8 operating points x 9."""
    rows = []
    for m in range(8):
        phi = 45.0 * m
        s = math.sin(math.radians(phi))
        e = [x * (1.0 + 0.5 * s) for x in E_BASE]
        ed = [x * math.cos(math.radians(phi)) for x in EDOT_BASE]
        base = condition(e, ed, phi_deg=phi, p_in=p_in_trapezoid(math.radians(phi)))
        rows.append(fd_conditions(base))
    return np.concatenate(rows)


def c4_step_conditions(step: int, q: int) -> np.ndarray:
    """Replayed synthetic orbit for C4: shaft angle step*1 deg,
    Picard iterate q scales e by (1 + 10^-(q+2))."""
    phi = math.radians(float(step))
    s, c = math.sin(phi), math.cos(phi)
    f = 1.0 + 10.0 ** (-(q + 2))
    e = [x * (1.0 + 0.5 * s) * f for x in E_BASE]
    ed = [x * 0.5 * OMEGA_S * c for x in E_BASE]
    base = condition(e, ed, phi_deg=float(step), p_in=p_in_trapezoid(phi))
    return fd_conditions(base)


def config(name: str) -> Config:
    """BASELINE.json configs C1..C5."""
    base = condition()
    if name == "C1":
        return Config("C1", grid(64, 32), base[None].copy(), 1.8, 1e-10,
                      "smooth 64x32, K=1, rtol 1e-10")
    if name == "C2":
        return Config("C2", grid(512, 256), fd_conditions(base), 1.8, 1e-10,
                      "smooth 512x256, K=9")
    if name == "C3":
        return Config("C3", grid(2048, 1024, "short"), fd_conditions(base), 1.6, 1e-10,
                      "short-textured 2048x1024, K=9")
    if name == "C4":
        return Config("C4", grid(1024, 512, "short"), c4_step_conditions(0, 0), 1.6, 1e-10,
                      "short-textured 1024x512, K=9 per Picard step")
    if name == "C5":
        return Config("C5", grid(4096, 2048, "short"), c5_conditions(), 1.6, 1e-10,
                      "short-textured 4096x2048, K=72")
    raise KeyError(name)


def table_case(n_theta: int, n_y: int, texture: str, K: int = 1) -> Config:
    """Paper Tables 4-6 analogues: omega 1.8 smooth, 1.6 textured, tol 1e-6."""
    base = condition()
    conds = fd_conditions(base) if K == 9 else base[None].copy()
    omega = 1.8 if texture == "smooth" else 1.6
    return Config(f"{texture}{n_theta}x{n_y}", grid(n_theta, n_y, texture), conds, omega, 1e-6)
