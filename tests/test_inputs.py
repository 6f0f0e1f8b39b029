"""The shared input generator: Table 8 values (golden fixture) and the 9
working conditions of Eqs. 2.17-2.19."""
import json
import math
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(__file__), "golden", "table8.json")


def test_table8_values(gi):
    t8 = json.load(open(GOLD))
    assert gi.R_K == t8["R_k"] and abs(gi.R_C - t8["R_c"]) < 1e-17
    assert gi.R_B == t8["R_b"] and gi.L_FMIN == t8["L_Fmin"]
    assert abs(gi.BETA - math.radians(t8["beta_deg"])) < 1e-15
    assert list(gi.E_BASE) == t8["e"] and list(gi.EDOT_BASE) == t8["edot"]
    assert gi.DE == t8["delta_e"] and gi.DEDOT == t8["delta_edot"]
    assert gi.TEX_DEPTH == t8["tex_depth"]
    assert list(gi.TEXTURES["short"][:2]) == t8["short_texture"]
    assert list(gi.TEXTURES["long"][:2]) == t8["long_texture"]


def test_kinematics_readings(gi):
    """R-A20: L_F(90 deg) = 3.71412e-2 m, U_y(90 deg) = 0.44870 m/s; L_F(180) = L_Fmin."""
    assert abs(gi.coupling_length(math.pi / 2) - 3.71412e-2) < 1e-7
    assert abs(gi.stroke_speed(math.pi / 2) - 0.44870) < 1e-5
    assert abs(gi.coupling_length(math.pi) - gi.L_FMIN) < 1e-15
    assert abs(gi.OMEGA_S - 62.8319) < 1e-4


def test_fd_conditions_structure(gi):
    base = gi.condition()
    c = gi.fd_conditions(base)
    assert c.shape == (9, 13)
    assert np.array_equal(c[0], base)
    for j in range(4):
        d = c[1 + j] - base
        assert np.count_nonzero(d) == 1 and abs(d[j] - 1e-9) < 1e-21
        d = c[5 + j] - base
        assert np.count_nonzero(d) == 1 and abs(d[4 + j] - 1e-8) < 1e-20


def test_configs(gi):
    for name, shape, K in [("C1", (64, 32), 1), ("C2", (512, 256), 9), ("C3", (2048, 1024), 9),
                           ("C4", (1024, 512), 9), ("C5", (4096, 2048), 72)]:
        cfg = gi.config(name)
        assert (cfg.grid["n_theta"], cfg.grid["n_y"]) == shape and cfg.K == K
    assert gi.config("C3").grid["tex_band_rows"] == 256


def test_random_conditions_seeded(gi):
    a = gi.random_conditions(7, 3)
    b = gi.random_conditions(7, 3)
    assert np.array_equal(a, b) and not np.array_equal(a, gi.random_conditions(8, 3))
