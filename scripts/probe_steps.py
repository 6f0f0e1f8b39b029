"""Where a row step's cycles go (timing-only build: GMAF_NVCC_EXTRA=-DGMAF_STEP_PROBE): per warp,
the mean clock() cycles per row step of [wait for the TMA data | phase A up to barrier 1 |
barrier 1 | phases B-D up to barrier 2 | barrier 2 | phases E-G], for a seam CTA (strip 0) and a
plain CTA (strip 1), C3 persistent solve, 400 fixed iterations."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

cfg = gi.config("C3")
S = P.JointSolver(cfg.grid, 9, max_matrices=5)
S.thickness(cfg.conds)
S.assemble()
S.solve_fixed(40, omega=cfg.omega)
L = P.lib()
n = 2048 * 16 * 8
buf = (C.c_uint * n)()
L.gmaf_debug_step_probe(buf, n, 1)
iters = 400
st = S.solve_fixed(iters, omega=cfg.omega)
L.gmaf_debug_step_probe(buf, n, 0)
a = np.array(buf, dtype=np.float64).reshape(2048, 16, 8)[:, :, :6]
t = S.tile_config()
steps = (t["th"] + 8) * iters
print("solve", round(st.solve_ms * 1e3 / iters, 1), "us/iter;", t, "steps per pass", t["th"] + 8)
names = ["data", "A", "bar1", "B-D", "bar2", "E-G"]
for cta, lab in ((0, "seam CTA (strip 0)"), (9, "plain CTA (strip 1)")):
    print(lab)
    for w in range(9):
        v = a[cta, w] / steps
        print(f"  warp {w}: " + "  ".join(f"{nm} {x:6.0f}" for nm, x in zip(names, v)) + f"  total {v.sum():6.0f}")
S.close()
