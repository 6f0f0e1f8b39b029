"""Picard time march on the GPU (Sec. 2.3; SURVEY 8(d) C4 "ms per Picard step"): C4's mesh
(short-textured 1024x512, K = 9 per Picard iteration), Table 8 pump, 1-degree time steps from
phi0, general scheme, eps_dyn 1e-3 (R-A31).  Writes gpurun_out/picard_march.json."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import gmaf_inputs as gi
import paper_2511_06824_b200 as P

n_theta, n_y = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (1024, 512)))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
scheme = sys.argv[4] if len(sys.argv) > 4 else "general"
g = gi.grid(n_theta, n_y, "short")
pump = gi.pump()
dt = 2 * math.pi / gi.OMEGA_S / 360.0
S = P.JointSolver(g, 9)
state = gi.condition(phi_deg=0.0, p_in=gi.p_in_trapezoid(0.0))
rows = []
for s in range(1, steps + 1):
    phi = s * math.pi / 180.0
    state = state.copy()
    state[8:13] = [gi.coupling_length(phi), 0.0, gi.stroke_speed(phi), gi.p_in_trapezoid(phi), gi.P_OUT]
    t0 = time.perf_counter()
    new, n_pic, res, pcg, code = S.picard_step(pump, state, phi, dt, scheme, eps_dyn=1e-3, max_picard=20,
                                               tol=1e-10, omega=1.6, raise_on_error=False)
    ms = 1e3 * (time.perf_counter() - t0)
    rows.append(dict(step=s, phi_deg=s, picard_iterations=n_pic, residual=res, pcg_iterations=pcg,
                     status=code, ms=ms, e=new[0:4].tolist(), edot=new[4:8].tolist()))
    print(f"step {s}: {n_pic} Picard iterations, residual {res:.2e}, {pcg} PCG iterations, "
          f"{ms:.1f} ms ({ms / max(n_pic, 1):.1f} ms per Picard iteration), status {code}", flush=True)
    state = new
S.close()
out = dict(mesh=[n_theta, n_y], texture="short", K=9, scheme=scheme, dt=dt, eps_dyn=1e-3,
           steps=rows, ms_per_picard_iteration=float(np.sum([r["ms"] for r in rows]) /
                                                     max(1, sum(r["picard_iterations"] for r in rows))))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/picard_march.json", "w"), indent=1)
print("ms per Picard iteration:", round(out["ms_per_picard_iteration"], 2))
