"""A/B timing of two builds of the library on the same GPU (same box, same clocks): per-iteration
time of fixed-iteration solves at C3 and at the 128-row slab (the strong-scaling unit), each
build in its own subprocess.  Usage: probe_ab.py ROOT_A ROOT_B ... (repository roots holding a built
paper_2511_06824_b200 package)."""
import os
import subprocess
import sys

CODE = r'''
import sys; sys.path.insert(0, sys.argv[1])
import gmaf_inputs as gi, paper_2511_06824_b200 as P
cfg = gi.config("C3")
out = []
for ny in (1024, 128):
    g = dict(cfg.grid, n_y=ny, tex_band_rows=max(ny // 4, 2 * cfg.grid["tex_n_y"]))
    S = P.JointSolver(g, 9, max_matrices=5)
    S.thickness(cfg.conds); S.assemble()
    S.solve_fixed(40, omega=cfg.omega)
    sts = [S.solve_fixed(400, omega=cfg.omega) for _ in range(3)]
    t = min(st.solve_ms * 1e3 / max(st.iterations, 1) for st in sts)   # per executed iteration
    out.append(round(t, 1)); S.close()
print(out)
'''
roots = sys.argv[1:]
for rep in range(2):
    for r in roots:
        res = subprocess.run([sys.executable, "-c", CODE, r], capture_output=True, text=True)
        print(rep, r, res.stdout.strip(), res.stderr.strip()[-300:], flush=True)
