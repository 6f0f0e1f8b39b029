"""Per-iteration time of the single-pass solve for C3-like row slabs on ONE GPU: the work one rank
of an N-way row split of C3 (2048 x 1024/N, K = 9, short texture) does per iteration, without the
exchange -- the compute side of the strong-scaling budget.  GMAF_SR_TW picks
the strip width."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

cfg = gi.config("C3")
for ny in (1024, 512, 256, 128):
    g = dict(cfg.grid, n_y=ny, tex_band_rows=max(ny // 4, 2 * cfg.grid["tex_n_y"]))
    S = P.JointSolver(g, 9)
    S.thickness(cfg.conds)
    S.assemble()
    S.solve_fixed(40, omega=cfg.omega)
    t = min(S.solve_fixed(400, omega=cfg.omega).solve_ms for _ in range(2)) * 1e3 / 400
    print(f"tw={os.environ.get('GMAF_SR_TW', '256')} n_y={ny}: {t:.1f} us/iter "
          f"({9 * 2048 * ny / t / 1e3:.1f} G DOF*iter/s)", flush=True)
    S.close()
