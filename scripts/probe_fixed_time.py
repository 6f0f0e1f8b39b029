"""Per-iteration time of a fixed-iteration C3 solve (graph launch, CUDA events)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P
cfg = gi.config("C3")
S = P.JointSolver(cfg.grid, 9)
S.thickness(cfg.conds)
S.assemble()
S.solve_fixed(40, omega=cfg.omega)
ts = [S.solve_fixed(800, omega=cfg.omega).solve_ms for _ in range(3)]
print(os.environ.get("GMAF_LIB", "main"), "us/iter", [round(t * 1e3 / 800, 1) for t in ts])
