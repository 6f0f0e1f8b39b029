"""ncu target (one GPU): C3 (short-textured 2048x1024, K = 9), thickness -> assembly -> one
fixed-iteration solve of N iterations (default 40) -- so that the persistent iteration kernel
k_srp of that solve can be captured and its DRAM bytes divided by N (per PCG iteration, the
unit of bench.py's roofline)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = gi.config(os.environ.get("CFG", "C3"))
S = P.JointSolver(cfg.grid, cfg.K, max_matrices=5 * (cfg.K // 9))
S.thickness(cfg.conds)
S.assemble()
st = S.solve_fixed(n_iter, omega=cfg.omega)
print("iterations", st.iterations, "solve_ms", round(st.solve_ms, 3), S.tile_config())
S.close()
