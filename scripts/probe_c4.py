import sys; sys.path.insert(0, sys.argv[1])
import gmaf_inputs as gi, paper_2511_06824_b200 as P
cfg = gi.config("C4")
S = P.JointSolver(cfg.grid, 9, max_matrices=5)
S.thickness(cfg.conds); S.assemble(); S.solve_fixed(40, omega=1.6)
sts = [S.solve_fixed(400, omega=1.6) for _ in range(3)]
print(sys.argv[1], "C4 us/iter", round(min(st.solve_ms * 1e3 / st.iterations for st in sts), 2))
