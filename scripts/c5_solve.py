"""C5 on ONE B200 (4096x2048 short-textured, K = 72 = 8 operating points x 9):
one full joint solve to rtol 1e-10, coupled and lockstep.  Writes gpurun_out/c5_solve.json."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

cfg = gi.config("C5")
S = P.JointSolver(cfg.grid, cfg.K)
out = {"dof": cfg.dof, "K": cfg.K}
for coupling in sys.argv[1:] or ["coupled"]:
    t0 = time.perf_counter()
    st, W = S.step(cfg.conds, tol=cfg.tol, omega=cfg.omega, coupling=coupling)
    wall = time.perf_counter() - t0
    out[coupling] = dict(iterations=st.iterations, converged=st.converged, solve_ms=st.solve_ms, wall_s=wall,
                         rel=st.rel_residual, true_rel=st.true_rel_residual,
                         dof_iter_per_s=cfg.dof * st.iterations / (st.solve_ms * 1e-3))
    print(coupling, out[coupling], flush=True)
S.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c5_solve.json", "w"), indent=1)
