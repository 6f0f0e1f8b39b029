"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

for sched in ("single", "table1"):
    g = gi.grid(96, 24, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8)
    S = P.JointSolver(g, 3)
    S.set_schedule(sched)
    st, W = S.step(gi.random_conditions(5, 3), tol=1e-8, omega=1.6, max_iter=3000)
    st2 = S.solve(tol=1e-8, omega=1.6, coupling="lockstep", max_iter=60, warm=True, raise_on_error=False)
    if sched == "single":
        st3 = S.solve(tol=1e-8, omega=1.6, coupling="async", max_iter=20, raise_on_error=False)
    print(sched, st.iterations, st.converged, st2.iterations)
    S.close()
# the persistent kernel's split seam loops (long row chunks; forced on a small mesh)
os.environ["GMAF_SEAM_SPLIT"] = "1"
g = gi.grid(96, 24, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8)
S = P.JointSolver(g, 3)
st, W = S.step(gi.random_conditions(5, 3), tol=1e-8, omega=1.6, max_iter=3000)
print("split seam", st.iterations, st.converged, S.tile_config())
S.close()
os.environ.pop("GMAF_SEAM_SPLIT")
# the compile-time strip widths of the persistent kernel (256 for 256 <= n_theta < 1024, 512 above)
for nt, ny in ((256, 12), (1024, 10)):
    g = gi.grid(nt, ny, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8)
    S = P.JointSolver(g, 2)
    S.thickness(gi.random_conditions(7, 2))
    S.assemble()
    st = S.solve(tol=1e-8, omega=1.6, max_iter=40, raise_on_error=False)
    print("tw", S.tile_config()["tw"], st.iterations, S.tile_config()["persistent"])
    S.close()
print("sanitize run done")
