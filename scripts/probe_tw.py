"""Per-iteration time of the persistent solve for strip widths with and without a partial compute
warp: n_theta = 4 x 512 (tw 512: 8 full compute warps + one with 4 lanes) against n_theta =
4 x 496 (tw 496: 8 full compute warps), same n_y and K -- is the third compute warp on SM
sub-partition 0 what paces the row pipeline?"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

cfg = gi.config("C3")
for nt, tw in ((2048, None), (1984, "496"), (2048, None), (1984, "496")):
    if tw:
        os.environ["GMAF_SR_TW"] = tw
    g = dict(cfg.grid, n_theta=nt)
    S = P.JointSolver(g, 9, max_matrices=5)
    os.environ.pop("GMAF_SR_TW", None)
    S.thickness(cfg.conds)
    S.assemble()
    S.solve_fixed(40, omega=cfg.omega)
    t = min(S.solve_fixed(400, omega=cfg.omega).solve_ms for _ in range(3)) * 1e3 / 400
    tc = S.tile_config()
    print(f"n_theta={nt} tw={tc['tw']} ctas={tc['n_ctas']}: {t:.1f} us/iter, "
          f"{9 * nt * g['n_y'] / t / 1e3:.1f} G DOF*iter/s", flush=True)
    S.close()
