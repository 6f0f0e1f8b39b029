"""Per-iteration time of a ONE-rank row-slab / peer-to-peer context (the exchange code paths of
the multi-rank solve without peers: local barrier + gather of the per-condition sums + scalar
stage inside the persistent kernel) against the plain single-rank solve, C3-like slabs."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

cfg = gi.config("C3")
for ny in (1024, 128):
    g = dict(cfg.grid, n_y=ny, tex_band_rows=max(ny // 4, 2 * cfg.grid["tex_n_y"]))
    out = []
    for mode in ("single", "rows", "p2p", "rows_per_launch"):
        kw = {} if mode == "single" else ({"rank": 0, "world": 1, "shard": "rows"} if mode.startswith("rows")
                                          else {"rank": 0, "world": 1, "p2p": True})
        if mode == "rows_per_launch":
            os.environ["GMAF_PERSIST"] = "0"   # the per-iteration kernels + exchange kernels
        S = P.JointSolver(g, 9, **kw)
        os.environ.pop("GMAF_PERSIST", None)
        if mode != "single":
            S.p2p_connect([S.p2p_handle()])
        S.thickness(cfg.conds)
        S.assemble()
        S.solve_fixed(40, omega=cfg.omega)
        t = min(S.solve_fixed(400, omega=cfg.omega).solve_ms for _ in range(3)) * 1e3 / 400
        out.append(f"{mode} {t:.1f} us/iter (persistent {S.tile_config()['persistent']})")
        S.close()
    print(f"n_y={ny}: " + "; ".join(out), flush=True)
