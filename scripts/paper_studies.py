#!/usr/bin/env python
"""B200 analogues of the paper's comparisons (context studies, not the bench line):

  table3: synchronized (coupled / lockstep) vs asynchronous strategy, textured 2000x1600-like
          (C3 2048x1024 short, K=9, omega 1.6)                       -- Table 3
  table4: GMAF (one joint K=9 solve) vs SGA (nine K=1 solves in sequence), smooth and short,
          400x360 and 800x760, tol 1e-6                               -- Tables 4-6
  assor_vs_jacobi: iterations and time of ASSOR-II vs Jacobi (the "36%", Table 2)
  omega: ASSOR-II iterations vs omega = 0.18 i + 0.1 (Fig. 2b)
  fig2a: none / Jacobi / ASSOR-I / ASSOR-II at 2000x1600 smooth, rtol 1e-12, omega 1.8 (Fig. 2a,
         P:277-281: 6352 / 6519 / 3738 iterations for Jacobi / ASSOR-I / ASSOR-II)
Writes one JSON document to stdout.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gmaf_inputs as gi  # noqa: E402
import paper_2511_06824_b200 as P  # noqa: E402


def timed_step(S, conds, reps=2, **kw):
    S.step(conds, **kw)                                # warm-up (graph build)
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        st, W = S.step(conds, **kw)
        dt = time.perf_counter() - t0
        best = dt if best is None or dt < best else best
    return st, best


def table3():
    cfg = gi.config("C3")
    S = P.JointSolver(cfg.grid, 9)
    out = {}
    for coupling in ("coupled", "lockstep", "async"):
        for pc in ("assor2", "jacobi"):
            st, dt = timed_step(S, cfg.conds, reps=1, tol=1e-6, omega=cfg.omega, precond=pc, coupling=coupling)
            its = S.cond_iterations().tolist()
            out[f"{coupling}/{pc}"] = dict(iterations=st.iterations, per_condition=its,
                                           total_block_iterations=int(sum(its)), seconds=dt,
                                           ms_per_iteration=1e3 * dt / max(st.iterations, 1))
    S.close()
    return out


def table4():
    out = {}
    for tex in ("smooth", "short"):
        for nt, ny in ((400, 360), (800, 760)):
            case = gi.table_case(nt, ny, tex, K=9)
            S = P.JointSolver(case.grid, 9)
            res = {}
            for pc in ("assor2", "jacobi"):
                st, dt = timed_step(S, case.conds, tol=case.tol, omega=case.omega, precond=pc)
                res[f"gmaf/{pc}"] = dict(iterations=st.iterations, seconds=dt)
            S.close()
            S1 = P.JointSolver(case.grid, 1)
            for pc in ("assor2", "jacobi"):
                tot, its = 0.0, []
                for k in range(9):
                    st, dt = timed_step(S1, case.conds[k][None], reps=1, tol=case.tol, omega=case.omega, precond=pc)
                    tot += dt
                    its.append(st.iterations)
                res[f"sga/{pc}"] = dict(iterations_mean=float(np.mean(its)), seconds=tot)
                res[f"speedup/{pc}"] = tot / res[f"gmaf/{pc}"]["seconds"]
            S1.close()
            out[f"{tex}{nt}x{ny}"] = res
    return out


def omega_sweep():
    case = gi.table_case(800, 760, "smooth", K=1)
    S = P.JointSolver(case.grid, 1)
    out = {}
    for i in range(1, 11):
        w = 0.18 * i + 0.1
        st, dt = timed_step(S, case.conds, reps=1, tol=1e-6, omega=w)
        out[f"{w:.2f}"] = st.iterations
    S.close()
    return out


def fig2a():
    case = gi.table_case(2000, 1600, "smooth", K=1)
    S = P.JointSolver(case.grid, 1)
    out = {}
    for pc in ("none", "jacobi", "assor1", "assor2"):
        st, dt = timed_step(S, case.conds, reps=1, tol=1e-12, omega=1.8, precond=pc)
        out[pc] = dict(iterations=st.iterations, seconds=dt, ms_per_iteration=1e3 * dt / max(st.iterations, 1))
    out["paper"] = dict(jacobi=6352, ssor=6352, assor1=6519, assor2=3738,
                        seconds=dict(ssor=1680.10, assor1=215.21, assor2=226.57, jacobi=246.41))
    S.close()
    return out


def main():
    if len(sys.argv) > 1:   # one study by name
        print(json.dumps({sys.argv[1]: globals()[sys.argv[1]]()}, indent=1))
        return
    doc = {"device": torch.cuda.get_device_name(0), "table3": table3(), "table4": table4(),
           "omega_sweep_800x760_smooth_tol1e-6": omega_sweep(), "fig2a": fig2a()}
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
