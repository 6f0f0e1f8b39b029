import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import gmaf_inputs as gi, oracle
g = gi.grid(60, 25, "short", tex_n_theta=6, tex_n_y=2, tex_band_rows=8)
conds = gi.random_conditions(43, 2)
AP, AE, AN, SS = oracle.assemble_joint(g, conds)
for k in range(2):
    h, hd = oracle.thickness(g, conds[k])
    print("k", k, "h range um", h.min() * 1e6, h.max() * 1e6, "AP range", AP[k].min(), AP[k].max())
for sched in ("table1", "single"):
    for coup in ("coupled", "lockstep"):
        r = oracle.pcg_joint(AP, AE, AN, SS, tol=1e-10, omega=1.6, schedule=sched, coupling=coup, history=True)
        print(sched, coup, "iters", r.iterations, "status", r.status, "conv", r.converged,
              "min rel", float(np.min(r.history)), "last", float(r.history[-1]))
try:
    import paper_2511_06824_b200 as P
    S = P.JointSolver(g, 2)
    st, W = S.step(conds, tol=1e-10, omega=1.6)
    print("gpu", st)
except Exception as e:
    print("gpu error", e)
