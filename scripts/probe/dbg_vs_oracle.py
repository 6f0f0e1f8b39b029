import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, gmaf_inputs as gi, oracle
import paper_2511_06824_b200 as P
for K in (2, 3):
    g = gi.grid(60, 25)
    conds = gi.random_conditions(43, K)
    AP, AE, AN, SS = oracle.assemble_joint(g, conds)
    S = P.JointSolver(g, K)
    S.thickness(conds); S.assemble()
    for j in (3, 4, 5):
        st = S.solve(tol=1e-30, omega=1.6, max_iter=j, raise_on_error=False)
        ref = oracle.pcg_joint(AP, AE, AN, SS, tol=1e-30, omega=1.6, max_iter=j, schedule="single")
        pg = np.stack([S.get("p", k) for k in range(K)])
        print("K", K, "iters", j, "gpu rel %.6e oracle rel %.6e" % (st.rel_residual, ref.rel_residual),
              "p err %.2e" % (np.linalg.norm(pg - ref.p) / np.linalg.norm(ref.p)))
    S.close()
