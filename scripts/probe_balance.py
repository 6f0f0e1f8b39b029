"""Load balance of the persistent solve at C3 (GMAF_DIAG): per-CTA arrival times at the grid
barrier, grouped by condition k (coefficient set shared or private), strip and chunk."""
import os
import sys
os.environ["GMAF_DIAG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

cfg = gi.config(os.environ.get("CFG", "C3"))
S = P.JointSolver(cfg.grid, cfg.K, max_matrices=5 * (cfg.K // 9))
S.thickness(cfg.conds)
S.assemble()
S.solve_fixed(40, omega=cfg.omega)
S.solve_fixed(40, omega=cfg.omega)
t = S.tile_config()
A = S.cta_arrivals().astype(np.float64)
S.close()
K = cfg.K
lat = (A - A.max(axis=1, keepdims=True)) / 1e3          # us before the last arrival (<= 0)
lat = lat[4:]                                           # skip the first iterations
b = np.arange(t["n_ctas"])
k, tile = b % K, b // K
strip, chunk = tile % t["n_strips"], tile // t["n_strips"]
print("tiles", t, "iterations", lat.shape[0])
print("mean wait per CTA (us): %.2f  (max %.2f)" % (-lat.mean(), -lat.min()))
for name, key, n in (("k", k, K), ("strip", strip, t["n_strips"]), ("chunk", chunk, t["n_chunks"])):
    print(name, [round(float(-lat[:, key == v].mean()), 2) for v in range(n)])
last = np.argmax(A[4:], axis=1)
print("last CTA k:", np.bincount(last % K, minlength=K).tolist(), "strip:",
      np.bincount((last // K) % t["n_strips"], minlength=t["n_strips"]).tolist(), "chunk:",
      np.bincount((last // K) // t["n_strips"], minlength=t["n_chunks"]).tolist())
