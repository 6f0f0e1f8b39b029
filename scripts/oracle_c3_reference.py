"""Write tests/golden/c3_oracle_samples.json (or c4_... with the argument C4): the ORACLE's full
solve of BASELINE config C3 (short-textured 2048x1024, K = 9) or C4 (short-textured 1024x512,
the 9 conditions of the first Picard iterate of the trajectory), omega 1.6, rtol 1e-10, ASSOR-II,
coupled synchronized convergence -- Table 1; Eqs. 3.5-3.6, 3.7, 3.9 -- and its
quadrature (Sec. 2.4-III).

Calls oracle/ only (plain C FP64, Table-1 schedule, one host core; ~40 min).  The stored values
are what test_gpu_parity.py::test_c3_converged_vs_full_oracle_solve compares the GPU's
bench-configuration solve against: p at 4096 seeded nodes, the per-condition L2 norms of p, the
9 wrenches and the iteration count.  The sample positions are drawn from a seeded generator
(not method arithmetic).

    python scripts/oracle_c3_reference.py [C3|C4]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gmaf_inputs as gi  # noqa: E402
import oracle  # noqa: E402

TOL, OMEGA, N_SAMPLES, SEED = 1e-10, 1.6, 4096, 20251106


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    cfg = gi.config(name)
    t0 = time.time()
    AP, AE, AN, S = oracle.assemble_joint(cfg.grid, cfg.conds)
    t1 = time.time()
    res = oracle.pcg_joint(AP, AE, AN, S, tol=TOL, omega=OMEGA)
    t2 = time.time()
    K, ny, nt = res.p.shape
    rng = np.random.default_rng(SEED)
    ks = rng.integers(0, K, N_SAMPLES)
    js = rng.integers(0, ny, N_SAMPLES)
    is_ = rng.integers(0, nt, N_SAMPLES)
    samples = [[int(k), int(j), int(i), float(res.p[k, j, i])] for k, j, i in zip(ks, js, is_)]
    W = [oracle.wrench(cfg.grid, cfg.conds[k], res.p[k]).tolist() for k in range(K)]
    out = {
        "source": "scripts/oracle_c3_reference.py (oracle/ only: orc_assemble, orc_pcg_joint Table-1 "
                  "schedule, orc_wrench)",
        "config": f"{name}: {cfg.note} (Eqs. 2.17-2.19), ASSOR-II, coupled",
        "tol": TOL, "omega": OMEGA,
        "iterations": int(res.iterations), "converged": bool(res.converged),
        "rel_residual": float(res.rel_residual), "true_rel_residual": float(res.true_rel_residual),
        "p_norm": [float(np.linalg.norm(res.p[k])) for k in range(K)],
        "wrench": W,
        "samples": samples,
        "oracle_seconds": {"assemble": t1 - t0, "solve": t2 - t1},
    }
    path = os.path.join(ROOT, "tests", "golden", f"{name.lower()}_oracle_samples.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"wrote {path}: {res.iterations} iterations, converged {res.converged}, "
          f"solve {t2 - t1:.0f} s")


if __name__ == "__main__":
    main()
