"""Fixed-iteration throughput probe: C3 (or argv[1]) joint solve, N iterations, per-kernel times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

cfg = gi.config(sys.argv[1] if len(sys.argv) > 1 else "C3")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
K = cfg.conds.shape[0]
if os.environ.get("PROBE_P2P"):
    S = P.JointSolver(cfg.grid, K, world=1, p2p=True)
    S.p2p_connect([S.p2p_handle()])
else:
    S = P.JointSolver(cfg.grid, K)
S.thickness(cfg.conds); S.assemble()
try:
    S.solve_fixed(20, omega=cfg.omega)
except P.GmafError as e:
    print("warm-up:", e)
S.reset_kernel_times()
try:
    st = S.solve_fixed(n, omega=cfg.omega)
    print(f"{cfg.name}: {n} iterations in {st.solve_ms:.2f} ms")
except P.GmafError as e:
    print("timed:", e)
dof = cfg.grid["n_theta"] * cfg.grid["n_y"] * K
for kt in S.kernel_times():
    if kt["launches"]:
        us = 1000 * kt["total_ms"] / kt["launches"]
        print(f"  {kt['name']:16s} {kt['launches']:6d} launches {us:9.2f} us  ({dof / us / 1e3:.1f} G DOF/s per launch)")
