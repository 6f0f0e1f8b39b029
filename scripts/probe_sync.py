"""Per-iteration sync kernels at one rank (ncu launch list in stream mode): C3, 12 fixed
iterations through the condition-sharded peer-to-peer path and the row-slab path."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gmaf_inputs as gi
import paper_2511_06824_b200 as P

mode = sys.argv[1]
cfg = gi.config("C3")
if mode == "rows":
    S = P.JointSolver(cfg.grid, 9, shard="rows", world=1)
else:
    S = P.JointSolver(cfg.grid, 9, p2p=True, world=1)
S.p2p_connect([S.p2p_handle()])
S.thickness(cfg.conds)
S.assemble()
st = S.solve_fixed(12, omega=cfg.omega)
torch.cuda.synchronize()
print(mode, st.iterations, st.solve_ms)
