"""Peer-to-peer condition sharding (include/gmaf.h gmaf_p2p_*): two ranks --
here two processes time-sharing ONE GPU, bootstrapped over gloo -- each owning a block of the 9
conditions, with the per-iteration gather fused into the iteration kernel over IPC-mapped peer
memory.  The sharded solve must reproduce the single-process joint solve bit for bit (same sums
in the same global condition order), including the gathered wrenches of all conditions."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi
    import paper_2511_06824_b200 as P
    from paper_2511_06824_b200.dist import connect_p2p, shard_range
    g = gi.grid(96, 40, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8)
    conds = gi.random_conditions(11, 9)
    S = P.JointSolver(g, 9, device=0, rank=rank, world=world, p2p=True)
    connect_p2p(S)
    st, W = S.step(conds, tol=1e-10, omega=1.6)
    lo, hi = shard_range(9, world, rank)
    p = np.stack([S.get("p", k) for k in range(lo, hi)])   # global condition indices
    st2 = S.solve(tol=1e-10, omega=1.6, warm=True)          # a second solve reuses the connection
    out[rank] = (st.iterations, st.converged, st.rel_residual, st.true_rel_residual, p, W, lo, hi,
                 st2.iterations, S.cond_rel.tolist() if hasattr(S, "cond_rel") else None)
    S.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_p2p_two_ranks_reproduce_the_joint_solve():
    import torch
    assert torch.cuda.is_available()
    from paper_2511_06824_b200 import build as B
    B.build()
    import gmaf_inputs as gi
    import paper_2511_06824_b200 as P
    g = gi.grid(96, 40, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8)
    conds = gi.random_conditions(11, 9)
    S = P.JointSolver(g, 9)
    st, W = S.step(conds, tol=1e-10, omega=1.6)
    pref = np.stack([S.get("p", k) for k in range(9)])
    S.close()
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(world, _port(), out), nprocs=world, join=True)
    for r in range(world):
        it, conv, rel, trel, p, Wr, lo, hi, it2, _ = out[r]
        assert conv and it == st.iterations, (r, it, st.iterations)
        assert rel == st.rel_residual and trel == st.true_rel_residual
        assert np.array_equal(p, pref[lo:hi])
        assert np.array_equal(Wr, W)                   # all 9 wrenches on every rank
        assert it2 == 0                                 # warm start from the converged p
