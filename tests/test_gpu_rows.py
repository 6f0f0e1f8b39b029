"""Row-slab sharding (include/gmaf.h GMAF_SHARD_ROWS_P2P, gmaf_slab):
three ranks -- here three processes time-sharing ONE GPU, bootstrapped over gloo -- each owning a
contiguous block of the unknown rows of all 9 conditions, with the halo rows of r and of the
search direction pushed into the neighbours' inboxes over IPC-mapped peer memory after every
iteration.  The middle rank has both neighbours; the slabs span several row chunks each.

The per-condition sums are added per rank and then over the ranks, so the scalars differ from
the one-process solve in the last bits only: the j-th iterate must agree to 1e-12 (any halo error
is O(1)), the converged p with the oracle to 1e-8 (R-A23), the wrenches to 1e-9."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    import gmaf_inputs as gi
    g = gi.grid(128, 96, "short", tex_n_theta=8, tex_n_y=3, tex_band_rows=24)
    return g, gi.random_conditions(5, 9)


def _rank(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_06824_b200 as P
    from paper_2511_06824_b200.dist import connect_p2p
    g, conds = _case()
    S = P.JointSolver(g, 9, device=0, rank=rank, world=world, shard="rows")
    connect_p2p(S)
    y0, y1 = S.slab
    S.thickness(conds)
    S.assemble()
    fx = S.solve(tol=1e-30, omega=1.6, max_iter=7, raise_on_error=False)    # 7 iterates
    p7 = np.stack([S.get("p", k)[y0:y1] for k in range(9)])
    st = S.solve(tol=1e-10, omega=1.6)
    W = S.integrate()
    p = np.stack([S.get("p", k)[y0:y1] for k in range(9)])
    st2 = S.solve(tol=1e-10, omega=1.6, warm=True)          # warm start: halo of p0, residual
    out[rank] = (y0, y1, fx.iterations, p7, st.iterations, st.converged, st.rel_residual,
                 st.true_rel_residual, p, W, st2.iterations, st.cond_rel)
    S.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_row_slabs_three_ranks_match_the_joint_solve():
    import torch
    assert torch.cuda.is_available()
    from paper_2511_06824_b200 import build as B
    B.build()
    import oracle as orc
    import paper_2511_06824_b200 as P
    g, conds = _case()
    S = P.JointSolver(g, 9)
    S.thickness(conds)
    S.assemble()
    S.solve(tol=1e-30, omega=1.6, max_iter=7, raise_on_error=False)
    p7ref = np.stack([S.get("p", k) for k in range(9)])
    st = S.solve(tol=1e-10, omega=1.6)
    W = S.integrate()
    pref = np.stack([S.get("p", k) for k in range(9)])
    S.close()
    AP, AE, AN, SS = orc.assemble_joint(g, conds)
    ref = orc.pcg_joint(AP, AE, AN, SS, tol=1e-10, omega=1.6)

    out = mp.Manager().dict()
    mp.spawn(_rank, args=(WORLD, _port(), out), nprocs=WORLD, join=True)
    rows = []
    for r in range(WORLD):
        y0, y1, it7, p7, it, conv, rel, trel, p, Wr, it2, crel = out[r]
        rows.append((y0, y1))
        assert it7 == 7
        err7 = np.linalg.norm(p7 - p7ref[:, y0:y1]) / np.linalg.norm(p7ref[:, y0:y1])
        assert err7 <= 1e-12, (r, err7)
        assert conv and abs(it - st.iterations) <= 2, (r, it, st.iterations)
        assert rel <= 1e-10 and trel <= 1e-9
        assert np.linalg.norm(p - ref.p[:, y0:y1]) <= 1e-8 * np.linalg.norm(ref.p[:, y0:y1]), r
        assert np.linalg.norm(p - pref[:, y0:y1]) <= 1e-9 * np.linalg.norm(pref[:, y0:y1]), r
        for k in range(9):
            assert np.linalg.norm(Wr[k] - W[k]) <= 1e-9 * np.linalg.norm(W[k]), (r, k)
        assert np.array_equal(Wr, out[0][9])            # the same wrenches on every rank
        assert it2 == 0                                 # warm start from the converged p
        # per-condition ||r_k||/||S_k|| at exit: both runs stop at the same global test; the
        # recursive residuals at 1e-10 carry the rounding noise of the different summation order
        assert np.all(crel <= 1e-9) and np.allclose(crel, st.cond_rel, rtol=0.1), (crel, st.cond_rel)
    assert rows[0][0] == 0 and rows[-1][1] == g["n_y"]
    assert all(rows[r][1] == rows[r + 1][0] for r in range(WORLD - 1))
