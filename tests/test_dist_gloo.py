"""Multi-process host logic on CPU (gloo, world_size 2): sharding, max-over-ranks timing
aggregation, and that sharded independent joint analyses reproduce the unsharded ones
(computed here with the oracle, which tests may use)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2511_06824_b200.dist import aggregate, operating_point_of, shard_range


def test_shard_range_tiles_exactly():
    for n in (0, 1, 7, 9, 72):
        for w in (1, 2, 3, 8):
            blocks = [shard_range(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(72, 8, 3) == (27, 36)      # C5: 9 conditions per GPU
    with pytest.raises(ValueError):
        shard_range(9, 2, 2)


def test_aggregate_single_process():
    a = aggregate(10.0, 12.0, 5e9)
    assert a.device_ms_max == 10.0 and a.dof_iters_total == 5e9
    assert abs(a.rate() - 5e11) < 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi
    import oracle
    # each rank: its own operating point, a small K=9 joint analysis through the oracle
    g = gi.grid(32, 16)
    conds = gi.fd_conditions(gi.condition(phi_deg=operating_point_of(rank)))
    res, W = oracle.joint_step(g, conds, tol=1e-10, omega=1.8)
    agg = aggregate(10.0 + rank, 20.0 + rank, float(9 * 32 * 16 * res.iterations))
    out[rank] = (res.iterations, W.tolist(), agg.device_ms_max, agg.wall_ms_max, agg.dof_iters_total,
                 [r[2] for r in agg.per_rank])
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_independent_points():
    import gmaf_inputs as gi
    import oracle
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    iters = []
    for rank in range(world):
        it, W, dmax, wmax, tot, per = out[rank]
        assert dmax == 11.0 and wmax == 21.0                 # max over ranks
        assert tot == sum(per)                               # sum of the ranks' work
        # the sharded result equals the same operating point analysed alone
        g = gi.grid(32, 16)
        conds = gi.fd_conditions(gi.condition(phi_deg=operating_point_of(rank)))
        ref, Wref = oracle.joint_step(g, conds, tol=1e-10, omega=1.8)
        assert it == ref.iterations and np.array_equal(np.array(W), Wref)
        iters.append(it)
    assert out[0][4] == out[1][4]                            # every rank sees the same total


def _slab_worker(rank, world, port, out):
    """One rank of a row-slab split (include/gmaf.h gmaf_slab_rows): it holds the stored rows
    [yb, ye) of r and of the previous search direction -- own rows + the 4 halo rows the device
    exchange delivers -- and evaluates one single-pass iteration's chain (z = M^-1 r, pd, s = A pd,
    r' = r - alpha s, z' = M^-1 r', A z') with the oracle's primitives on that data alone; the
    per-rank sums over OWN rows are all-reduced over gloo."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi
    import oracle
    import paper_2511_06824_b200 as P
    g = gi.grid(48, 40, "short", tex_n_theta=6, tex_n_y=2, tex_band_rows=10)
    cond = gi.random_conditions(3, 1)[0]
    AP, AE, AN, S = oracle.assemble(g, cond)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(S.shape) * 1e-9
    pd_old = rng.standard_normal(S.shape) * 1e5
    alpha, beta, omega = 0.37, 0.61, 1.6
    y0, y1, yb, ye = P.gmaf_slab_rows(g["n_y"], world, rank)
    res = {}
    for halo in (4, 3):                       # the library's depth, and one row less
        lo, hi = max(y0 - halo, 0), min(y1 + halo, g["n_y"])
        if halo == 4:
            assert (lo, hi) == (yb, ye)
        m = np.zeros_like(S)
        m[lo:hi] = 1.0
        rl, pl = r * m, pd_old * m             # rows outside the stored ones are never seen
        z = oracle.precond_apply(AP, AE, AN, rl, "assor2", omega)
        pd = z + beta * pl
        r1 = rl - alpha * oracle.spmv(AP, AE, AN, pd)
        z1 = oracle.precond_apply(AP, AE, AN, r1, "assor2", omega)
        w1 = oracle.spmv(AP, AE, AN, z1)
        own = slice(y0, y1)
        t = torch.tensor([np.sum(r1[own] * z1[own]), np.sum(z1[own] * w1[own]), np.sum(r1[own] ** 2)],
                         dtype=torch.float64)
        dist.all_reduce(t)
        res[halo] = t.tolist()
    out[rank] = ((y0, y1, yb, ye), res)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_row_slab_halo_depth():
    """Row-slab partition of the library (gmaf_slab_rows) on two gloo ranks: slabs tile the rows,
    and 4 halo rows (SLAB_HALO) are exactly what one single-pass iteration needs -- with them the
    all-reduced gamma = r'.z', delta = z'.A z' and r'.r' equal the unsplit computation (to the
    summation order); with 3 they do not (delta reaches 4 rows across the slab edge)."""
    import gmaf_inputs as gi
    import oracle
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_slab_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    (a0, a1, b0, b1), _ = out[0]
    (c0, c1, d0, d1), _ = out[1]
    assert a0 == 0 and a1 == c0 and c1 == 40 and (b0, b1) == (0, a1 + 4) and (d0, d1) == (c0 - 4, 40)
    g = gi.grid(48, 40, "short", tex_n_theta=6, tex_n_y=2, tex_band_rows=10)
    cond = gi.random_conditions(3, 1)[0]
    AP, AE, AN, S = oracle.assemble(g, cond)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(S.shape) * 1e-9
    pd_old = rng.standard_normal(S.shape) * 1e5
    alpha, beta, omega = 0.37, 0.61, 1.6
    z = oracle.precond_apply(AP, AE, AN, r, "assor2", omega)
    r1 = r - alpha * oracle.spmv(AP, AE, AN, z + beta * pd_old)
    z1 = oracle.precond_apply(AP, AE, AN, r1, "assor2", omega)
    full = [np.sum(r1 * z1), np.sum(z1 * oracle.spmv(AP, AE, AN, z1)), np.sum(r1 ** 2)]
    for rank in range(world):
        res = out[rank][1]
        for q in range(3):
            assert abs(res[4][q] - full[q]) <= 1e-12 * abs(full[q]), (rank, q, res[4][q], full[q])
        assert abs(res[3][1] - full[1]) > 1e-9 * abs(full[1])    # one halo row less breaks delta
