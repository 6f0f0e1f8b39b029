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
