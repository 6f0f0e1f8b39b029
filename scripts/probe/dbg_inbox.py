"""Row-slab debugging: after fixed-budget solves, compare rank 1's inbox (rows received from rank 0)
with rank 0's own field rows (latest residual)."""
import os, sys, socket, ctypes as C
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch.multiprocessing as mp

K = int(os.environ.get("KK", "2")); NT, NY = 60, 16

def rank_fn(rank, world, port, res):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi, paper_2511_06824_b200 as P
    from paper_2511_06824_b200.dist import connect_p2p
    S = P.JointSolver(gi.grid(NT, NY), K, device=0, rank=rank, world=world, shard="rows")
    connect_p2p(S)
    y0, y1 = S.slab
    S.thickness(gi.random_conditions(43, K)); S.assemble()
    L = P.lib()
    L.gmaf_debug_inbox.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_ulonglong)]
    out = []
    for j in (1, 2, 3):
        S.solve(tol=1e-30, omega=1.6, max_iter=j, raise_on_error=False)
        nb = 8 * 4 * K * NT
        ns_rows = min(y1 + 4, NY) - max(y0 - 4, 0)
        nf = K * ns_rows * NT
        box = np.zeros(nb + 2 * nf); seq = C.c_ulonglong()
        L.gmaf_debug_inbox(S.ctx, box.ctypes.data_as(C.POINTER(C.c_double)), C.byref(seq))
        r = np.stack([S.get("r", k) for k in range(K)])
        u = box[nb:].reshape(2, K, ns_rows, NT)
        out.append((seq.value, box[:nb].reshape(2, 2, 2, K, 4, NT), r, u, max(y0 - 4, 0)))
    res[rank] = ((y0, y1), out)
    S.close(); dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    res = mp.Manager().dict()
    mp.spawn(rank_fn, args=(2, port, res), nprocs=2, join=True)
    (a0, a1), o0 = res[0]; (b0, b1), o1 = res[1]
    for q, j in enumerate((1, 2, 3)):
        seq1, box1, r1, u1, yb1 = o1[q]; seq0, box0, r0, u0, yb0 = o0[q]
        for par in (0, 1):
            for slot in (0, 1):
                got = box1[slot, 0, 1]                                   # pd rows a1-4..a1-1 from rank 0
                want = u0[par][:, a1 - 4 - yb0:a1 - yb0, :]
                e = [float(np.abs(got[k] - want[k]).max() / max(np.abs(want[k]).max(), 1e-300)) for k in range(K)]
                print(f"   iters {j} pd u[{par}] vs slot {slot} up err {['%.1e' % x for x in e]}")
        # after the solve: the last iteration's push landed in slot (seq - 2) & 1 (then p and the
        # true-residual gathers followed): compare vec 0 (r) side 0 of rank 1 with rank 0's rows
        for slot in (0, 1):
            got = box1[slot, 0, 0]                       # [K][4][NT] rows a1-4 .. a1-1 of r
            want = r0[:, a1 - 4:a1, :]
            err = [float(np.abs(got[k] - want[k]).max() / max(np.abs(want[k]).max(), 1e-300)) for k in range(K)]
            got1 = box0[slot, 1, 0]; want1 = r1[:, b0:b0 + 4, :]
            err1 = [float(np.abs(got1[k] - want1[k]).max() / max(np.abs(want1[k]).max(), 1e-300)) for k in range(K)]
            print(f"iters {j} seq {seq0},{seq1} slot {slot}: up (rank0->1) err per k {['%.1e' % e for e in err]}  down (rank1->0) {['%.1e' % e for e in err1]}")
