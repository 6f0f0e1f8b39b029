"""Row-slab debugging: a sequence of fixed-budget solves on the same context, each compared with
the one-process context running the same sequence."""
import os, sys, socket
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch.multiprocessing as mp

CASE = tuple(eval(os.environ.get("CASE", "(3, 60, 25, 'short', 2, 43)")))
SEQ = [int(x) for x in os.environ.get("SEQ", "7,3,3,4,3,2,5,3,1,3").split(",")]

def grid(gi, nt, ny, tex):
    if tex == "short":
        return gi.grid(nt, ny, tex, tex_n_theta=max(2, nt // 10), tex_n_y=2, tex_band_rows=max(4, ny // 3))
    return gi.grid(nt, ny)

def run(S, K, rows):
    import paper_2511_06824_b200 as P
    import gmaf_inputs as gi
    c = gi.random_conditions(CASE[5], K)
    if os.environ.get("SAMEC"):
        c = np.repeat(c[:1], K, axis=0)
    if os.environ.get("DUP2"):           # the 2 conditions of K=2, repeated to K rows
        c2 = gi.random_conditions(CASE[5], 2)
        c = np.concatenate([c2] * (K // 2))
    S.thickness(c); S.assemble()
    out = []
    for j in SEQ:
        st = S.solve(tol=1e-30, omega=1.6, max_iter=j, raise_on_error=False,
                     coupling=os.environ.get("COUPLING", "coupled"), precond=os.environ.get("PRECOND", "assor2"))
        out.append((st.iterations, st.rel_residual, np.stack([S.get("r", k)[rows] for k in range(K)])))
    return out

def rank_fn(rank, world, port, res):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi, paper_2511_06824_b200 as P
    from paper_2511_06824_b200.dist import connect_p2p
    w, nt, ny, tex, K, seed = CASE
    shard = os.environ.get("SHARD", "rows")
    S = P.JointSolver(grid(gi, nt, ny, tex), K, device=0, rank=rank, world=world, shard=shard, p2p=True)
    connect_p2p(S)
    y0, y1 = S.slab
    if shard == "conditions":   # every rank reports its own conditions' full fields: compare rank 0's block
        res[rank] = ((0, ny), run(S, K, slice(None)))
    else:
        res[rank] = ((y0, y1), run(S, K, slice(y0, y1)))
    S.close(); dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    import gmaf_inputs as gi, paper_2511_06824_b200 as P
    w, nt, ny, tex, K, seed = CASE
    S = P.JointSolver(grid(gi, nt, ny, tex), K)
    ref = run(S, K, slice(None))
    S.close()
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    res = mp.Manager().dict()
    mp.spawn(rank_fn, args=(w, port, res), nprocs=w, join=True)
    for q, j in enumerate(SEQ):
        errs = []
        for r in range(w):
            (y0, y1), out = res[r]
            p = out[q][2]; pr = ref[q][2][:, y0:y1]
            errs.append(np.linalg.norm(p - pr) / np.linalg.norm(pr))
        (y0, y1), out = res[min(1, w - 1)]
        p = out[q][2]; pr = ref[q][2][:, y0:y1]
        rowe = [float(np.abs(p[:, i] - pr[:, i]).max() / np.abs(pr).max()) for i in range(y1 - y0)]
        cole = [float(np.abs(p[:, :, c] - pr[:, :, c]).max() / np.abs(pr).max()) for c in range(p.shape[2])]
        for r in range(w):
            (y0, y1), out = res[r]
            p = out[q][2]; pr = ref[q][2][:, y0:y1]
            print("  rank", r, "r row err", ['%.0e' % (np.abs(p[:, i] - pr[:, i]).max() / np.abs(ref[q][2]).max()) for i in range(y1 - y0)],
                  "per k", ['%.0e' % (np.abs(p[k] - pr[k]).max() / np.abs(ref[q][2]).max()) for k in range(p.shape[0])])
        print(f"solve {q} max_iter {j}: iters {res[0][1][q][0]} rel {res[0][1][q][1]:.4e} ref {ref[q][1]:.4e} p err per rank {['%.1e' % e for e in errs]}")
