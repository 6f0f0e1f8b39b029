import os, sys, socket
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch.multiprocessing as mp

CASE = (3, 60, 25, "short", 2, 43)

def grid(gi, nt, ny, tex):
    if tex == "short":
        return gi.grid(nt, ny, tex, tex_n_theta=max(2, nt // 10), tex_n_y=2, tex_band_rows=max(4, ny // 3))
    return gi.grid(nt, ny)

def run(S, K, rows, out):
    import gmaf_inputs as gi
    S.thickness(gi.random_conditions(CASE[5], K)); S.assemble()
    S.solve(tol=1e-30, omega=1.6, max_iter=7, raise_on_error=False)   # as in the test: 7 first
    for j in (0, 1, 2, 3):
        st = S.solve(tol=1e-30, omega=1.6, max_iter=j, raise_on_error=False)
        out[j] = (st.status, st.rel_residual, np.stack([S.get("p", k)[rows] for k in range(K)]),
                  np.stack([S.get("r", k)[rows] for k in range(K)]))

def rank_fn(rank, world, port, res):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi, paper_2511_06824_b200 as P
    from paper_2511_06824_b200.dist import connect_p2p
    w, nt, ny, tex, K, seed = CASE
    S = P.JointSolver(grid(gi, nt, ny, tex), K, device=0, rank=rank, world=world, shard="rows")
    connect_p2p(S)
    y0, y1 = S.slab
    out = {}
    run(S, K, slice(y0, y1), out)
    res[rank] = ((y0, y1), out)
    S.close(); dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    import gmaf_inputs as gi, paper_2511_06824_b200 as P
    w, nt, ny, tex, K, seed = CASE
    S = P.JointSolver(grid(gi, nt, ny, tex), K)
    ref = {}
    run(S, K, slice(None), ref)
    S.close()
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    res = mp.Manager().dict()
    mp.spawn(rank_fn, args=(w, port, res), nprocs=w, join=True)
    for r in range(w):
        (y0, y1), out = res[r]
        for j in (0, 1, 2, 3):
            st, rel, p, rr = out[j]
            pe = np.linalg.norm(p - ref[j][2][:, y0:y1]) / max(np.linalg.norm(ref[j][2][:, y0:y1]), 1e-300)
            re = np.linalg.norm(rr - ref[j][3][:, y0:y1]) / max(np.linalg.norm(ref[j][3][:, y0:y1]), 1e-300)
            rowerr = [float(np.abs(rr[:, i] - ref[j][3][:, y0 + i]).max()) for i in range(y1 - y0)]
            print(f"rank {r} slab {y0}-{y1} iter {j}: status {st} rel {rel:.3e} (ref {ref[j][1]:.3e}) p err {pe:.2e} r err {re:.2e} rowmax {['%.1e' % x for x in rowerr]}")
