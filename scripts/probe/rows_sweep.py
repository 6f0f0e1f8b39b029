"""Random sweep of the row-slab path: world 2..4 processes on one GPU, random mesh / K / texture,
7 fixed iterations compared with the one-process context (<= 1e-12 relative)."""
import os, sys, socket
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch.multiprocessing as mp

def cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        w = int(rng.integers(2, 5)); nt = int(rng.integers(6, 100)) * 2; ny = int(rng.integers(8 * w, 8 * w + 60))
        K = int(rng.integers(1, 10)); tex = "short" if rng.random() < 0.5 else "smooth"
        if nt < 12:
            continue
        out.append((w, nt, ny, tex, K, int(rng.integers(0, 1000))))
    return out

def grid(gi, nt, ny, tex):
    if tex == "short":
        return gi.grid(nt, ny, tex, tex_n_theta=max(2, nt // 10), tex_n_y=2, tex_band_rows=max(4, ny // 3))
    return gi.grid(nt, ny)

def run(S, K, rows, seed):
    import gmaf_inputs as gi
    S.thickness(gi.random_conditions(seed, K)); S.assemble()
    S.solve(tol=1e-30, omega=1.6, max_iter=7, raise_on_error=False)
    return np.stack([S.get("p", k)[rows] for k in range(K)])

def rank_fn(rank, world, port, case, res):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi, paper_2511_06824_b200 as P
    from paper_2511_06824_b200.dist import connect_p2p
    w, nt, ny, tex, K, seed = case
    S = P.JointSolver(grid(gi, nt, ny, tex), K, device=0, rank=rank, world=world, shard="rows")
    connect_p2p(S)
    y0, y1 = S.slab
    res[rank] = ((y0, y1), run(S, K, slice(y0, y1), seed))
    S.close(); dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    import gmaf_inputs as gi, paper_2511_06824_b200 as P
    bad = 0
    for case in cases(int(os.environ.get("N", "16")), int(os.environ.get("SEED", "5"))):
        w, nt, ny, tex, K, seed = case
        S = P.JointSolver(grid(gi, nt, ny, tex), K)
        ref = run(S, K, slice(None), seed); S.close()
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        res = mp.Manager().dict()
        mp.spawn(rank_fn, args=(w, port, case, res), nprocs=w, join=True)
        errs = []
        for r in range(w):
            (y0, y1), p = res[r]
            errs.append(float(np.linalg.norm(p - ref[:, y0:y1]) / np.linalg.norm(ref[:, y0:y1])))
        ok = max(errs) <= 1e-12
        bad += not ok
        print("OK " if ok else "BAD", case, ["%.1e" % e for e in errs], flush=True)
    print("bad cases:", bad)
