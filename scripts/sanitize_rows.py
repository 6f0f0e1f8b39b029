"""Row-slab sharding under compute-sanitizer: two ranks (processes on one GPU, gloo bootstrap),
a tiny textured case, cold + warm solve + quadrature, stream launch mode (set by the caller)."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _rank(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gmaf_inputs as gi
    import paper_2511_06824_b200 as P
    from paper_2511_06824_b200.dist import connect_p2p
    nt, ny, K, seed = (int(x) for x in os.environ.get("SAN_CASE", "96,40,3,5").split(","))
    g = gi.grid(nt, ny, "short", tex_n_theta=8, tex_n_y=2, tex_band_rows=8) if nt == 96 else gi.grid(nt, ny)
    S = P.JointSolver(g, K, device=0, rank=rank, world=world, shard="rows")
    connect_p2p(S)
    S.thickness(gi.random_conditions(seed, K))
    S.assemble()
    st = S.solve(tol=1e-8, omega=1.6, max_iter=3000, raise_on_error=False)
    W = S.integrate()
    st2 = S.solve(tol=1e-8, omega=1.6, warm=True, raise_on_error=False)
    print(f"rank {rank}: slab {S.slab} iterations {st.iterations} warm {st2.iterations}", flush=True)
    S.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    if len(sys.argv) > 2:        # one rank per top-level process: sanitize_rows.py RANK PORT
        _rank(int(sys.argv[1]), int(os.environ.get('SAN_WORLD', '2')), int(sys.argv[2]))
        print("sanitize rows run done", flush=True)
        sys.exit(0)
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_rank, args=(int(os.environ.get('SAN_WORLD', '2')), port), nprocs=int(os.environ.get('SAN_WORLD', '2')), join=True)
    print("sanitize rows run done")
