"""stress: 2 processes, alternating fused / p2p / generic decomposed solves"""
import os, sys, socket, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def proc(rank, port, q, mode):
    import torch, torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    import paper_2111_09859_b200 as W
    from paper_2111_09859_b200 import dist
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    import test_gpu_dist as T
    comm = dist.TorchComm()
    g, cfg, phi0 = T._channel(n0=32, arith="fast", steps=4)
    g2, cfg2, p2 = T._cylinder("hj_curvature", "exact", 3)
    first = {}
    bad = []
    for it in range(6):
        for kind in mode.split(","):
            t0 = time.time()
            if kind == "p2p": os.environ["WD_DIST_P2P"] = "1"
            if kind == "generic":
                rep = W.solve_steady(g2, W.BoundarySpec(T.CYL), cfg2, phi0=p2, comm=comm)
            else:
                rep = W.solve_steady(g, W.BoundarySpec(T.FACES), cfg, phi0=phi0, comm=comm)
            os.environ.pop("WD_DIST_P2P", None)
            h = rep.residual_history
            if kind not in first: first[kind] = h
            elif not np.array_equal(first[kind], h): bad.append((it, kind))
            if rank == 0: print(it, kind, round(time.time() - t0, 3), flush=True)
    q.put((rank, bad))
    tdist.destroy_process_group()

if __name__ == "__main__":
    import torch.multiprocessing as mp
    mode = sys.argv[1] if len(sys.argv) > 1 else "fused,p2p,generic"
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=proc, args=(r, port, q, mode)) for r in range(2)]
    [p.start() for p in ps]
    res = [q.get(timeout=150) for _ in ps]
    [p.join(60) for p in ps]
    print(mode, res)
