import os, sys, socket
import numpy as np
sys.path.insert(0, ".")
import oracle

def worker(rank, world, port, n, k):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    import torch, torch.distributed as dist
    import paper_1204_3052_b200 as mx
    from paper_1204_3052_b200 import distributed as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    eng = mx.Engine(0)
    a_np = oracle.scaled_input(n, np.float32, 42)
    a = torch.from_numpy(a_np).cuda()
    got = D.exponentiate_row_sharded_fused(a, k, engine=eng).cpu().numpy()
    ref = eng.power(a_np, k)
    rows = n // world
    for r in range(world):
        blk = slice(r * rows, (r + 1) * rows)
        same = np.array_equal(got[blk], ref[blk])
        err = oracle.compare(got[blk], ref[blk])[2]
        print(f"rank {rank}: rows of rank {r}: bitwise {same} fro {err:.3e} zeros {np.mean(got[blk]==0):.3f}", flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ps = [mp.get_context("spawn").Process(target=worker, args=(r, 2, port, 1024, k)) for r in range(2)]
    [p.start() for p in ps]; [p.join(300) for p in ps]
