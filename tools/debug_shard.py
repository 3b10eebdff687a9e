"""Partitioned product on P gloo ranks sharing one GPU: per case, the rank, success and memory."""
import os, sys, socket
import numpy as np
import torch.multiprocessing as mp
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

def worker(rank, world, port, names):
    import torch, torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if rank == 0 and os.environ.get("MEM0"):
        os.environ["H2G_DEBUG_MEM"] = "1"  # engine memory marks of rank 0 only
    sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2309_09061_b200 as P
    from paper_2309_09061_b200.device import Context, DeviceH2
    from paper_2309_09061_b200.shard import Sharding
    from helpers import load, rebuild_raw, rel
    ctx = Context(0); sh = Sharding(ctx)
    for name in names:
        d = load(name); eps = float(d["eps"][0])
        xr, yr = rebuild_raw(d)
        dx = P.recompress(DeviceH2.upload(xr, ctx), eps, ctx=ctx)
        dy = dx if yr is xr else P.recompress(DeviceH2.upload(yr, ctx), eps, ctx=ctx)
        ctx.synchronize(); print(rank, name, "inputs", ctx.memory(reset=True), flush=True)
        g = P.multiply(dx, dy, eps, ctx=ctx); ctx.synchronize(); print(rank, name, "multiply", flush=True)
        z = P.coarsen(g, dx.block_tree, eps, ctx=ctx); ctx.synchronize(); print(rank, name, "coarsen", ctx.memory(), flush=True)
        zr, zc = z.ranks()
        ok = list(zr) == list(d["rank.final_row"])
        print(rank, name, "final ranks equal", ok, flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    names = sys.argv[1:]
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(worker, args=(2, port, names), nprocs=2)
