"""Matvec call timing in the bench's setting (reserved pool, after the error estimate)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("H2G_POOL_RESERVE_GB", "120")
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
ctx = Context(0)
dxr, dyr, spec = build_config_device(cfg, ctx=ctx)
dx = P.recompress(dxr, spec["eps"], ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, spec["eps"], ctx=ctx)
del dxr, dyr
z = P.coarsen(P.multiply(dx, dy, spec["eps"], ctx=ctx), dx.block_tree, spec["eps"], ctx=ctx)
v = torch.randn(z.shape[1], dtype=torch.float64, device="cuda")
def timed(tag):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter(); e0.record()
    for _ in range(10): z.matvec(v)
    e1.record(); h1 = time.perf_counter(); torch.cuda.synchronize()
    print(tag, "device ms/call", e0.elapsed_time(e1) / 10, "host ms/call", (h1 - h0) * 100, flush=True)
timed("fresh")
timed("again")
est = P.estimate_relative_spectral_error(dx, dy, z, steps=20, seed=0)
timed("after estimate")
