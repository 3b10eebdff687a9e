"""Per-step device times of repeated products (variance check)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config
xr, yr, spec = build_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
ctx = Context(0)
eps = spec["eps"]
dx = P.recompress(DeviceH2.upload(xr, ctx), eps, ctx=ctx)
bt = dx.block_tree
ts = []
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    z = P.coarsen(P.multiply(dx, dx, eps, ctx=ctx), bt, eps, ctx=ctx)
    e1.record(ctx.stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(" ".join(f"{t:.1f}" for t in ts))
