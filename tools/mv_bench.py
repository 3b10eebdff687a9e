"""Time GPU matvecs of the c-config product Z (profile mode per launch)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
xr, yr, spec = build_config(cfg)
ctx = Context(0)
dx = P.recompress(DeviceH2.upload(xr, ctx), spec["eps"], ctx=ctx)
z = P.coarsen(P.multiply(dx, dx, spec["eps"], ctx=ctx), dx.block_tree, spec["eps"], ctx=ctx)
v = torch.randn(z.shape[1], dtype=torch.float64, device="cuda")
for _ in range(5):
    z.matvec(v)
torch.cuda.synchronize()
for _ in range(3):
    z.matvec(v)
torch.cuda.synchronize()
