"""Kernel-class device ms (profile mode) of one product of a config built on the GPU:
python tools/class_times.py c4 [warmup]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = Context(0)
dxr, dyr, spec = build_config_device(cfg, ctx=ctx)
eps = spec["eps"]
dx = P.recompress(dxr, eps, ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, eps, ctx=ctx)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
ctx.synchronize()
ctx.set_profile(True)
ctx.kernel_stats(reset=True)
P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
ks = ctx.kernel_stats(reset=True)
print({k: round(v["ms"], 1) for k, v in ks.items() if v["ms"] > 0})
