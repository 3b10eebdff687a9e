"""Chrome trace + stage times of one product of a config built on the GPU.
usage: H2G_TRACE=out.json python tools/trace_config.py c4 [n]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device
cfg = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
import torch as _t
os.environ.setdefault("H2G_POOL_RESERVE_GB", f"{0.7 * _t.cuda.get_device_properties(0).total_memory / 1e9:.0f}")
ctx = Context(0)
dxr, dyr, spec = build_config_device(cfg, n=n, ctx=ctx)
dx = P.recompress(dxr, spec["eps"], ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, spec["eps"], ctx=ctx)
eps = spec["eps"]
for _ in range(int(os.environ.get("WARMUP", "3"))):  # steady state (host allocations, pools)
    z = P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
ctx.synchronize()
ctx.set_timing(True)
g = P.multiply(dx, dy, eps, ctx=ctx)
s1 = ctx.stage_times()
z = P.coarsen(g, dx.block_tree, eps, ctx=ctx)
ctx.synchronize()
s2 = ctx.stage_times()
print({k: round(s1[k] * 1e3, 1) for k in ("t_setup", "t1_row", "t1_mat")}, {k: round(s2[k] * 1e3, 1) for k in ("t2_row", "t2_mat")})
print("host ms", {k: round(v, 1) for k, v in ctx.host_times().items()})
if os.environ.get("H2G_TRACE"):
    ctx.trace_begin()
    g = P.multiply(dx, dy, eps, ctx=ctx)
    z = P.coarsen(g, dx.block_tree, eps, ctx=ctx)
    ctx.trace_dump(os.environ["H2G_TRACE"])
