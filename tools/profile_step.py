"""One product step on a BASELINE config for profiling (ncu / nsight): build, recompress, 1 warm-up, 1 step."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = (int(sys.argv[2]) or None) if len(sys.argv) > 2 else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
xr, yr, spec = build_config(cfg, n=n)
ctx = Context(0)
dx = P.recompress(DeviceH2.upload(xr, ctx), spec["eps"], ctx=ctx)
dy = dx if yr is xr else P.recompress(DeviceH2.upload(yr, ctx), spec["eps"], ctx=ctx)
for i in range(1 + steps):
    ctx.set_timing(i == steps)
    t0 = time.perf_counter()
    g = P.multiply(dx, dy, spec["eps"], ctx=ctx)
    s1 = ctx.stage_times()
    z = P.coarsen(g, dx.block_tree, spec["eps"], ctx=ctx)
    ctx.synchronize()
    t = time.perf_counter() - t0
s2 = ctx.stage_times()
print(f"step {t*1e3:.1f} ms", {k: round(s1[k] * 1e3, 2) for k in ("t_setup", "t1_row", "t1_col", "t1_mat")},
      {k: round(s2[k] * 1e3, 2) for k in ("t2_row", "t2_col", "t2_mat")})
print("host ms", {k: round(v, 1) for k, v in ctx.host_times().items()})
if os.environ.get("H2G_TRACE"):
    ctx.trace_begin()
    g = P.multiply(dx, dy, spec["eps"], ctx=ctx)
    z = P.coarsen(g, dx.block_tree, spec["eps"], ctx=ctx)
    ctx.trace_dump(os.environ["H2G_TRACE"])
