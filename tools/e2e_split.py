import os, sys, time
sys.path.insert(0, "/root/repo")
import ctypes as C
import numpy as np, torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200 import _native as N, api
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config
xr, yr, spec = build_config("c2")
ctx = Context(0); eps = spec["eps"]
dx = P.recompress(DeviceH2.upload(xr, ctx), eps, ctx=ctx)
pk = dx.download_packed(); bt = dx.block_tree
xp = {}
for k, v in pk.items():
    t = torch.empty(len(v), dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True)
    a = t.numpy(); a[:] = v; xp[k] = a
z = P.coarsen(P.multiply(dx, dx, eps, ctx=ctx), bt, eps, ctx=ctx)
zs = z.packed_shapes()
zout = {k: torch.empty(n, dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True).numpy() for k, n in zs.items()}
del z
for it in range(6):
    ctx.synchronize()
    T = {}; t0 = time.perf_counter()
    d = DeviceH2.upload_packed(xp, bt, ctx, asynchronous=True); T["upload"] = time.perf_counter() - t0
    g = P.multiply(d, d, eps, ctx=ctx); T["multiply"] = time.perf_counter() - t0
    nh = zout["near_data"]; h = N.P()
    N.check(ctx.lib.h2g_coarsen_prefetch(ctx.h, g.h, ctx.blocks(bt), float(eps), -1, 1, nh.ctypes.data_as(N.F64P), nh.size, C.byref(h)))
    T["coarsen"] = time.perf_counter() - t0
    zz = P.DeviceH2(ctx, h, bt, bt.rows, bt.cols)
    del g
    ctx.synchronize(); T["sync"] = time.perf_counter() - t0
    out = zz.download_packed(zout); T["download"] = time.perf_counter() - t0
    del zz, d
    T["free"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 1) for k, v in T.items()})
