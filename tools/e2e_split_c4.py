"""Host timeline of the e2e call (multiply_coarsen_packed) at c4: upload X / Y (asynchronous
nearfield), multiply, coarsen (with Z's nearfield prefetch), download -- against the device-only product."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("H2G_POOL_RESERVE_GB", "120")
import ctypes as C
import numpy as np, torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200 import _native as N
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config_device
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
ctx = Context(0)
dxr, dyr, spec = build_config_device(cfg, ctx=ctx)
eps = spec["eps"]
dx = P.recompress(dxr, eps, ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, eps, ctx=ctx)
del dxr, dyr
def pinned(d):
    out = {}
    for k, v in d.items():
        if k.startswith(("rows.", "cols.", "bt.")):
            continue
        t = torch.empty(len(v), dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True)
        a = t.numpy(); a[:] = v; out[k] = a
    return out
xp, yp = pinned(dx.download_packed()), pinned(dy.download_packed())
btx, bty = dx.block_tree, dy.block_tree
print({k: round(v.nbytes / 1e9, 3) for k, v in xp.items() if v.nbytes > 1e7})
z = P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), btx, eps, ctx=ctx)
zs = z.packed_shapes()
zout = {k: torch.empty(n, dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True).numpy() for k, n in zs.items()}
del z
for it in range(5):
    ctx.synchronize()
    T = {}; t0 = time.perf_counter()
    a = DeviceH2.upload_packed(xp, btx, ctx, asynchronous=True); T["upload_x"] = time.perf_counter() - t0
    b = DeviceH2.upload_packed(yp, bty, ctx, asynchronous=True); T["upload_y"] = time.perf_counter() - t0
    g = P.multiply(a, b, eps, ctx=ctx); T["multiply"] = time.perf_counter() - t0
    nh = zout["near_data"]; h = N.P()
    N.check(ctx.lib.h2g_coarsen_prefetch(ctx.h, g.h, ctx.blocks(btx), float(eps), -1, 1, nh.ctypes.data_as(N.F64P), nh.size, C.byref(h)))
    T["coarsen"] = time.perf_counter() - t0
    zz = DeviceH2(ctx, h, btx, btx.rows, btx.cols)
    del g
    zz.download_packed(zout); T["download"] = time.perf_counter() - t0
    del zz, a, b
    print({k: round(1e3 * v, 1) for k, v in T.items()}, flush=True)
ctx.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(ctx.stream)
for _ in range(3):
    zz = P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), btx, eps, ctx=ctx)
ev1.record(ctx.stream); torch.cuda.synchronize()
print("device-only ms", ev0.elapsed_time(ev1) / 3)
