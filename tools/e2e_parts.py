"""Time the parts of the packed host-buffer product: upload (sync / async), product, download."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config
xr, yr, spec = build_config("c2")
ctx = Context(0)
eps = spec["eps"]
dx = P.recompress(DeviceH2.upload(xr, ctx), eps, ctx=ctx)
pk = dx.download_packed()
xp = {}
for k, v in pk.items():
    t = torch.empty(len(v), dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True)
    a = t.numpy(); a[:] = v; xp[k] = a
bt = dx.block_tree
print("bytes", {k: v.nbytes // 1000000 for k, v in xp.items() if v.nbytes > 1e6})
z = P.coarsen(P.multiply(dx, dx, eps, ctx=ctx), bt, eps, ctx=ctx)
zs = z.packed_shapes()
zout = {k: torch.empty(n, dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True).numpy() for k, n in zs.items()}
for it in range(4):
    T = {}
    t0 = time.perf_counter(); d1 = DeviceH2.upload_packed(xp, bt, ctx); ctx.synchronize(); T["upload_sync"] = time.perf_counter() - t0
    t0 = time.perf_counter(); d2 = DeviceH2.upload_packed(xp, bt, ctx, asynchronous=True); T["upload_async_return"] = time.perf_counter() - t0
    ctx.synchronize(); T["upload_async_total"] = time.perf_counter() - t0
    t0 = time.perf_counter(); zz = P.coarsen(P.multiply(d1, d1, eps, ctx=ctx), bt, eps, ctx=ctx); ctx.synchronize(); T["product"] = time.perf_counter() - t0
    t0 = time.perf_counter(); zz.download_packed(zout); T["download"] = time.perf_counter() - t0
    t0 = time.perf_counter(); P.multiply_coarsen_packed(xp, bt, None, None, eps, coarse=bt, out=zout, ctx=ctx); T["e2e"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 2) for k, v in T.items()})
