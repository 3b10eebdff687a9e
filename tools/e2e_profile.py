"""Break the end-to-end (host H2Matrix in -> host H2Matrix out) product into its host/device parts."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.packed import pack_h2, unpack_h2
from paper_2309_09061_b200.problems import build_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
xr, yr, spec = build_config(cfg)
ctx = Context(0)
dx = P.recompress(DeviceH2.upload(xr, ctx), spec["eps"], ctx=ctx)
xh = dx.download()
eps = spec["eps"]
for it in range(3):
    T = {}
    t = time.perf_counter()
    d = pack_h2(xh); T["pack"] = time.perf_counter() - t
    t = time.perf_counter()
    dxx = DeviceH2.upload(xh, ctx); ctx.synchronize(); T["upload(incl pack)"] = time.perf_counter() - t
    t = time.perf_counter()
    g = P.multiply(dxx, dxx, eps, ctx=ctx); z = P.coarsen(g, dxx.block_tree, eps, ctx=ctx); ctx.synchronize()
    T["product"] = time.perf_counter() - t
    t = time.perf_counter()
    pk = z.to_packed(); T["to_packed"] = time.perf_counter() - t
    t = time.perf_counter()
    zh = unpack_h2(pk, rows=z.rows, cols=z.cols); T["unpack"] = time.perf_counter() - t
    t = time.perf_counter()
    zz = P.multiply_coarsen(xh, xh, eps, ctx=ctx); T["multiply_coarsen(host)"] = time.perf_counter() - t
    print({k: round(v * 1e3, 1) for k, v in T.items()})
