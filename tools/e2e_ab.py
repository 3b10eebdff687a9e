"""A/B of the packed host-buffer product with and without the nearfield prefetch (H2G_NO_PREFETCH)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200 import api
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
xr, yr, spec = build_config(cfg)
ctx = Context(0)
eps = spec["eps"]
dx = P.recompress(DeviceH2.upload(xr, ctx), eps, ctx=ctx)
pk = dx.download_packed()
xp = {}
for k, v in pk.items():
    t = torch.empty(len(v), dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True)
    a = t.numpy(); a[:] = v; xp[k] = a
bt = dx.block_tree
z = P.coarsen(P.multiply(dx, dx, eps, ctx=ctx), bt, eps, ctx=ctx)
zs = z.packed_shapes()
zout = {k: torch.empty(n, dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True).numpy()
        for k, n in zs.items()}
del z
res = {0: [], 1: []}
for it in range(24):
    mode = it % 2
    api._NO_PREFETCH = bool(mode)
    ctx.synchronize()
    t0 = time.perf_counter()
    P.multiply_coarsen_packed(xp, bt, None, None, eps, coarse=bt, out=zout, ctx=ctx)
    res[mode].append((time.perf_counter() - t0) * 1e3)
for m, name in ((0, "prefetch"), (1, "no-prefetch")):
    v = np.array(res[m][2:])
    print(f"{name:12s} median {np.median(v):7.2f} ms  min {v.min():7.2f}  max {v.max():7.2f}")
