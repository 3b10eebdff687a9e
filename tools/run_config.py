"""Full-size product of a BASELINE config on the GPU: device-built inputs, recompress, timed
multiply + coarsen, power-iteration accuracy (reference estimator on GPU matvecs).
usage: python tools/run_config.py c3 [n] [steps]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
import torch as _t
os.environ.setdefault("H2G_POOL_RESERVE_GB", f"{0.7 * _t.cuda.get_device_properties(0).total_memory / 1e9:.0f}")
ctx = Context(0)
t0 = time.perf_counter()
dxr, dyr, spec = build_config_device(cfg, n=n, ctx=ctx)
ctx.synchronize()
t_build = time.perf_counter() - t0
t0 = time.perf_counter()
dx = P.recompress(dxr, spec["eps"], ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, spec["eps"], ctx=ctx)
ctx.synchronize()
t_rec = time.perf_counter() - t0
del dxr, dyr
eps = spec["eps"]
for _ in range(3):  # warm-up: host allocations and memory pools reach steady state (as bench.py)
    z = P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
ctx.synchronize()
per = []
for _ in range(steps):  # per-product device time; the median is reported (box-to-box host noise)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    z = P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
    e1.record(ctx.stream)
    e1.synchronize()
    per.append(e0.elapsed_time(e1))
ms = sorted(per)[len(per) // 2]
est = P.estimate_relative_spectral_error(dx, dy, z, steps=20, seed=0)
zs = z.sizes()
out = {"config": cfg, "n": spec["n"], "eps": eps, "ms_per_product": ms, "ms_each": [round(t, 2) for t in per], "dof_per_s": spec["n"] / (ms / 1e3),
       "eps2_power_iteration": est, "build_s": t_build, "recompress_s": t_rec,
       "z_packed_mb": z.packed_bytes() / 1e6, "x_packed_mb": dx.packed_bytes() / 1e6,
       "mem_peak_gb": torch.cuda.max_memory_allocated() / 1e9}
print(json.dumps(out))
