"""Per-step device times of back-to-back products as bench.py runs them (no host sync between steps),
and with a sync between steps: python tools/step_loop.py c4 [steps] [sync]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device
cfg = sys.argv[1]; steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sync = len(sys.argv) > 3 and sys.argv[3] == "sync"
import torch as _t
os.environ.setdefault("H2G_POOL_RESERVE_GB", f"{0.7 * _t.cuda.get_device_properties(0).total_memory / 1e9:.0f}")
ctx = Context(0)
dxr, dyr, spec = build_config_device(cfg, ctx=ctx)
eps = spec["eps"]
dx = P.recompress(dxr, eps, ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, eps, ctx=ctx)
del dxr, dyr
def step():
    return P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
for _ in range(3):
    z = step()
ctx.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
host = []
stages = []
timing = os.environ.get("STAGES") is not None
if timing:
    ctx.set_timing(True)
evs[0].record(ctx.stream)
for i in range(steps):
    t0 = time.perf_counter()
    g = P.multiply(dx, dy, eps, ctx=ctx)
    s1 = ctx.stage_times() if timing else {}
    z = P.coarsen(g, dx.block_tree, eps, ctx=ctx)
    del g
    s2 = ctx.stage_times() if timing else {}
    evs[i + 1].record(ctx.stream)
    if sync:
        ctx.synchronize()
    host.append(time.perf_counter() - t0)
    if timing:
        ht = ctx.host_times(reset=True)
        stages.append({"host_top": sorted(((round(v, 1), k) for k, v in ht.items()), reverse=True)[:8]})
        stages.append({k: round(1e3 * v, 1) for k, v in {**{k: s1[k] for k in ("t_setup", "t1_span", "t1_mat")},
                                                        **{k: s2[k] for k in ("t2_norms", "t2_span", "t2_mat")}}.items()})
torch.cuda.synchronize()
dev = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
for st in stages:
    print("  stages ms", st)
print(cfg, "sync" if sync else "nosync", "device ms", [round(d, 1) for d in dev], "mean", round(sum(dev) / steps, 1),
      "host s", [round(h, 3) for h in host], "mem", {k: round(v / 1e9, 1) for k, v in ctx.memory().items()})
