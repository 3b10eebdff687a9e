"""Time GPU matvecs of the c-config product Z the way bench.py does (profile-mode events per launch)
and print achieved GB/s for Z v and Z^T v."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from paper_2309_09061_b200.problems import build_config_device
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = Context(0)
dxr, dyr, spec = build_config_device(cfg, ctx=ctx)
dx = P.recompress(dxr, spec["eps"], ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, spec["eps"], ctx=ctx)
del dxr, dyr
z = P.coarsen(P.multiply(dx, dy, spec["eps"], ctx=ctx), dx.block_tree, spec["eps"], ctx=ctx)
v = torch.randn(z.shape[1], dtype=torch.float64, device="cuda")
for trans in (False, True):
    for _ in range(3):
        z.matvec(v, trans=trans)
    torch.cuda.synchronize()
    ctx.kernel_stats(reset=True)
    ctx.set_profile(True)
    for _ in range(10):
        z.matvec(v, trans=trans)
    ctx.synchronize()
    ctx.set_profile(False)
    s = ctx.kernel_stats(reset=True)["mv"]
    ms, by = s["ms"] / 10, s["bytes"] / 10
    # whole-call device time (streams overlap; no per-launch events), torch events around 10 calls
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        z.matvec(v, trans=trans)
    e1.record()
    torch.cuda.synchronize()
    wall = e0.elapsed_time(e1) / 10
    print(json.dumps({"config": cfg, "trans": trans, "kernel_ms_sum": ms, "launches": s["launches"] // 10,
                      "gb": by / 1e9, "gbs_kernel_sum": by / ms / 1e6, "call_ms": wall,
                      "gbs_call": by / wall / 1e6}))
