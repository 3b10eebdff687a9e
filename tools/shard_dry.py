"""Per-rank work of the partitioned product on ONE GPU (a projection, not a multi-GPU measurement):
the context is told it is rank r of P with an all-gather that zero-fills the other ranks'
segments, so it computes only its own subtrees (other ranks' clusters come back with rank 0 and
zero blocks: a lower bound for the boundary work of the column passes).
Device time per product for every (P, r); the max over r estimates the compute part of a P-GPU
step without the exchanges.

    python tools/shard_dry.py [config] [P ...]
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2309_09061_b200 as P  # noqa: E402
from paper_2309_09061_b200 import _native as N  # noqa: E402
from paper_2309_09061_b200.device import Context, DeviceH2  # noqa: E402
from paper_2309_09061_b200.problems import build_config  # noqa: E402
from paper_2309_09061_b200.shard import _ALLGATHER, _DeviceBytes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
Ps = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
xr, yr, spec = build_config(cfg)
eps = spec["eps"]
ctx = Context(0)
dx = P.recompress(DeviceH2.upload(xr, ctx), eps, ctx=ctx)
dy = dx if yr is xr else P.recompress(DeviceH2.upload(yr, ctx), eps, ctx=ctx)
state = {"rank": 0}


def _zero_others(user, channel, dbuf, off, nseg, stream):
    offs = [int(off[i]) for i in range(nseg + 1)]
    if offs[-1] == 0:
        return 0
    buf = torch.as_tensor(_DeviceBytes(dbuf, offs[-1]), device="cuda:0")
    with torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device="cuda:0")):
        for i in range(nseg):
            if i != state["rank"] and offs[i + 1] > offs[i]:
                buf[offs[i]:offs[i + 1]].zero_()
    return 0


noop = _ALLGATHER(_zero_others)


def timed(reps=5):
    for _ in range(2):
        P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    t0 = time.perf_counter()
    for _ in range(reps):
        P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), dx.block_tree, eps, ctx=ctx)
    e1.record(ctx.stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


for nparts in Ps:
    per = []
    for r in range(nparts):
        state["rank"] = r
        N.check(ctx.lib.h2g_ctx_set_comm(ctx.h, r if nparts > 1 else 0, nparts, C.cast(noop, C.c_void_p) if nparts > 1 else None, None))
        per.append(timed())
    worst = max(p[0] for p in per)
    print(f"{cfg} P={nparts}: per-rank ms {[round(p[0], 1) for p in per]}  max {worst:.1f}  "
          f"(P=1-relative speed-up of the compute part: see first line)", flush=True)
N.check(ctx.lib.h2g_ctx_set_comm(ctx.h, 0, 1, None, None))
