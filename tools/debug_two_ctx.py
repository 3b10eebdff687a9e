"""Two native contexts in one process, products on each in turn (regression check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from helpers import load
from test_gpu_parity import _inputs
for it in range(3):
    for name in ["rand_s0_tol1e-3", "rand_s2_2d", "c1"]:
        d = load(name)
        x, y, eps = _inputs(d)
        a = Context(0)
        ax = DeviceH2.upload(x, a); ay = ax if y is x else DeviceH2.upload(y, a)
        a.synchronize(); b0 = a.memory(reset=True)["payload"]
        za = P.coarsen(P.multiply(ax, ay, eps, ctx=a), ax.block_tree, eps, ctx=a)
        a.synchronize(); pa = a.memory()["payload_high"] - b0
        zah = za.download()
        solo = Context(0)
        sx = DeviceH2.upload(x, solo); sy = sx if y is x else DeviceH2.upload(y, solo)
        zs = P.coarsen(P.multiply(sx, sy, eps, ctx=solo), sx.block_tree, eps, ctx=solo).download()
        print(it, name, "ok", pa, flush=True)
