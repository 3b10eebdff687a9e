import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context, DeviceH2
from helpers import load
from test_gpu_parity import _inputs
d = load("rand_s0_tol1e-3")
x, y, eps = _inputs(d)
a = Context(0)
ax = DeviceH2.upload(x, a); ay = DeviceH2.upload(y, a)
za = P.coarsen(P.multiply(ax, ay, eps, ctx=a), ax.block_tree, eps, ctx=a)
zah = za.download()
print("a ok", flush=True)
solo = Context(0)
sx = DeviceH2.upload(x, solo); sy = DeviceH2.upload(y, solo)
g = P.multiply(sx, sy, eps, ctx=solo)
print("mult ok", flush=True)
z = P.coarsen(g, sx.block_tree, eps, ctx=solo)
print("coarsen ok", flush=True)
del g
print("del g ok", flush=True)
zh = z.download()
print("solo ok", flush=True)
