"""sigma_1 of every leaf block of a product G (block_norms, the NormBatch kernels) against host SVDs:
max relative error and the worst blocks' shapes.  usage: python tools/norm_check.py [config] [n]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2309_09061_b200 as P
from helpers import load, rebuild_raw
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
d = load(cfg)
eps = float(d["eps"][0])
xr, yr = rebuild_raw(d)
x = P.recompress(xr, eps)
y = x if yr is xr else P.recompress(yr, eps)
g = P.multiply(x, y, eps)
gh = g.download() if hasattr(g, "download") else g
cn, nn = P.coupling_norms(g), P.nearfield_norms(g)
for name, got, mats in (("coupling", cn, gh.coupling), ("nearfield", nn, gh.nearfield)):
    errs = []
    for b, m in mats.items():
        ref = np.linalg.norm(m, 2)
        errs.append((abs(got[b] - ref) / max(ref, 1e-300), b, m.shape, got[b], ref))
    errs.sort(reverse=True)
    print(name, len(errs), "max rel err", errs[0][0] if errs else None)
    for e in errs[:5]:
        print("   ", e)
