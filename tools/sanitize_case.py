"""Small product for compute-sanitizer (one tool per call): a golden random case through multiply,
coarsen and the matvec, ranks checked against the reference fixture."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2309_09061_b200 as P
from helpers import load
from paper_2309_09061_b200.packed import unpack_h2
name = sys.argv[1] if len(sys.argv) > 1 else "rand_s2_2d"
d = load(name)
eps = float(d["eps"][0])
x = unpack_h2(d, "x/")
y = unpack_h2(d, "y/", rows=x.block_tree.cols)
dx, dy = P.DeviceH2.upload(x), P.DeviceH2.upload(y)
g = P.multiply(dx, dy, eps)
z = P.coarsen(g, dx.block_tree, eps)
import torch
v = torch.randn(z.shape[1], dtype=torch.float64, device="cuda")
z.matvec(v); z.matvec(v, trans=True)
zh = z.download()
ok = list(zh.row_basis.rank) == list(d["rank.final_row"]) and list(zh.col_basis.rank) == list(d["rank.final_col"])
print("ranks equal to the reference:", ok)
sys.exit(0 if ok else 1)
