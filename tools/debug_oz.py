"""Compare Gram-path outputs (R^T R of basis / total weights) of the integer tensor-core partial
Grams against the FP64 double-double ones: python tools/debug_oz.py out.npz (env selects the path)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device
ctx = Context(0)
out = {}
for cfg, n in (("c2", 2048), ("c4", 4096)):
    dxr, dyr, spec = build_config_device(cfg, n=n, ctx=ctx)
    rw = P.basis_weights(dxr.col_basis, ctx=ctx).r
    for s, m in rw.items():
        out[f"{cfg}.rw.{s}"] = m.T @ m
    zy = P.total_weights(dxr, P.basis_weights(dxr.col_basis, ctx=ctx), ctx=ctx).z
    for s, m in zy.items():
        out[f"{cfg}.z.{s}"] = m.T @ m
    dx = P.recompress(dxr, spec["eps"], ctx=ctx)
    out[f"{cfg}.xrank"] = np.asarray(dx.ranks()[0])
np.savez(sys.argv[1], **out)
