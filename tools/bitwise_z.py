"""Write Z (packed) of one product of a config to an npz, for bitwise comparison between builds:
H2G_LIB=a.so python tools/bitwise_z.py c2 out_a.npz; H2G_LIB=b.so ... out_b.npz; then compare."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device
if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise identical" if not bad else f"differ: {bad}")
    for k in bad:
        if a[k].shape == b[k].shape and a[k].dtype.kind == "f":
            print(k, "max rel", float(np.max(np.abs(a[k] - b[k])) / max(1e-300, np.max(np.abs(a[k])))))
        else:
            print(k, a[k].shape, b[k].shape)
    sys.exit(0)
ctx = Context(0)
dxr, dyr, spec = build_config_device(sys.argv[1], ctx=ctx)
dx = P.recompress(dxr, spec["eps"], ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, spec["eps"], ctx=ctx)
z = P.coarsen(P.multiply(dx, dy, spec["eps"], ctx=ctx), dx.block_tree, spec["eps"], ctx=ctx)
np.savez(sys.argv[2], **z.download_packed())
