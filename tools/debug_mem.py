"""Arena payload over the stages of one single-GPU product (H2G_DEBUG_MEM=1): python tools/debug_mem.py c2 [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.device import Context
from paper_2309_09061_b200.problems import build_config_device
cfg = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else None
ctx = Context(0)
dxr, dyr, spec = build_config_device(cfg, n=n, ctx=ctx)
dx = P.recompress(dxr, spec["eps"], ctx=ctx)
dy = dx if dyr is dxr else P.recompress(dyr, spec["eps"], ctx=ctx)
del dxr, dyr
ctx.synchronize()
print("inputs", ctx.memory(reset=True), file=sys.stderr)
z = P.coarsen(P.multiply(dx, dy, spec["eps"], ctx=ctx), dx.block_tree, spec["eps"], ctx=ctx)
ctx.synchronize()
print("after", ctx.memory(), file=sys.stderr)
print("sizes X", dx.packed_bytes() / 1e6, "Z", z.packed_bytes() / 1e6, file=sys.stderr)
