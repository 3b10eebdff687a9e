"""Debug driver: GPU multiply/coarsen/recompress vs the golden fixtures, verbose diagnostics."""
import os, sys, time, traceback
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import load, rebuild_raw, rel
import paper_2309_09061_b200 as P
from paper_2309_09061_b200.packed import unpack_h2
from paper_2309_09061_b200.h2 import h2_matvec_host

def diff_ranks(name, got, want):
    got, want = list(got), list(want)
    if got == want:
        return "ok"
    bad = [(i, g, w) for i, (g, w) in enumerate(zip(got, want)) if g != w]
    return f"MISMATCH {len(bad)} first {bad[:6]} (len {len(got)} vs {len(want)})"

def run(name):
    d = load(name)
    eps = float(d["eps"][0])
    t0 = time.time()
    if "x/bt.row" in d:
        x = unpack_h2(d, "x/")
        y = unpack_h2(d, "y/", rows=x.block_tree.cols)
    else:
        xr, yr = rebuild_raw(d)
        x = P.recompress(xr, eps)
        y = x if yr is xr else P.recompress(yr, eps)
        print(f"  recompress x ranks: {diff_ranks('x', x.row_basis.rank, d['rank.x_row'])}")
    dx = P.DeviceH2.upload(x)
    dy = dx if y is x else P.DeviceH2.upload(y)
    g = P.multiply(dx, dy, eps)
    gh = g.download()
    print(f"  pt rows: {'ok' if list(gh.block_tree.row) == list(d['pt.row']) and list(gh.block_tree.col) == list(d['pt.col']) else 'MISMATCH'}")
    print(f"  induced row ranks: {diff_ranks('r', gh.row_basis.rank, d['rank.induced_row'])}")
    print(f"  induced col ranks: {diff_ranks('c', gh.col_basis.rank, d['rank.induced_col'])}")
    errs = [rel(h2_matvec_host(gh, v), d['probe.gv'][i]) for i, v in enumerate(d['probe.v'])]
    print(f"  G v rel err vs ref: {max(errs):.3e}")
    z = P.coarsen(g, x.block_tree, eps)
    zh = z.download()
    print(f"  final row ranks: {diff_ranks('r', zh.row_basis.rank, d['rank.final_row'])}")
    print(f"  final col ranks: {diff_ranks('c', zh.col_basis.rank, d['rank.final_col'])}")
    errs = [rel(h2_matvec_host(zh, v), d['probe.zv'][i]) for i, v in enumerate(d['probe.v'])]
    xy = [rel(h2_matvec_host(zh, v), d['probe.xyv'][i]) for i, v in enumerate(d['probe.v'])]
    print(f"  Z v rel err vs ref: {max(errs):.3e}   |Zv - X(Yv)|/|X(Yv)|: {max(xy):.3e}  (eps {eps:g})  {time.time()-t0:.1f}s")

if __name__ == "__main__":
    names = sys.argv[1:] or ["rand_s0_tol1e-3", "rand_s1_tol0", "rand_s2_2d", "rand_s3_2d_tol0", "c1", "c2", "c3", "c4", "c5"]
    for n in names:
        print(f"== {n}", flush=True)
        try:
            run(n)
        except Exception:
            traceback.print_exc()
        sys.stdout.flush()
