"""GPU parity at the BASELINE sizes against fixtures produced by the REFERENCE itself
(tests/golden/make_golden_full.py: h2mul run stage by stage exactly as its harness does,
bench.py:195-237, at c2 n = 16,384, c3 n = 32,768, c4 n = 65,536 and 262,144, c5 n = 32,768,
plus scaling=False / scale_blocks=False cases).

Inputs are built on the GPU by the repo's interpolation builder and pinned to the reference's raw
inputs through X_raw v / Y_raw v at the same n (<= 1e-13).  Gates (BASELINE north_star): identical
T^XY, every per-cluster rank equal (input recompression, induced row/col, final row/col),
||(Z_gpu - Z_ref) v|| / ||Z_ref v|| <= 10 eps (also G v and Z^T v), ||Z_gpu v - X(Y v)|| / ||X(Y v)||
<= max(eps, 1.1 x the reference's own value), and the power-iteration estimate within 1e-4
relative of the reference's.
"""

import glob
import os

import numpy as np
import pytest

from helpers import GOLDEN, rel

pytestmark = pytest.mark.gpu

FULL_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                    if "meta.case" in np.load(p).files)


def _structure(dg):
    s = dg.sizes()
    nb = int(s[0])
    import ctypes as C  # noqa: F401
    from paper_2309_09061_b200 import _native as N
    row, col = np.zeros(nb, np.int64), np.zeros(nb, np.int64)
    ptr, idx = np.zeros(nb + 1, np.int64), np.zeros(int(s[7]), np.int64)
    adm = np.zeros(nb, np.uint8)
    N.check(dg.ctx.lib.h2g_h2_structure(dg.h, row.ctypes.data_as(N.I64P), col.ctypes.data_as(N.I64P),
                                        ptr.ctypes.data_as(N.I64P), idx.ctypes.data_as(N.I64P),
                                        adm.ctypes.data_as(N.U8P)))
    return row, col, ptr, idx, adm


@pytest.mark.parametrize("case", FULL_CASES)
def test_fullsize_parity(case):
    import torch
    import paper_2309_09061_b200 as P
    from paper_2309_09061_b200.device import Context
    from paper_2309_09061_b200.problems import build_config_device
    d = dict(np.load(os.path.join(GOLDEN, f"{case}.npz")))
    name, n = str(d["meta.config"][0]), int(d["meta.n"][0])
    scaling = bool(d["meta.scaling"][0])
    eps = float(d["eps"][0])
    ctx = Context(0)
    dev = torch.device("cuda", 0)
    v = np.random.default_rng(123).standard_normal(n)
    vt = torch.from_numpy(v).to(dev)
    dxr, dyr, _ = build_config_device(name, n=n, ctx=ctx)
    # the GPU-built raw inputs are the reference's raw inputs (problems.py:295-332)
    assert rel(dxr.matvec(vt).cpu().numpy(), d["probe.xraw_v"][0]) <= 1e-13
    assert rel(dyr.matvec(vt).cpu().numpy(), d["probe.yraw_v"][0]) <= 1e-13
    dx = P.recompress(dxr, eps, ctx=ctx)
    dy = dx if dyr is dxr else P.recompress(dyr, eps, ctx=ctx)
    del dxr, dyr
    xr, xc = dx.ranks()
    yr, yc = dy.ranks()
    assert np.array_equal(xr, d["rank.x_row"]) and np.array_equal(xc, d["rank.x_col"])
    assert np.array_equal(yr, d["rank.y_row"]) and np.array_equal(yc, d["rank.y_col"])

    g = P.multiply(dx, dy, eps, scaling=scaling, ctx=ctx)
    row, col, ptr, idx, adm = _structure(g)
    assert np.array_equal(row, d["pt.row"]) and np.array_equal(col, d["pt.col"])
    assert np.array_equal(ptr, d["pt.child_ptr"]) and np.array_equal(idx, d["pt.child_idx"])
    assert np.array_equal(adm, d["pt.adm"])
    gr, gc = g.ranks()
    assert np.array_equal(gr, d["rank.induced_row"]), np.flatnonzero(gr != d["rank.induced_row"])[:10]
    assert np.array_equal(gc, d["rank.induced_col"]), np.flatnonzero(gc != d["rank.induced_col"])[:10]
    z = P.coarsen(g, dx.block_tree, eps, scale_blocks=scaling, ctx=ctx)
    zr, zc = z.ranks()
    assert np.array_equal(zr, d["rank.final_row"]), np.flatnonzero(zr != d["rank.final_row"])[:10]
    assert np.array_equal(zc, d["rank.final_col"]), np.flatnonzero(zc != d["rank.final_col"])[:10]

    tol = 10 * eps
    gv = g.matvec(vt).cpu().numpy()
    del g
    zv = z.matvec(vt).cpu().numpy()
    ztv = z.matvec(vt, trans=True).cpu().numpy()
    assert rel(gv, d["probe.gv"][0].astype(np.float64)) <= tol
    assert rel(zv, d["probe.zv"][0].astype(np.float64)) <= tol
    assert rel(ztv, d["probe.ztv"][0].astype(np.float64)) <= tol
    xyv = d["probe.xyv"][0]
    assert rel(zv, xyv) <= max(eps, 1.1 * float(d["probe.ref_xy_rel"][0]), 1e-12)
    est = P.estimate_relative_spectral_error(dx, dy, z, steps=20, seed=0)
    ref = float(d["est.eps2"][0])
    if ref <= 1e-12:
        assert est <= 1e-12
    else:
        assert abs(est - ref) <= 1e-4 * ref, (est, ref)
