"""Drop-in entry points of the hot path (reference h2mul multiply / coarsen / recompress).

Each function accepts host `H2Matrix` objects (the reference container interface; data is
uploaded, computed on the GPU and downloaded back) or `DeviceH2` handles (device-resident; no
host traffic).  Keyword arguments and error behaviour follow the reference:
  multiply(x, y, tol, *, max_rank=None, scaling=True)          induced.py:358-372
  coarsen(g, coarse, tol, *, max_rank=None, scale_blocks=True) coarsening.py:408-422
  recompress(g, tol, *, max_rank=None)                          coarsening.py:437-445
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
import os as _os
from .device import Context, DeviceH2, default_context
from .errors import InvalidInputError
from .h2 import H2Matrix
from .trees import BlockTree, same_cluster_tree

__all__ = ["multiply", "coarsen", "recompress", "multiply_coarsen", "multiply_coarsen_packed"]


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


def _dev(g, ctx):
    if isinstance(g, DeviceH2):
        return g, False
    if isinstance(g, H2Matrix):
        return DeviceH2.upload(g, ctx), True
    raise InvalidInputError(f"expected an H2Matrix or DeviceH2, got {type(g).__name__}")


def _check_tol(tol):
    if tol < 0:
        raise InvalidInputError(f"tolerance must be >= 0, got {tol}")


def _mr(max_rank):
    return -1 if max_rank is None else max(0, int(max_rank))


def multiply(x, y, tol: float, *, max_rank: int | None = None, scaling: bool = True,
             ctx: Context | None = None):
    """Phase 1: X*Y over the refined product tree with compressed induced bases."""
    _check_tol(tol)
    ctx = _ctx(ctx)
    if isinstance(x, H2Matrix) and isinstance(y, H2Matrix):
        if not same_cluster_tree(x.block_tree.cols, y.block_tree.rows):
            raise InvalidInputError("x and y do not share the middle cluster tree")
    dx, hx = _dev(x, ctx)
    dy, hy = _dev(y, ctx) if y is not x else (dx, hx)
    h = N.P()
    N.check(ctx.lib.h2g_multiply(ctx.h, dx.h, dy.h, float(tol), _mr(max_rank), 1 if scaling else 0,
                                 C.byref(h)))
    g = DeviceH2(ctx, h, None, dx.rows, dy.cols)
    return g.download() if hx else g


def coarsen(g, coarse: BlockTree, tol: float, *, max_rank: int | None = None, scale_blocks: bool = True,
            ctx: Context | None = None):
    """Phase 2: re-compression of the phase-1 product onto `coarse`."""
    _check_tol(tol)
    ctx = _ctx(ctx)
    dg, hg = _dev(g, ctx)
    h = N.P()
    N.check(ctx.lib.h2g_coarsen(ctx.h, dg.h, ctx.blocks(coarse), float(tol), _mr(max_rank),
                                1 if scale_blocks else 0, C.byref(h)))
    z = DeviceH2(ctx, h, coarse, coarse.rows, coarse.cols)
    return z.download() if hg else z


def recompress(g, tol: float, *, max_rank: int | None = None, ctx: Context | None = None):
    """Adaptive-rank recompression on the matrix's own block tree (input preparation)."""
    _check_tol(tol)
    ctx = _ctx(ctx)
    dg, hg = _dev(g, ctx)
    h = N.P()
    N.check(ctx.lib.h2g_recompress(ctx.h, dg.h, float(tol), _mr(max_rank), C.byref(h)))
    z = DeviceH2(ctx, h, dg.block_tree, dg.rows, dg.cols)
    return z.download() if hg else z


def multiply_coarsen(x, y, tol: float, *, coarse: BlockTree | None = None, max_rank: int | None = None,
                     ctx: Context | None = None):
    """The full product path the reference harness times (bench.py:201-237): multiply, then
    coarsen onto `coarse` (default: X's block tree, `--coarsen input-tree`)."""
    ctx = _ctx(ctx)
    dx, hx = _dev(x, ctx)
    dy = dx if y is x else _dev(y, ctx)[0]
    g = multiply(dx, dy, tol, max_rank=max_rank, ctx=ctx)
    z = coarsen(g, coarse if coarse is not None else dx.block_tree, tol, max_rank=max_rank, ctx=ctx)
    return z.download() if hx else z


_NO_PREFETCH = _os.environ.get("H2G_NO_PREFETCH", "") not in ("", "0")  # A/B switch for the e2e tools


def multiply_coarsen_packed(xp: dict, x_tree: BlockTree, yp: dict | None = None, y_tree: BlockTree | None = None,
                            tol: float = 0.0, *, coarse: BlockTree | None = None, max_rank: int | None = None,
                            out: dict | None = None, ctx: Context | None = None) -> dict:
    """The product on HOST buffers in the packed layout (packed.py; the arrays the C ABI
    h2g_h2_upload / h2g_h2_download take): upload X (and Y; None = Y is X), multiply, coarsen onto
    `coarse` (default X's block tree), download Z into `out` (preallocated, e.g. pinned, arrays of
    DeviceH2.packed_shapes() length) or fresh arrays.  Z's block tree is `coarse`."""
    _check_tol(tol)
    ctx = _ctx(ctx)
    # nearfield arrays stream in on the copy stream while the weights and bases are computed
    dx = DeviceH2.upload_packed(xp, x_tree, ctx, asynchronous=True)
    dy = dx if yp is None else DeviceH2.upload_packed(yp, y_tree if y_tree is not None else x_tree, ctx,
                                                      asynchronous=True)
    g = multiply(dx, dy, tol, max_rank=max_rank, ctx=ctx)
    coarse = coarse if coarse is not None else dx.block_tree
    nh = None if out is None else out.get("near_data")
    h = N.P()
    if nh is not None and not _NO_PREFETCH and nh.dtype == np.float64 and nh.flags.c_contiguous and nh.ndim == 1:
        # Z's dense blocks shared with G stream into out["near_data"] while phase 2 runs
        N.check(ctx.lib.h2g_coarsen_prefetch(ctx.h, g.h, ctx.blocks(coarse), float(tol), _mr(max_rank), 1,
                                             nh.ctypes.data_as(N.F64P), nh.size, C.byref(h)))
    else:
        N.check(ctx.lib.h2g_coarsen(ctx.h, g.h, ctx.blocks(coarse), float(tol), _mr(max_rank), 1, C.byref(h)))
    z = DeviceH2(ctx, h, coarse, coarse.rows, coarse.cols)
    del g
    return z.download_packed(out)
