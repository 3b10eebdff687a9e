"""Host-side structure through the native planner (no GPU needed).

`product_tree(bx, by)` builds T^XY with the C++ planner that the GPU product itself uses
(csrc/engine.cu `product_tree`, reference trees.py:314-359) and returns it as a `BlockTree`.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .trees import BlockTree

__all__ = ["product_tree", "NativeBlocks"]


class NativeBlocks:
    """Owning handles (cluster trees + block tree) for host-only native calls."""

    def __init__(self, bt: BlockTree):
        lib = N.load()
        self.lib = lib
        self.bt = bt
        self._trees = []
        th = {}
        for tree in (bt.rows, bt.cols):
            if id(tree) in th:
                continue
            f = tree.flat()
            arrs = [N.i64(tree.start), N.i64(tree.stop), N.i64(f["child_ptr"]), N.i64(f["child_idx"])]
            h = N.P()
            N.check(lib.h2g_tree_create(None, tree.nnodes, *[a[1] for a in arrs], C.byref(h)))
            th[id(tree)] = h
            self._trees.append(h)
        f = bt.flat()
        arrs = [N.i64(f["row"]), N.i64(f["col"]), N.i64(f["child_ptr"]), N.i64(f["child_idx"])]
        a8 = N.u8(np.asarray(bt.admissible, dtype=np.uint8))
        h = N.P()
        N.check(lib.h2g_blocks_create(None, th[id(bt.rows)], th[id(bt.cols)], bt.nblocks, *[a[1] for a in arrs],
                                      a8[1], C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.lib.h2g_blocks_destroy(self.h)
            for t in self._trees:
                self.lib.h2g_tree_destroy(t)
        except Exception:
            pass


def _structure(lib, h):
    sz = np.zeros(2, np.int64)
    N.check(lib.h2g_blocks_structure(h, sz.ctypes.data_as(N.I64P), None, None, None, None, None))
    nb, nk = int(sz[0]), int(sz[1])
    row, col = np.zeros(nb, np.int64), np.zeros(nb, np.int64)
    ptr, idx, adm = np.zeros(nb + 1, np.int64), np.zeros(nk, np.int64), np.zeros(nb, np.uint8)
    N.check(lib.h2g_blocks_structure(h, sz.ctypes.data_as(N.I64P), row.ctypes.data_as(N.I64P),
                                     col.ctypes.data_as(N.I64P), ptr.ctypes.data_as(N.I64P),
                                     idx.ctypes.data_as(N.I64P), adm.ctypes.data_as(N.U8P)))
    return row, col, ptr, idx, adm


def product_tree(bx: BlockTree, by: BlockTree, with_counts: bool = False):
    """T^XY of X's and Y's block trees, built by the native planner."""
    nx, ny = NativeBlocks(bx), NativeBlocks(by)
    lib = nx.lib
    out = N.P()
    cnt = np.zeros(3, np.int64)
    N.check(lib.h2g_product_tree(nx.h, ny.h, C.byref(out), cnt.ctypes.data_as(N.I64P)))
    try:
        row, col, ptr, idx, adm = _structure(lib, out)
    finally:
        lib.h2g_blocks_destroy(out)
    kids = [tuple(int(c) for c in idx[ptr[b]:ptr[b + 1]]) for b in range(len(row))]
    bt = BlockTree(bx.rows, by.cols, row, col, kids, adm.astype(bool))
    if with_counts:
        return bt, {"a": int(cnt[0]), "b": int(cnt[1]), "c": int(cnt[2])}
    return bt
