"""Packed interchange layout for H^2 matrices (host <-> device <-> fixtures).

One flat float64 array per matrix family plus int64 offset tables, all
row-major (reference storage convention, h2mul/dense.py:3-4):

  rows./cols.  start, stop, child_ptr, child_idx           cluster trees
  bt.          row, col, child_ptr, child_idx, adm (u8)     block tree (preorder)
  rb./cb.      rank, leaf_off, xfer_off, data               bases: leaf (size x k),
                                                            transfer (k_c x k_parent)
  coup_off, coup_data                                       k_t x k_s per admissible leaf
  near_off, near_data                                       size_t x size_s per inadmissible leaf

Offsets are -1 where a block / cluster carries no matrix.  This replaces the
reference's JSON fixture format (h2mul/h2.py:314-397) with a binary one.
"""

from __future__ import annotations

import numpy as np

from .h2 import ClusterBasis, H2Matrix
from .trees import BlockTree, ClusterTree

__all__ = ["pack_h2", "unpack_h2", "pack_tree", "unpack_tree", "pack_structure", "unpack_structure",
           "save_h2", "load_h2", "save_packed", "load_packed", "FORMAT"]

FORMAT = "h2g-packed-1"  # on-disk: one .npz (uncompressed) holding the packed layout below


def pack_tree(tree, p, out):
    out[p + "start"] = np.asarray(tree.start, dtype=np.int64)
    out[p + "stop"] = np.asarray(tree.stop, dtype=np.int64)
    f = tree.flat()
    out[p + "child_ptr"] = f["child_ptr"]
    out[p + "child_idx"] = f["child_idx"]


def unpack_tree(d, p) -> ClusterTree:
    ptr, idx = np.asarray(d[p + "child_ptr"]), np.asarray(d[p + "child_idx"])
    kids = [tuple(int(c) for c in idx[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)]
    return ClusterTree(None, None, d[p + "start"], d[p + "stop"], kids, None, None, None)


def _pack_basis(basis, p, out):
    tree = basis.tree
    f = tree.flat()
    rank = np.asarray(basis.rank, dtype=np.int64)
    size = (tree.stop - tree.start).astype(np.int64)
    loff = np.full(tree.nnodes, -1, np.int64)
    xoff = np.full(tree.nnodes, -1, np.int64)
    leaves = np.nonzero(f["is_leaf"])[0]
    nonroot = np.nonzero(f["parent"] >= 0)[0]
    lsz = size[leaves] * rank[leaves]
    xsz = rank[nonroot] * rank[f["parent"][nonroot]]
    loff[leaves] = np.concatenate([[0], np.cumsum(lsz)[:-1]]) if len(leaves) else []
    base = int(lsz.sum())
    xoff[nonroot] = base + (np.concatenate([[0], np.cumsum(xsz)[:-1]]) if len(nonroot) else [])
    data = np.empty(base + int(xsz.sum()))
    for t in leaves:
        data[loff[t]:loff[t] + lsz[np.searchsorted(leaves, t)]] = np.asarray(basis.leaf_matrix[t]).ravel()
    for i, t in enumerate(nonroot):
        data[xoff[t]:xoff[t] + xsz[i]] = np.asarray(basis.transfer[t]).ravel()
    out[p + "rank"] = rank
    out[p + "leaf_off"] = loff
    out[p + "xfer_off"] = xoff
    out[p + "data"] = data


def pack_basis_arrays(basis):
    """(rank, leaf_off, xfer_off, data) of one basis in the packed layout."""
    out = {}
    _pack_basis(basis, "", out)
    return out["rank"], out["leaf_off"], out["xfer_off"], out["data"]


def _unpack_basis(d, p, tree) -> ClusterBasis:
    rank = [int(v) for v in d[p + "rank"]]
    data = d[p + "data"]
    loff, xoff = d[p + "leaf_off"], d[p + "xfer_off"]
    par = tree.flat()["parent"]
    leaf, xfer = {}, {}
    for t in range(tree.nnodes):
        if tree.is_leaf(t):
            n = tree.size(t) * rank[t]
            leaf[t] = data[loff[t]:loff[t] + n].reshape(tree.size(t), rank[t])
        if par[t] >= 0:
            n = rank[t] * rank[par[t]]
            xfer[t] = data[xoff[t]:xoff[t] + n].reshape(rank[t], rank[par[t]])
    return ClusterBasis(tree, rank, leaf, xfer)


def pack_structure(bt: BlockTree, prefix: str = "", out: dict | None = None) -> dict:
    """Cluster trees + block tree of the packed layout (rows., cols., bt. keys)."""
    out = {} if out is None else out
    p = prefix
    pack_tree(bt.rows, p + "rows.", out)
    pack_tree(bt.cols, p + "cols.", out)
    f = bt.flat()
    out[p + "bt.row"], out[p + "bt.col"] = f["row"], f["col"]
    out[p + "bt.child_ptr"], out[p + "bt.child_idx"] = f["child_ptr"], f["child_idx"]
    out[p + "bt.adm"] = np.asarray(bt.admissible, dtype=np.uint8)
    return out


def unpack_structure(d, prefix: str = "", rows=None, cols=None) -> BlockTree:
    p = prefix
    rows = rows if rows is not None else unpack_tree(d, p + "rows.")
    cols = cols if cols is not None else unpack_tree(d, p + "cols.")
    ptr, idx = np.asarray(d[p + "bt.child_ptr"]), np.asarray(d[p + "bt.child_idx"])
    kids = [tuple(int(c) for c in idx[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)]
    return BlockTree(rows, cols, d[p + "bt.row"], d[p + "bt.col"], kids, np.asarray(d[p + "bt.adm"]).astype(bool))


def pack_h2(g: H2Matrix, prefix: str = "") -> dict:
    out = {}
    p = prefix
    bt = g.block_tree
    pack_structure(bt, p, out)
    _pack_basis(g.row_basis, p + "rb.", out)
    _pack_basis(g.col_basis, p + "cb.", out)
    for name, store in (("coup", g.coupling), ("near", g.nearfield)):
        off = np.full(bt.nblocks, -1, np.int64)
        keys = sorted(store)
        sizes = [store[b].size for b in keys]
        starts = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64) if keys else []
        off[keys] = starts
        out[p + name + "_off"] = off
        out[p + name + "_data"] = (np.concatenate([np.asarray(store[b]).ravel() for b in keys])
                                   if keys else np.zeros(0))
    return out


def unpack_h2(d, prefix: str = "", rows=None, cols=None) -> H2Matrix:
    p = prefix
    bt = unpack_structure(d, p, rows, cols)
    rows, cols = bt.rows, bt.cols
    rb = _unpack_basis(d, p + "rb.", rows)
    cb = _unpack_basis(d, p + "cb.", cols)
    coup, near = {}, {}
    coff, noff = d[p + "coup_off"], d[p + "near_off"]
    cdat, ndat = d[p + "coup_data"], d[p + "near_data"]
    for b in range(bt.nblocks):
        if not bt.children[b]:
            t, s = bt.row[b], bt.col[b]
            if bt.admissible[b]:
                n = rb.rank[t] * cb.rank[s]
                coup[b] = cdat[coff[b]:coff[b] + n].reshape(rb.rank[t], cb.rank[s])
            else:
                n = rows.size(t) * cols.size(s)
                near[b] = ndat[noff[b]:noff[b] + n].reshape(rows.size(t), cols.size(s))
    return H2Matrix(bt, rb, cb, coup, near)


def save_packed(path, packed: dict, block_tree: BlockTree | None = None):
    """Write a packed-layout dict (e.g. DeviceH2.download_packed()) to one binary .npz; the
    structure keys come from `block_tree` when the dict lacks them.  Replaces the reference's
    JSON serialisation (h2mul/h2.py:314-397) for matrices of GB size."""
    d = dict(packed)
    if "bt.row" not in d:
        if block_tree is None:
            raise ValueError("packed dict without structure: pass its block_tree")
        pack_structure(block_tree, "", d)
    np.savez(path, __format__=np.array([FORMAT]), **d)


def load_packed(path):
    """(packed dict, BlockTree) of a file written by save_packed / save_h2."""
    with np.load(path) as z:
        if "__format__" not in z.files or str(z["__format__"][0]) != FORMAT:
            raise ValueError(f"{path}: not an {FORMAT} file")
        d = {k: z[k] for k in z.files if k != "__format__"}
    return d, unpack_structure(d)


def save_h2(path, g: H2Matrix):
    """Host H2Matrix -> binary packed file (h2mul.h2_to_json's role, h2.py:362-381)."""
    save_packed(path, pack_h2(g))


def load_h2(path) -> H2Matrix:
    """Binary packed file -> host H2Matrix (h2mul.h2_from_json's role, h2.py:384-397)."""
    d, bt = load_packed(path)
    return unpack_h2(d, rows=bt.rows, cols=bt.cols)
