"""Cluster trees, block trees, the product block tree T^XY and column trees (host side).

Mirrors the reference interface in h2mul/trees.py (same class names, attribute
names and preorder id conventions, trees.py:1-6) so callers can switch.  The
product block tree -- the only structure built inside the timed product -- is
built by the native planner (csrc/engine.cu `product_tree`, exported as
h2g_product_tree); `build_product_block_tree` below wraps it.
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidInputError, StructureError

__all__ = [
    "ClusterTree", "BlockTree", "ColumnTree", "build_cluster_tree", "admissible",
    "admissible_boxes", "box_diameter", "box_distance", "build_block_tree",
    "build_product_block_tree", "same_cluster_tree", "sparsity_constant",
    "KIND_A", "KIND_B", "KIND_C", "KIND_N",
]

KIND_A, KIND_B, KIND_C, KIND_N = "a", "b", "c", "n"


class ClusterTree:
    """Binary geometric cluster tree; nodes in preorder with contiguous index ranges
    into a recorded permutation (reference trees.py:34-97)."""

    def __init__(self, points, perm, start, stop, children, split_axis, bbox_min, bbox_max):
        self.points = points
        self.perm = perm
        self.start = np.asarray(start, dtype=np.int64)
        self.stop = np.asarray(stop, dtype=np.int64)
        self.children = [tuple(int(c) for c in k) for k in children]
        self.split_axis = split_axis
        self.bbox_min = bbox_min
        self.bbox_max = bbox_max
        self.root = 0
        self._flat = None

    @property
    def nnodes(self) -> int:
        return len(self.start)

    @property
    def npoints(self) -> int:
        return int(self.stop[0] - self.start[0]) if self.points is None else self.points.shape[0]

    @property
    def dim(self) -> int:
        return self.points.shape[1]

    def size(self, t: int) -> int:
        return int(self.stop[t] - self.start[t])

    def is_leaf(self, t: int) -> bool:
        return not self.children[t]

    def leaves(self) -> list[int]:
        return [t for t in range(self.nnodes) if not self.children[t]]

    def index_range(self, t: int) -> slice:
        return slice(int(self.start[t]), int(self.stop[t]))

    def diameter(self, t: int) -> float:
        return box_diameter(self.bbox_min[t], self.bbox_max[t])

    def depth(self) -> int:
        return int(self.flat()["level"].max()) if self.nnodes else 0

    def flat(self) -> dict:
        """Flat topology arrays: parent, level, child CSR, per-level node lists."""
        if self._flat is None:
            n = self.nnodes
            parent = np.full(n, -1, np.int64)
            level = np.zeros(n, np.int64)
            lens = np.array([len(k) for k in self.children], dtype=np.int64)
            ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            idx = np.fromiter((c for k in self.children for c in k), dtype=np.int64,
                              count=int(ptr[-1]))
            for t in range(n):
                for c in self.children[t]:
                    parent[c] = t
                    level[c] = level[t] + 1
            self._flat = {"parent": parent, "level": level, "child_ptr": ptr, "child_idx": idx,
                          "is_leaf": lens == 0}
        return self._flat


def build_cluster_tree(points, leaf_size: int) -> ClusterTree:
    """Median bisection along the longest box axis, stable ties (reference trees.py:100-144)."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    if pts.ndim != 2 or pts.shape[0] == 0:
        raise InvalidInputError("point set must be a non-empty (n, d) array")
    if leaf_size < 1:
        raise InvalidInputError(f"leaf_size must be >= 1, got {leaf_size}")
    n = pts.shape[0]
    work = pts.copy()
    perm = np.arange(n)
    start, stop, kids, axis_of, bmin, bmax = [], [], [], [], [], []
    # explicit stack in preorder: (lo, hi, parent, slot)
    stack = [(0, n, -1, 0)]
    while stack:
        lo, hi, par, slot = stack.pop()
        node = len(start)
        if par >= 0:
            kids[par][slot] = node
        start.append(lo); stop.append(hi); kids.append(None); axis_of.append(-1)
        lo_box = work[lo:hi].min(axis=0)
        hi_box = work[lo:hi].max(axis=0)
        bmin.append(lo_box); bmax.append(hi_box)
        if hi - lo > leaf_size:
            ax = int(np.argmax(hi_box - lo_box))
            order = np.argsort(work[lo:hi, ax], kind="stable")
            work[lo:hi] = work[lo:hi][order]
            perm[lo:hi] = perm[lo:hi][order]
            mid = lo + (hi - lo + 1) // 2
            axis_of[node] = ax
            kids[node] = [0, 0]
            stack.append((mid, hi, node, 1))
            stack.append((lo, mid, node, 0))
        else:
            kids[node] = []
    return ClusterTree(work, perm, start, stop, [tuple(k) for k in kids], axis_of,
                       np.asarray(bmin), np.asarray(bmax))


def box_diameter(bmin, bmax) -> float:
    return float(np.linalg.norm(np.asarray(bmax) - np.asarray(bmin)))


def box_distance(amin, amax, bmin, bmax) -> float:
    gap = np.maximum(0.0, np.maximum(np.asarray(bmin) - np.asarray(amax),
                                     np.asarray(amin) - np.asarray(bmax)))
    return float(np.linalg.norm(gap))


def admissible_boxes(amin, amax, bmin, bmax, eta: float) -> bool:
    """max(diam) <= eta * dist and dist > 0 (reference trees.py:157-168)."""
    if eta <= 0:
        raise InvalidInputError(f"eta must be > 0, got {eta}")
    diam = max(box_diameter(amin, amax), box_diameter(bmin, bmax))
    dist = box_distance(amin, amax, bmin, bmax)
    return dist > 0.0 and diam <= eta * dist


def admissible(rows, t, cols, s, eta) -> bool:
    return admissible_boxes(rows.bbox_min[t], rows.bbox_max[t], cols.bbox_min[s], cols.bbox_max[s], eta)


class BlockTree:
    """Tree of (row cluster, column cluster) pairs whose leaves tile I x J
    (reference trees.py:176-227); ids in preorder, `admissible` True on admissible leaves."""

    def __init__(self, rows, cols, row, col, children, admissible_flags):
        self.rows = rows
        self.cols = cols
        self.row = [int(v) for v in row]
        self.col = [int(v) for v in col]
        self.children = [tuple(int(c) for c in k) for k in children]
        self.admissible = [bool(a) for a in admissible_flags]
        self.root = 0
        self.index = {(r, c): b for b, (r, c) in enumerate(zip(self.row, self.col))}
        self._flat = None

    @property
    def nblocks(self) -> int:
        return len(self.row)

    def is_leaf(self, b: int) -> bool:
        return not self.children[b]

    def is_admissible_leaf(self, b: int) -> bool:
        return not self.children[b] and self.admissible[b]

    def is_inadmissible_leaf(self, b: int) -> bool:
        return not self.children[b] and not self.admissible[b]

    def leaves(self) -> list[int]:
        return [b for b in range(self.nblocks) if not self.children[b]]

    def admissible_leaves(self) -> list[int]:
        return [b for b in self.leaves() if self.admissible[b]]

    def inadmissible_leaves(self) -> list[int]:
        return [b for b in self.leaves() if not self.admissible[b]]

    def transposed(self) -> "BlockTree":
        """Row/column roles swapped, block ids kept (reference trees.py:211-214)."""
        bt = BlockTree.__new__(BlockTree)
        bt.rows, bt.cols = self.cols, self.rows
        bt.row, bt.col = self.col, self.row
        bt.children, bt.admissible = self.children, self.admissible
        bt.root = 0
        bt.index = {(r, c): b for b, (r, c) in enumerate(zip(bt.row, bt.col))}
        bt._flat = None
        return bt

    def flat(self) -> dict:
        """Flat arrays: row, col, kind (0 adm leaf, 1 inadm leaf, 2 inner), child CSR, parent."""
        if self._flat is None:
            nb = self.nblocks
            lens = np.array([len(k) for k in self.children], dtype=np.int64)
            ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            idx = np.fromiter((c for k in self.children for c in k), dtype=np.int64, count=int(ptr[-1]))
            adm = np.asarray(self.admissible, dtype=bool)
            kind = np.where(lens > 0, 2, np.where(adm, 0, 1)).astype(np.int64)
            parent = np.full(nb, -1, np.int64)
            parent[idx] = np.repeat(np.arange(nb, dtype=np.int64), lens)
            self._flat = {"row": np.asarray(self.row, np.int64), "col": np.asarray(self.col, np.int64),
                          "kind": kind, "child_ptr": ptr, "child_idx": idx, "parent": parent}
        return self._flat


def same_cluster_tree(a, b) -> bool:
    if a is b:
        return True
    return (a.nnodes == b.nnodes and np.array_equal(a.start, b.start)
            and np.array_equal(a.stop, b.stop) and a.children == b.children)


def build_block_tree(rows: ClusterTree, cols: ClusterTree, eta: float) -> BlockTree:
    """Recursive eta-admissible block partition (reference trees.py:246-274)."""
    if rows.npoints == 0 or cols.npoints == 0:
        raise InvalidInputError("cluster trees must be non-empty")
    if eta <= 0:
        raise InvalidInputError(f"eta must be > 0, got {eta}")
    rmin, rmax = np.asarray(rows.bbox_min), np.asarray(rows.bbox_max)
    cmin, cmax = np.asarray(cols.bbox_min), np.asarray(cols.bbox_max)
    # per-node 1-D norms, rounded exactly like box_diameter (boundary cases diam == eta*dist)
    rdiam = [box_diameter(rmin[t], rmax[t]) for t in range(rows.nnodes)]
    cdiam = [box_diameter(cmin[s], cmax[s]) for s in range(cols.nnodes)]
    row, col, kids, adm = [], [], [], []
    stack = [(0, 0, -1, 0)]
    while stack:
        t, s, par, slot = stack.pop()
        b = len(row)
        if par >= 0:
            kids[par][slot] = b
        row.append(t); col.append(s); kids.append([])
        gap = np.maximum(0.0, np.maximum(cmin[s] - rmax[t], rmin[t] - cmax[s]))
        dist = float(np.linalg.norm(gap))
        ok = dist > 0.0 and max(rdiam[t], cdiam[s]) <= eta * dist
        if ok:
            adm.append(True)
        elif not rows.children[t] and not cols.children[s]:
            adm.append(False)
        else:
            adm.append(False)
            pairs = [(a, c) for a in (rows.children[t] or (t,)) for c in (cols.children[s] or (s,))]
            kids[b] = [0] * len(pairs)
            for slot2 in reversed(range(len(pairs))):
                stack.append((pairs[slot2][0], pairs[slot2][1], b, slot2))
    return BlockTree(rows, cols, row, col, [tuple(k) for k in kids], adm)


def sparsity_constant(bt: BlockTree) -> int:
    """max_t #{s : (t, s) in the tree} (reference trees.py:438-443)."""
    return int(np.bincount(np.asarray(bt.row)).max())


class ColumnTree:
    """Projection of a product-tree sub-block onto its column component (trees.py:362-406)."""

    __slots__ = ("cluster", "children", "admissible", "matrix")

    def __init__(self, cluster: int, children=(), admissible: bool = True, matrix=None):
        self.cluster = cluster
        self.children = tuple(children)
        self.admissible = admissible
        self.matrix = matrix

    def is_leaf(self) -> bool:
        return not self.children

    def leaves(self):
        if not self.children:
            yield self
        else:
            for c in self.children:
                yield from c.leaves()


def build_product_block_tree(bx: BlockTree, by: BlockTree) -> BlockTree:
    """Minimal block tree on which X*Y is exact (reference trees.py:314-359).

    Built by the native planner; see planner.product_tree for the flat result
    (block ids, kinds and the classified triples the assembly consumes).
    """
    from . import planner
    if not same_cluster_tree(bx.cols, by.rows):
        raise InvalidInputError("factors do not share the middle cluster tree")
    return planner.product_tree(bx, by)
