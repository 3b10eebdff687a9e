"""Host containers with the reference's interface (h2mul/h2.py:32-194).

`ClusterBasis`, `BasisProduct` and `H2Matrix` keep the reference's attribute
names (rank / leaf_matrix / transfer; block_tree / row_basis / col_basis /
coupling / nearfield) so code written against h2mul reads them unchanged.
The GPU path never computes on these dicts: `packed.py` flattens them into
device arenas (`device.DeviceH2`) and back.
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidInputError

__all__ = ["ClusterBasis", "BasisProduct", "H2Matrix", "storage_bytes", "to_dense",
           "h2_matvec_host", "expand_basis"]

DENSE_GUARD = 16384


class ClusterBasis:
    """Nested basis: explicit leaf matrices, transfers E_c (k_c x k_parent) above
    (reference h2.py:32-72).  Ranks may be zero."""

    def __init__(self, tree, rank, leaf_matrix, transfer):
        self.tree = tree
        self.rank = [int(k) for k in rank]
        self.leaf_matrix = leaf_matrix
        self.transfer = transfer

    def expand(self, t: int) -> np.ndarray:
        if self.tree.is_leaf(t):
            return self.leaf_matrix[t]
        return np.vstack([self.expand(c) @ self.transfer[c] for c in self.tree.children[t]])

    def max_rank(self) -> int:
        return max(self.rank) if self.rank else 0

    def storage_bytes(self) -> int:
        return (sum(m.nbytes for m in self.leaf_matrix.values())
                + sum(m.nbytes for m in self.transfer.values()))


def expand_basis(basis: ClusterBasis, t: int) -> np.ndarray:
    return basis.expand(t)


class BasisProduct:
    """P_s = W_s^T V_s per cluster (reference h2.py:116-124)."""

    def __init__(self, tree, p):
        self.tree = tree
        self.p = p

    def transposed(self) -> "BasisProduct":
        return BasisProduct(self.tree, {s: m.T for s, m in self.p.items()})


class H2Matrix:
    """Block tree + bases + couplings (admissible leaves) + nearfield (inadmissible
    leaves) (reference h2.py:148-194)."""

    def __init__(self, block_tree, row_basis, col_basis, coupling, nearfield):
        self.block_tree = block_tree
        self.row_basis = row_basis
        self.col_basis = col_basis
        self.coupling = coupling
        self.nearfield = nearfield

    @property
    def shape(self):
        return (self.block_tree.rows.npoints, self.block_tree.cols.npoints)

    def transposed(self) -> "H2Matrix":
        return H2Matrix(self.block_tree.transposed(), self.col_basis, self.row_basis,
                        {b: s.T for b, s in self.coupling.items()},
                        {b: m.T for b, m in self.nearfield.items()})

    def validate(self):
        """Placement and dimension checks (reference h2.py:175-194)."""
        bt = self.block_tree
        for b in range(bt.nblocks):
            t, s = bt.row[b], bt.col[b]
            if bt.is_admissible_leaf(b):
                if b not in self.coupling:
                    raise InvalidInputError(f"admissible leaf {b} lacks coupling")
                if self.coupling[b].shape != (self.row_basis.rank[t], self.col_basis.rank[s]):
                    raise InvalidInputError(f"coupling {b} has wrong shape")
            elif bt.is_inadmissible_leaf(b):
                if b not in self.nearfield:
                    raise InvalidInputError(f"inadmissible leaf {b} lacks nearfield")
                if self.nearfield[b].shape != (bt.rows.size(t), bt.cols.size(s)):
                    raise InvalidInputError(f"nearfield {b} has wrong shape")


def storage_bytes(g: H2Matrix) -> int:
    """Bytes of bases, couplings and nearfield (reference h2.py:307-311)."""
    return (g.row_basis.storage_bytes() + g.col_basis.storage_bytes()
            + sum(m.nbytes for m in g.coupling.values())
            + sum(m.nbytes for m in g.nearfield.values()))


def h2_matvec_host(g: H2Matrix, x) -> np.ndarray:
    """y = G x on the host (verification helper; reference h2.py:224-244)."""
    bt = g.block_tree
    rows, cols = bt.rows, bt.cols
    x = np.asarray(x, dtype=np.float64)
    xh = [None] * cols.nnodes
    for s in reversed(range(cols.nnodes)):
        if cols.is_leaf(s):
            xh[s] = g.col_basis.leaf_matrix[s].T @ x[cols.index_range(s)]
        else:
            xh[s] = sum((g.col_basis.transfer[c].T @ xh[c] for c in cols.children[s]),
                        np.zeros(g.col_basis.rank[s]))
    yh = [np.zeros(k) for k in g.row_basis.rank]
    for b, m in g.coupling.items():
        yh[bt.row[b]] = yh[bt.row[b]] + m @ xh[bt.col[b]]
    y = np.zeros(rows.npoints)
    for t in range(rows.nnodes):
        if rows.is_leaf(t):
            y[rows.index_range(t)] += g.row_basis.leaf_matrix[t] @ yh[t]
        else:
            for c in rows.children[t]:
                yh[c] = yh[c] + g.row_basis.transfer[c] @ yh[t]
    for b, m in g.nearfield.items():
        y[rows.index_range(bt.row[b])] += m @ x[cols.index_range(bt.col[b])]
    return y


def to_dense(g: H2Matrix, guard: int = DENSE_GUARD) -> np.ndarray:
    """Explicit dense matrix, guarded (reference h2.py:270-286)."""
    if max(g.shape) > guard:
        raise InvalidInputError(f"dense conversion of size {g.shape} refused (guard {guard})")
    bt = g.block_tree
    out = np.zeros(g.shape)
    for b, s in g.coupling.items():
        t, c = bt.row[b], bt.col[b]
        out[bt.rows.index_range(t), bt.cols.index_range(c)] += \
            g.row_basis.expand(t) @ s @ g.col_basis.expand(c).T
    for b, m in g.nearfield.items():
        out[bt.rows.index_range(bt.row[b]), bt.cols.index_range(bt.col[b])] += m
    return out
