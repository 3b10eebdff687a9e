"""NumPy restatement of the reference's adaptive H^2 product (oracle; test infrastructure).

Reference: /root/reference/pkg/src/h2mul/{dense,trees,h2,weights,induced,coarsening}.py.
Each function below names the reference lines it restates.  Data model:
dict-of-matrices keyed by cluster / block id, like the reference, so the
restatement stays close to the algorithm's text; the GPU path uses packed
arenas instead (see paper_2309_09061_b200/packed.py).

Conventions shared with the reference (dense.py:3-4): float64, row-major,
cluster and block ids in preorder with the root at 0.
"""

from __future__ import annotations

import time
from functools import reduce

import numpy as np

__all__ = [
    "OTree", "OBlocks", "OBasis", "OH2", "OCol",
    "o_qr_r", "o_full_qr", "o_tsvd", "o_norm2", "o_norms2",
    "o_basis_product", "o_basis_weights", "o_total_weights",
    "o_product_tree", "o_induced_rows", "o_induced_cols", "o_assemble",
    "o_multiply", "o_coverage", "o_coarse_rows", "o_coarse_cols", "o_coupling_norms", "o_nearfield_norms",
    "o_project_final", "o_coarsen", "o_orthogonalize", "o_recompress",
    "o_matvec", "o_matvec_t", "o_to_dense", "o_from_packed", "o_to_packed",
    "o_spectral_norm_est", "o_relative_spectral_error",
    "o_run_stages", "OracleError",
]

EPS64 = float(np.finfo(np.float64).eps)


class OracleError(RuntimeError):
    """Structural inconsistency seen by the oracle (reference StructureError)."""


# ----------------------------------------------------------------------------
# containers
# ----------------------------------------------------------------------------

class OTree:
    """Cluster-tree topology: preorder ids, contiguous [start, stop) ranges (trees.py:34-97)."""

    def __init__(self, start, stop, kids):
        self.start = np.asarray(start, dtype=np.int64)
        self.stop = np.asarray(stop, dtype=np.int64)
        self.kids = [tuple(int(c) for c in k) for k in kids]
        self.n = len(self.start)

    def size(self, t):
        return int(self.stop[t] - self.start[t])

    def leaf(self, t):
        return not self.kids[t]

    def same(self, other):
        return (self is other) or (self.n == other.n and np.array_equal(self.start, other.start)
                                   and np.array_equal(self.stop, other.stop) and self.kids == other.kids)


class OBlocks:
    """Block tree over (rows x cols) (trees.py:176-227); `adm` is True on admissible leaves."""

    def __init__(self, rows, cols, row, col, kids, adm):
        self.rows, self.cols = rows, cols
        self.row = [int(v) for v in row]
        self.col = [int(v) for v in col]
        self.kids = [tuple(int(c) for c in k) for k in kids]
        self.adm = [bool(a) for a in adm]
        self.index = {(self.row[b], self.col[b]): b for b in range(len(self.row))}
        self.nb = len(self.row)

    def leaf(self, b):
        return not self.kids[b]

    def adm_leaf(self, b):
        return not self.kids[b] and self.adm[b]

    def near_leaf(self, b):
        return not self.kids[b] and not self.adm[b]

    def T(self):
        return OBlocks(self.cols, self.rows, self.col, self.row, self.kids, self.adm)


class OBasis:
    """Nested cluster basis: leaf matrices + transfers (h2.py:32-72)."""

    def __init__(self, tree, rank, leaf, xfer):
        self.tree = tree
        self.rank = [int(k) for k in rank]
        self.leaf = leaf
        self.xfer = xfer

    def expand(self, t):
        if self.tree.leaf(t):
            return self.leaf[t]
        return np.vstack([self.expand(c) @ self.xfer[c] for c in self.tree.kids[t]])


class OH2:
    """Block tree + bases + couplings (adm leaves) + nearfield (inadm leaves) (h2.py:148-194)."""

    def __init__(self, bt, rb, cb, coup, near):
        self.bt, self.rb, self.cb, self.coup, self.near = bt, rb, cb, coup, near

    @property
    def shape(self):
        return (int(self.bt.rows.stop[0] - self.bt.rows.start[0]),
                int(self.bt.cols.stop[0] - self.bt.cols.start[0]))

    def T(self):
        """Transposed view, block ids kept (h2.py:169-173)."""
        return OH2(self.bt.T(), self.cb, self.rb,
                   {b: m.T for b, m in self.coup.items()},
                   {b: m.T for b, m in self.near.items()})


class OCol:
    """Column-tree node with an optional representation matrix (trees.py:362-406)."""

    __slots__ = ("cl", "kids", "adm", "mat")

    def __init__(self, cl, kids=(), adm=True, mat=None):
        self.cl, self.kids, self.adm, self.mat = cl, tuple(kids), adm, mat

    def leaves(self):
        if not self.kids:
            yield self
        else:
            for k in self.kids:
                yield from k.leaves()

    def shape_only(self):
        return OCol(self.cl, [k.shape_only() for k in self.kids], self.adm)


# ----------------------------------------------------------------------------
# dense kernels (dense.py)
# ----------------------------------------------------------------------------

def o_qr_r(m):
    """R factor only (dense.py:145-150): empty -> (min dim) x cols zeros."""
    m = np.asarray(m, dtype=np.float64)
    if min(m.shape) == 0:
        return np.zeros((min(m.shape), m.shape[1]))
    return np.linalg.qr(m, mode="r")


def o_full_qr(m):
    """Complete QR (dense.py:69-74): zero columns -> (I, zeros)."""
    if m.shape[1] == 0:
        return np.eye(m.shape[0]), np.zeros(m.shape)
    return np.linalg.qr(m, mode="complete")


def o_tsvd(m, tol, cap=None):
    """Truncated SVD with the reference rank rule (dense.py:77-101).

    thr = max(tol, max(rows, cols) * eps * sigma_1); k = #{sigma > thr};
    k = min(k, max(0, cap)).  Returns (u_k, sigma_k, v_k, k, sigma_all).
    """
    if tol < 0:
        raise ValueError("tolerance must be >= 0")
    if min(m.shape) == 0:
        return np.zeros((m.shape[0], 0)), np.zeros(0), np.zeros((m.shape[1], 0)), 0, np.zeros(0)
    u, s, vt = np.linalg.svd(m, full_matrices=False)
    thr = max(tol, max(m.shape) * EPS64 * s[0])
    k = int(np.count_nonzero(s > thr))
    if cap is not None:
        k = min(k, max(0, int(cap)))
    return np.ascontiguousarray(u[:, :k]), s[:k].copy(), np.ascontiguousarray(vt[:k].T), k, s


def o_norm2(m):
    """sigma_1 (dense.py:104-119): Gram eigvalsh on the short side if <= 64, else SVD."""
    if min(m.shape) == 0:
        return 0.0
    if min(m.shape) <= 64:
        g = m @ m.T if m.shape[0] <= m.shape[1] else m.T @ m
        return float(np.sqrt(max(np.linalg.eigvalsh(g)[-1], 0.0)))
    return float(np.linalg.svd(m, compute_uv=False)[0])


def o_norms2(mats):
    """Shape-batched sigma_1 (dense.py:122-142)."""
    mats = list(mats)
    out = [0.0] * len(mats)
    by_shape = {}
    for i, m in enumerate(mats):
        by_shape.setdefault(m.shape, []).append(i)
    for shp, ids in by_shape.items():
        if min(shp) == 0 or min(shp) > 64:
            for i in ids:
                out[i] = o_norm2(mats[i])
            continue
        st = np.stack([mats[i] for i in ids])
        g = st @ st.transpose(0, 2, 1) if shp[0] <= shp[1] else st.transpose(0, 2, 1) @ st
        top = np.linalg.eigvalsh(g)[:, -1]
        for i, v in zip(ids, top):
            out[i] = float(np.sqrt(max(v, 0.0)))
    return out


# ----------------------------------------------------------------------------
# basis products and weights (h2.py:127-145, weights.py:37-101)
# ----------------------------------------------------------------------------

def o_basis_product(wx, vy):
    """P_s = W_s^T V_s, bottom-up via transfers (h2.py:127-145)."""
    tr = wx.tree
    p = {}
    for s in reversed(range(tr.n)):  # children have larger preorder ids
        if tr.leaf(s):
            p[s] = wx.leaf[s].T @ vy.leaf[s]
        else:
            acc = np.zeros((wx.rank[s], vy.rank[s]))
            for c in tr.kids[s]:
                acc += wx.xfer[c].T @ p[c] @ vy.xfer[c]
            p[s] = acc
    return p


def o_basis_weights(w):
    """R_r of a bottom-up QR of the basis (weights.py:37-57)."""
    tr = w.tree
    r = {}
    for c in reversed(range(tr.n)):
        if tr.leaf(c):
            r[c] = o_qr_r(w.leaf[c])
        else:
            r[c] = o_qr_r(np.vstack([r[k] @ w.xfer[k] for k in tr.kids[c]]))
    return r


def o_total_weights(h, rw, scaling=True):
    """Top-down condensed weights Z_s (weights.py:60-101)."""
    bt = h.bt
    tr = bt.rows
    by_row = {s: [] for s in range(tr.n)}
    for b in range(bt.nb):
        if bt.adm_leaf(b):
            by_row[bt.row[b]].append(b)
    z = {}
    parent = _parents(tr)
    for s in range(tr.n):  # preorder: parent before child
        parts = []
        if parent[s] >= 0:
            parts.append(z[parent[s]] @ h.rb.xfer[s].T)
        for b in by_row[s]:
            blk = rw[bt.col[b]] @ h.coup[b].T
            if scaling:
                nrm = o_norm2(blk)
                if nrm == 0.0:
                    continue
                blk = blk / nrm
            parts.append(blk)
        st = np.vstack(parts) if parts else np.zeros((0, h.rb.rank[s]))
        z[s] = o_qr_r(st)
    return z


def _parents(tr):
    par = [-1] * tr.n
    for t in range(tr.n):
        for c in tr.kids[t]:
            par[c] = t
    return par


def _depths(tr):
    d = [0] * tr.n
    for t in range(tr.n):
        for c in tr.kids[t]:
            d[c] = d[t] + 1
    return d


# ----------------------------------------------------------------------------
# product block tree (trees.py:288-359)
# ----------------------------------------------------------------------------

def _kind(bx, by, t, s, r):
    """Triple kind a > b > c > n (trees.py:288-300)."""
    bts = bx.index.get((t, s))
    bsr = by.index.get((s, r))
    if bts is None or bsr is None:
        raise OracleError(f"triple ({t},{s},{r}) not covered")
    if by.adm_leaf(bsr):
        return "a"
    if bx.adm_leaf(bts):
        return "b"
    if bx.leaf(bts) and by.leaf(bsr):
        return "c"
    return "n"


def _submid(bx, by, mid, t, s, r):
    """trees.py:303-311."""
    if (not bx.leaf(bx.index[(t, s)]) and not by.leaf(by.index[(s, r)]) and mid.kids[s]):
        return mid.kids[s]
    return (s,)


def _kid_pairs(rows, cols, t, r):
    return [(a, b) for a in (rows.kids[t] or (t,)) for b in (cols.kids[r] or (r,))]


def o_product_tree(bx, by):
    """T^XY (trees.py:314-359)."""
    if not bx.cols.same(by.rows):
        raise ValueError("factors do not share the middle cluster tree")
    rows, cols, mid = bx.rows, by.cols, bx.cols
    row, col, kids, adm = [], [], [], []

    def visit(t, r, middles):
        b = len(row)
        row.append(t); col.append(r); kids.append(()); adm.append(True)
        pending = list(middles)
        open_mid = []
        dense = False
        while pending:
            s = pending.pop()
            k = _kind(bx, by, t, s, r)
            if k == "c":
                dense = True
            elif k == "n":
                if rows.leaf(t) and cols.leaf(r):
                    pending.extend(mid.kids[s])
                else:
                    open_mid.append(s)
        if open_mid:
            subs = [q for s in open_mid for q in _submid(bx, by, mid, t, s, r)]
            kids[b] = tuple(visit(t2, r2, subs) for t2, r2 in _kid_pairs(rows, cols, t, r))
        elif dense:
            adm[b] = False
        return b

    visit(0, 0, [0])
    return OBlocks(rows, cols, row, col, kids, adm)


# ----------------------------------------------------------------------------
# phase 1 (induced.py)
# ----------------------------------------------------------------------------

def _xv(x, y, pxy, t, s):
    """X|ts V_Y,s for a leaf row cluster t by block descent (induced.py:59-73)."""
    bx = x.bt
    b = bx.index[(t, s)]
    if bx.adm_leaf(b):
        return x.rb.leaf[t] @ x.coup[b] @ pxy[s]
    if bx.leaf(b):
        return x.near[b] @ y.rb.leaf[s]
    acc = np.zeros((bx.rows.size(t), y.rb.rank[s]))
    for b2 in bx.kids[b]:
        s2 = bx.col[b2]
        part = _xv(x, y, pxy, t, s2)
        acc += part @ y.rb.xfer[s2] if s2 != s else part
    return acc


class OInduced:
    """Compressed induced basis result (induced.py:33-46)."""

    def __init__(self, q, bc, proj):
        self.q, self.bc, self.proj = q, bc, proj


def o_induced_rows(x, y, zy, pxy, tol, max_rank=None, scale_blocks=True, level_decay=1.0):
    """Fig. 3 bottom-up compression of the induced row basis (induced.py:76-184)."""
    bx = x.bt
    if not bx.cols.same(y.bt.rows):
        raise ValueError("x and y do not share the middle cluster tree")
    tr = bx.rows
    vx, vy = x.rb, y.rb
    mids_of = {t: [] for t in range(tr.n)}       # induced.py:49-56
    for b in range(bx.nb):
        if not bx.adm_leaf(b):
            mids_of[bx.row[b]].append(bx.col[b])
    depth = _depths(tr)
    rank = [0] * tr.n
    leaf_q, xfer_q, bc, proj = {}, {}, {}, {}
    svals = {}

    def compress(t, vx_t, blocks, middles, is_leaf):     # induced.py:115-146
        m = vx_t.shape[0]
        cols = []
        for s, blk in zip(middles, blocks):
            w = blk @ zy[s].T
            if scale_blocks:
                nrm = o_norm2(blk)
                if nrm == 0.0:
                    continue
                w = w / nrm
            cols.append(w)
        stacked = np.hstack(cols) if cols else np.zeros((m, 0))
        qf, rf = o_full_qr(vx_t)
        k1 = min(vx_t.shape)
        rem = qf[:, k1:].T @ stacked
        cap = None if max_rank is None else max(0, max_rank - k1)
        u, _, _, k2, sv = o_tsvd(rem, tol * level_decay ** depth[t], cap)
        svals[t] = (sv, max(rem.shape) if min(rem.shape) else 0)
        q_t = np.hstack([qf[:, :k1], qf[:, k1:] @ u])
        rank[t] = k1 + k2
        bc[t] = np.vstack([rf[:k1], np.zeros((k2, vx_t.shape[1]))])
        for s, blk in zip(middles, blocks):
            proj[(t, s)] = q_t.T @ blk
        if is_leaf:
            leaf_q[t] = q_t
        else:
            off = 0
            for c in tr.kids[t]:
                xfer_q[c] = q_t[off:off + rank[c]]
                off += rank[c]

    def proj_block(t2, s2):                               # induced.py:148-153
        b2 = bx.index[(t2, s2)]
        if bx.adm_leaf(b2):
            return bc[t2] @ x.coup[b2] @ pxy[s2]
        return proj[(t2, s2)]

    def ahat(t, s):                                       # induced.py:155-167
        b = bx.index[(t, s)]
        acc = np.zeros((sum(rank[c] for c in tr.kids[t]), vy.rank[s]))
        grouped = {}
        for b2 in bx.kids[b]:
            grouped.setdefault(bx.col[b2], []).append(proj_block(bx.row[b2], bx.col[b2]))
        for s2, parts in grouped.items():
            blk = np.vstack(parts)
            acc += blk @ vy.xfer[s2] if s2 != s else blk
        return acc

    # bottom-up in reverse preorder == children before parents (induced.py:169-180)
    for t in reversed(range(tr.n)):
        middles = mids_of[t]
        if tr.leaf(t):
            compress(t, vx.leaf[t], [_xv(x, y, pxy, t, s) for s in middles], middles, True)
        else:
            vhat = np.vstack([bc[c] @ vx.xfer[c] for c in tr.kids[t]])
            compress(t, vhat, [ahat(t, s) for s in middles], middles, False)
    res = OInduced(OBasis(tr, rank, leaf_q, xfer_q), bc, proj)
    res.svals = svals
    return res


def o_induced_cols(x, y, zxt, pxy, tol, **kw):
    """Row algorithm on Y^T X^T (induced.py:187-200)."""
    return o_induced_rows(y.T(), x.T(), zxt, {s: m.T for s, m in pxy.items()}, tol, **kw)


def _wyl(x, y, pxy, s, r):
    """Y|sr^T W_X,s for a leaf column cluster r (induced.py:203-217)."""
    by = y.bt
    b = by.index[(s, r)]
    if by.adm_leaf(b):
        return y.cb.leaf[r] @ y.coup[b].T @ pxy[s].T
    if by.leaf(b):
        return y.near[b].T @ x.cb.leaf[s]
    acc = np.zeros((by.cols.size(r), x.cb.rank[s]))
    for b2 in by.kids[b]:
        s2 = by.row[b2]
        part = _wyl(x, y, pxy, s2, r)
        acc += part @ x.cb.xfer[s2] if s2 != s else part
    return acc


def o_assemble(x, y, qrow, qcol, pxy, pt=None):
    """Product over T^XY in the induced bases + push-down (induced.py:220-355)."""
    bx, by = x.bt, y.bt
    if not bx.cols.same(by.rows):
        raise ValueError("x and y do not share the middle cluster tree")
    if pt is None:
        pt = o_product_tree(bx, by)
    rows, mid, cols = bx.rows, bx.cols, by.cols
    vx, wy = x.rb, y.cb
    qr_, qc_ = qrow.q, qcol.q
    coup, near = {}, {}
    xv_memo, wy_memo = {}, {}

    def xv(t, s):
        if (t, s) not in xv_memo:
            xv_memo[(t, s)] = _xv(x, y, pxy, t, s)
        return xv_memo[(t, s)]

    def wyl(s, r):
        if (s, r) not in wy_memo:
            wy_memo[(s, r)] = _wyl(x, y, pxy, s, r)
        return wy_memo[(s, r)]

    def rowf(t, s):
        b = bx.index[(t, s)]
        if bx.adm_leaf(b):
            return qrow.bc[t] @ x.coup[b] @ pxy[s]
        return qrow.proj[(t, s)]

    def colf(r, s):
        b = by.index[(s, r)]
        if by.adm_leaf(b):
            return qcol.bc[r] @ y.coup[b].T @ pxy[s].T
        return qcol.proj[(r, s)]

    def acc(store, key, val):
        store[key] = store[key] + val if key in store else val

    def visit(node, middles):
        t, r = pt.row[node], pt.col[node]
        is_leaf = pt.leaf(node)
        dense = is_leaf and not pt.adm[node]
        pending = list(middles)
        open_mid = []
        while pending:
            s = pending.pop()
            k = _kind(bx, by, t, s, r)
            if k == "a":
                sy = y.coup[by.index[(s, r)]]
                if dense:
                    acc(near, node, xv(t, s) @ sy @ wy.leaf[r].T)
                else:
                    acc(coup, node, rowf(t, s) @ sy @ qcol.bc[r].T)
            elif k == "b":
                sx = x.coup[bx.index[(t, s)]]
                if dense:
                    acc(near, node, vx.leaf[t] @ sx @ wyl(s, r).T)
                else:
                    acc(coup, node, qrow.bc[t] @ sx @ colf(r, s).T)
            elif k == "c":
                acc(near, node, x.near[bx.index[(t, s)]] @ y.near[by.index[(s, r)]])
            elif is_leaf:
                pending.extend(mid.kids[s])
            else:
                open_mid.append(s)
        if open_mid:
            subs = [q for s in open_mid for q in _submid(bx, by, mid, t, s, r)]
            for ch in pt.kids[node]:
                visit(ch, subs)
        elif not is_leaf:
            for ch in pt.kids[node]:
                visit(ch, [])

    visit(0, [0])

    for node in range(pt.nb):                             # induced.py:329-344
        if pt.leaf(node) or node not in coup:
            continue
        s_tr = coup.pop(node)
        t, r = pt.row[node], pt.col[node]
        for ch in pt.kids[node]:
            t2, r2 = pt.row[ch], pt.col[ch]
            part = qr_.xfer[t2] @ s_tr if t2 != t else s_tr
            part = part @ qc_.xfer[r2].T if r2 != r else part
            if pt.near_leaf(ch):
                acc(near, ch, qr_.leaf[t2] @ part @ qc_.leaf[r2].T)
            else:
                acc(coup, ch, part)
    for node in range(pt.nb):                             # induced.py:346-353
        if pt.adm_leaf(node) and node not in coup:
            coup[node] = np.zeros((qr_.rank[pt.row[node]], qc_.rank[pt.col[node]]))
        if pt.near_leaf(node) and node not in near:
            near[node] = np.zeros((rows.size(pt.row[node]), cols.size(pt.col[node])))
    return OH2(pt, qr_, qc_, coup, near)


def o_multiply(x, y, tol, max_rank=None, scaling=True):
    """Phase-1 driver (induced.py:358-372)."""
    pxy = o_basis_product(x.cb, y.rb)
    zy = o_total_weights(y, o_basis_weights(y.cb), scaling)
    zxt = o_total_weights(x.T(), o_basis_weights(x.rb), scaling)
    qrow = o_induced_rows(x, y, zy, pxy, tol, max_rank=max_rank, scale_blocks=scaling)
    qcol = o_induced_cols(x, y, zxt, pxy, tol, max_rank=max_rank, scale_blocks=scaling)
    return o_assemble(x, y, qrow, qcol, pxy)


# ----------------------------------------------------------------------------
# phase 2 (coarsening.py)
# ----------------------------------------------------------------------------

def _union(a, b):
    """Structure-only union of two column trees (coarsening.py:89-105)."""
    if a is None:
        return b.shape_only()
    if b is None:
        return a.shape_only()
    if a.cl != b.cl:
        raise OracleError("column trees rooted at different clusters")
    if a.kids and b.kids:
        return OCol(a.cl, [_union(p, q) for p, q in zip(a.kids, b.kids)])
    if a.kids:
        return a.shape_only()
    if b.kids:
        return b.shape_only()
    return OCol(a.cl, adm=a.adm and b.adm)


def _match(ct, target, w):
    """Refine a representation to the target structure (coarsening.py:108-136)."""
    if ct.cl != target.cl:
        raise ValueError("representation and target roots differ")
    if ct.kids:
        if not target.kids:
            return ct
        return OCol(ct.cl, [_match(c, tc, w) for c, tc in zip(ct.kids, target.kids)], ct.adm, ct.mat)
    if target.kids:
        out = []
        for tc in target.kids:
            out.append(_match(OCol(tc.cl, (), True, ct.mat @ w.xfer[tc.cl].T), tc, w))
        return OCol(ct.cl, out, True)
    if ct.adm and not target.adm:
        return OCol(ct.cl, (), False, ct.mat @ w.leaf[ct.cl].T)
    return ct


def _stack(reps):
    """coarsening.py:139-146."""
    f = reps[0]
    if f.kids:
        return OCol(f.cl, [_stack([r.kids[i] for r in reps]) for i in range(len(f.kids))], f.adm)
    return OCol(f.cl, (), f.adm, np.vstack([r.mat for r in reps]))


def _mapm(ct, fn):
    """coarsening.py:149-153."""
    if not ct.kids:
        return OCol(ct.cl, (), ct.adm, fn(ct.mat))
    return OCol(ct.cl, [_mapm(c, fn) for c in ct.kids], ct.adm)


def _flat(ct):
    """coarsening.py:156-157."""
    return np.hstack([lf.mat for lf in ct.leaves()])


def _check_coarse(pt, coarse):
    """coarsening.py:160-168."""
    if not (pt.rows.same(coarse.rows) and pt.cols.same(coarse.cols)):
        raise ValueError("coarse tree lives on different cluster trees")
    for b in range(coarse.nb):
        if (coarse.row[b], coarse.col[b]) not in pt.index:
            raise ValueError("coarse block finer than the product tree")


def o_coverage(pt, coarse):
    """cov[pb]: an ancestor-or-self coarse leaf is admissible (coarsening.py:171-184)."""
    cov = [False] * pt.nb
    stack = [(0, 0, None)]
    while stack:
        pb, cb, state = stack.pop()
        if state is None and cb is not None and coarse.leaf(cb):
            state = coarse.adm[cb]
        cov[pb] = state is True
        for ch in pt.kids[pb]:
            key = (pt.row[ch], pt.col[ch])
            stack.append((ch, coarse.index.get(key) if state is None else None, state))
    return cov


class OCoarse:
    """Coarse-basis state (coarsening.py:36-50)."""

    def __init__(self, q, r, z, reps):
        self.q, self.r, self.z, self.reps = q, r, z, reps


def o_coupling_norms(g):
    keys = list(g.coup)
    return dict(zip(keys, o_norms2([g.coup[b] for b in keys])))


def o_nearfield_norms(g):
    keys = list(g.near)
    return dict(zip(keys, o_norms2([g.near[b] for b in keys])))


def o_coarse_rows(g, coarse, tol, max_rank=None, scale_blocks=True, cnorms=None, nnorms=None):
    """Fig. 5 adaptive coarse row basis (coarsening.py:187-332)."""
    pt = g.bt
    _check_coarse(pt, coarse)
    cov = o_coverage(pt, coarse)
    tr = pt.rows
    v1, w1 = g.rb, g.cb
    adm_of = {t: [] for t in range(tr.n)}
    near_of = {t: [] for t in range(tr.n)}
    sub_of = {t: [] for t in range(tr.n)}
    for b in range(pt.nb):
        t = pt.row[b]
        if pt.adm_leaf(b):
            adm_of[t].append(b)
        elif pt.near_leaf(b):
            if cov[b]:
                near_of[t].append(b)
        elif cov[b]:
            sub_of[t].append(b)
    if scale_blocks and cnorms is None:
        cnorms = o_coupling_norms(g)
    if scale_blocks and nnorms is None:
        nnorms = o_nearfield_norms(g)
    rank = [0] * tr.n
    leaf_q, xfer_q, rmap, zmap, reps = {}, {}, {}, {}, {}
    svals = {}
    parent = _parents(tr)

    def zstep(t):                                         # coarsening.py:231-245
        parts = []
        zp = zmap[parent[t]] if parent[t] >= 0 else None
        if zp is not None and zp.shape[0] > 0:
            parts.append(zp @ v1.xfer[t].T)
        for b in adm_of[t]:
            blk = g.coup[b].T
            if scale_blocks:
                nrm = cnorms[b]
                if nrm == 0.0:
                    continue
                blk = blk / nrm
            parts.append(blk)
        if not parts:
            return np.zeros((0, v1.rank[t]))
        return o_qr_r(np.vstack(parts))

    def scaled(m, nrm=None):                              # coarsening.py:247-252
        if not scale_blocks:
            return m
        if nrm is None:
            nrm = o_norm2(m)
        return m / nrm if nrm > 0.0 else m

    def child_rep(b):                                     # coarsening.py:254-258
        if pt.adm_leaf(b):
            return OCol(pt.col[b], (), True, rmap[pt.row[b]] @ g.coup[b])
        return reps[b]

    def merged_rep(b):                                    # coarsening.py:260-279
        groups, order = {}, []
        for b2 in pt.kids[b]:
            r2 = pt.col[b2]
            if r2 not in groups:
                groups[r2] = []
                order.append(r2)
            groups[r2].append(child_rep(b2))
        merged = {}
        for r2 in order:
            parts = groups[r2]
            target = reduce(_union, parts, None)
            merged[r2] = _stack([_match(p, target, w1) for p in parts])
        r = pt.col[b]
        if order == [r]:
            return merged[r]
        return OCol(r, [merged[r2] for r2 in order], True)

    def leaf_rep(b, t):                                   # coarsening.py:281-290
        if pt.adm_leaf(b):
            return OCol(pt.col[b], (), True, rmap[t] @ g.coup[b])
        if pt.near_leaf(b):
            return reps[b]
        rep = OCol(pt.col[b], [leaf_rep(b2, t) for b2 in pt.kids[b]], True)
        reps[b] = rep
        return rep

    for t in range(tr.n):                                 # top-down Z (preorder)
        zmap[t] = zstep(t)
    for t in reversed(range(tr.n)):                       # bottom-up bases (coarsening.py:292-328)
        if tr.leaf(t):
            vl = v1.leaf[t]
            cols = [vl @ zmap[t].T]
            cols += [scaled(g.near[b], nnorms[b] if scale_blocks else None) for b in near_of[t]]
            st = np.hstack(cols)
            u, _, _, k, sv = o_tsvd(st, tol, max_rank)
            svals[t] = (sv, max(st.shape) if min(st.shape) else 0)
            rank[t] = k
            leaf_q[t] = u
            rmap[t] = u.T @ vl
            for b in near_of[t]:
                reps[b] = OCol(pt.col[b], (), False, u.T @ g.near[b])
            for b in sub_of[t]:
                leaf_rep(b, t)
        else:
            vhat = np.vstack([rmap[c] @ v1.xfer[c] for c in tr.kids[t]])
            merged = [merged_rep(b) for b in sub_of[t]]
            cols = [vhat @ zmap[t].T] + [scaled(_flat(rep)) for rep in merged]
            st = np.hstack(cols)
            u, _, _, k, sv = o_tsvd(st, tol, max_rank)
            svals[t] = (sv, max(st.shape) if min(st.shape) else 0)
            rank[t] = k
            off = 0
            for c in tr.kids[t]:
                xfer_q[c] = u[off:off + rank[c]]
                off += rank[c]
            rmap[t] = u.T @ vhat
            for b, rep in zip(sub_of[t], merged):
                reps[b] = _mapm(rep, lambda m, u=u: u.T @ m)
    st = OCoarse(OBasis(tr, rank, leaf_q, xfer_q), rmap, zmap, reps)
    st.svals = svals
    return st


def o_coarse_cols(g, coarse, tol, **kw):
    """coarsening.py:335-339."""
    return o_coarse_rows(g.T(), coarse.T(), tol, **kw)


def o_project_final(g, rs, cs, coarse):
    """Final projection onto the coarse tree (coarsening.py:354-405)."""
    pt = g.bt
    _check_coarse(pt, coarse)
    qr_, qc_ = rs.q, cs.q

    def row_rep(b):
        if pt.adm_leaf(b):
            return OCol(pt.col[b], (), True, rs.r[pt.row[b]] @ g.coup[b])
        return rs.reps[b]

    def lift(node, chain, out):
        if not node.kids:
            if node.adm:
                out += node.mat @ cs.r[node.cl].T @ chain
            else:
                out += node.mat @ qc_.leaf[node.cl] @ chain
            return
        for c in node.kids:
            lift(c, qc_.xfer[c.cl] @ chain, out)

    coup, near = {}, {}
    for b in range(coarse.nb):
        if not coarse.leaf(b):
            continue
        t, r = coarse.row[b], coarse.col[b]
        pb = pt.index[(t, r)]
        if coarse.adm[b]:
            s = np.zeros((qr_.rank[t], qc_.rank[r]))
            lift(row_rep(pb), np.eye(qc_.rank[r]), s)
            coup[b] = s
        elif pt.near_leaf(pb):
            near[b] = g.near[pb].copy()
        elif pt.adm_leaf(pb):
            near[b] = g.rb.leaf[t] @ g.coup[pb] @ g.cb.leaf[r].T
        else:
            raise OracleError("inadmissible coarse leaf is subdivided in the product tree")
    return OH2(coarse, qr_, qc_, coup, near)


def o_coarsen(g, coarse, tol, max_rank=None, scale_blocks=True):
    """Phase-2 driver (coarsening.py:408-422)."""
    cn = o_coupling_norms(g) if scale_blocks else None
    nn = o_nearfield_norms(g) if scale_blocks else None
    rs = o_coarse_rows(g, coarse, tol, max_rank=max_rank, scale_blocks=scale_blocks, cnorms=cn, nnorms=nn)
    cs = o_coarse_cols(g, coarse, tol, max_rank=max_rank, scale_blocks=scale_blocks, cnorms=cn, nnorms=nn)
    return o_project_final(g, rs, cs, coarse)


def o_orthogonalize(basis):
    """Isometric re-factorisation, exact-zero directions dropped (h2.py:79-113)."""
    tr = basis.tree
    rank = [0] * tr.n
    leaf, xfer, rmap = {}, {}, {}
    for t in reversed(range(tr.n)):
        if tr.leaf(t):
            st = basis.leaf[t]
        else:
            st = np.vstack([rmap[c] @ basis.xfer[c] for c in tr.kids[t]])
        u, s, v, k, _ = o_tsvd(st, 0.0)
        rmap[t] = s[:, None] * v.T
        rank[t] = k
        if tr.leaf(t):
            leaf[t] = u
        else:
            off = 0
            for c in tr.kids[t]:
                xfer[c] = u[off:off + rank[c]]
                off += rank[c]
    return OBasis(tr, rank, leaf, xfer), rmap


def o_recompress(g, tol, max_rank=None):
    """Input preparation: orthogonalise, then coarsen onto the own tree (coarsening.py:425-445)."""
    qr_, rr = o_orthogonalize(g.rb)
    qc_, rc = o_orthogonalize(g.cb)
    bt = g.bt
    coup = {b: rr[bt.row[b]] @ s @ rc[bt.col[b]].T for b, s in g.coup.items()}
    return o_coarsen(OH2(bt, qr_, qc_, coup, g.near), bt, tol, max_rank=max_rank)


# ----------------------------------------------------------------------------
# verification kernels (h2.py:197-286)
# ----------------------------------------------------------------------------

def _fwd(basis, x):
    tr = basis.tree
    out = [None] * tr.n
    for s in reversed(range(tr.n)):
        if tr.leaf(s):
            out[s] = basis.leaf[s].T @ x[tr.start[s]:tr.stop[s]]
        else:
            acc = np.zeros(basis.rank[s])
            for c in tr.kids[s]:
                acc += basis.xfer[c].T @ out[c]
            out[s] = acc
    return out


def _bwd(basis, yhat, y):
    tr = basis.tree
    for t in range(tr.n):
        if tr.leaf(t):
            y[tr.start[t]:tr.stop[t]] += basis.leaf[t] @ yhat[t]
        else:
            for c in tr.kids[t]:
                yhat[c] = yhat[c] + basis.xfer[c] @ yhat[t]


def o_matvec(g, x):
    """y = G x (h2.py:224-244)."""
    bt = g.bt
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros(g.shape[0])
    xh = _fwd(g.cb, x)
    yh = [np.zeros(k) for k in g.rb.rank]
    for b, s in g.coup.items():
        yh[bt.row[b]] = yh[bt.row[b]] + s @ xh[bt.col[b]]
    _bwd(g.rb, yh, y)
    for b, m in g.near.items():
        t, s = bt.row[b], bt.col[b]
        y[bt.rows.start[t]:bt.rows.stop[t]] += m @ x[bt.cols.start[s]:bt.cols.stop[s]]
    return y


def o_matvec_t(g, x):
    """y = G^T x (h2.py:247-267)."""
    return o_matvec(g.T(), x)


def o_spectral_norm_est(apply, apply_t, dim, steps, rng):
    """Power iteration on A^T A, sigma_1 estimate |A v| (bench.py:126-144)."""
    v = rng.standard_normal(dim)
    nv = np.linalg.norm(v)
    if nv == 0 or dim == 0:
        return 0.0
    v = v / nv
    sigma = 0.0
    for _ in range(steps):
        w = apply(v)
        sigma = float(np.linalg.norm(w))
        if sigma == 0.0:
            return 0.0
        v = apply_t(w)
        nv = float(np.linalg.norm(v))
        if nv == 0.0:
            return sigma
        v = v / nv
    return sigma


def o_relative_spectral_error(x, y, g, steps=20, seed=0):
    """|XY - G|_2 / |XY|_2 by the same power iteration for both norms (bench.py:147-174)."""
    rng = np.random.default_rng(seed)
    n_k = y.shape[1]

    def xy(v):
        return o_matvec(x, o_matvec(y, v))

    def xy_t(v):
        return o_matvec_t(y, o_matvec_t(x, v))

    denom = o_spectral_norm_est(xy, xy_t, n_k, steps, rng)
    numer = o_spectral_norm_est(lambda v: xy(v) - o_matvec(g, v), lambda v: xy_t(v) - o_matvec_t(g, v),
                                n_k, steps, rng)
    if denom == 0.0:
        return 0.0 if numer == 0.0 else float("inf")
    return numer / denom


def o_to_dense(g):
    """Explicit dense matrix (h2.py:270-286), small instances only."""
    bt = g.bt
    out = np.zeros(g.shape)
    for b, s in g.coup.items():
        t, c = bt.row[b], bt.col[b]
        out[bt.rows.start[t]:bt.rows.stop[t], bt.cols.start[c]:bt.cols.stop[c]] += \
            g.rb.expand(t) @ s @ g.cb.expand(c).T
    for b, m in g.near.items():
        t, c = bt.row[b], bt.col[b]
        out[bt.rows.start[t]:bt.rows.stop[t], bt.cols.start[c]:bt.cols.stop[c]] += m
    return out


# ----------------------------------------------------------------------------
# packed interchange format (shared with the GPU path and the golden fixtures)
# ----------------------------------------------------------------------------

def _tree_from(d, p):
    ptr, idx = d[p + "child_ptr"], d[p + "child_idx"]
    kids = [tuple(idx[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)]
    return OTree(d[p + "start"], d[p + "stop"], kids)


def _basis_from(d, p, tree):
    rank = [int(v) for v in d[p + "rank"]]
    data = d[p + "data"]
    loff, xoff = d[p + "leaf_off"], d[p + "xfer_off"]
    par = _parents(tree)
    leaf, xfer = {}, {}
    for t in range(tree.n):
        if tree.leaf(t):
            n = tree.size(t) * rank[t]
            leaf[t] = data[loff[t]:loff[t] + n].reshape(tree.size(t), rank[t])
        if par[t] >= 0:
            n = rank[t] * rank[par[t]]
            xfer[t] = data[xoff[t]:xoff[t] + n].reshape(rank[t], rank[par[t]])
    return OBasis(tree, rank, leaf, xfer)


def o_from_packed(d, prefix="", rows=None, cols=None):
    """Build an oracle H^2 matrix from the packed npz layout (see paper_2309_09061_b200/packed.py)."""
    p = prefix
    rows = rows if rows is not None else _tree_from(d, p + "rows.")
    cols = cols if cols is not None else _tree_from(d, p + "cols.")
    ptr, idx = d[p + "bt.child_ptr"], d[p + "bt.child_idx"]
    kids = [tuple(idx[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)]
    bt = OBlocks(rows, cols, d[p + "bt.row"], d[p + "bt.col"], kids, d[p + "bt.adm"].astype(bool))
    rb = _basis_from(d, p + "rb.", rows)
    cb = _basis_from(d, p + "cb.", cols)
    coup, near = {}, {}
    coff, noff = d[p + "coup_off"], d[p + "near_off"]
    cdat, ndat = d[p + "coup_data"], d[p + "near_data"]
    for b in range(bt.nb):
        t, s = bt.row[b], bt.col[b]
        if bt.adm_leaf(b):
            n = rb.rank[t] * cb.rank[s]
            coup[b] = cdat[coff[b]:coff[b] + n].reshape(rb.rank[t], cb.rank[s])
        elif bt.near_leaf(b):
            n = rows.size(t) * cols.size(s)
            near[b] = ndat[noff[b]:noff[b] + n].reshape(rows.size(t), cols.size(s))
    return OH2(bt, rb, cb, coup, near)


def _tree_to(tree, p, out):
    out[p + "start"] = np.asarray(tree.start, dtype=np.int64)
    out[p + "stop"] = np.asarray(tree.stop, dtype=np.int64)
    lens = [len(k) for k in tree.kids]
    out[p + "child_ptr"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out[p + "child_idx"] = np.asarray([c for k in tree.kids for c in k], dtype=np.int64)


def _basis_to(basis, p, out):
    tr = basis.tree
    par = _parents(tr)
    chunks, loff, xoff, pos = [], np.full(tr.n, -1, np.int64), np.full(tr.n, -1, np.int64), 0
    for t in range(tr.n):
        if tr.leaf(t):
            m = np.ascontiguousarray(basis.leaf[t], dtype=np.float64)
            loff[t] = pos; chunks.append(m.ravel()); pos += m.size
    for t in range(tr.n):
        if par[t] >= 0:
            m = np.ascontiguousarray(basis.xfer[t], dtype=np.float64)
            xoff[t] = pos; chunks.append(m.ravel()); pos += m.size
    out[p + "rank"] = np.asarray(basis.rank, dtype=np.int64)
    out[p + "leaf_off"], out[p + "xfer_off"] = loff, xoff
    out[p + "data"] = np.concatenate(chunks) if chunks else np.zeros(0)


def o_to_packed(g, prefix=""):
    """Inverse of o_from_packed."""
    out = {}
    p = prefix
    _tree_to(g.bt.rows, p + "rows.", out)
    _tree_to(g.bt.cols, p + "cols.", out)
    bt = g.bt
    out[p + "bt.row"] = np.asarray(bt.row, dtype=np.int64)
    out[p + "bt.col"] = np.asarray(bt.col, dtype=np.int64)
    lens = [len(k) for k in bt.kids]
    out[p + "bt.child_ptr"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out[p + "bt.child_idx"] = np.asarray([c for k in bt.kids for c in k], dtype=np.int64)
    out[p + "bt.adm"] = np.asarray(bt.adm, dtype=np.uint8)
    _basis_to(g.rb, p + "rb.", out)
    _basis_to(g.cb, p + "cb.", out)
    for name, store in (("coup", g.coup), ("near", g.near)):
        off = np.full(bt.nb, -1, np.int64)
        chunks, pos = [], 0
        for b in range(bt.nb):
            if b in store:
                m = np.ascontiguousarray(store[b], dtype=np.float64)
                off[b] = pos; chunks.append(m.ravel()); pos += m.size
        out[p + name + "_off"] = off
        out[p + name + "_data"] = np.concatenate(chunks) if chunks else np.zeros(0)
    return out


# ----------------------------------------------------------------------------
# stage runner mirroring the reference harness (bench.py:195-237)
# ----------------------------------------------------------------------------

def o_run_stages(x, y, coarse, tol, max_rank=None):
    """Run the product stage by stage with wall-clock timers (bench.py:201-237).

    Returns (final, induced, times) where times holds t_setup, t1_row, t1_col,
    t1_mat, t2_row, t2_col, t2_mat and t_total (bench.py:265).
    """
    tm = {}
    c0 = time.perf_counter()
    pxy = o_basis_product(x.cb, y.rb)
    zy = o_total_weights(y, o_basis_weights(y.cb))
    zxt = o_total_weights(x.T(), o_basis_weights(x.rb))
    tm["t_setup"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    qrow = o_induced_rows(x, y, zy, pxy, tol, max_rank=max_rank)
    tm["t1_row"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    qcol = o_induced_cols(x, y, zxt, pxy, tol, max_rank=max_rank)
    tm["t1_col"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    pt = o_product_tree(x.bt, y.bt)
    induced = o_assemble(x, y, qrow, qcol, pxy, pt)
    tm["t1_mat"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    cn = o_coupling_norms(induced)
    nn = o_nearfield_norms(induced)
    rs = o_coarse_rows(induced, coarse, tol, max_rank=max_rank, cnorms=cn, nnorms=nn)
    tm["t2_row"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    cs = o_coarse_cols(induced, coarse, tol, max_rank=max_rank, cnorms=cn, nnorms=nn)
    tm["t2_col"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    final = o_project_final(induced, rs, cs, coarse)
    tm["t2_mat"] = time.perf_counter() - c0
    tm["t_total"] = sum(tm[k] for k in ("t1_row", "t1_col", "t1_mat", "t2_row", "t2_col", "t2_mat"))
    info = {"qrow": qrow, "qcol": qcol, "rows": rs, "cols": cs}
    return final, induced, tm, info
