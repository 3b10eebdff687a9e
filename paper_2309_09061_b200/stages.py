"""Stage-level drop-ins: the reference's stage functions one call at a time, on the GPU.

The reference harness times the product stage by stage (h2mul/bench.py:195-237) and the package
exports every stage (h2mul/__init__.py:11-32).  Each function here has the reference's name,
positional arguments and keyword arguments, runs its stage through the C ABI
(include/h2g.h, "Stage-level entry points") and returns a device-resident result with the
reference container's attribute names:

  cluster_basis_product(wx, vy)                        h2.py:127-145      -> BasisProduct (.p)
  basis_weights(w)                                     weights.py:37-57   -> BasisWeights (.r)
  total_weights(y, rw, scaling=True)                   weights.py:60-101  -> TotalWeights (.z)
  compress_induced_row_basis(x, y, zy, pxy, tol, *, max_rank=None, scale_blocks=True,
                             level_decay=1.0)          induced.py:76-184  -> InducedBasisResult
  compress_induced_col_basis(x, y, zx_adjoint, pxy, tol, **kw)  induced.py:187-200
  assemble_product(x, y, qrow, qcol, pxy, product_tree=None)   induced.py:220-355 -> DeviceH2
  coupling_norms(g) / nearfield_norms(g)               coarsening.py:342-351 (_coupling_norms ...)
  build_coarse_row_basis(g, coarse, tol, *, max_rank=None, scale_blocks=True,
                         coupling_norms=None, nearfield_norms=None)  coarsening.py:187-332
  build_coarse_col_basis(g, coarse, tol, **kw)         coarsening.py:335-339 -> CoarsenState
  project_final(g, rowstate, colstate, coarse)         coarsening.py:354-405 -> DeviceH2

Matrix arguments are `DeviceH2` (or host `H2Matrix`, uploaded); bases are `DeviceBasis` views
(`DeviceH2.row_basis` / `.col_basis`) or host `ClusterBasis` objects (uploaded).  Per-cluster
results (`.p`, `.r`, `.z`, `.basis_change`, `.block_projections`) download lazily into dicts keyed
like the reference's (cluster id; (t, s) for block projections).  Norms are device tensors indexed
by block id (or dicts {block: norm}, as the reference passes them).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .device import Context, DeviceH2, default_context
from .errors import InvalidInputError
from .h2 import ClusterBasis, H2Matrix
from .packed import pack_basis_arrays
from .trees import BlockTree, ClusterTree, build_product_block_tree, same_cluster_tree

__all__ = ["DeviceBasis", "DeviceMats", "BasisProduct", "BasisWeights", "TotalWeights", "InducedBasisResult",
           "CoarsenState", "cluster_basis_product", "basis_weights", "total_weights",
           "compress_induced_row_basis", "compress_induced_col_basis", "assemble_product", "coupling_norms",
           "nearfield_norms", "block_norms", "build_coarse_row_basis", "build_coarse_col_basis", "project_final",
           "build_product_block_tree"]


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


def _mr(max_rank):
    return -1 if max_rank is None else max(0, int(max_rank))


def _check_tol(tol):
    if tol < 0:
        raise InvalidInputError(f"tolerance must be >= 0, got {tol}")


def _dev_h2(g, ctx):
    if isinstance(g, DeviceH2):
        return g
    if isinstance(g, H2Matrix):
        return DeviceH2.upload(g, ctx)
    raise InvalidInputError(f"expected an H2Matrix or DeviceH2, got {type(g).__name__}")


class _Handle:
    """Owns one native handle; `_destroy` names its h2g_*_destroy function."""

    _destroy = None

    def __init__(self, ctx: Context, h, *keep):
        self.ctx, self.h, self._keep = ctx, h, keep

    def __del__(self):
        try:
            if getattr(self, "h", None) and self._destroy:
                getattr(self.ctx.lib, self._destroy)(self.h)
                self.h = None
        except Exception:
            pass


class DeviceBasis(_Handle):
    """A cluster basis on the device (reference ClusterBasis, h2.py:32-72)."""

    _destroy = "h2g_basis_destroy"

    def __init__(self, ctx, h, tree: ClusterTree, *keep):
        super().__init__(ctx, h, *keep)
        self.tree = tree
        self._host = None

    @classmethod
    def of(cls, b, ctx=None) -> "DeviceBasis":
        if isinstance(b, DeviceBasis):
            return b
        if isinstance(b, ClusterBasis):
            ctx = _ctx(ctx)
            rank, loff, xoff, data = pack_basis_arrays(b)
            h = N.P()
            N.check(ctx.lib.h2g_basis_upload(ctx.h, ctx.tree(b.tree), N.i64(rank)[1], N.i64(loff)[1],
                                             N.i64(xoff)[1], N.f64(data)[1], len(data), C.byref(h)))
            return cls(ctx, h, b.tree)
        raise InvalidInputError(f"expected a ClusterBasis or DeviceBasis, got {type(b).__name__}")

    def download(self) -> ClusterBasis:
        if self._host is None:
            s = np.zeros(2, np.int64)
            N.check(self.ctx.lib.h2g_basis_sizes(self.h, s.ctypes.data_as(N.I64P)))
            n = int(s[0])
            rank, loff, xoff = (np.zeros(n, np.int64) for _ in range(3))
            data = np.zeros(max(1, int(s[1])))
            N.check(self.ctx.lib.h2g_basis_download(self.ctx.h, self.h, rank.ctypes.data_as(N.I64P),
                                                    loff.ctypes.data_as(N.I64P), xoff.ctypes.data_as(N.I64P),
                                                    data.ctypes.data_as(N.F64P)))
            tr = self.tree
            leaf = {t: data[loff[t]:loff[t] + tr.size(t) * rank[t]].reshape(tr.size(t), rank[t])
                    for t in range(n) if tr.is_leaf(t)}
            par = tr.flat()["parent"]
            xf = {t: data[xoff[t]:xoff[t] + rank[t] * rank[par[t]]].reshape(rank[t], rank[par[t]])
                  for t in range(n) if par[t] >= 0}
            self._host = ClusterBasis(tr, rank, leaf, xf)
        return self._host

    @property
    def rank(self):
        return self.download().rank

    @property
    def leaf_matrix(self):
        return self.download().leaf_matrix

    @property
    def transfer(self):
        return self.download().transfer


class DeviceMats(_Handle):
    """Small device matrices indexed by cluster (or block) id; `.to_dict()` downloads them."""

    _destroy = "h2g_mats_destroy"

    def __init__(self, ctx, h, *keep, keys=None):
        super().__init__(ctx, h, *keep)
        self._dict = None
        self._keys = keys

    def shapes(self):
        n = C.c_int(0)
        N.check(self.ctx.lib.h2g_mats_shapes(self.h, C.byref(n), None, None))
        r, c = np.zeros(n.value, np.int64), np.zeros(n.value, np.int64)
        N.check(self.ctx.lib.h2g_mats_shapes(self.h, C.byref(n), r.ctypes.data_as(N.I64P),
                                             c.ctypes.data_as(N.I64P)))
        return r, c

    def to_dict(self, present=None) -> dict:
        """{id: matrix} for the entries `present(id)` selects (default: every entry)."""
        if self._dict is None:
            r, c = self.shapes()
            off = np.zeros(len(r), np.int64)
            data = np.zeros(max(1, int((r * c).sum())))
            N.check(self.ctx.lib.h2g_mats_download(self.ctx.h, self.h, off.ctypes.data_as(N.I64P),
                                                   data.ctypes.data_as(N.F64P)))
            self._dict = {i: data[off[i]:off[i] + r[i] * c[i]].reshape(r[i], c[i])
                          for i in range(len(r)) if off[i] >= 0}
        d = self._dict
        if present is not None:
            d = {i: m for i, m in d.items() if present(i)}
        return d

    @classmethod
    def upload(cls, mats: dict, n: int, ctx=None) -> "DeviceMats":
        ctx = _ctx(ctx)
        rows, cols, off = np.zeros(n, np.int64), np.zeros(n, np.int64), np.full(n, -1, np.int64)
        chunks, pos = [], 0
        for i, m in mats.items():
            m = np.ascontiguousarray(m, dtype=np.float64)
            rows[i], cols[i] = m.shape
            off[i] = pos
            chunks.append(m.ravel())
            pos += m.size
        data = np.concatenate(chunks) if chunks else np.zeros(1)
        h = N.P()
        N.check(ctx.lib.h2g_mats_upload(ctx.h, n, N.i64(rows)[1], N.i64(cols)[1], N.i64(off)[1], N.f64(data)[1],
                                        pos, C.byref(h)))
        return cls(ctx, h)


class BasisProduct:
    """P_s = W_X,s^T V_Y,s per cluster s (reference h2.py:116-124), on the device."""

    def __init__(self, tree, mats: DeviceMats):
        self.tree, self.mats = tree, mats

    @property
    def p(self) -> dict:
        return self.mats.to_dict()


class BasisWeights:
    """R_r with W_r = Q_r R_r per cluster (reference weights.py:20-25), on the device."""

    def __init__(self, tree, mats: DeviceMats):
        self.tree, self.mats = tree, mats

    @property
    def r(self) -> dict:
        return self.mats.to_dict()


class TotalWeights:
    """Z_s per cluster (reference weights.py:28-34), on the device."""

    def __init__(self, tree, mats: DeviceMats, scaled: bool):
        self.tree, self.mats, self.scaled = tree, mats, scaled

    @property
    def z(self) -> dict:
        return self.mats.to_dict()


class InducedBasisResult(_Handle):
    """Compressed induced basis (reference induced.py:33-46): q, basis_change[t] = Q_t^T V_t and
    block_projections[(t, s)] = Q_t^T X|ts V_Y,s for every non-admissible-leaf block."""

    _destroy = "h2g_induced_destroy"

    def __init__(self, ctx, h, tree, blocks: BlockTree, col: bool, *keep):
        super().__init__(ctx, h, *keep)
        self.tree, self._blocks, self.col = tree, blocks, col
        self._parts = None

    def _get(self):
        if self._parts is None:
            q, bc, pr = N.P(), N.P(), N.P()
            N.check(self.ctx.lib.h2g_induced_parts(self.h, C.byref(q), C.byref(bc), C.byref(pr)))
            self._parts = (DeviceBasis(self.ctx, q, self.tree, self), DeviceMats(self.ctx, bc, self),
                           DeviceMats(self.ctx, pr, self))
        return self._parts

    @property
    def q(self) -> DeviceBasis:
        return self._get()[0]

    @property
    def basis_change(self) -> dict:
        return self._get()[1].to_dict()

    @property
    def block_projections(self) -> dict:
        bt = self._blocks
        got = self._get()[2].to_dict(lambda b: not (bt.is_leaf(b) and bt.admissible[b]))
        return {(bt.row[b], bt.col[b]): m for b, m in got.items()}

    @classmethod
    def from_parts(cls, q, basis_change: dict, block_projections: dict, blocks: BlockTree, col: bool = False,
                   ctx=None) -> "InducedBasisResult":
        """An induced basis computed elsewhere (e.g. by the CPU oracle), for assemble_product.
        `blocks` is X's block tree (Y^T's for a column basis); projections keyed (t, s)."""
        ctx = _ctx(ctx)
        dq = DeviceBasis.of(q, ctx)
        bc = DeviceMats.upload(basis_change, dq.tree.nnodes, ctx)
        idx = {(blocks.row[b], blocks.col[b]): b for b in range(blocks.nblocks)}
        pr = DeviceMats.upload({idx[k]: m for k, m in block_projections.items()}, blocks.nblocks, ctx)
        h = N.P()
        N.check(ctx.lib.h2g_induced_create(ctx.h, dq.h, bc.h, pr.h, 1 if col else 0, C.byref(h)))
        return cls(ctx, h, dq.tree, blocks, col, dq, bc, pr)


class CoarsenState(_Handle):
    """One adaptive coarse-basis construction (reference coarsening.py:36-50): q, r, z on the
    device; `nreps` counts the stored column-tree representations."""

    _destroy = "h2g_cstate_destroy"

    def __init__(self, ctx, h, tree, col: bool, g, coarse, *keep):
        super().__init__(ctx, h, g, *keep)
        self.tree, self.col, self.g, self.coarse = tree, col, g, coarse
        self._parts = None

    def _get(self):
        if self._parts is None:
            q, r, z = N.P(), N.P(), N.P()
            nreps = C.c_longlong(0)
            N.check(self.ctx.lib.h2g_cstate_parts(self.h, C.byref(q), C.byref(r), C.byref(z), C.byref(nreps)))
            self._parts = (DeviceBasis(self.ctx, q, self.tree, self), DeviceMats(self.ctx, r, self),
                           DeviceMats(self.ctx, z, self), int(nreps.value))
        return self._parts

    @property
    def q(self) -> DeviceBasis:
        return self._get()[0]

    @property
    def r(self) -> dict:
        return self._get()[1].to_dict()

    @property
    def z(self) -> dict:
        return self._get()[2].to_dict()

    @property
    def nreps(self) -> int:
        return self._get()[3]


# ------------------------------------------------------------------------------------------------

def _basis(b, ctx):
    return DeviceBasis.of(b, ctx)


def cluster_basis_product(wx, vy, *, ctx: Context | None = None) -> BasisProduct:
    """W_X,s^T V_Y,s for every cluster s (reference h2.py:127-145)."""
    ctx = _ctx(ctx)
    w, v = _basis(wx, ctx), _basis(vy, ctx)
    if not same_cluster_tree(w.tree, v.tree):
        raise InvalidInputError("bases live on different cluster trees")
    h = N.P()
    N.check(ctx.lib.h2g_cluster_basis_product(ctx.h, w.h, v.h, C.byref(h)))
    return BasisProduct(w.tree, DeviceMats(ctx, h, w, v))


def basis_weights(w, *, ctx: Context | None = None) -> BasisWeights:
    """R_r of W_r = Q_r R_r, bottom-up (reference weights.py:37-57)."""
    ctx = _ctx(ctx)
    b = _basis(w, ctx)
    h = N.P()
    N.check(ctx.lib.h2g_basis_weights(ctx.h, b.h, C.byref(h)))
    return BasisWeights(b.tree, DeviceMats(ctx, h, b))


def total_weights(y, rw: BasisWeights, scaling: bool = True, *, ctx: Context | None = None) -> TotalWeights:
    """Top-down condensation weights Z_s (reference weights.py:60-101).  `y` is a DeviceH2 / H2Matrix
    or its transposed view (`g.transposed()`), as the reference passes x.transposed()."""
    ctx = _ctx(ctx)
    transposed = isinstance(y, _Transposed)
    g = _dev_h2(y.g if transposed else y, ctx)
    h = N.P()
    N.check(ctx.lib.h2g_total_weights(ctx.h, g.h, 1 if transposed else 0, rw.mats.h, 1 if scaling else 0,
                                      C.byref(h)))
    tree = g.cols if transposed else g.rows
    return TotalWeights(tree, DeviceMats(ctx, h, g, rw.mats), bool(scaling))


class _Transposed:
    """g.transposed() for the stage functions that take a transposed matrix (total_weights)."""

    def __init__(self, g):
        self.g = g

    def transposed(self):
        return self.g


def transposed(g):
    return _Transposed(g)


def _induced(x, y, z: TotalWeights, pxy: BasisProduct, tol, max_rank, scale_blocks, level_decay, col, ctx):
    _check_tol(tol)
    ctx = _ctx(ctx)
    dx, dy = _dev_h2(x, ctx), _dev_h2(y, ctx)
    if not same_cluster_tree(dx.cols, dy.rows):
        raise InvalidInputError("x and y do not share the middle cluster tree")
    h = N.P()
    fn = ctx.lib.h2g_compress_induced_col_basis if col else ctx.lib.h2g_compress_induced_row_basis
    N.check(fn(ctx.h, dx.h, dy.h, z.mats.h, pxy.mats.h, float(tol), _mr(max_rank), 1 if scale_blocks else 0,
               float(level_decay), C.byref(h)))
    tree = dy.cols if col else dx.rows
    blocks = dy.block_tree.transposed() if col else dx.block_tree
    return InducedBasisResult(ctx, h, tree, blocks, col, dx, dy, z.mats, pxy.mats)


def compress_induced_row_basis(x, y, zy: TotalWeights, pxy: BasisProduct, tol: float, *,
                               max_rank: int | None = None, scale_blocks: bool = True, level_decay: float = 1.0,
                               ctx: Context | None = None) -> InducedBasisResult:
    """Adaptive isometric basis spanning the products X|ts Y|sr row-wise (reference induced.py:76-184)."""
    return _induced(x, y, zy, pxy, tol, max_rank, scale_blocks, level_decay, False, ctx)


def compress_induced_col_basis(x, y, zx_adjoint: TotalWeights, pxy: BasisProduct, tol: float, *,
                               max_rank: int | None = None, scale_blocks: bool = True, level_decay: float = 1.0,
                               ctx: Context | None = None) -> InducedBasisResult:
    """Induced column basis: the row algorithm applied to Y^T X^T (reference induced.py:187-200)."""
    return _induced(x, y, zx_adjoint, pxy, tol, max_rank, scale_blocks, level_decay, True, ctx)


def assemble_product(x, y, qrow: InducedBasisResult, qcol: InducedBasisResult, pxy: BasisProduct,
                     product_tree: BlockTree | None = None, *, ctx: Context | None = None) -> DeviceH2:
    """X*Y over the product block tree in the induced bases (reference induced.py:220-355).  T^XY is
    built natively; a given `product_tree` must equal it (trees.py:314-359)."""
    ctx = _ctx(ctx)
    dx, dy = _dev_h2(x, ctx), _dev_h2(y, ctx)
    if not same_cluster_tree(dx.cols, dy.rows):
        raise InvalidInputError("x and y do not share the middle cluster tree")
    h = N.P()
    N.check(ctx.lib.h2g_assemble_product(ctx.h, dx.h, dy.h, qrow.h, qcol.h, pxy.mats.h, C.byref(h)))
    g = DeviceH2(ctx, h, None, dx.rows, dy.cols)
    if product_tree is not None:
        bt = g.block_tree
        if not (list(bt.row) == list(product_tree.row) and list(bt.col) == list(product_tree.col)):
            raise InvalidInputError("product_tree is not the product block tree of x and y")
    g._keep = (qrow, qcol, pxy)
    return g


def block_norms(g, *, ctx: Context | None = None):
    """(coupling norms, nearfield norms) of g's leaves as device tensors indexed by block id
    (reference coarsening.py:342-351, _coupling_norms / _nearfield_norms)."""
    import torch
    ctx = _ctx(ctx)
    dg = _dev_h2(g, ctx)
    nb = int(dg.sizes()[0])
    dev = torch.device("cuda", ctx.device)
    cn = torch.zeros(max(1, nb), dtype=torch.float64, device=dev)
    nn = torch.zeros(max(1, nb), dtype=torch.float64, device=dev)
    torch.cuda.current_stream(dev).synchronize()
    N.check(ctx.lib.h2g_block_norms(ctx.h, dg.h, C.c_void_p(cn.data_ptr()), C.c_void_p(nn.data_ptr())))
    return cn, nn


def _norm_dict(g, which):
    cn, nn = block_norms(g)
    bt = g.block_tree
    v = (cn if which == "c" else nn).cpu().numpy()
    want = bt.admissible_leaves() if which == "c" else bt.inadmissible_leaves()
    return {b: float(v[b]) for b in want}


def coupling_norms(g) -> dict:
    """{block: sigma_1(S_b)} over admissible leaves (reference coarsening.py:342-345)."""
    return _norm_dict(g, "c")


def nearfield_norms(g) -> dict:
    """{block: sigma_1(N_b)} over inadmissible leaves (reference coarsening.py:348-351)."""
    return _norm_dict(g, "n")


def _norm_arg(v, nb, ctx):
    """Norms given as a device tensor (block-indexed) or as the reference's {block: norm} dict."""
    if v is None:
        return None, None
    import torch
    dev = torch.device("cuda", ctx.device)
    if isinstance(v, dict):
        a = np.zeros(max(1, nb))
        for b, x in v.items():
            a[int(b)] = float(x)
        v = torch.from_numpy(a).to(dev)
    v = torch.as_tensor(v, dtype=torch.float64, device=dev).contiguous()
    if v.numel() < nb:
        raise InvalidInputError("norm array shorter than the number of blocks")
    torch.cuda.current_stream(dev).synchronize()
    return C.c_void_p(v.data_ptr()), v


def _coarse(g, coarse, tol, max_rank, scale_blocks, cn, nn, col, ctx):
    _check_tol(tol)
    ctx = _ctx(ctx)
    dg = _dev_h2(g, ctx)
    nb = int(dg.sizes()[0])
    pc, kc = _norm_arg(cn, nb, ctx)
    pn, kn = _norm_arg(nn, nb, ctx)
    h = N.P()
    fn = ctx.lib.h2g_build_coarse_col_basis if col else ctx.lib.h2g_build_coarse_row_basis
    N.check(fn(ctx.h, dg.h, ctx.blocks(coarse), float(tol), _mr(max_rank), 1 if scale_blocks else 0, pc, pn,
               C.byref(h)))
    tree = coarse.cols if col else coarse.rows
    return CoarsenState(ctx, h, tree, col, dg, coarse, kc, kn)


def build_coarse_row_basis(g, coarse: BlockTree, tol: float, *, max_rank: int | None = None,
                           scale_blocks: bool = True, coupling_norms=None, nearfield_norms=None,
                           ctx: Context | None = None) -> CoarsenState:
    """Adaptive row basis for re-compressing g onto `coarse` (reference coarsening.py:187-332)."""
    return _coarse(g, coarse, tol, max_rank, scale_blocks, coupling_norms, nearfield_norms, False, ctx)


def build_coarse_col_basis(g, coarse: BlockTree, tol: float, *, max_rank: int | None = None,
                           scale_blocks: bool = True, coupling_norms=None, nearfield_norms=None,
                           ctx: Context | None = None) -> CoarsenState:
    """Adaptive column basis: the row construction on G^T (reference coarsening.py:335-339)."""
    return _coarse(g, coarse, tol, max_rank, scale_blocks, coupling_norms, nearfield_norms, True, ctx)


def project_final(g, rowstate: CoarsenState, colstate: CoarsenState, coarse: BlockTree, *,
                  ctx: Context | None = None) -> DeviceH2:
    """Project the phase-1 product onto the coarse tree and the new bases (coarsening.py:354-405)."""
    ctx = _ctx(ctx)
    dg = rowstate.g
    h = N.P()
    N.check(ctx.lib.h2g_project_final(ctx.h, dg.h, rowstate.h, colstate.h, ctx.blocks(coarse), C.byref(h)))
    z = DeviceH2(ctx, h, coarse, coarse.rows, coarse.cols)
    z._keep = (rowstate, colstate)
    return z
