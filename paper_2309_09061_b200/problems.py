"""Input construction for the BASELINE configs (setup, not the timed product).

Restates the reference's interpolation builder (h2mul/problems.py:218-332)
for point-kernel problems and adds the seeded generators and kernels that
BASELINE.json's configs name but the reference lacks:
uniform 2-D / 3-D points, the Fibonacci sphere, 1/r and exp(-r)/r.
Everything here is host NumPy and runs once before the product; the
product itself (multiply / coarsen) runs on the GPU.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import InvalidInputError
from .h2 import ClusterBasis, H2Matrix
from .trees import build_block_tree, build_cluster_tree

__all__ = ["CONFIGS", "KERNEL_FNS", "make_points", "build_interpolation_h2", "build_config", "build_config_device"]

_FLAT_AXIS = 1e-8  # reference problems.py:40


def _k_log(r):
    return -np.log(r)


def _k_slp(r):
    return 1.0 / (4.0 * np.pi * r)


def _k_inv(r):
    return 1.0 / r


def _k_yukawa(r):
    return np.exp(-r) / r


KERNEL_FNS = {"log": _k_log, "slp": _k_slp, "inv_r": _k_inv, "exp_r": _k_yukawa}

# BASELINE.json "configs" 1..5; golden_n is the reduced size used for reference fixtures
CONFIGS = {
    "c1": dict(geometry="interval", n=2048, kernel_x="log", kernel_y="log", leaf=32, eta=1.0,
               order=4, eps=1e-6, golden_n=2048),
    "c2": dict(geometry="uniform2d", n=16384, kernel_x="log", kernel_y="log", leaf=64, eta=1.0,
               order=4, eps=1e-6, golden_n=2048),
    "c3": dict(geometry="fibonacci", n=32768, kernel_x="slp", kernel_y="slp", leaf=64, eta=2.0,
               order=3, eps=1e-5, golden_n=2048),
    "c4": dict(geometry="fibonacci", n=262144, kernel_x="inv_r", kernel_y="exp_r", leaf=128,
               eta=2.0, order=4, eps=1e-6, golden_n=4096),
    "c5": dict(geometry="uniform3d", n=2097152, kernel_x="inv_r", kernel_y="inv_r", leaf=128,
               eta=2.0, order=3, eps=1e-4, golden_n=4096),
}


def make_points(geometry: str, n: int, seed: int = 0):
    """Seeded point sets and quadrature weights for the configs."""
    if geometry == "interval":
        # reference problems.py:153-155: midpoints of a uniform grid, weights 1/n
        return ((np.arange(n) + 0.5) / n)[:, None], np.full(n, 1.0 / n)
    if geometry == "uniform2d":
        return np.random.default_rng(seed).uniform(size=(n, 2)), np.ones(n)
    if geometry == "uniform3d":
        return np.random.default_rng(seed).uniform(size=(n, 3)), np.ones(n)
    if geometry == "fibonacci":
        i = np.arange(n) + 0.5
        phi = np.arccos(1.0 - 2.0 * i / n)
        theta = np.pi * (1.0 + math.sqrt(5.0)) * i
        pts = np.stack([np.cos(theta) * np.sin(phi), np.sin(theta) * np.sin(phi), np.cos(phi)], axis=1)
        return pts, np.ones(n)
    raise InvalidInputError(f"unknown geometry {geometry!r}")


def _kernel(fn, xi, xj):
    """g(x_i, x_j) with zero where the points coincide (reference problems.py:175-189)."""
    diff = np.atleast_2d(xi)[:, None, :] - np.atleast_2d(xj)[None, :, :]
    r = np.linalg.norm(diff, axis=-1)
    mask = r > 0
    safe = np.where(mask, r, 1.0)
    return np.where(mask, fn(safe), 0.0)


def _cheb(a, b, m):
    """Chebyshev-Lobatto nodes (reference problems.py:218-222)."""
    if m == 1:
        return np.array([0.5 * (a + b)])
    j = np.arange(m)
    return 0.5 * (a + b) + 0.5 * (b - a) * np.cos(np.pi * j / (m - 1))


def _lagrange(nodes, x):
    """l_nu(x_i), product accumulated in the reference's order (problems.py:225-235)."""
    m = len(nodes)
    if m == 1:
        return np.ones((len(x), 1))
    out = np.ones((len(x), m))
    for nu in range(m):
        for mu in range(m):
            if mu != nu:
                out[:, nu] *= (x - nodes[mu]) / (nodes[nu] - nodes[mu])
    return out


class _TensorInterp:
    """Per-cluster tensor Chebyshev grids on the bounding boxes (problems.py:238-266)."""

    def __init__(self, tree, order):
        self.axes, self.points = [], []
        for t in range(tree.nnodes):
            ext = tree.bbox_max[t] - tree.bbox_min[t]
            top = ext.max()
            ax = []
            for a in range(tree.dim):
                m = order if top > 0 and ext[a] > _FLAT_AXIS * top else 1
                ax.append(_cheb(tree.bbox_min[t][a], tree.bbox_max[t][a], m))
            self.axes.append(ax)
            grid = np.meshgrid(*ax, indexing="ij")
            self.points.append(np.stack([g.ravel() for g in grid], axis=-1))

    def eval(self, t, x):
        out = np.ones((x.shape[0], 1))
        for a, nodes in enumerate(self.axes[t]):
            la = _lagrange(nodes, x[:, a])
            out = (out[:, :, None] * la[:, None, :]).reshape(x.shape[0], -1)
        return out


def build_interpolation_h2(tree, blocks, weights_perm, kernel_fn, order) -> H2Matrix:
    """H^2 approximation by tensor Chebyshev interpolation (reference problems.py:295-332).

    ``weights_perm`` are the quadrature weights in tree (permuted) order; the
    nearfield is g(x_i, x_j) w_i w_j and the leaf bases carry w_i.
    """
    interp = _TensorInterp(tree, order)
    rank = [interp.points[t].shape[0] for t in range(tree.nnodes)]
    leaf, xfer = {}, {}
    for t in range(tree.nnodes):
        if tree.is_leaf(t):
            sl = tree.index_range(t)
            leaf[t] = interp.eval(t, tree.points[sl]) * weights_perm[sl, None]
        for c in tree.children[t]:
            xfer[c] = interp.eval(t, interp.points[c])
    basis = ClusterBasis(tree, rank, leaf, xfer)
    coup, near = {}, {}
    for b in range(blocks.nblocks):
        t, s = blocks.row[b], blocks.col[b]
        if blocks.is_admissible_leaf(b):
            coup[b] = _kernel(kernel_fn, interp.points[t], interp.points[s])
        elif blocks.is_inadmissible_leaf(b):
            st, ss = tree.index_range(t), tree.index_range(s)
            near[b] = _kernel(kernel_fn, tree.points[st], tree.points[ss]) * \
                np.outer(weights_perm[st], weights_perm[ss])
    return H2Matrix(blocks, basis, basis, coup, near)


def build_config(name: str, n: int | None = None, seed: int = 0):
    """Raw (not yet recompressed) inputs X, Y for a BASELINE config at size n.

    Returns (x_raw, y_raw, spec); y_raw is x_raw when X = Y.
    """
    spec = dict(CONFIGS[name])
    n = spec["n"] if n is None else int(n)
    spec["n"] = n
    pts, wts = make_points(spec["geometry"], n, seed)
    tree = build_cluster_tree(pts, spec["leaf"])
    blocks = build_block_tree(tree, tree, spec["eta"])
    w = wts[tree.perm]
    x = build_interpolation_h2(tree, blocks, w, KERNEL_FNS[spec["kernel_x"]], spec["order"])
    if spec["kernel_y"] == spec["kernel_x"]:
        y = x
    else:
        y = build_interpolation_h2(tree, blocks, w, KERNEL_FNS[spec["kernel_y"]], spec["order"])
    return x, y, spec


KERNEL_IDS = {"log": 0, "slp": 1, "inv_r": 2, "exp_r": 3}  # h2g_h2_build_kernel ids


def _interp_basis_packed(tree, weights_perm, order):
    """Host interpolation basis in the packed layout plus the per-cluster Chebyshev grids."""
    interp = _TensorInterp(tree, order)
    rank = np.asarray([interp.points[t].shape[0] for t in range(tree.nnodes)], dtype=np.int64)
    f = tree.flat()
    loff = np.full(tree.nnodes, -1, np.int64)
    xoff = np.full(tree.nnodes, -1, np.int64)
    chunks, off = [], 0
    for t in range(tree.nnodes):
        if tree.is_leaf(t):
            sl = tree.index_range(t)
            m = interp.eval(t, tree.points[sl]) * weights_perm[sl, None]
            loff[t] = off
            chunks.append(m.ravel())
            off += m.size
    for t in range(tree.nnodes):
        p = f["parent"][t]
        if p >= 0:
            m = interp.eval(p, interp.points[t])
            xoff[t] = off
            chunks.append(m.ravel())
            off += m.size
    data = np.concatenate(chunks) if chunks else np.zeros(0)
    noff = np.zeros(tree.nnodes, np.int64)
    grids, o = [], 0
    for t in range(tree.nnodes):
        noff[t] = o
        grids.append(np.ascontiguousarray(interp.points[t], dtype=np.float64).ravel())
        o += interp.points[t].size
    return rank, loff, xoff, data, noff, np.concatenate(grids)


def build_config_device(name: str, n: int | None = None, seed: int = 0, ctx=None):
    """Raw inputs X, Y of a BASELINE config built on the GPU: structure and the
    small interpolation bases on the host, the couplings and nearfield blocks evaluated by
    h2g_h2_build_kernel.  Returns (dx_raw, dy_raw, spec) as DeviceH2 (dy is dx when X = Y)."""
    import ctypes as C
    from . import _native as N
    from .device import DeviceH2, default_context
    spec = dict(CONFIGS[name])
    n = spec["n"] if n is None else int(n)
    spec["n"] = n
    ctx = ctx or default_context()
    pts, wts = make_points(spec["geometry"], n, seed)
    tree = build_cluster_tree(pts, spec["leaf"])
    blocks = build_block_tree(tree, tree, spec["eta"])
    w = np.ascontiguousarray(wts[tree.perm], dtype=np.float64)
    P = np.ascontiguousarray(tree.points, dtype=np.float64)
    rank, loff, xoff, data, noff, nodes = _interp_basis_packed(tree, w, spec["order"])
    hb = ctx.blocks(blocks)

    def make(kernel):
        h = N.P()
        N.check(ctx.lib.h2g_h2_build_kernel(
            ctx.h, hb, KERNEL_IDS[kernel], P.shape[1], N.f64(P)[1], N.f64(w)[1], N.i64(rank)[1], N.i64(loff)[1],
            N.i64(xoff)[1], N.f64(data)[1], len(data), N.i64(noff)[1], N.f64(nodes)[1], len(nodes), C.byref(h)))
        return DeviceH2(ctx, h, blocks, tree, tree)

    dx = make(spec["kernel_x"])
    dy = dx if spec["kernel_y"] == spec["kernel_x"] else make(spec["kernel_y"])
    return dx, dy, spec
