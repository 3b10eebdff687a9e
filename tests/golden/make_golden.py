"""Generate the golden fixtures by running the REFERENCE implementation (h2mul).

Run in the build container only (it imports /root/reference read-only):

    python tests/golden/make_golden.py

Every fixture holds, in the packed layout of paper_2309_09061_b200/packed.py
(x/, y/, z/ only for c1 and the random cases; the reduced-size c2-c5 cases
keep structure, ranks and probes, and their inputs are rebuilt by
paper_2309_09061_b200.problems, pinned by probe.xraw_v):
  x/..., y/...        the recompressed inputs, exactly as the reference harness
                      prepares them (bench.py:198-199, coarsening.py:437-445)
  z/...               the reference's final product Z (coarsening.py:408-422)
  pt.*                the refined product block tree T^XY (trees.py:314-359)
  rank.*              per-cluster ranks: induced row/col (induced.py:76-200),
                      final row/col (coarsening.py:187-339)
  probe.*             v, X_raw v, Y_raw v, G v, Z v, X (Y v), Z^T v for probe vectors
  gap.*               min |sigma - thr| / thr over every truncation (rank-parity margin)

Kernels and geometries that the reference lacks (uniform 2-D/3-D points,
Fibonacci sphere, 1/r, exp(-r)/r) are injected the way SURVEY.md 8(d)
prescribes: points through build_h2_by_interpolation(..., geometry=...) and
the kernel by wrapping h2mul.problems._kernel_values in memory.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import paper_2309_09061_b200.problems as myprob  # noqa: E402  (geometry generators only)


def _ref():
    sys.path.insert(0, REF)
    import h2mul
    import h2mul.problems as hp
    return h2mul, hp


def pack_tree(tree, p, out):
    out[p + "start"] = np.asarray(tree.start, dtype=np.int64)
    out[p + "stop"] = np.asarray(tree.stop, dtype=np.int64)
    lens = [len(c) for c in tree.children]
    out[p + "child_ptr"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out[p + "child_idx"] = np.asarray([c for k in tree.children for c in k], dtype=np.int64)


def pack_basis(basis, p, out):
    tree = basis.tree
    par = [-1] * tree.nnodes
    for t in range(tree.nnodes):
        for c in tree.children[t]:
            par[c] = t
    chunks, pos = [], 0
    loff = np.full(tree.nnodes, -1, np.int64)
    xoff = np.full(tree.nnodes, -1, np.int64)
    for t in range(tree.nnodes):
        if tree.is_leaf(t):
            m = np.ascontiguousarray(basis.leaf_matrix[t])
            loff[t] = pos; chunks.append(m.ravel()); pos += m.size
    for t in range(tree.nnodes):
        if par[t] >= 0:
            m = np.ascontiguousarray(basis.transfer[t])
            xoff[t] = pos; chunks.append(m.ravel()); pos += m.size
    out[p + "rank"] = np.asarray(basis.rank, dtype=np.int64)
    out[p + "leaf_off"] = loff
    out[p + "xfer_off"] = xoff
    out[p + "data"] = np.concatenate(chunks) if chunks else np.zeros(0)


def pack_h2(g, p, out):
    bt = g.block_tree
    pack_tree(bt.rows, p + "rows.", out)
    pack_tree(bt.cols, p + "cols.", out)
    out[p + "bt.row"] = np.asarray(bt.row, dtype=np.int64)
    out[p + "bt.col"] = np.asarray(bt.col, dtype=np.int64)
    lens = [len(c) for c in bt.children]
    out[p + "bt.child_ptr"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out[p + "bt.child_idx"] = np.asarray([c for k in bt.children for c in k], dtype=np.int64)
    out[p + "bt.adm"] = np.asarray(bt.admissible, dtype=np.uint8)
    pack_basis(g.row_basis, p + "rb.", out)
    pack_basis(g.col_basis, p + "cb.", out)
    for name, store in (("coup", g.coupling), ("near", g.nearfield)):
        off = np.full(bt.nblocks, -1, np.int64)
        chunks, pos = [], 0
        for b in range(bt.nblocks):
            if b in store:
                m = np.ascontiguousarray(store[b])
                off[b] = pos; chunks.append(m.ravel()); pos += m.size
        out[p + name + "_off"] = off
        out[p + name + "_data"] = np.concatenate(chunks) if chunks else np.zeros(0)


class GapLog:
    """Wrap the reference truncated_svd to log min |sigma - thr| / thr per call."""

    def __init__(self, h2mul):
        self.vals = []
        import h2mul.dense as hd
        import h2mul.induced as hi
        import h2mul.coarsening as hc
        self.orig = hd.truncated_svd
        log = self

        def wrapped(a, tol, max_rank=None, relative=False):
            m = np.asarray(a, dtype=np.float64)
            if min(m.shape) > 0:
                s = np.linalg.svd(m, compute_uv=False)
                thr = max(tol, max(m.shape) * np.finfo(float).eps * s[0])
                if thr > 0:
                    log.vals.append(float(np.min(np.abs(s - thr)) / thr))
            return log.orig(a, tol, max_rank=max_rank, relative=relative)

        self.mods = (hi, hc)
        for mod in self.mods:
            mod.truncated_svd = wrapped

    def restore(self):
        for mod in self.mods:
            mod.truncated_svd = self.orig


def ref_instance(h2mul, hp, points, weights, kernel_fn, leaf, eta, order, base_kernel):
    """Reference tree / block tree / interpolation with an injected kernel."""
    orig = hp._kernel_values

    def kv(kernel, xi, xj, normals_i=None):
        if kernel_fn is None:
            return orig(kernel, xi, xj, normals_i)
        diff = np.atleast_2d(xi)[:, None, :] - np.atleast_2d(xj)[None, :, :]
        r = np.linalg.norm(diff, axis=-1)
        mask = r > 0
        safe = np.where(mask, r, 1.0)
        return np.where(mask, kernel_fn(safe), 0.0)

    hp._kernel_values = kv
    try:
        tree = h2mul.build_cluster_tree(points, leaf)
        blocks = h2mul.build_block_tree(tree, tree, eta)
        prob = h2mul.KernelProblem("sphere", base_kernel, len(points), order)
        geo = h2mul.Geometry(points, weights, None)
        g = h2mul.build_h2_by_interpolation(prob, tree, blocks, geo)
    finally:
        hp._kernel_values = orig
    return tree, blocks, g


def run_reference(h2mul, x, y, eps, out, probes, x_raw=None, y_raw=None, keep_z=True,
                  keep_inputs=True):
    from h2mul.coarsening import _coupling_norms, _nearfield_norms
    gaps = GapLog(h2mul)
    try:
        pxy = h2mul.cluster_basis_product(x.col_basis, y.row_basis)
        zy = h2mul.total_weights(y, h2mul.basis_weights(y.col_basis))
        zxt = h2mul.total_weights(x.transposed(), h2mul.basis_weights(x.row_basis))
        qrow = h2mul.compress_induced_row_basis(x, y, zy, pxy, eps)
        qcol = h2mul.compress_induced_col_basis(x, y, zxt, pxy, eps)
        pt = h2mul.build_product_block_tree(x.block_tree, y.block_tree)
        g = h2mul.assemble_product(x, y, qrow, qcol, pxy, pt)
        n1 = len(gaps.vals)
        coarse = x.block_tree
        cn, nn = _coupling_norms(g), _nearfield_norms(g)
        rs = h2mul.build_coarse_row_basis(g, coarse, eps, coupling_norms=cn, nearfield_norms=nn)
        cs = h2mul.build_coarse_col_basis(g, coarse, eps, coupling_norms=cn, nearfield_norms=nn)
        z = h2mul.project_final(g, rs, cs, coarse)
    finally:
        gaps.restore()
    if keep_inputs:
        pack_h2(x, "x/", out)
        pack_h2(y, "y/", out)
    if keep_z:
        pack_h2(z, "z/", out)
    out["pt.row"] = np.asarray(pt.row, dtype=np.int64)
    out["pt.col"] = np.asarray(pt.col, dtype=np.int64)
    lens = [len(c) for c in pt.children]
    out["pt.child_ptr"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out["pt.child_idx"] = np.asarray([c for k in pt.children for c in k], dtype=np.int64)
    out["pt.adm"] = np.asarray(pt.admissible, dtype=np.uint8)
    out["rank.x_row"] = np.asarray(x.row_basis.rank, dtype=np.int64)
    out["rank.x_col"] = np.asarray(x.col_basis.rank, dtype=np.int64)
    out["rank.y_row"] = np.asarray(y.row_basis.rank, dtype=np.int64)
    out["rank.y_col"] = np.asarray(y.col_basis.rank, dtype=np.int64)
    out["rank.induced_row"] = np.asarray(qrow.q.rank, dtype=np.int64)
    out["rank.induced_col"] = np.asarray(qcol.q.rank, dtype=np.int64)
    out["rank.final_row"] = np.asarray(rs.q.rank, dtype=np.int64)
    out["rank.final_col"] = np.asarray(cs.q.rank, dtype=np.int64)
    gv = np.asarray(gaps.vals) if gaps.vals else np.ones(1)
    out["gap.phase1"] = np.asarray([gv[:n1].min() if n1 else 1.0])
    out["gap.phase2"] = np.asarray([gv[n1:].min() if len(gv) > n1 else 1.0])
    out["eps"] = np.asarray([eps])
    vs, zv, gv_, xyv, ztv, xr, yr = [], [], [], [], [], [], []
    for v in probes:
        vs.append(v)
        zv.append(h2mul.h2_matvec(z, v))
        gv_.append(h2mul.h2_matvec(g, v))
        xyv.append(h2mul.h2_matvec(x, h2mul.h2_matvec(y, v)))
        ztv.append(h2mul.h2_matvec_adjoint(z, v))
        if x_raw is not None:
            xr.append(h2mul.h2_matvec(x_raw, v))
            yr.append(h2mul.h2_matvec(y_raw, v))
    # the reference's own power-iteration error estimate |XY - Z|_2 / |XY|_2 (bench.py:147-174)
    from h2mul.bench import estimate_relative_spectral_error
    out["est.eps2"] = np.asarray([estimate_relative_spectral_error(x, y, z, steps=20, seed=0)])
    out["probe.v"] = np.asarray(vs)
    out["probe.zv"] = np.asarray(zv)
    out["probe.gv"] = np.asarray(gv_)
    out["probe.xyv"] = np.asarray(xyv)
    out["probe.ztv"] = np.asarray(ztv)
    if xr:
        out["probe.xraw_v"] = np.asarray(xr)
        out["probe.yraw_v"] = np.asarray(yr)
    return z, g


def config_case(name, h2mul, hp):
    """Seeded instances with the BASELINE configs' generators (reduced n where noted)."""
    spec = myprob.CONFIGS[name]
    n = spec["golden_n"]
    pts, wts = myprob.make_points(spec["geometry"], n, seed=0)
    kx = myprob.KERNEL_FNS[spec["kernel_x"]]
    ky = myprob.KERNEL_FNS[spec["kernel_y"]]
    if spec["geometry"] == "interval":
        # c1 is the reference's own log-1d problem with weights 1/n (problems.py:153-155)
        inst = h2mul.build_problem(h2mul.KernelProblem.log_1d(n, order=spec["order"]),
                                   eta=spec["eta"], leaf_size=spec["leaf"])
        x_raw = inst.h2
        y_raw = x_raw
    else:
        _, _, x_raw = ref_instance(h2mul, hp, pts, wts, kx, spec["leaf"], spec["eta"], spec["order"],
                                   "single-layer")
        if spec["kernel_y"] == spec["kernel_x"]:
            y_raw = x_raw
        else:
            _, _, y_raw = ref_instance(h2mul, hp, pts, wts, ky, spec["leaf"], spec["eta"],
                                       spec["order"], "single-layer")
    eps = spec["eps"]
    x = h2mul.recompress(x_raw, eps)
    y = x if y_raw is x_raw else h2mul.recompress(y_raw, eps)
    rng = np.random.default_rng(123)
    probes = [rng.standard_normal(n) for _ in range(3)]
    out = {"meta.n": np.asarray([n]), "meta.config": np.asarray([name])}
    small = name == "c1"   # full packed X/Y/Z only where they stay small (~2 MB)
    run_reference(h2mul, x, y, eps, out, probes, x_raw=x_raw, y_raw=y_raw,
                  keep_z=small, keep_inputs=small)
    return out


def random_pair_case(h2mul, seed, n, leaf, dim, tol, rank=3):
    """Unbalanced random X (I x J), Y (J x K) on three different trees (tests/util.py:9-48)."""
    rng = np.random.default_rng(seed)
    trees = [h2mul.build_cluster_tree(rng.uniform(0.0, 1.0, size=(n, dim)), leaf) for _ in range(3)]

    def basis(tree):
        leafm, xfer = {}, {}
        for t in range(tree.nnodes):
            if tree.is_leaf(t):
                leafm[t] = rng.standard_normal((tree.size(t), rank))
            for c in tree.children[t]:
                xfer[c] = rng.standard_normal((rank, rank))
        return h2mul.ClusterBasis(tree, [rank] * tree.nnodes, leafm, xfer)

    def h2(rows, cols):
        bt = h2mul.build_block_tree(rows, cols, 1.0)
        rb, cb = basis(rows), basis(cols)
        coup, near = {}, {}
        for b in range(bt.nblocks):
            if bt.is_admissible_leaf(b):
                coup[b] = rng.standard_normal((rank, rank))
            elif bt.is_inadmissible_leaf(b):
                near[b] = rng.standard_normal((rows.size(bt.row[b]), cols.size(bt.col[b])))
        return h2mul.H2Matrix(bt, rb, cb, coup, near)

    x = h2(trees[0], trees[1])
    y = h2(trees[1], trees[2])
    probes = [rng.standard_normal(n) for _ in range(3)]
    out = {"meta.n": np.asarray([n]), "meta.config": np.asarray([f"random-s{seed}"])}
    z, g = run_reference(h2mul, x, y, tol, out, probes)
    if n <= 256:
        out["dense.z"] = h2mul.to_dense(z)
        out["dense.g"] = h2mul.to_dense(g)
        out["dense.xy"] = h2mul.to_dense(x) @ h2mul.to_dense(y)
    return out


def main():
    h2mul, hp = _ref()
    out_dir = os.environ.get("GOLDEN_OUT", HERE)
    os.makedirs(out_dir, exist_ok=True)
    cases = {}
    for name in ("c1", "c2", "c3", "c4", "c5"):
        cases[name] = config_case(name, h2mul, hp)
    cases["rand_s0_tol1e-3"] = random_pair_case(h2mul, 0, 48, 4, 1, 1e-3)
    cases["rand_s1_tol0"] = random_pair_case(h2mul, 1, 40, 4, 1, 0.0)
    cases["rand_s2_2d"] = random_pair_case(h2mul, 2, 96, 6, 2, 1e-4)
    cases["rand_s3_2d_tol0"] = random_pair_case(h2mul, 3, 64, 5, 2, 0.0)
    for name, out in cases.items():
        path = os.path.join(out_dir, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB, ranks induced "
              f"{out['rank.induced_row'].max()} final {out['rank.final_row'].max()}, "
              f"gaps {out['gap.phase1'][0]:.1e}/{out['gap.phase2'][0]:.1e}")


if __name__ == "__main__":
    main()
