"""GPU parity: the CUDA product path (through the C ABI) against the reference's golden vectors
and the live CPU oracle.

Bars (BASELINE.json north_star): identical block structure; per-cluster ranks equal; relative
error ||(Z_gpu - Z_ref) v|| / ||Z_ref v|| <= 10 eps on probe vectors (tol = 0 cases: <= 1e-10);
||Z_gpu v - X(Y v)|| / ||X(Y v)|| within the reference's own value x 1.1 (or eps).
"""

import os

import numpy as np
import pytest

from helpers import CONFIG_CASES, RANDOM_CASES, load, rebuild_raw, rel

pytestmark = pytest.mark.gpu


def _P():
    import paper_2309_09061_b200 as P
    return P


def _probe_tol(eps):
    return 1e-10 if eps == 0 else 10 * eps


def _inputs(d):
    P = _P()
    from paper_2309_09061_b200.packed import unpack_h2
    eps = float(d["eps"][0])
    if "x/bt.row" in d:
        x = unpack_h2(d, "x/")
        y = unpack_h2(d, "y/", rows=x.block_tree.cols)
        return x, y, eps
    xr, yr = rebuild_raw(d)
    x = P.recompress(xr, eps)
    y = x if yr is xr else P.recompress(yr, eps)
    assert list(x.row_basis.rank) == list(d["rank.x_row"])   # GPU recompress = reference recompress
    assert list(y.col_basis.rank) == list(d["rank.y_col"])
    return x, y, eps


@pytest.mark.parametrize("name", RANDOM_CASES + CONFIG_CASES)
def test_golden_parity(name):
    P = _P()
    from paper_2309_09061_b200.h2 import h2_matvec_host
    d = load(name)
    x, y, eps = _inputs(d)
    g = P.multiply(x, y, eps)
    bt = g.block_tree
    assert bt.row == list(d["pt.row"]) and bt.col == list(d["pt.col"])
    assert [int(a) for a in bt.admissible] == list(d["pt.adm"])
    assert list(g.row_basis.rank) == list(d["rank.induced_row"])
    assert list(g.col_basis.rank) == list(d["rank.induced_col"])
    z = P.coarsen(g, x.block_tree, eps)
    assert list(z.row_basis.rank) == list(d["rank.final_row"])
    assert list(z.col_basis.rank) == list(d["rank.final_col"])
    tol = _probe_tol(eps)
    for i, v in enumerate(d["probe.v"]):
        assert rel(h2_matvec_host(g, v), d["probe.gv"][i]) <= tol
        assert rel(h2_matvec_host(z, v), d["probe.zv"][i]) <= tol
        ref_xy = rel(d["probe.zv"][i], d["probe.xyv"][i])
        assert rel(h2_matvec_host(z, v), d["probe.xyv"][i]) <= max(eps, 1.1 * ref_xy, 1e-12)


def _oracle_pair(seed, n=64, leaf=4, dim=2, rank=3, zero=False):
    """Random unbalanced pair on three trees (reference tests/util.py:9-48), in package containers."""
    from paper_2309_09061_b200.h2 import ClusterBasis, H2Matrix
    from paper_2309_09061_b200.trees import build_block_tree, build_cluster_tree
    rng = np.random.default_rng(seed)
    trees = [build_cluster_tree(rng.uniform(size=(n, dim)), leaf) for _ in range(3)]

    def basis(tree):
        lm = {t: rng.standard_normal((tree.size(t), rank)) for t in range(tree.nnodes) if tree.is_leaf(t)}
        xf = {c: rng.standard_normal((rank, rank)) for t in range(tree.nnodes) for c in tree.children[t]}
        return ClusterBasis(tree, [rank] * tree.nnodes, lm, xf)

    def h2(r, c):
        bt = build_block_tree(r, c, 1.0)
        s = 0.0 if zero else 1.0
        cp = {b: s * rng.standard_normal((rank, rank)) for b in bt.admissible_leaves()}
        nf = {b: s * rng.standard_normal((r.size(bt.row[b]), c.size(bt.col[b]))) for b in bt.inadmissible_leaves()}
        return H2Matrix(bt, basis(r), basis(c), cp, nf)

    return h2(trees[0], trees[1]), h2(trees[1], trees[2])


@pytest.mark.parametrize("seed,tol", [(11, 1e-3), (12, 0.0), (13, 1e-6)])
def test_live_oracle_random(seed, tol):
    import oracle as O
    from helpers import to_oracle
    P = _P()
    from paper_2309_09061_b200.h2 import h2_matvec_host
    x, y = _oracle_pair(seed)
    ox, oy = to_oracle(x), to_oracle(y)
    og = O.o_multiply(ox, oy, tol)
    oz = O.o_coarsen(og, ox.bt, tol)
    z = P.multiply_coarsen(x, y, tol)
    assert list(z.row_basis.rank) == oz.rb.rank and list(z.col_basis.rank) == oz.cb.rank
    rng = np.random.default_rng(seed)
    for _ in range(3):
        v = rng.standard_normal(x.shape[1])
        assert rel(h2_matvec_host(z, v), O.o_matvec(oz, v)) <= _probe_tol(tol)


def test_exact_at_zero_tolerance_dense():
    """tol = 0 reproduces the dense product (reference test_acceptance.py:35-49)."""
    P = _P()
    from paper_2309_09061_b200.h2 import to_dense
    from paper_2309_09061_b200.problems import build_config
    x, _, _ = build_config("c1", n=512)
    dx = to_dense(x)
    ref = dx @ dx
    g = P.multiply(x, x, 0.0)
    z = P.coarsen(g, x.block_tree, 0.0)
    nref = np.linalg.norm(ref, 2)
    assert np.linalg.norm(to_dense(g) - ref, 2) / nref <= 1e-10
    assert np.linalg.norm(to_dense(z) - ref, 2) / nref <= 1e-10


def test_zero_inputs_give_zero_product():
    """Exact zero-norm skips (weights.py:88, induced.py:123, coarsening.py:239)."""
    P = _P()
    from paper_2309_09061_b200.h2 import to_dense
    x, y = _oracle_pair(21, zero=True)
    z = P.multiply_coarsen(x, y, 1e-4)
    assert np.abs(to_dense(z)).max() == 0.0


def test_max_rank_cap():
    """max_rank caps every induced and final rank (dense.py:99-100, induced.py:131)."""
    P = _P()
    import oracle as O
    from helpers import to_oracle
    x, y = _oracle_pair(31)
    g = P.multiply(x, y, 1e-8, max_rank=5)
    assert max(g.row_basis.rank) <= max(5, 3) and max(g.col_basis.rank) <= max(5, 3)
    og = O.o_multiply(to_oracle(x), to_oracle(y), 1e-8, max_rank=5)
    assert list(g.row_basis.rank) == og.rb.rank
    z = P.coarsen(g, x.block_tree, 1e-8, max_rank=4)
    assert max(z.row_basis.rank) <= 4 and max(z.col_basis.rank) <= 4


def test_error_behaviour():
    P = _P()
    from paper_2309_09061_b200 import InvalidInputError
    from paper_2309_09061_b200.trees import build_block_tree, build_cluster_tree
    x, y = _oracle_pair(41)
    with pytest.raises(InvalidInputError):
        P.multiply(x, y, -1.0)
    with pytest.raises(InvalidInputError):
        P.multiply(y, _oracle_pair(42, n=70)[0], 1e-3)   # middle trees differ
    g = P.multiply(x, y, 1e-3)
    other = build_cluster_tree(np.random.default_rng(1).uniform(size=(70, 2)), 4)
    with pytest.raises(InvalidInputError):
        P.coarsen(g, build_block_tree(other, other, 1.0), 1e-3)


def test_native_library_loaded_from_repo():
    P = _P()
    from paper_2309_09061_b200 import _native
    x, y = _oracle_pair(51)
    P.multiply_coarsen(x, y, 1e-3)
    maps = open("/proc/self/maps").read()
    assert os.path.realpath(_native.LIB_PATH) in maps


def test_packed_host_buffer_path():
    """multiply_coarsen_packed (packed host buffers over the C ABI) equals the object path."""
    P = _P()
    import torch
    from paper_2309_09061_b200.packed import pack_h2, unpack_h2
    d = load("rand_s0_tol1e-3")
    x, y, eps = _inputs(d)
    z = P.multiply_coarsen(x, y, eps)
    xp, yp = pack_h2(x), pack_h2(y)
    pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in xp.items() if k.endswith("data")}
    xp.update(pinned)
    zp = P.multiply_coarsen_packed(xp, x.block_tree, yp, y.block_tree, eps)
    zp.update({"bt.row": d["x/bt.row"], "bt.col": d["x/bt.col"], "bt.child_ptr": d["x/bt.child_ptr"],
               "bt.child_idx": d["x/bt.child_idx"], "bt.adm": d["x/bt.adm"]})
    z2 = unpack_h2(zp, rows=x.block_tree.rows, cols=x.block_tree.cols)
    assert list(z2.row_basis.rank) == list(z.row_basis.rank)
    v = np.random.default_rng(3).standard_normal(x.shape[1])
    from paper_2309_09061_b200.h2 import h2_matvec_host
    assert rel(h2_matvec_host(z2, v), h2_matvec_host(z, v)) <= 1e-13
    # preallocated output: Z's dense blocks shared with G are prefetched into out["near_data"]
    # during phase 2 (h2g_coarsen_prefetch); the result must be bit-identical, every entry written
    keys = [k for k in zp if not k.startswith("bt.")]
    for pad in (7, 0):
        out = {k: torch.full((zp[k].size + pad,), float("nan") if k.endswith("data") else -7,
                             dtype=torch.float64 if k.endswith("data") else torch.int64).pin_memory().numpy()
               for k in keys}
        z3 = P.multiply_coarsen_packed(xp, x.block_tree, yp, y.block_tree, eps, out=out)
        for k in keys:
            assert np.array_equal(z3[k], zp[k]), k
    # a nearfield buffer too small for Z: no prefetch, a fresh array is returned
    out = {"near_data": np.zeros(max(0, zp["near_data"].size - 1))}
    z4 = P.multiply_coarsen_packed(xp, x.block_tree, yp, y.block_tree, eps, out=out)
    assert np.array_equal(z4["near_data"], zp["near_data"])


def test_deferred_nearfield_upload_first_uses():
    """An asynchronous upload defers the nearfield copy to the matrix's first use (H2::start_near): every
    first use -- matvec, download, coarsen, recompress, multiply -- must see the complete matrix."""
    P = _P()
    import torch
    from paper_2309_09061_b200.packed import pack_h2
    d = load("rand_s0_tol1e-3")
    x, y, eps = _inputs(d)
    xp = pack_h2(x)
    xp.update({k: torch.from_numpy(v).pin_memory().numpy() for k, v in xp.items() if k.endswith("data")})
    ref = P.DeviceH2.upload_packed(xp, x.block_tree)
    v = np.random.default_rng(11).standard_normal(x.shape[1])
    want = ref.matvec(v)
    up = lambda: P.DeviceH2.upload_packed(xp, x.block_tree, asynchronous=True)
    assert torch.equal(up().matvec(v), want)
    got = up().download_packed()
    for k, a in ref.download_packed().items():
        assert np.array_equal(got[k], a), k
    zr = P.coarsen(ref, x.block_tree, eps)
    assert torch.equal(P.coarsen(up(), x.block_tree, eps).matvec(v), zr.matvec(v))
    assert torch.equal(P.recompress(up(), eps).matvec(v), P.recompress(ref, eps).matvec(v))
    a, b = up(), up()
    g = P.multiply(a, b, eps)
    assert torch.equal(g.matvec(v), P.multiply(ref, ref, eps).matvec(v))
    # the host array may be released after a synchronising call even if the matrix was not used yet
    # (include/h2g.h): the deferred copy starts, and the copy stream drains, inside ctx.synchronize()
    near = xp["near_data"]
    xq = dict(xp)
    xq["near_data"] = torch.from_numpy(near.copy()).pin_memory().numpy()
    late = P.DeviceH2.upload_packed(xq, x.block_tree, asynchronous=True)
    late.ctx.synchronize()
    xq["near_data"][:] = np.nan  # stands for freed memory
    assert torch.equal(late.matvec(v), want)


@pytest.mark.parametrize("name", ["rand_s0_tol1e-3", "c1"])
def test_gpu_matvec_matches_host(name):
    """GPU h2_matvec / adjoint (h2.py:224-267) against the host restatement on Z and X."""
    P = _P()
    import torch
    from paper_2309_09061_b200.h2 import h2_matvec_host
    d = load(name)
    x, y, eps = _inputs(d)
    dx = P.DeviceH2.upload(x)
    z = P.coarsen(P.multiply(dx, P.DeviceH2.upload(y) if y is not x else dx, eps), dx.block_tree, eps)
    zh = z.download()
    rng = np.random.default_rng(5)
    for g, gh in ((dx, x), (z, zh)):
        nr, nc = g.shape
        v = rng.standard_normal(nc)
        u = rng.standard_normal(nr)
        gv = g.matvec(torch.from_numpy(v).cuda()).cpu().numpy()
        assert rel(gv, h2_matvec_host(gh, v)) <= 1e-13
        gtu = g.matvec(torch.from_numpy(u).cuda(), trans=True).cpu().numpy()
        # adjoint identity <G v, u> = <v, G^T u>
        assert abs(gv @ u - v @ gtu) <= 1e-12 * np.linalg.norm(gv) * np.linalg.norm(u)


@pytest.mark.parametrize("name", ["c1"] + RANDOM_CASES)
def test_gpu_matvec_on_reference_z(name):
    """The GPU matvec / adjoint (csrc/matvec.cu) applied to the reference's OWN product Z (stored
    packed in the fixture) reproduces the reference's own h2_matvec / h2_matvec_adjoint outputs
    (h2.py:224-267, recorded as probe.zv / probe.ztv by make_golden.py:198-215): the same matrix, so
    only the summation order differs (<= 1e-13)."""
    P = _P()
    import torch
    from paper_2309_09061_b200.packed import unpack_h2
    d = load(name)
    if "z/bt.row" not in d:
        pytest.skip("fixture without the reference Z")
    x = unpack_h2(d, "x/") if "x/bt.row" in d else None
    zr = unpack_h2(d, "z/", rows=x.block_tree.rows if x is not None else None,
                   cols=x.block_tree.cols if x is not None else None)
    dz = P.DeviceH2.upload(zr)
    for i, v in enumerate(d["probe.v"]):
        vt = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        assert rel(dz.matvec(vt).cpu().numpy(), d["probe.zv"][i]) <= 1e-13
        assert rel(dz.matvec(vt, trans=True).cpu().numpy(), d["probe.ztv"][i]) <= 1e-13


@pytest.mark.parametrize("name", RANDOM_CASES + CONFIG_CASES)
def test_gpu_error_estimate_matches_reference(name):
    """GPU power-iteration |XY - Z|_2 / |XY|_2 (bench.py:147-174) against the reference's own value."""
    P = _P()
    d = load(name)
    x, y, eps = _inputs(d)
    dx = P.DeviceH2.upload(x)
    dy = dx if y is x else P.DeviceH2.upload(y)
    z = P.coarsen(P.multiply(dx, dy, eps), dx.block_tree, eps)
    est = P.estimate_relative_spectral_error(dx, dy, z, steps=20, seed=0)
    ref = float(d["est.eps2"][0])
    if ref <= 1e-12:  # exact product (tol 0 or ranks below the tolerance): rounding noise only
        assert est <= 1e-12
    else:
        assert abs(est - ref) <= 1e-4 * ref


@pytest.mark.parametrize("name,n", [("c2", 2048), ("c3", 2048), ("c4", 4096)])
def test_gpu_input_builder_matches_host(name, n):
    """GPU kernel evaluation (h2g_h2_build_kernel) reproduces the host builder (problems.py:295-332),
    and its recompressed input has the reference's per-cluster ranks."""
    P = _P()
    import torch
    from paper_2309_09061_b200.problems import build_config, build_config_device
    xr, yr, spec = build_config(name, n=n)
    dxr, dyr, _ = build_config_device(name, n=n)
    hx = P.DeviceH2.upload(xr)
    v = torch.from_numpy(np.random.default_rng(7).standard_normal(n)).cuda()
    assert rel(dxr.matvec(v).cpu().numpy(), hx.matvec(v).cpu().numpy()) <= 1e-13
    if yr is not xr:
        hy = P.DeviceH2.upload(yr)
        assert rel(dyr.matvec(v).cpu().numpy(), hy.matvec(v).cpu().numpy()) <= 1e-13
    d = load(name)
    x = P.recompress(dxr, spec["eps"])
    assert list(x.download().row_basis.rank) == list(d["rank.x_row"])


def test_device_save_load_roundtrip(tmp_path):
    """DeviceH2.save / DeviceH2.load through the binary packed file: bit-identical Z."""
    P = _P()
    d = load("rand_s2_2d")
    x, y, eps = _inputs(d)
    dx = P.DeviceH2.upload(x)
    z = P.coarsen(P.multiply(dx, P.DeviceH2.upload(y), eps), dx.block_tree, eps)
    path = tmp_path / "z.npz"
    z.save(path)
    z2 = P.DeviceH2.load(path)
    a, b = z.download_packed(), z2.download_packed()
    assert set(a) == set(b) and all(np.array_equal(a[k], b[k]) for k in a)


def _expand(basis, t):
    from paper_2309_09061_b200.h2 import expand_basis
    return expand_basis(basis, t)


@pytest.mark.parametrize("seed,tol", [(30, 0.1), (31, 1e-3), (32, 0.0)])
def test_induced_and_final_bases_are_isometric(seed, tol):
    """Q_t^T Q_t = I for every cluster of the induced (phase 1) and final (phase 2) bases
    (reference test_induced.py:97-104, test_coarsening.py:153-166)."""
    P = _P()
    x, y = _oracle_pair(seed)
    g = P.multiply(x, y, tol)
    z = P.coarsen(g, x.block_tree, tol)
    for basis in (g.row_basis, g.col_basis, z.row_basis, z.col_basis):
        for t in range(basis.tree.nnodes):
            q = _expand(basis, t)
            assert np.linalg.norm(q.T @ q - np.eye(q.shape[1])) <= 1e-11


@pytest.mark.parametrize("seed", range(3))
def test_induced_bases_protect_the_input_bases(seed):
    """span V_X,t is inside the induced row basis Q_t, span W_Y,r inside the column basis
    (reference test_induced.py:85-94: Q_t basis_change_t = V_X,t)."""
    P = _P()
    x, y = _oracle_pair(seed + 20)
    g = P.multiply(x, y, 0.3)
    for q_basis, v_basis in ((g.row_basis, x.row_basis), (g.col_basis, y.col_basis)):
        for t in range(q_basis.tree.nnodes):
            q, v = _expand(q_basis, t), _expand(v_basis, t)
            assert np.linalg.norm(v - q @ (q.T @ v)) <= 1e-12 * (1 + np.linalg.norm(v))


def test_block_relative_error_per_coarse_leaf():
    """Coarsening onto a coarser admissibility: every coarse admissible leaf within 10 eps of the
    product block (reference test_coarsening.py:190-206)."""
    P = _P()
    from paper_2309_09061_b200.h2 import to_dense
    from paper_2309_09061_b200.trees import build_block_tree
    eps = 1e-4
    x, y = _oracle_pair(13)
    g = P.multiply(x, y, eps)
    coarse = build_block_tree(g.block_tree.rows, g.block_tree.cols, 1.0)
    z = P.coarsen(g, coarse, eps)
    ref, got = to_dense(g), to_dense(z)
    rows, cols = coarse.rows, coarse.cols
    checked = 0
    for b in range(coarse.nblocks):
        if coarse.children[b] or not coarse.admissible[b]:
            continue
        t, r = coarse.row[b], coarse.col[b]
        sr = slice(int(rows.start[t]), int(rows.stop[t]))
        sc = slice(int(cols.start[r]), int(cols.stop[r]))
        blk_ref, blk_got = ref[sr, sc], got[sr, sc]
        assert np.linalg.norm(blk_got - blk_ref, 2) <= 10 * eps * np.linalg.norm(blk_ref, 2) + 1e-13
        checked += 1
    assert checked > 0


@pytest.mark.parametrize("env", [{"H2G_NO_GRAM": "1", "H2G_NO_GRAM_QR": "1"},  # Householder TSQR everywhere
                                 {"H2G_GRAM_PROT": "1"},                         # Gram for protected SVDs too
                                 {"H2G_GRAM_TILED": "1", "H2G_NORM_CTA": "1"},   # 64x64 Gram tiles, smem Lanczos
                                 {"H2G_SYNC_EXPAND": "1", "H2G_SERIAL": "1"}])   # expansions / passes in line
def test_alternative_factorisation_paths(env):
    """The factorisation paths selected by environment switches (read once per process) keep every
    golden gate: the Householder TSQR + QRCP path that the double-double Gram path replaced by
    default, the opt-in Gram path for the protected-basis SVDs of phase 1, the 64 x 64-tile Gram
    decomposition and shared-memory Lanczos norms the block-list Gram and register-tile norms
    replaced, and the push-down expansions / row and column passes on the main stream."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", os.path.join(here, "test_gpu_parity.py"),
           "-k", "test_golden_parity", "-m", "gpu"]
    r = subprocess.run(cmd, env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
