"""Host logic: packed layout round trip, cluster/block tree builders vs the fixtures, error types."""

import numpy as np
import pytest

from helpers import load
from paper_2309_09061_b200 import InvalidInputError
from paper_2309_09061_b200.h2 import h2_matvec_host, to_dense
from paper_2309_09061_b200.packed import pack_h2, unpack_h2
from paper_2309_09061_b200.problems import build_config, make_points
from paper_2309_09061_b200.trees import build_block_tree, build_cluster_tree


def test_packed_roundtrip():
    d = load("rand_s2_2d")
    x = unpack_h2(d, "x/")
    d2 = pack_h2(x)
    for k, v in d2.items():
        assert np.array_equal(v, d["x/" + k]), k
    x2 = unpack_h2(d2)
    v = d["probe.v"][0]
    assert np.array_equal(h2_matvec_host(x, v), h2_matvec_host(x2, v))


def test_cluster_tree_known_answer():
    # 8 points, leaf size 1 -> 15 nodes in preorder (reference test_trees.py:12-26)
    t = build_cluster_tree(np.arange(8.0), 1)
    assert t.nnodes == 15
    assert t.children[0] == (1, 8)
    assert [t.size(i) for i in t.leaves()] == [1] * 8


def test_block_tree_tiles_the_matrix():
    rng = np.random.default_rng(3)
    rows = build_cluster_tree(rng.uniform(size=(60, 2)), 5)
    cols = build_cluster_tree(rng.uniform(size=(50, 2)), 4)
    bt = build_block_tree(rows, cols, 1.0)
    cover = np.zeros((60, 50), int)
    for b in bt.leaves():
        cover[rows.index_range(bt.row[b]), cols.index_range(bt.col[b])] += 1
    assert (cover == 1).all()


def test_invalid_inputs_raise_reference_errors():
    with pytest.raises(InvalidInputError):
        build_cluster_tree(np.zeros((0, 2)), 4)
    with pytest.raises(InvalidInputError):
        build_cluster_tree(np.zeros((4, 2)), 0)
    t = build_cluster_tree(np.arange(8.0), 2)
    with pytest.raises(InvalidInputError):
        build_block_tree(t, t, 0.0)
    with pytest.raises(InvalidInputError):
        make_points("torus", 10)


def test_interpolation_is_accurate_small():
    x, _, spec = build_config("c1", n=256)
    dense = to_dense(x)
    pts = x.block_tree.rows.points[:, 0]
    w = 1.0 / 256
    r = np.abs(pts[:, None] - pts[None, :])
    ref = np.where(r > 0, -np.log(np.where(r > 0, r, 1.0)), 0.0) * w * w
    assert np.linalg.norm(dense - ref, 2) / np.linalg.norm(ref, 2) < 1e-3


def test_binary_packed_file_roundtrip(tmp_path):
    """save_h2 / load_h2 (the binary replacement of h2_to_json / h2_from_json, h2.py:314-397)."""
    from paper_2309_09061_b200.packed import load_h2, load_packed, save_h2, FORMAT
    d = load("rand_s0_tol1e-3")
    g = unpack_h2(d, "x/")
    path = tmp_path / "x.npz"
    save_h2(path, g)
    g2 = load_h2(path)
    assert g2.block_tree.row == g.block_tree.row and g2.block_tree.col == g.block_tree.col
    assert list(g2.row_basis.rank) == list(g.row_basis.rank)
    v = np.random.default_rng(0).standard_normal(g.shape[1])
    assert np.array_equal(h2_matvec_host(g2, v), h2_matvec_host(g, v))
    p1, p2 = pack_h2(g), load_packed(path)[0]
    assert set(p1) == set(p2) and all(np.array_equal(p1[k], p2[k]) for k in p1)
    bad = tmp_path / "bad.npz"
    np.savez(bad, x=np.zeros(1))
    with pytest.raises(ValueError, match=FORMAT):
        load_h2(bad)
