"""CPU-tier checks of the native library: it loads, exports every symbol include/h2g.h declares,
and its host-only planner builds the reference's product block tree (trees.py:314-359)."""

import os
import re

import numpy as np
import pytest

from helpers import CONFIG_CASES, RANDOM_CASES, load, rebuild_raw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "h2g.h")).read()
    return sorted(set(re.findall(r"\b(h2g_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2309_09061_b200 import _native as N
    lib = N.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.SIGNATURES), set(syms) ^ set(N.SIGNATURES)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2309_09061_b200", "libh2g.so")
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("name", RANDOM_CASES + ["c1"])
def test_native_product_tree_matches_reference(name):
    from paper_2309_09061_b200.packed import unpack_h2
    from paper_2309_09061_b200.planner import product_tree
    d = load(name)
    x = unpack_h2(d, "x/")
    y = unpack_h2(d, "y/", rows=x.block_tree.cols)
    pt, cnt = product_tree(x.block_tree, y.block_tree, with_counts=True)
    assert pt.row == list(d["pt.row"]) and pt.col == list(d["pt.col"])
    assert [int(a) for a in pt.admissible] == list(d["pt.adm"])
    f = pt.flat()
    assert np.array_equal(f["child_ptr"], d["pt.child_ptr"]) and np.array_equal(f["child_idx"], d["pt.child_idx"])
    assert cnt["a"] + cnt["b"] + cnt["c"] > 0


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_native_product_tree_configs(name):
    from paper_2309_09061_b200.planner import product_tree
    d = load(name)
    xr, yr = rebuild_raw(d)
    pt = product_tree(xr.block_tree, yr.block_tree)
    assert pt.row == list(d["pt.row"]) and pt.col == list(d["pt.col"])
    assert [int(a) for a in pt.admissible] == list(d["pt.adm"])


def test_product_tree_rejects_mismatched_middle_tree():
    from paper_2309_09061_b200 import InvalidInputError
    from paper_2309_09061_b200.trees import build_block_tree, build_cluster_tree, build_product_block_tree
    rng = np.random.default_rng(0)
    a = build_cluster_tree(rng.uniform(size=(40, 1)), 4)
    b = build_cluster_tree(rng.uniform(size=(44, 1)), 4)
    with pytest.raises(InvalidInputError):
        build_product_block_tree(build_block_tree(a, a, 1.0), build_block_tree(b, b, 1.0))
