"""Shared test helpers: fixtures, host <-> oracle bridges, probe comparisons."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CONFIG_CASES = ["c1", "c2", "c3", "c4", "c5"]
RANDOM_CASES = ["rand_s0_tol1e-3", "rand_s1_tol0", "rand_s2_2d", "rand_s3_2d_tol0", "rand_s5_zero_coup",
                "rand_s6_zero_coup_tol0"]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def to_oracle(g):
    """Package H2Matrix -> oracle OH2 through the packed layout."""
    from oracle import o_from_packed
    from paper_2309_09061_b200.packed import pack_h2
    return o_from_packed(pack_h2(g))


def golden_inputs_oracle(d):
    """Oracle X, Y of a fixture: packed inputs when stored, else rebuilt + recompressed."""
    from oracle import o_from_packed, o_recompress
    if "x/bt.row" in d:
        x = o_from_packed(d, "x/")
        y = o_from_packed(d, "y/", rows=x.bt.cols) if "y/bt.row" in d else x
        return x, y
    xr, yr = rebuild_raw(d)
    x = o_recompress(to_oracle(xr), float(d["eps"][0]))
    y = x if yr is xr else o_recompress(to_oracle(yr), float(d["eps"][0]))
    return x, y


def rebuild_raw(d):
    from paper_2309_09061_b200.problems import build_config
    name = str(d["meta.config"][0])
    xr, yr, _ = build_config(name, n=int(d["meta.n"][0]))
    return xr, yr


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
