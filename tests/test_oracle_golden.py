"""Pin the CPU oracle (oracle/h2_oracle.py) against golden vectors produced by the
reference h2mul itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import oracle as O
from helpers import CONFIG_CASES, RANDOM_CASES, golden_inputs_oracle, load, rebuild_raw, rel, to_oracle


@pytest.mark.parametrize("name", CONFIG_CASES)
def test_problem_builder_matches_reference(name):
    """paper_2309_09061_b200.problems rebuilds the reference's raw interpolation inputs."""
    d = load(name)
    xr, yr = rebuild_raw(d)
    from paper_2309_09061_b200.h2 import h2_matvec_host
    for i, v in enumerate(d["probe.v"]):
        assert rel(h2_matvec_host(xr, v), d["probe.xraw_v"][i]) < 1e-13
        assert rel(h2_matvec_host(yr, v), d["probe.yraw_v"][i]) < 1e-13


def _check_case(d, x, y):
    eps = float(d["eps"][0])
    pt = O.o_product_tree(x.bt, y.bt)
    assert pt.row == list(d["pt.row"]) and pt.col == list(d["pt.col"])
    assert [int(a) for a in pt.adm] == list(d["pt.adm"])
    final, induced, _, info = O.o_run_stages(x, y, x.bt, eps)
    assert info["qrow"].q.rank == list(d["rank.induced_row"])
    assert info["qcol"].q.rank == list(d["rank.induced_col"])
    assert info["rows"].q.rank == list(d["rank.final_row"])
    assert info["cols"].q.rank == list(d["rank.final_col"])
    for i, v in enumerate(d["probe.v"]):
        assert rel(O.o_matvec(final, v), d["probe.zv"][i]) < 1e-11
        assert rel(O.o_matvec(induced, v), d["probe.gv"][i]) < 1e-11
        assert rel(O.o_matvec_t(final, v), d["probe.ztv"][i]) < 1e-11
    return final


@pytest.mark.parametrize("name", RANDOM_CASES + ["c1"])
def test_oracle_matches_reference_packed_inputs(name):
    d = load(name)
    x, y = golden_inputs_oracle(d)
    final = _check_case(d, x, y)
    if "dense.z" in d:
        assert rel(O.o_to_dense(final), d["dense.z"]) < 1e-11


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_oracle_matches_reference_rebuilt_inputs(name):
    d = load(name)
    x, y = golden_inputs_oracle(d)
    assert x.rb.rank == list(d["rank.x_row"]) and y.cb.rank == list(d["rank.y_col"])
    _check_case(d, x, y)


@pytest.mark.parametrize("name", ["c1", "rand_s0_tol1e-3", "rand_s2_2d"])
def test_oracle_error_estimate_matches_reference(name):
    """The oracle's power-iteration estimate (bench.py:147-174) on the reference's own X, Y, Z."""
    import oracle as O
    d = load(name)
    x, y, z = O.o_from_packed(d, "x/"), O.o_from_packed(d, "y/"), O.o_from_packed(d, "z/")
    est = O.o_relative_spectral_error(x, y, z, steps=20, seed=0)
    assert abs(est - float(d["est.eps2"][0])) <= 1e-8 * float(d["est.eps2"][0])
