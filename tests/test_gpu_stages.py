"""Stage-level drop-ins (paper_2309_09061_b200/stages.py, C ABI "Stage-level entry points") against
the reference's golden vectors and the CPU oracle, one stage at a time.

* The stage-by-stage replay of the reference harness (bench.py:195-237) gives every per-cluster
  rank of the golden fixtures and the same Z as the fused multiply / coarsen.
* Per-stage results against the oracle: basis products entrywise, basis / total weights through
  their Gram (R^T R: the factors are unique up to row signs), induced bases' defining identities
  (reference test_induced.py:85-118), block norms entrywise.
* the ORACLE's induced bases and basis product fed to the GPU assembly give the
  oracle's G entrywise (couplings and nearfield, <= 1e-13), so assembly parity is pinned without
  any basis-sign ambiguity.
"""

import numpy as np
import pytest

from helpers import load, rel, to_oracle

pytestmark = pytest.mark.gpu


def _P():
    import paper_2309_09061_b200 as P
    return P


def _case(name="rand_s2_2d"):
    from paper_2309_09061_b200.packed import unpack_h2
    d = load(name)
    x = unpack_h2(d, "x/")
    y = unpack_h2(d, "y/", rows=x.block_tree.cols)
    return d, x, y, float(d["eps"][0])


def _replay(P, dx, dy, eps, scaling=True):
    """The reference harness's stage sequence (bench.py:201-237) through the stage drop-ins."""
    pxy = P.cluster_basis_product(dx.col_basis, dy.row_basis)
    zy = P.total_weights(dy, P.basis_weights(dy.col_basis), scaling=scaling)
    zxt = P.total_weights(dx.transposed(), P.basis_weights(dx.row_basis), scaling=scaling)
    qrow = P.compress_induced_row_basis(dx, dy, zy, pxy, eps, scale_blocks=scaling)
    qcol = P.compress_induced_col_basis(dx, dy, zxt, pxy, eps, scale_blocks=scaling)
    g = P.assemble_product(dx, dy, qrow, qcol, pxy)
    coarse = dx.block_tree
    cn, nn = P.block_norms(g) if scaling else (None, None)
    rs = P.build_coarse_row_basis(g, coarse, eps, scale_blocks=scaling, coupling_norms=cn, nearfield_norms=nn)
    cs = P.build_coarse_col_basis(g, coarse, eps, scale_blocks=scaling, coupling_norms=cn, nearfield_norms=nn)
    z = P.project_final(g, rs, cs, coarse)
    return dict(pxy=pxy, zy=zy, zxt=zxt, qrow=qrow, qcol=qcol, g=g, rs=rs, cs=cs, z=z)


@pytest.mark.parametrize("name", ["rand_s2_2d", "rand_s0_tol1e-3", "c1"])
def test_stage_replay_matches_golden_and_fused(name):
    import torch
    P = _P()
    from paper_2309_09061_b200.device import DeviceH2
    d, x, y, eps = _case(name)
    dx, dy = DeviceH2.upload(x), DeviceH2.upload(y)
    r = _replay(P, dx, dy, eps)
    assert list(r["qrow"].q.rank) == list(d["rank.induced_row"])
    assert list(r["qcol"].q.rank) == list(d["rank.induced_col"])
    assert list(r["rs"].q.rank) == list(d["rank.final_row"])
    assert list(r["cs"].q.rank) == list(d["rank.final_col"])
    zr, zc = r["z"].ranks()
    assert list(zr) == list(d["rank.final_row"]) and list(zc) == list(d["rank.final_col"])
    zf = P.coarsen(P.multiply(dx, dy, eps), dx.block_tree, eps)
    for i, v in enumerate(d["probe.v"]):
        vt = torch.from_numpy(v).cuda()
        zv = r["z"].matvec(vt).cpu().numpy()
        assert rel(zv, d["probe.zv"][i]) <= 10 * eps
        assert rel(zv, zf.matvec(vt).cpu().numpy()) <= 1e-13
        assert rel(r["g"].matvec(vt).cpu().numpy(), d["probe.gv"][i]) <= 10 * eps


def test_stages_against_oracle():
    P = _P()
    import oracle as O
    from paper_2309_09061_b200.device import DeviceH2
    from paper_2309_09061_b200.h2 import expand_basis
    d, x, y, eps = _case("rand_s2_2d")
    ox, oy = to_oracle(x), to_oracle(y)
    dx, dy = DeviceH2.upload(x), DeviceH2.upload(y)
    r = _replay(P, dx, dy, eps)
    # basis product (h2.py:127-145): unique, entrywise
    opxy = O.o_basis_product(ox.cb, oy.rb)
    gp = r["pxy"].p
    for s, m in opxy.items():
        assert np.abs(gp[s] - m).max() <= 1e-13 * max(1.0, np.abs(m).max())
    # basis weights / total weights: R and Z are unique up to row signs -> compare R^T R
    orw = O.o_basis_weights(oy.cb)
    grw = P.basis_weights(dy.col_basis).r
    for s, m in orw.items():
        a, b = grw[s], m
        assert np.linalg.norm(a.T @ a - b.T @ b) <= 1e-12 * max(1.0, np.linalg.norm(b.T @ b))
    ozy = O.o_total_weights(oy, orw)
    gzy = r["zy"].z
    for s, m in ozy.items():
        a = gzy[s]
        assert np.linalg.norm(a.T @ a - m.T @ m) <= 1e-11 * max(1.0, np.linalg.norm(m.T @ m))
    # induced bases: ranks equal the oracle's; Q isometric; Q basis_change = V_X (induced.py:33-46);
    # A_ts = Q_t^T X|ts V_Y,s reproduces the oracle's Q_t A_ts (both project onto the same span)
    oqr = O.o_induced_rows(ox, oy, ozy, opxy, eps)
    qr = r["qrow"]
    assert list(qr.q.rank) == oqr.q.rank
    qb = qr.q.download()
    bc = qr.basis_change
    for t in range(x.block_tree.rows.nnodes):
        q = expand_basis(qb, t)
        assert np.linalg.norm(q.T @ q - np.eye(q.shape[1])) <= 1e-11
        v = expand_basis(x.row_basis, t)
        assert np.linalg.norm(q @ bc[t] - v) <= 1e-11 * max(1.0, np.linalg.norm(v))
    gproj = qr.block_projections
    assert set(gproj) == set(oqr.proj)
    for (t, s), m in oqr.proj.items():
        qo = oqr.q.expand(t)
        a = expand_basis(qb, t) @ gproj[(t, s)]
        b = qo @ m
        assert np.linalg.norm(a - b) <= max(10 * eps, 1e-12) * max(1.0, np.linalg.norm(b))
    # block norms (coarsening.py:342-351): exact against the norms of the GPU's own G (host SVD),
    # and within the truncation level against the oracle's G (other, equally valid induced bases)
    og = O.o_multiply(ox, oy, eps)
    gh = r["g"].download()
    cn, nn = P.coupling_norms(r["g"]), P.nearfield_norms(r["g"])
    assert set(cn) == set(gh.coupling) and set(nn) == set(gh.nearfield)
    for b, m in gh.coupling.items():
        assert abs(cn[b] - np.linalg.norm(m, 2)) <= 1e-13 * max(1.0, cn[b])
    for b, m in gh.nearfield.items():
        assert abs(nn[b] - np.linalg.norm(m, 2)) <= 1e-13 * max(1.0, nn[b])
    for b, val in O.o_coupling_norms(og).items():
        assert abs(cn[b] - val) <= 10 * eps * max(1.0, val)
    for b, val in O.o_nearfield_norms(og).items():
        assert abs(nn[b] - val) <= 10 * eps * max(1.0, val)


def test_oracle_bases_through_gpu_assembly_entrywise():
    """the oracle's qrow / qcol / pxy fed to the GPU assembly (induced.py:220-355)."""
    P = _P()
    import oracle as O
    from paper_2309_09061_b200.device import DeviceH2
    from paper_2309_09061_b200.h2 import ClusterBasis
    from paper_2309_09061_b200.stages import BasisProduct, DeviceMats, InducedBasisResult
    for name in ("rand_s2_2d", "rand_s0_tol1e-3", "rand_s3_2d_tol0"):
        d, x, y, eps = _case(name)
        ox, oy = to_oracle(x), to_oracle(y)
        opxy = O.o_basis_product(ox.cb, oy.rb)
        ozy = O.o_total_weights(oy, O.o_basis_weights(oy.cb))
        ozxt = O.o_total_weights(ox.T(), O.o_basis_weights(ox.rb))
        oqr = O.o_induced_rows(ox, oy, ozy, opxy, eps)
        oqc = O.o_induced_cols(ox, oy, ozxt, opxy, eps)
        og = O.o_assemble(ox, oy, oqr, oqc, opxy)
        dx, dy = DeviceH2.upload(x), DeviceH2.upload(y)

        def basis(ob, tree):
            return ClusterBasis(tree, ob.rank, ob.leaf, ob.xfer)

        qrow = InducedBasisResult.from_parts(basis(oqr.q, x.block_tree.rows), oqr.bc, oqr.proj, x.block_tree)
        qcol = InducedBasisResult.from_parts(basis(oqc.q, y.block_tree.cols), oqc.bc, oqc.proj,
                                             y.block_tree.transposed(), col=True)
        nmid = x.block_tree.cols.nnodes
        pxy = BasisProduct(x.block_tree.cols, DeviceMats.upload(opxy, nmid))
        g = P.assemble_product(dx, dy, qrow, qcol, pxy).download()
        assert list(g.block_tree.row) == og.bt.row and list(g.block_tree.col) == og.bt.col
        for b, m in og.coup.items():
            assert np.abs(g.coupling[b] - m).max() <= 1e-13 * max(1.0, np.abs(m).max()), (name, b)
        for b, m in og.near.items():
            assert np.abs(g.nearfield[b] - m).max() <= 1e-13 * max(1.0, np.abs(m).max()), (name, b)


def test_stage_errors():
    P = _P()
    from paper_2309_09061_b200 import InvalidInputError
    from paper_2309_09061_b200.device import DeviceH2
    d, x, y, eps = _case("rand_s2_2d")
    dx, dy = DeviceH2.upload(x), DeviceH2.upload(y)
    r = _replay(P, dx, dy, eps)
    with pytest.raises(InvalidInputError):
        P.compress_induced_row_basis(dx, dy, r["zy"], r["pxy"], -1.0)
    with pytest.raises(InvalidInputError):  # a row state where the column state belongs
        P.project_final(r["g"], r["rs"], r["rs"], dx.block_tree)
    _, x2, _, _ = _case("rand_s0_tol1e-3")  # n = 48 against n = 96
    with pytest.raises(InvalidInputError):  # bases on different trees
        P.cluster_basis_product(DeviceH2.upload(x2).row_basis, dy.col_basis)


def test_level_decay_and_scaling_flags():
    """level_decay (induced.py:76-81) and scaling / scale_blocks = False (induced.py:358-372,
    coarsening.py:408-422) through the stage drop-ins, against the oracle's ranks."""
    P = _P()
    import oracle as O
    from paper_2309_09061_b200.device import DeviceH2
    d, x, y, eps = _case("rand_s0_tol1e-3")
    ox, oy = to_oracle(x), to_oracle(y)
    dx, dy = DeviceH2.upload(x), DeviceH2.upload(y)
    opxy = O.o_basis_product(ox.cb, oy.rb)
    for scaling, decay in ((True, 0.5), (False, 1.0), (False, 2.0)):
        ozy = O.o_total_weights(oy, O.o_basis_weights(oy.cb), scaling=scaling)
        oq = O.o_induced_rows(ox, oy, ozy, opxy, eps, scale_blocks=scaling, level_decay=decay)
        pxy = P.cluster_basis_product(dx.col_basis, dy.row_basis)
        zy = P.total_weights(dy, P.basis_weights(dy.col_basis), scaling=scaling)
        q = P.compress_induced_row_basis(dx, dy, zy, pxy, eps, scale_blocks=scaling, level_decay=decay)
        assert list(q.q.rank) == oq.q.rank, (scaling, decay)
    r = _replay(P, dx, dy, eps, scaling=False)
    oz = O.o_coarsen(O.o_multiply(ox, oy, eps, scaling=False), ox.bt, eps, scale_blocks=False)
    assert list(r["rs"].q.rank) == oz.rb.rank and list(r["cs"].q.rank) == oz.cb.rank
