"""Golden fixtures at the BASELINE sizes, produced by running the REFERENCE (h2mul).

Run in the build container only (imports /root/reference read-only), one case per process:

    python tests/golden/make_golden_full.py c2_full      # n = 16,384   (~2 min, 3 GB)
    python tests/golden/make_golden_full.py c3_full      # n = 32,768   (~3 min, 4 GB)
    python tests/golden/make_golden_full.py c4_n65536    # n = 65,536   (~6 min, 12 GB)
    python tests/golden/make_golden_full.py c4_full      # n = 262,144  (~30 min, ~45 GB)
    python tests/golden/make_golden_full.py c5_n32768    # n = 32,768   (~8 min, 12 GB)
    python tests/golden/make_golden_full.py c2_noscale   # n = 2,048, scaling=False / scale_blocks=False

The reference's stage sequence is replayed exactly as its harness does
(bench.py:195-237, coarsening.py:408-422; recompress bench.py:198-199). The
inputs are not stored: the GPU tests rebuild them with the repo's generator and
interpolation builder (on the device), pinned by probe.xraw_v / probe.yraw_v
(the reference's raw X v and Y v at this very n). Stored, per case:
  pt.*            T^XY (trees.py:314-359): row, col, children, admissibility
  rank.*          every per-cluster rank: inputs after recompress, induced row/col,
                  final row/col
  gap.*           min |sigma - thr| / thr over every truncation (rank-parity margin)
  probe.*         one N(0,1) probe v (default_rng(123)): X_raw v, Y_raw v (float64),
                  G v, Z v, Z^T v (float32: the gates are 10 eps >= 1e-5 relative,
                  float32 storage adds <= 6e-8), X (Y v) (float64), and the
                  reference's own ||Z v - X(Y v)|| / ||X(Y v)|| computed in float64
  est.eps2        the reference's power-iteration estimate (bench.py:147-174)
  stages.*        the reference's stage times on this container (1 BLAS thread)
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")        # reference cli.py:12-15
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import make_golden as mg  # noqa: E402
import paper_2309_09061_b200.problems as myprob  # noqa: E402

CASES = {
    "c2_full": ("c2", 16384, True),
    "c3_full": ("c3", 32768, True),
    "c4_n65536": ("c4", 65536, True),
    "c4_full": ("c4", 262144, True),
    "c5_n32768": ("c5", 32768, True),
    "c5_n65536": ("c5", 65536, True),
    "c2_noscale": ("c2", 2048, False),
    "c4_noscale": ("c4", 4096, False),
}


def run(case: str) -> dict:
    h2mul, hp = mg._ref()
    from h2mul.coarsening import _coupling_norms, _nearfield_norms
    from h2mul.bench import estimate_relative_spectral_error
    name, n, scaling = CASES[case]
    spec = myprob.CONFIGS[name]
    pts, wts = myprob.make_points(spec["geometry"], n, seed=0)
    kx = myprob.KERNEL_FNS[spec["kernel_x"]]
    ky = myprob.KERNEL_FNS[spec["kernel_y"]]
    t0 = time.perf_counter()
    _, _, x_raw = mg.ref_instance(h2mul, hp, pts, wts, kx, spec["leaf"], spec["eta"], spec["order"],
                                  "single-layer")
    if spec["kernel_y"] == spec["kernel_x"]:
        y_raw = x_raw
    else:
        _, _, y_raw = mg.ref_instance(h2mul, hp, pts, wts, ky, spec["leaf"], spec["eta"],
                                      spec["order"], "single-layer")
    t_build = time.perf_counter() - t0
    eps = spec["eps"]
    x = h2mul.recompress(x_raw, eps)
    y = x if y_raw is x_raw else h2mul.recompress(y_raw, eps)
    rng = np.random.default_rng(123)
    v = rng.standard_normal(n)
    out = {"meta.n": np.asarray([n]), "meta.config": np.asarray([name]),
           "meta.case": np.asarray([case]), "meta.scaling": np.asarray([int(scaling)]),
           "eps": np.asarray([eps])}
    out["probe.xraw_v"] = h2mul.h2_matvec(x_raw, v)[None]
    out["probe.yraw_v"] = h2mul.h2_matvec(y_raw, v)[None]
    del x_raw, y_raw

    gaps = mg.GapLog(h2mul)
    st = {}
    try:
        t = time.perf_counter()
        pxy = h2mul.cluster_basis_product(x.col_basis, y.row_basis)
        zy = h2mul.total_weights(y, h2mul.basis_weights(y.col_basis), scaling=scaling)
        zxt = h2mul.total_weights(x.transposed(), h2mul.basis_weights(x.row_basis), scaling=scaling)
        st["t_setup"] = time.perf_counter() - t
        t = time.perf_counter()
        qrow = h2mul.compress_induced_row_basis(x, y, zy, pxy, eps, scale_blocks=scaling)
        st["t1_row"] = time.perf_counter() - t
        t = time.perf_counter()
        qcol = h2mul.compress_induced_col_basis(x, y, zxt, pxy, eps, scale_blocks=scaling)
        st["t1_col"] = time.perf_counter() - t
        t = time.perf_counter()
        pt = h2mul.build_product_block_tree(x.block_tree, y.block_tree)
        g = h2mul.assemble_product(x, y, qrow, qcol, pxy, pt)
        st["t1_mat"] = time.perf_counter() - t
        del zy, zxt
        n1 = len(gaps.vals)
        coarse = x.block_tree
        t = time.perf_counter()
        cn = _coupling_norms(g) if scaling else None
        nn = _nearfield_norms(g) if scaling else None
        rs = h2mul.build_coarse_row_basis(g, coarse, eps, scale_blocks=scaling,
                                          coupling_norms=cn, nearfield_norms=nn)
        st["t2_row"] = time.perf_counter() - t
        t = time.perf_counter()
        cs = h2mul.build_coarse_col_basis(g, coarse, eps, scale_blocks=scaling,
                                          coupling_norms=cn, nearfield_norms=nn)
        st["t2_col"] = time.perf_counter() - t
        t = time.perf_counter()
        z = h2mul.project_final(g, rs, cs, coarse)
        st["t2_mat"] = time.perf_counter() - t
    finally:
        gaps.restore()
    out["pt.row"] = np.asarray(pt.row, dtype=np.int32)
    out["pt.col"] = np.asarray(pt.col, dtype=np.int32)
    lens = [len(c) for c in pt.children]
    out["pt.child_ptr"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out["pt.child_idx"] = np.asarray([c for k in pt.children for c in k], dtype=np.int32)
    out["pt.adm"] = np.asarray(pt.admissible, dtype=np.uint8)
    for key, basis in (("x_row", x.row_basis), ("x_col", x.col_basis), ("y_row", y.row_basis),
                       ("y_col", y.col_basis), ("induced_row", qrow.q), ("induced_col", qcol.q),
                       ("final_row", rs.q), ("final_col", cs.q)):
        out["rank." + key] = np.asarray(basis.rank, dtype=np.int32)
    gv = np.asarray(gaps.vals) if gaps.vals else np.ones(1)
    out["gap.phase1"] = np.asarray([gv[:n1].min() if n1 else 1.0])
    out["gap.phase2"] = np.asarray([gv[n1:].min() if len(gv) > n1 else 1.0])
    out["gap.count"] = np.asarray([len(gv)])
    zv = h2mul.h2_matvec(z, v)
    xyv = h2mul.h2_matvec(x, h2mul.h2_matvec(y, v))
    out["probe.zv"] = zv.astype(np.float32)[None]
    out["probe.gv"] = h2mul.h2_matvec(g, v).astype(np.float32)[None]
    out["probe.ztv"] = h2mul.h2_matvec_adjoint(z, v).astype(np.float32)[None]
    out["probe.xyv"] = xyv[None]
    out["probe.ref_xy_rel"] = np.asarray([np.linalg.norm(zv - xyv) / np.linalg.norm(xyv)])
    del g
    t = time.perf_counter()
    out["est.eps2"] = np.asarray([estimate_relative_spectral_error(x, y, z, steps=20, seed=0)])
    t_est = time.perf_counter() - t
    for k, val in st.items():
        out["stages." + k] = np.asarray([val])
    out["stages.t_total"] = np.asarray([sum(st[k] for k in st if k != "t_setup")])
    out["meta.t_build_s"] = np.asarray([t_build])
    out["meta.t_est_s"] = np.asarray([t_est])
    return out


def main():
    case = sys.argv[1]
    out_dir = os.environ.get("GOLDEN_OUT", HERE)
    t0 = time.perf_counter()
    out = run(case)
    path = os.path.join(out_dir, f"{case}.npz")
    np.savez_compressed(path, **out)
    print(f"{case}: {os.path.getsize(path) / 1e6:.2f} MB in {time.perf_counter() - t0:.0f} s; "
          f"ranks induced {out['rank.induced_row'].max()}/{out['rank.induced_col'].max()} "
          f"final {out['rank.final_row'].max()}/{out['rank.final_col'].max()}; gaps "
          f"{out['gap.phase1'][0]:.1e}/{out['gap.phase2'][0]:.1e}; eps2 {out['est.eps2'][0]:.3e}; "
          f"t_total {out['stages.t_total'][0]:.1f} s", flush=True)


if __name__ == "__main__":
    main()
