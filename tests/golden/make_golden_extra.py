"""Extra golden fixtures produced by running the REFERENCE (h2mul): edge cases of the zero-norm
skips (weights.py:86-89, induced.py:121-125, coarsening.py:237-241).

    python tests/golden/make_golden_extra.py

rand_s5_zero_coup / rand_s6_zero_coup_tol0: unbalanced random pairs on three trees
(tests/util.py:9-48 style, as make_golden.random_pair_case) in which a third of X's and Y's
coupling blocks (and one nearfield block) are exactly zero, at tol = 1e-3 and tol = 0 (where the
eps * max(rows, cols) floor of the truncation -- which depends on the stacks' row counts --
decides the ranks).  Same stored keys as make_golden.random_pair_case.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402


def zero_coupling_case(h2mul, seed, n, leaf, dim, tol, rank=3):
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
        adm = [b for b in range(bt.nblocks) if bt.is_admissible_leaf(b)]
        zero = set(adm[::3])
        for b in adm:
            coup[b] = np.zeros((rank, rank)) if b in zero else rng.standard_normal((rank, rank))
        inadm = [b for b in range(bt.nblocks) if bt.is_inadmissible_leaf(b)]
        for i, b in enumerate(inadm):
            shape = (rows.size(bt.row[b]), cols.size(bt.col[b]))
            near[b] = np.zeros(shape) if i == 1 else rng.standard_normal(shape)
        return h2mul.H2Matrix(bt, rb, cb, coup, near)

    x = h2(trees[0], trees[1])
    y = h2(trees[1], trees[2])
    probes = [rng.standard_normal(n) for _ in range(3)]
    out = {"meta.n": np.asarray([n]), "meta.config": np.asarray([f"zero-coupling-s{seed}"])}
    mg.run_reference(h2mul, x, y, tol, out, probes)
    return out


def main():
    h2mul, _ = mg._ref()
    out_dir = os.environ.get("GOLDEN_OUT", HERE)
    cases = {"rand_s5_zero_coup": zero_coupling_case(h2mul, 5, 96, 6, 2, 1e-3),
             "rand_s6_zero_coup_tol0": zero_coupling_case(h2mul, 6, 80, 5, 2, 0.0)}
    for name, out in cases.items():
        path = os.path.join(out_dir, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB, ranks induced "
              f"{out['rank.induced_row'].max()} final {out['rank.final_row'].max()}")


if __name__ == "__main__":
    main()
