"""Multi-GPU partition, host side (no GPU): the engine's row-subtree split (csrc/shard.cu
make_part, via h2g_tree_partition) and the in-place segment all-gather over gloo, world_size 2."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2309_09061_b200.problems import make_points
from paper_2309_09061_b200.shard import tree_partition
from paper_2309_09061_b200.trees import build_cluster_tree


def _restated_partition(tree, P):
    """Python restatement of make_part: first level with >= P clusters, contiguous deal-out."""
    kids = tree.children
    level = np.zeros(tree.nnodes, np.int64)
    parent = np.full(tree.nnodes, -1)
    for t in range(tree.nnodes):
        for c in kids[t]:
            level[c] = level[t] + 1
            parent[c] = t
    owner = np.full(tree.nnodes, -1)
    if P <= 1:
        return owner, -1
    for lev in range(int(level.max()) + 1):
        L = [t for t in range(tree.nnodes) if level[t] == lev]
        if len(L) >= P:
            for i, t in enumerate(L):
                owner[t] = i * P // len(L)
            for t in range(tree.nnodes):
                if level[t] > lev:
                    owner[t] = owner[parent[t]]
            return owner, lev
    return owner, -1


@pytest.mark.parametrize("geom,n,leaf", [("interval", 2048, 32), ("uniform2d", 4096, 64), ("fibonacci", 3000, 40)])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_matches_restatement_and_is_subtree_contiguous(geom, n, leaf, P):
    pts, _ = make_points(geom, n, seed=1)
    tree = build_cluster_tree(pts, leaf)
    owner, level = tree_partition(tree, P)
    ref_owner, ref_level = _restated_partition(tree, P)
    assert level == ref_level
    assert np.array_equal(owner, ref_owner)
    if level < 0:
        return
    # each rank owns a contiguous index range of the points, the ranges tile [0, n) in rank order
    lo = {}
    hi = {}
    for t in range(tree.nnodes):
        o = int(owner[t])
        if o < 0:
            continue
        lo[o] = min(lo.get(o, n), int(tree.start[t]))
        hi[o] = max(hi.get(o, 0), int(tree.stop[t]))
    assert sorted(lo) == list(range(P))
    edges = [(lo[o], hi[o]) for o in range(P)]
    assert edges[0][0] == 0 and edges[-1][1] == n
    for a, b in zip(edges, edges[1:]):
        assert a[1] == b[0]
    # children inherit their parent's owner below the partition level; top levels are replicated
    for t in range(tree.nnodes):
        for c in tree.children[t]:
            if owner[t] >= 0:
                assert owner[c] == owner[t]


def test_balanced_tree_partition_level_is_log2_p():
    tree = build_cluster_tree(make_points("uniform2d", 16384, seed=0)[0], 64)
    for P, lev in ((2, 1), (4, 2), (8, 3)):
        owner, level = tree_partition(tree, P)
        assert level == lev
        sizes = np.bincount(owner[owner >= 0], minlength=P)
        assert sizes.min() == sizes.max()  # balanced: equal cluster counts per rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2309_09061_b200.shard import allgather_segments
    sizes = [5, 0, 11][:world] if world == 3 else [7, 3]
    off = np.concatenate([[0], np.cumsum(sizes)])
    buf = torch.zeros(int(off[-1]), dtype=torch.uint8)
    buf[off[rank]:off[rank + 1]] = torch.arange(sizes[rank], dtype=torch.uint8) + 10 * (rank + 1)
    g = dist.new_group(backend="gloo")
    allgather_segments(buf, off, g)
    q.put((rank, buf.tolist()))
    dist.destroy_process_group()


def test_segment_allgather_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=5) for _ in range(2))
    want = [10, 11, 12, 13, 14, 15, 16, 20, 21, 22]
    assert res[0] == want and res[1] == want
