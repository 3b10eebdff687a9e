"""Multi-GPU product: torch.distributed plumbing for the engine's row-subtree partition.

SURVEY 8(e) / BASELINE north star: one process per GPU; the row cluster tree (and the column tree
for the column passes) is split into subtrees at level log2(P); each rank computes its subtrees'
clusters and product blocks plus the replicated top levels, and the per-cluster results are
exchanged by an all-gather over NVLink.  The engine (csrc/shard.cu) lays the results out as one
device buffer with one segment per rank; this module supplies the collective that fills the other
ranks' segments (h2g_ctx_set_comm):

* backend "nccl": one broadcast per segment on the context's CUDA stream (torch's NCCL stream
  waits on it and it waits on the collective) -- no host synchronisation;
* backend "gloo": host staging (device -> host, gloo broadcasts, host -> device), used by the
  tests, including two ranks sharing one GPU.

Every rank must hold the whole of X and Y (upload them on every rank); the product Z comes back
complete on every rank.  Channel 0 / 1 are the row / column passes, which run on two host threads:
each has its own process group so their collectives never interleave.
"""

from __future__ import annotations

import ctypes as C
import traceback

import numpy as np

from . import _native as N

__all__ = ["Sharding", "allgather_segments", "tree_partition"]

_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_longlong), C.c_int,
                         C.c_void_p)
_ALLTOALL = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_longlong), C.c_void_p,
                        C.POINTER(C.c_longlong), C.c_int, C.c_void_p)


class _DeviceBytes:
    """__cuda_array_interface__ over a raw device pointer (zero-copy view for torch.as_tensor)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def allgather_segments(buf, off, group=None):
    """In-place variable all-gather: bytes [off[i], off[i+1]) of the 1-D uint8 tensor `buf` are
    valid on rank i of `group` on entry and on every rank on return (one broadcast per segment)."""
    import torch.distributed as dist
    nseg = len(off) - 1
    if nseg != dist.get_world_size(group):
        raise ValueError("one segment per rank expected")
    for i in range(nseg):
        lo, hi = int(off[i]), int(off[i + 1])
        if hi > lo:
            src = dist.get_global_rank(group, i) if group is not None else i
            dist.broadcast(buf[lo:hi], src=src, group=group)


class Sharding:
    """Attach the ranks of the current process group to a Context: its products are partitioned.

    All ranks must construct it in the same order (it creates two process groups)."""

    def __init__(self, ctx, group=None):
        import torch.distributed as dist
        self.ctx = ctx
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group))
        ranks = None if group is None else dist.get_process_group_ranks(group)
        # one communicator per host thread of the engine (row / column passes)
        self.groups = [dist.new_group(ranks=ranks, backend=self.backend) for _ in range(2)]
        self.calls = 0
        self.bytes = 0
        self._cb = _ALLGATHER(self._allgather)  # keep the trampolines alive
        self._cb2 = _ALLTOALL(self._alltoall)
        self.a2a_calls = 0
        self.a2a_bytes = 0
        N.check(ctx.lib.h2g_ctx_set_comm(ctx.h, self.rank, self.size, C.cast(self._cb, C.c_void_p), None))
        N.check(ctx.lib.h2g_ctx_set_alltoall(ctx.h, C.cast(self._cb2, C.c_void_p), None))

    def close(self):
        """Back to single-GPU products on this context."""
        N.check(self.ctx.lib.h2g_ctx_set_alltoall(self.ctx.h, None, None))
        N.check(self.ctx.lib.h2g_ctx_set_comm(self.ctx.h, 0, 1, None, None))

    def _allgather(self, user, channel, dbuf, off, nseg, stream):
        try:
            import torch
            offs = [int(off[i]) for i in range(nseg + 1)]
            self.calls += 1
            self.bytes += offs[-1]
            if offs[-1] == 0:
                return 0
            dev = torch.device("cuda", self.ctx.device)
            buf = torch.as_tensor(_DeviceBytes(dbuf, offs[-1]), device=dev)
            group = self.groups[channel]
            ext = torch.cuda.ExternalStream(int(stream) if stream else 0, device=dev)
            if self.backend == "nccl":
                with torch.cuda.device(dev), torch.cuda.stream(ext):
                    allgather_segments(buf, offs, group)
            else:  # host staging
                ext.synchronize()
                host = buf.cpu()
                allgather_segments(host, offs, group)
                with torch.cuda.device(dev), torch.cuda.stream(ext):
                    buf.copy_(host)
                ext.synchronize()
            return 0
        except BaseException:  # never unwind through the C frames
            traceback.print_exc()
            return 1


    def _alltoall(self, user, channel, sbuf, soff, rbuf, roff, nseg, stream):
        """Variable all-to-all of the engine's halo / transpose exchanges (one collective)."""
        try:
            import torch
            import torch.distributed as dist
            so = [int(soff[i]) for i in range(nseg + 1)]
            ro = [int(roff[i]) for i in range(nseg + 1)]
            self.a2a_calls += 1
            self.a2a_bytes += so[-1]
            dev = torch.device("cuda", self.ctx.device)
            ssplit = [so[i + 1] - so[i] for i in range(nseg)]
            rsplit = [ro[i + 1] - ro[i] for i in range(nseg)]
            sb = torch.as_tensor(_DeviceBytes(sbuf or 0, so[-1]), device=dev) if so[-1] else \
                torch.empty(0, dtype=torch.uint8, device=dev)
            rb = torch.as_tensor(_DeviceBytes(rbuf or 0, ro[-1]), device=dev) if ro[-1] else \
                torch.empty(0, dtype=torch.uint8, device=dev)
            group = self.groups[channel]
            ext = torch.cuda.ExternalStream(int(stream) if stream else 0, device=dev)
            if self.backend == "nccl":
                with torch.cuda.device(dev), torch.cuda.stream(ext):
                    dist.all_to_all_single(rb, sb, rsplit, ssplit, group=group)
            else:  # host staging
                ext.synchronize()
                hs = sb.cpu()
                hr = torch.empty(ro[-1], dtype=torch.uint8)
                dist.all_to_all_single(hr, hs, rsplit, ssplit, group=group)
                with torch.cuda.device(dev), torch.cuda.stream(ext):
                    rb.copy_(hr)
                ext.synchronize()
            return 0
        except BaseException:  # never unwind through the C frames
            traceback.print_exc()
            return 1


def tree_partition(tree, nparts: int):
    """(owner per cluster, partition level) of the engine's row-subtree split (host only):
    owner -1 marks the replicated top levels; level -1 = no level has nparts clusters."""
    lib = N.load()
    f = tree.flat()
    arrs = [N.i64(tree.start), N.i64(tree.stop), N.i64(f["child_ptr"]), N.i64(f["child_idx"])]
    h = N.P()
    N.check(lib.h2g_tree_create(None, tree.nnodes, *[a[1] for a in arrs], C.byref(h)))
    try:
        owner = np.zeros(tree.nnodes, np.int64)
        level = C.c_int(0)
        N.check(lib.h2g_tree_partition(h, int(nparts), owner.ctypes.data_as(N.I64P), C.byref(level)))
    finally:
        lib.h2g_tree_destroy(h)
    return owner, int(level.value)
