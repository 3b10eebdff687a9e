"""Device-resident objects: context, cluster / block trees and H^2 matrices on the GPU.

`DeviceH2` is the GPU counterpart of h2mul.H2Matrix (reference h2.py:148-194): the block tree
and the bases / couplings / nearfield live in device arenas owned by the native library; the
host keeps the structure (trees, block tree) needed to rebuild an `H2Matrix` on download.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import CudaError, InvalidInputError
from .h2 import H2Matrix
from .packed import pack_h2, unpack_h2
from .trees import BlockTree

__all__ = ["Context", "DeviceH2", "default_context"]


class Context:
    """One native context per device: a CUDA stream plus pinned staging (h2g_ctx)."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise CudaError("no CUDA device: the B200 product path has no CPU fallback")
        self.lib = N.load()
        self.device = device
        # the native context runs on a torch-owned stream so torch CUDA events can time it
        # high priority: the engine queues work ahead on a low-priority stream (dense-target assembly)
        # that must not hold back the level-serial critical path
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device, priority=-5)
        h = N.P()
        N.check(self.lib.h2g_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h
        self._trees = {}
        self._blocks = {}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                for b in self._blocks.values():
                    self.lib.h2g_blocks_destroy(b[0])
                for t in self._trees.values():
                    self.lib.h2g_tree_destroy(t[0])
                self.lib.h2g_ctx_destroy(self.h)
        except Exception:
            pass

    def set_timing(self, on: bool):
        N.check(self.lib.h2g_ctx_set_timing(self.h, 1 if on else 0))

    STAGES = ("t_setup", "t1_row", "t1_col", "t1_mat", "t2_row", "t2_col", "t2_mat",
              "t_setup_col", "t1_span", "t2_span", "t2_norms")

    def stage_times(self) -> dict:
        """Device seconds of the last multiply / coarsen in the reference harness's stage split
        (bench.py:195-237).  Row and column passes of a phase run concurrently on two streams:
        t1_row / t1_col (t2_row / t2_col) are each pass's own span, t1_span / t2_span the joint one."""
        out = np.zeros(len(self.STAGES))
        N.check(self.lib.h2g_ctx_stage_times_ext(self.h, out.ctypes.data_as(N.F64P), len(out)))
        return {k: float(v) / 1e3 for k, v in zip(self.STAGES, out)}

    def memory(self, reset: bool = False) -> dict:
        """Bytes of the engine's device arenas (default cudaMallocAsync pool: high-water marks since
        the last reset; torch's allocator statistics cannot see these)."""
        out = np.zeros(6, np.int64)
        N.check(self.lib.h2g_ctx_mem(self.h, out.ctypes.data_as(N.I64P), 1 if reset else 0))
        return {"used_high": int(out[0]), "used": int(out[1]), "reserved_high": int(out[2]),
                "reserved": int(out[3]), "payload_high": int(out[4]), "payload": int(out[5])}

    def counters(self, reset: bool = False) -> dict:
        out = np.zeros(2, np.int64)
        N.check(self.lib.h2g_ctx_counters(self.h, out.ctypes.data_as(N.I64P), 1 if reset else 0))
        return {"launches": int(out[0]), "syncs": int(out[1])}

    KCLASSES = ("gsum", "qr_r", "svd", "norm", "gather", "mv")

    def set_profile(self, on: bool):
        N.check(self.lib.h2g_ctx_set_profile(self.h, 1 if on else 0))

    def set_serial(self, on: bool):
        """Process-wide serial mode (h2g_set_serial): a product's passes and auxiliary launches run one
        after the other on the main stream, so profile-mode events time every launch by itself."""
        N.check(self.lib.h2g_set_serial(1 if on else 0))

    def kernel_stats(self, reset: bool = True) -> dict:
        out = np.zeros(4 * len(self.KCLASSES))
        N.check(self.lib.h2g_ctx_kernel_stats(self.h, out.ctypes.data_as(N.F64P), 1 if reset else 0))
        return {k: {"launches": int(out[4 * i]), "ms": float(out[4 * i + 1]), "flops": float(out[4 * i + 2]),
                    "bytes": float(out[4 * i + 3])} for i, k in enumerate(self.KCLASSES)}

    def host_times(self, reset: bool = True) -> dict:
        buf = C.create_string_buffer(1 << 14)
        self.lib.h2g_ctx_host_times(self.h, buf, len(buf), 1 if reset else 0)
        out = {}
        for part in buf.value.decode().split(";"):
            if "=" in part:
                k, v = part.split("=")
                out[k] = float(v)
        return out

    def trace_begin(self):
        N.check(self.lib.h2g_ctx_trace_begin(self.h))

    def trace_dump(self, path: str):
        N.check(self.lib.h2g_ctx_trace_dump(self.h, path.encode()))

    def synchronize(self):
        N.check(self.lib.h2g_ctx_synchronize(self.h))

    # structure handles are cached per host object (trees and block trees are immutable)
    def tree(self, tree):
        key = id(tree)
        if key in self._trees and self._trees[key][1] is tree:
            return self._trees[key][0]
        f = tree.flat()
        arrs = [N.i64(tree.start), N.i64(tree.stop), N.i64(f["child_ptr"]), N.i64(f["child_idx"])]
        h = N.P()
        N.check(self.lib.h2g_tree_create(self.h, tree.nnodes, *[a[1] for a in arrs], C.byref(h)))
        self._trees[key] = (h, tree)
        return h

    def blocks(self, bt: BlockTree):
        key = id(bt)
        if key in self._blocks and self._blocks[key][1] is bt:
            return self._blocks[key][0]
        f = bt.flat()
        adm = np.asarray(bt.admissible, dtype=np.uint8)
        arrs = [N.i64(f["row"]), N.i64(f["col"]), N.i64(f["child_ptr"]), N.i64(f["child_idx"])]
        a8 = N.u8(adm)
        h = N.P()
        N.check(self.lib.h2g_blocks_create(self.h, self.tree(bt.rows), self.tree(bt.cols), bt.nblocks,
                                           *[a[1] for a in arrs], a8[1], C.byref(h)))
        self._blocks[key] = (h, bt)
        return h


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


class DeviceH2:
    """An H^2 matrix resident on the GPU (handle to a native h2g_h2)."""

    def __init__(self, ctx: Context, handle, block_tree: BlockTree | None, rows, cols):
        self.ctx = ctx
        self.h = handle
        self._bt = block_tree
        self.rows, self.cols = rows, cols

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.h2g_h2_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @classmethod
    def upload(cls, g: H2Matrix, ctx: Context | None = None) -> "DeviceH2":
        return cls.upload_packed(pack_h2(g), g.block_tree, ctx, share=g.row_basis is g.col_basis)

    @classmethod
    def upload_packed(cls, d: dict, block_tree: BlockTree, ctx: Context | None = None, *,
                      share: bool = False, asynchronous: bool = False) -> "DeviceH2":
        """Upload from the packed layout (packed.py keys rb.*, cb.*, coup_*, near_*) over the
        C ABI h2g_h2_upload.  Host arrays are copied as given; pinned arrays (e.g.
        torch.empty(..., pin_memory=True).numpy()) transfer at full link bandwidth."""
        ctx = ctx or default_context()
        a = {k: (N.f64(v) if k.endswith("data") else N.i64(v)) for k, v in d.items()
             if not k.startswith(("rows.", "cols.", "bt."))}
        if share and "cb.rank" not in a:
            for k in ("rank", "leaf_off", "xfer_off", "data"):
                a["cb." + k] = a["rb." + k]
        g = block_tree
        h = N.P()
        fn = ctx.lib.h2g_h2_upload_async if asynchronous else ctx.lib.h2g_h2_upload
        N.check(fn(
            ctx.h, ctx.blocks(g),
            a["rb.rank"][1], a["rb.leaf_off"][1], a["rb.xfer_off"][1], a["rb.data"][1], len(a["rb.data"][0]),
            a["cb.rank"][1], a["cb.leaf_off"][1], a["cb.xfer_off"][1], a["cb.data"][1], len(a["cb.data"][0]),
            1 if share else 0,
            a["coup_off"][1], a["coup_data"][1], len(a["coup_data"][0]),
            a["near_off"][1], a["near_data"][1], len(a["near_data"][0]), C.byref(h)))
        out = cls(ctx, h, g, g.rows, g.cols)
        if asynchronous:  # the nearfield copy reads these host arrays until the next synchronisation
            out._host_keep = a
        return out

    def sizes(self):
        out = np.zeros(8, np.int64)
        N.check(self.ctx.lib.h2g_h2_sizes(self.h, out.ctypes.data_as(N.I64P)))
        return out

    def ranks(self) -> tuple[np.ndarray, np.ndarray]:
        """Per-cluster ranks of the row and column bases (no device work, no download)."""
        s = self.sizes()
        rr, cr = np.zeros(int(s[1]), np.int64), np.zeros(int(s[2]), np.int64)
        N.check(self.ctx.lib.h2g_h2_ranks(self.h, rr.ctypes.data_as(N.I64P), cr.ctypes.data_as(N.I64P)))
        return rr, cr

    @property
    def block_tree(self) -> BlockTree:
        if self._bt is None:
            s = self.sizes()
            nb = int(s[0])
            row, col = np.zeros(nb, np.int64), np.zeros(nb, np.int64)
            ptr, idx = np.zeros(nb + 1, np.int64), np.zeros(int(s[7]), np.int64)
            adm = np.zeros(nb, np.uint8)
            N.check(self.ctx.lib.h2g_h2_structure(self.h, row.ctypes.data_as(N.I64P), col.ctypes.data_as(N.I64P),
                                                  ptr.ctypes.data_as(N.I64P), idx.ctypes.data_as(N.I64P),
                                                  adm.ctypes.data_as(N.U8P)))
            kids = [tuple(int(c) for c in idx[ptr[b]:ptr[b + 1]]) for b in range(nb)]
            self._bt = BlockTree(self.rows, self.cols, row, col, kids, adm.astype(bool))
        return self._bt

    def packed_shapes(self) -> dict:
        """Array lengths of the packed layout of this matrix (keys as in packed.py)."""
        s = self.sizes()
        nb, nr, nc = int(s[0]), int(s[1]), int(s[2])
        d = {}
        for p, n, ln in (("rb.", nr, s[3]), ("cb.", nc, s[4])):
            d[p + "rank"] = d[p + "leaf_off"] = d[p + "xfer_off"] = n
            d[p + "data"] = int(ln)
        d["coup_off"], d["coup_data"] = nb, int(s[5])
        d["near_off"], d["near_data"] = nb, int(s[6])
        return d

    def download_packed(self, out: dict | None = None) -> dict:
        """Download into the packed layout over the C ABI h2g_h2_download (device gather, one
        copy per family).  `out` may hold preallocated (e.g. pinned) arrays of at least
        packed_shapes() length; float64 for *data, int64 otherwise."""
        shp = self.packed_shapes()
        d = {}
        for k, n in shp.items():
            a = None if out is None else out.get(k)
            dt = np.float64 if k.endswith("data") else np.int64
            if a is None or a.dtype != dt or a.size < n or not a.flags.c_contiguous:
                a = np.zeros(n, dt)
            d[k] = a[:n]
        self._download_into(d)
        return d

    def _download_into(self, d: dict):
        def ip(k):
            return d[k].ctypes.data_as(N.I64P)

        def fp(k):
            return d[k].ctypes.data_as(N.F64P)

        N.check(self.ctx.lib.h2g_h2_download(
            self.ctx.h, self.h, ip("rb.rank"), ip("rb.leaf_off"), ip("rb.xfer_off"), fp("rb.data"),
            ip("cb.rank"), ip("cb.leaf_off"), ip("cb.xfer_off"), fp("cb.data"),
            ip("coup_off"), fp("coup_data"), ip("near_off"), fp("near_data")))

    def to_packed(self) -> dict:
        d = self.download_packed()
        bt = self.block_tree
        f = bt.flat()
        d["bt.row"], d["bt.col"] = f["row"], f["col"]
        d["bt.child_ptr"], d["bt.child_idx"] = f["child_ptr"], f["child_idx"]
        d["bt.adm"] = np.asarray(bt.admissible, dtype=np.uint8)
        return d

    def download(self) -> H2Matrix:
        """Host H2Matrix with the reference's container interface."""
        return unpack_h2(self.to_packed(), rows=self.rows, cols=self.cols)

    # stage-level views (stages.py): bases as DeviceBasis, the transposed view for total_weights
    @property
    def row_basis(self):
        from .stages import DeviceBasis
        h = N.P()
        N.check(self.ctx.lib.h2g_h2_basis(self.h, 0, C.byref(h)))
        return DeviceBasis(self.ctx, h, self.rows, self)

    @property
    def col_basis(self):
        from .stages import DeviceBasis
        h = N.P()
        N.check(self.ctx.lib.h2g_h2_basis(self.h, 1, C.byref(h)))
        return DeviceBasis(self.ctx, h, self.cols, self)

    def transposed(self):
        from .stages import transposed
        return transposed(self)

    @property
    def shape(self) -> tuple[int, int]:
        return (int(self.rows.stop[0] - self.rows.start[0]), int(self.cols.stop[0] - self.cols.start[0]))

    def matvec(self, x, *, trans: bool = False, alpha: float = 1.0, out=None, accumulate: bool = False):
        """op(G) x on the GPU through the C ABI h2g_matvec (reference h2_matvec / h2_matvec_adjoint,
        h2.py:224-267).  x: CUDA float64 tensor of length cols (rows if trans); returns a CUDA
        tensor (out, if given, accumulated into when accumulate=True)."""
        import torch
        nr, nc = self.shape
        nin, nout = (nr, nc) if trans else (nc, nr)
        dev = torch.device("cuda", self.ctx.device)
        x = torch.as_tensor(x, dtype=torch.float64, device=dev).contiguous()
        if x.shape != (nin,):
            raise InvalidInputError(f"x has shape {tuple(x.shape)}, expected ({nin},)")
        if out is None:
            if accumulate:
                raise InvalidInputError("accumulate=True needs out")
            out = torch.empty(nout, dtype=torch.float64, device=dev)
        elif out.shape != (nout,) or out.dtype != torch.float64 or not out.is_contiguous():
            raise InvalidInputError(f"out must be a contiguous float64 tensor of shape ({nout},)")
        cur = torch.cuda.current_stream(dev)
        self.ctx.stream.wait_stream(cur)
        x.record_stream(self.ctx.stream)
        out.record_stream(self.ctx.stream)
        N.check(self.ctx.lib.h2g_matvec(self.ctx.h, self.h, 1 if trans else 0, C.c_void_p(x.data_ptr()),
                                        C.c_void_p(out.data_ptr()), float(alpha), 1 if accumulate else 0))
        cur.wait_stream(self.ctx.stream)
        return out

    def save(self, path):
        """Write this matrix to a binary packed file (packed.save_packed; device gather + one copy
        per family, no host H2Matrix objects)."""
        from .packed import save_packed
        save_packed(path, self.download_packed(), self.block_tree)

    @classmethod
    def load(cls, path, ctx: Context | None = None) -> "DeviceH2":
        """Upload a binary packed file (packed.save_packed / save_h2) to the device."""
        from .packed import load_packed
        d, bt = load_packed(path)
        return cls.upload_packed(d, bt, ctx)

    def packed_bytes(self) -> int:
        """Bytes of the packed float64 payload (bases + couplings + nearfield)."""
        s = self.sizes()
        return int(8 * (s[3] + s[4] + s[5] + s[6]))


def check_same_trees(a, b):
    if not (a.nnodes == b.nnodes and np.array_equal(a.start, b.start) and np.array_equal(a.stop, b.stop)):
        raise InvalidInputError("cluster trees differ")
