"""Multi-GPU partition of the product through the C ABI: P ranks over gloo (host-staged
all-gathers) sharing the box's one GPU, each computing its row/column subtrees; Z on every rank must
meet the single-GPU golden bars (ranks equal to the reference's, probe errors <= 10 eps) and equal the
single-rank product.  (NCCL refuses two ranks on one device; the collective is the only difference of
the NCCL path, see paper_2309_09061_b200/shard.py.)"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, names, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, HERE)
        sys.path.insert(0, os.path.dirname(HERE))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2309_09061_b200 as P
        from helpers import load, rel
        from test_gpu_parity import _inputs, _probe_tol
        from paper_2309_09061_b200.device import Context, DeviceH2
        from paper_2309_09061_b200.h2 import h2_matvec_host
        from paper_2309_09061_b200.shard import Sharding
        ctx = Context(0)
        sh = Sharding(ctx)
        res = {}
        for name in names:
            if name.startswith("mem:"):  # memory of the partitioned product on a larger case
                res[name] = _memory_case(P, Context, DeviceH2, ctx, name[4:])
                continue
            d = load(name)
            x, y, eps = _inputs(d)  # (inputs prepared unpartitioned on the default context)
            dx = DeviceH2.upload(x, ctx)
            dy = dx if y is x else DeviceH2.upload(y, ctx)
            ctx.synchronize()
            base = ctx.memory(reset=True)["payload"]
            g = P.multiply(dx, dy, eps, ctx=ctx)
            zd = P.coarsen(g, dx.block_tree, eps, ctx=ctx)  # from the distributed G (own rows + halo)
            ctx.synchronize()
            part_bytes = ctx.memory()["payload_high"] - base
            gh = g.download()  # gathers the partitioned rows
            z = zd.download()
            del g, zd
            tol = _probe_tol(eps)
            r = {
                "induced_row": list(gh.row_basis.rank) == list(d["rank.induced_row"]),
                "induced_col": list(gh.col_basis.rank) == list(d["rank.induced_col"]),
                "final_row": list(z.row_basis.rank) == list(d["rank.final_row"]),
                "final_col": list(z.col_basis.rank) == list(d["rank.final_col"]),
                "gv": max(rel(h2_matvec_host(gh, v), d["probe.gv"][i]) for i, v in enumerate(d["probe.v"])),
                "zv": max(rel(h2_matvec_host(z, v), d["probe.zv"][i]) for i, v in enumerate(d["probe.v"])),
                "tol": tol,
            }
            # single rank on a context without the sharding, same device memory pool
            solo = Context(0)
            sx = DeviceH2.upload(x, solo)
            sy = sx if y is x else DeviceH2.upload(y, solo)
            solo.synchronize()
            base = solo.memory(reset=True)["payload"]
            zsd = P.coarsen(P.multiply(sx, sy, eps, ctx=solo), sx.block_tree, eps, ctx=solo)
            solo.synchronize()
            r["mem_ratio"] = part_bytes / max(1, solo.memory()["payload_high"] - base)
            zs = zsd.download()
            r["vs_single"] = max(rel(h2_matvec_host(z, v), h2_matvec_host(zs, v)) for v in d["probe.v"])
            res[name] = r
        q.put((rank, res, sh.calls + sh.a2a_calls, sh.bytes + sh.a2a_bytes))
        dist.destroy_process_group()
    except BaseException as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}, 0, 0))
        raise SystemExit(1) from e


def _memory_case(P, Context, DeviceH2, ctx, name):
    """Per-rank arena payload of the partitioned product against the single-rank product, and Z."""
    import torch
    from helpers import load, rebuild_raw, rel
    d = load(name)
    eps = float(d["eps"][0])
    xr, yr = rebuild_raw(d)
    out = {}
    zs = {}
    for tag, c in (("part", ctx), ("solo", Context(0))):
        dx = P.recompress(DeviceH2.upload(xr, c), eps, ctx=c)
        dy = dx if yr is xr else P.recompress(DeviceH2.upload(yr, c), eps, ctx=c)
        c.synchronize()
        base = c.memory(reset=True)["payload"]
        z = P.coarsen(P.multiply(dx, dy, eps, ctx=c), dx.block_tree, eps, ctx=c)
        c.synchronize()
        out[tag] = c.memory()["payload_high"] - base
        v = torch.from_numpy(np.random.default_rng(9).standard_normal(dx.shape[1])).cuda()
        zs[tag] = z.matvec(v).cpu().numpy()  # the partitioned Z is gathered for the matvec
        del z, dx, dy
    return {"mem_ratio": out["part"] / max(1, out["solo"]), "bytes": out, "vs_single": rel(zs["part"], zs["solo"])}


def _run(world, names):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, names, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res, calls, nbytes = q.get(timeout=600)
        assert "error" not in res, res.get("error")
        out[rank] = (res, calls, nbytes)
    for p in procs:
        p.join(60)
    return out


@pytest.mark.parametrize("world,names", [(2, ["rand_s0_tol1e-3", "rand_s2_2d", "c1", "c2", "mem:c2_full"]),
                                         (3, ["c1", "rand_s1_tol0"])])
def test_partitioned_product_meets_golden_bars(world, names):
    out = _run(world, names)
    for rank, (res, calls, nbytes) in out.items():
        assert calls > 0 and nbytes > 0  # the results really travelled between the ranks
        for name, r in res.items():
            if name.startswith("mem:"):
                assert r["vs_single"] <= 1e-12, (rank, name, r)
                continue
            for k in ("induced_row", "induced_col", "final_row", "final_col"):
                assert r[k], (rank, name, k)
            assert r["gv"] <= r["tol"], (rank, name, r)
            assert r["zv"] <= r["tol"], (rank, name, r)
            assert r["vs_single"] <= 1e-12, (rank, name, r)
    # G and Z stay distributed by block rows (transpose halo for the column passes): the per-rank
    # device memory of the product is well below the single-rank product's on the larger cases
    for rank, (res, _, _) in out.items():
        for name, r in res.items():
            print(rank, name, "memory ratio", round(r["mem_ratio"], 3), r.get("bytes", ""))
            if name == "mem:c2_full":  # n = 16,384 at P = 2: G, Z and the pass scratch halve; the
                # transpose halo of G (~35 % of G on this sphere), the exchanged bases and the top levels
                # do not.  Measured 0.72 (1.50 vs 2.07 GB) with per-level scratch arenas (0.68 = 1.79 vs
                # 2.63 GB before them: the single-rank peak fell further than the per-rank one).  The
                # single-rank product runs its push-down expansions on an auxiliary stream beside phase 2,
                # so its high-water mark depends on the stream schedule (2.00-2.22 GB measured): 0.71-0.75
                assert r["mem_ratio"] <= 0.78, (rank, r)


def _nccl_worker(port, q):
    try:
        import ctypes as C
        import numpy as np
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, os.path.dirname(HERE))
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        from paper_2309_09061_b200.device import Context
        from paper_2309_09061_b200.shard import Sharding
        ctx = Context(0)
        sh = Sharding(ctx)  # one rank: the engine never calls it, so call the trampoline directly
        buf = torch.arange(4096, dtype=torch.uint8, device="cuda")
        ref = buf.clone()
        off = (C.c_longlong * 2)(0, 4096)
        rc = sh._allgather(None, 1, buf.data_ptr(), off, 1, ctx.stream.cuda_stream)
        torch.cuda.synchronize()
        q.put((rc, bool(torch.equal(buf, ref)), sh.calls, sh.backend))
        dist.destroy_process_group()
    except BaseException:
        import traceback
        q.put(("error", traceback.format_exc(), 0, ""))


def test_nccl_allgather_trampoline_world1():
    """The NCCL branch of the engine's all-gather callback (broadcasts on the engine's stream via
    ExternalStream + __cuda_array_interface__) runs cleanly; world size 1 is all one GPU allows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(60)
    assert res[0] == 0, res
    assert res[1] and res[2] == 1 and res[3] == "nccl"
