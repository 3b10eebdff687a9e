"""Benchmark: the adaptive H^2 x H^2 product (multiply + coarsen) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--n N] [--impl ours|reference]

One step = one full product Z = X*Y on the largest BASELINE config that fits one B200 (default
configs[3] = c4: n = 262,144 Fibonacci-sphere points, X from 1/r and Y from exp(-r)/r, leaf 128,
eta 2, Chebyshev order 4 (rank 64), eps 1e-6), i.e. phase 1 (basis products + weights + induced
bases + assembly over T^XY) followed by phase 2 (re-compression onto X's block tree) -- the
stages the reference harness times (bench.py:195-237 of h2mul; its t_total excludes only the
weights, which we include).  Inputs are built on the GPU by the reference's interpolation recipe
(synthetic seeded points) and recompressed at eps before timing.  Metric: DOF/s = n / product time.

--impl reference times the reference's CPU path (the oracle port, oracle/h2_oracle.py: the
reference is pure Python, so nothing compiles into oracle/_ref; the port was measured to cost the
same as h2mul itself) with 1 BLAS thread -- the reference protocol pins it (cli.py:12-15) --
on a bounded sample: the same generator at a reduced n (--cpu-sample-n, default per config),
because 25 full-size c4 CPU products (~18 min each) cannot fit the driver's window.
Multi-GPU (N > 1, one process per GPU under torchrun): by default ONE product per step computed
jointly by all ranks -- the row (and column) cluster trees split into subtrees at level log2 N,
results all-gathered over NCCL (paper_2309_09061_b200/shard.py, csrc/shard.cu) -- so value =
n / (max-over-ranks step time), strong scaling.  --parallelism replicas runs N independent
products instead (weak scaling, value = N n / time).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=None,
                    help="n of the CPU (reference-arm / cpu_baseline) sample; default per config")
    ap.add_argument("--parallelism", default="shard", choices=["shard", "replicas"])
    ap.add_argument("--profile-json", default=None, help="write per-stage / per-kernel detail here")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def reduce_max(value: float, device) -> float:
    """Max over ranks (device timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def fp64_peak_tflops():
    """cuBLAS DGEMM 8192^3 on this GPU (MEASURED_PEAKS.json has no FP64 entry)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * n ** 3 / best / 1e9


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# CPU sample sizes: about 10-15 s of single-thread CPU work per product (c2 at 8,192: ~7 s;
# c4 at 4,096: ~12 s), the same generator as the GPU line
CPU_SAMPLE_N = {"c1": 2048, "c2": 8192, "c3": 8192, "c4": 4096, "c5": 4096}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def build_inputs(cfg, n):
    from paper_2309_09061_b200.problems import build_config
    xr, yr, spec = build_config(cfg, n=n)
    return xr, yr, spec


def _blas_threads(threads):
    os.environ["OMP_NUM_THREADS"] = os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=threads)
    except Exception:  # pragma: no cover
        return None


def cpu_oracle_prepare(cfg, n):
    """CPU oracle inputs at size n: the config's generator, recompressed at eps (untimed)."""
    import oracle as O
    from paper_2309_09061_b200.packed import pack_h2
    xr, yr, spec = build_inputs(cfg, n)
    x = O.o_recompress(O.o_from_packed(pack_h2(xr)), spec["eps"])
    y = x if yr is xr else O.o_recompress(O.o_from_packed(pack_h2(yr)), spec["eps"])
    return x, y, spec["eps"]


def cpu_oracle_time(x, y, eps):
    """One full CPU product (weights + phase 1 + phase 2); returns (seconds, stage detail)."""
    import oracle as O
    t0 = time.perf_counter()
    final, induced, tm, _ = O.o_run_stages(x, y, x.bt, eps)
    return time.perf_counter() - t0, tm   # includes the weights (t_setup), like our timed step


def cpu_oracle_run(cfg, n, threads):
    """Time the CPU oracle on the config's generator at size n; returns (seconds, detail)."""
    lim = _blas_threads(threads)
    try:
        x, y, eps = cpu_oracle_prepare(cfg, n)
        return cpu_oracle_time(x, y, eps)
    finally:
        if lim is not None:
            lim.__exit__(None, None, None)


def run_reference(args, rank, world):
    """Reference arm: the reference's CPU path (oracle port) at 1 BLAS thread as the reference
    protocol pins it (cli.py:12-15), bounded sample per step (same generator, reduced n)."""
    if rank != 0:
        return
    threads = 1
    n = args.cpu_sample_n or CPU_SAMPLE_N[args.config]
    lim = _blas_threads(threads)
    try:
        x, y, eps = cpu_oracle_prepare(args.config, n)
        for _ in range(args.warmup):
            cpu_oracle_time(x, y, eps)
        times = []
        for _ in range(args.steps):
            t, _ = cpu_oracle_time(x, y, eps)
            times.append(t)
    finally:
        if lim is not None:
            lim.__exit__(None, None, None)
    ms = 1e3 * sum(times) / len(times)
    value = n / (ms / 1e3)
    from paper_2309_09061_b200.problems import CONFIGS
    spec = CONFIGS[args.config]
    line = {
        "impl": "reference", "metric": "h2_product_dof_per_s", "value": value, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded points, BASELINE generator)",
        "config": {"workload": f"{args.config} product X*Y -> Z (multiply + coarsen onto X's tree)",
                   "n": spec["n"], "geometry": spec["geometry"], "kernel_x": spec["kernel_x"],
                   "kernel_y": spec["kernel_y"], "leaf": spec["leaf"], "eta": spec["eta"],
                   "order": spec["order"], "eps": spec["eps"], "sample_n": n},
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": (f"{args.config} generator at its full n={n}" if n == spec["n"] else
                                    f"{args.config} generator at reduced n={n} (the full n={spec['n']} product "
                                    f"takes minutes per step on one core)") +
                                   ", full product incl. weights, oracle/h2_oracle.py NumPy restatement of h2mul, "
                                   "1 BLAS thread (reference cli.py:12-15)"},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    # H2G_BENCH_BACKEND=gloo: functional check of the N > 1 path with ranks sharing the GPUs there
    # are (host-staged all-gathers; its timings are not a measurement)
    backend = os.environ.get("H2G_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2309_09061_b200 as P
    from paper_2309_09061_b200.device import Context, DeviceH2
    from paper_2309_09061_b200.problems import CONFIGS

    spec = dict(CONFIGS[args.config])
    n = args.n or spec["n"]
    eps = spec["eps"]
    # one process per GPU: map 70 % of the device into the engine's stream-ordered pool up front.
    # Growing the pool later happens inside whichever allocation needs it, on the host thread of a
    # level batch -- measured 5 ms to 1.2 s per call at c4, i.e. +100..1000 ms on ~30 % of the steps
    # (tools/step_loop.py with H2G_DEBUG_ALLOC=1); with the reservation every c4 step is 1.08-1.09 s.
    total_gb = torch.cuda.get_device_properties(local).total_memory / 1e9
    os.environ.setdefault("H2G_POOL_RESERVE_GB", f"{0.7 * total_gb:.0f}")
    ctx = Context(local)
    from paper_2309_09061_b200.problems import build_config_device
    t0 = time.perf_counter()
    # raw interpolation inputs built on the GPU (structure and the small interpolation bases on the
    # host, couplings / nearfield evaluated by h2g_h2_build_kernel; pinned to the reference's raw
    # inputs by tests/test_gpu_fullsize.py)
    dxr, dyr, spec = build_config_device(args.config, n=n, ctx=ctx)
    ctx.synchronize()
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    dx = P.recompress(dxr, eps, ctx=ctx)
    dy = dx if dyr is dxr else P.recompress(dyr, eps, ctx=ctx)
    del dxr, dyr
    ctx.synchronize()
    t_prep = time.perf_counter() - t0
    coarse = dx.block_tree
    stream = ctx.stream
    shard = world > 1 and args.parallelism == "shard"
    if shard:  # from here on every product on ctx is partitioned across the ranks
        from paper_2309_09061_b200.shard import Sharding
        sharding = Sharding(ctx)
    units = n if shard else world * n  # DOF of the products one step completes, all ranks together

    def step():
        g = P.multiply(dx, dy, eps, ctx=ctx)
        return P.coarsen(g, coarse, eps, ctx=ctx)

    for _ in range(max(3, args.warmup)):
        z = step()
    ctx.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.counters(reset=True)
    ctx.memory(reset=True)
    xc0 = (sharding.calls, sharding.bytes) if shard else (0, 0)
    clocks = ClockSampler(local)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # ncu --profile-from-start off captures exactly the launches between cudaProfilerStart / Stop, on
    # every engine thread and stream (NVTX ranges are per host thread and would miss the column
    # passes and the planner-queued launches)
    torch.cuda.profiler.start()
    torch.cuda.nvtx.range_push("timed")
    e0.record(stream)
    for _ in range(args.steps):
        z = step()
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    e1.synchronize()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    mem = ctx.memory()
    torch.cuda.synchronize()
    clk = clocks.stop()
    cnt = ctx.counters(reset=True)
    xchg = None
    if shard:
        xchg = {"allgathers_per_step": (sharding.calls - xc0[0]) / args.steps,
                "bytes_per_step": (sharding.bytes - xc0[1]) / args.steps, "backend": backend,
                "partition": "row/column cluster trees split at the first level with >= N clusters; "
                             "top levels replicated"}
    ms = reduce_max(e0.elapsed_time(e1) / args.steps, torch.device("cuda", local))
    value = units / (ms / 1e3)

    # stage split (reference harness stage names) and per-kernel-class accounting, untimed step
    ctx.set_timing(True)
    ctx.set_profile(True)
    ctx.kernel_stats(reset=True)
    g = P.multiply(dx, dy, eps, ctx=ctx)
    st1 = ctx.stage_times()
    z = P.coarsen(g, coarse, eps, ctx=ctx)
    st2 = ctx.stage_times()
    g_ranks = g.ranks()
    ks_conc = ctx.kernel_stats(reset=True)
    hts = ctx.host_times(reset=True)
    ctx.set_profile(False)
    ctx.set_timing(False)
    # per-kernel-class durations for the roofline from a serialized profiled product (every launch
    # on the main stream, CUDA events around each): in the concurrent step above the events of one
    # stream also cover the other streams' kernels running beside it
    del z
    ctx.set_serial(True)
    ctx.set_profile(True)
    ctx.kernel_stats(reset=True)
    z = P.coarsen(P.multiply(dx, dy, eps, ctx=ctx), coarse, eps, ctx=ctx)
    ctx.synchronize()
    ks = ctx.kernel_stats(reset=True)
    ctx.set_profile(False)
    ctx.set_serial(False)
    stages = {k: st1[k] for k in ("t_setup", "t_setup_col", "t1_row", "t1_col", "t1_span", "t1_mat")}
    stages.update({k: st2[k] for k in ("t2_norms", "t2_row", "t2_col", "t2_span", "t2_mat")})
    stages["note"] = ("device seconds of one product in the reference harness's split (bench.py:195-237); "
                      "row and column passes of each phase run concurrently on two streams, t*_row / t*_col "
                      "are each pass's own span and t*_span their joint span; t_setup = basis product + the "
                      "row pass's weights (t_setup_col: the column pass's, concurrent); t2_row includes "
                      "t2_norms as in the reference")
    zr = [int(r) for r in z.ranks()[0]]

    # end to end through the C-ABI boundary on HOST buffers: X (and Y) in the packed layout in
    # pinned host memory -> h2g_h2_upload -> multiply -> coarsen -> h2g_h2_download into pinned
    # host buffers; every step uploads its inputs and downloads Z
    def pinned_copy(d):
        out = {}
        for k, v in d.items():
            if k.startswith(("rows.", "cols.", "bt.")):
                continue
            t = torch.empty(len(v), dtype=torch.float64 if k.endswith("data") else torch.int64, pin_memory=True)
            a = t.numpy()
            a[:] = v
            out[k] = a
        return out

    def payload(d):  # every host array the step copies (data + offset tables)
        return sum(v.nbytes for v in d.values())

    xp = pinned_copy(dx.download_packed())
    yp = None if dy is dx else pinned_copy(dy.download_packed())
    bt_x = dx.block_tree
    bt_y = None if dy is dx else dy.block_tree
    zshape = z.packed_shapes()
    zout = {k: torch.empty(n, dtype=torch.float64 if k.endswith("data") else torch.int64,
                           pin_memory=True).numpy() for k, n in zshape.items()}
    for _ in range(max(2, args.warmup)):
        P.multiply_coarsen_packed(xp, bt_x, yp, bt_y, eps, coarse=bt_x, out=zout, ctx=ctx)
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        zp = P.multiply_coarsen_packed(xp, bt_x, yp, bt_y, eps, coarse=bt_x, out=zout, ctx=ctx)
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = reduce_max(sum(e2e_t) / len(e2e_t), torch.device("cuda", local))
    h2d = payload(xp) + (payload(yp) if yp is not None else 0)
    d2h = payload(zp)

    # roofline: dominant kernel class by device time in the profiled step
    peak_fp64 = fp64_peak_tflops()
    hbm, hbm_src = hbm_peak()
    # dominant kernel: gsum_pipe_kernel -- the "gsum" class is exactly that kernel (both template
    # instantiations: <1> is the dense-target assembly launch, <0> every other grouped GEMM); it is
    # the largest kernel by device time in the committed ncu launch list of the timed region
    # (profiles/r02_launches_c4_summary.txt: 33 % of kernel time), the other classes group several
    dom = "gsum"
    d = ks[dom]
    achieved = d["flops"] / (d["ms"] / 1e3) / 1e12 if d["ms"] > 0 else 0.0
    total_flops = sum(v["flops"] for v in ks.values())
    traffic, traffic_note = None, None
    tr_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_gsum_ncu.json")
    if os.path.exists(tr_path):
        with open(tr_path) as fh:
            tr = json.load(fh)
        traffic = tr.get("dram_bytes_per_launch")
        traffic_note = (f"dram read+write of the dense-target assembly launch ({tr.get('kernel', '')}, grid "
                        f"{tr.get('grid', '')}, the longest gsum launch of a c4 product) from one ncu --set full "
                        f"capture, profiles/r02_gsum_ncu.json")
    roofline = {"bound": "fp64", "kernel": "gsum_pipe_kernel", "achieved": achieved, "peak": peak_fp64,
                "unit": "TFLOP/s", "frac": achieved / peak_fp64, "traffic": traffic,
                "traffic_note": traffic_note,
                "flops_note": "reference-ledger flops of the terms (per-triple shapes); the grouped assembly "
                              "executes fewer",
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (no FP64 entry in MEASURED_PEAKS.json)",
                "launches": d["launches"], "kernel_ms": d["ms"], "kernel_flops": d["flops"],
                "timing_note": "kernel durations: CUDA events around every launch of one serialized "
                               "product (h2g_set_serial: all launches on the main stream, so no other "
                               "stream's kernels fall inside a launch's events); the timed steps run the "
                               "row and column passes and the auxiliary launches concurrently",
                "concurrent_kernel_ms": {k: v["ms"] for k, v in ks_conc.items()},
                "classes": {k: {"ms": v["ms"], "launches": v["launches"],
                                "achieved_tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] > 0 else 0.0}
                            for k, v in ks.items()},
                "phase_mix": {"ledger_flops": total_flops, "t_roof_ms": 1e3 * total_flops / (peak_fp64 * 1e12),
                              "frac_of_step": (1e3 * total_flops / (peak_fp64 * 1e12)) / ms},
                "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src}

    # accuracy of the full-size product: the reference's 20-step power-iteration estimate of
    # |XY - Z|_2 / |XY|_2 (bench.py:147-174), every matvec on the GPU
    eps2 = P.estimate_relative_spectral_error(dx, dy, z, steps=20, seed=0)
    eps2_induced = P.estimate_relative_spectral_error(dx, dy, g, steps=20, seed=0)
    del g
    # H^2 matvec: HBM bound, every stored entry of Z read once per product.  `ms` is
    # the device time of one whole Z v (CUDA events around 10 back-to-back calls on the stream the
    # calls are ordered on: the nearfield stream overlaps the transform chain inside a call);
    # `kernel_ms_sum` adds the per-launch event times of the same launches run serially (profile mode)
    vz = torch.randn(n, dtype=torch.float64, device=torch.device("cuda", local))
    yz = torch.empty_like(vz)  # the output buffer is reused (no allocator traffic inside the timing)
    for _ in range(3):
        z.matvec(vz, out=yz)
    torch.cuda.synchronize()
    mv_reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(mv_reps):
        z.matvec(vz, out=yz)
    e1.record()
    torch.cuda.synchronize()
    mv_call_ms = e0.elapsed_time(e1) / mv_reps
    ctx.kernel_stats(reset=True)
    ctx.set_profile(True)
    for _ in range(mv_reps):
        z.matvec(vz, out=yz)
    ctx.synchronize()
    ctx.set_profile(False)
    mvs = ctx.kernel_stats(reset=True)["mv"]
    mv_ms = mvs["ms"] / mv_reps
    mv_bytes = mvs["bytes"] / mv_reps
    matvec = {"kernel": "mv_warp_kernel", "ms": mv_call_ms, "launches": mvs["launches"] // mv_reps,
              "bytes": mv_bytes, "achieved_gbs": mv_bytes / (mv_call_ms / 1e3) / 1e9 if mv_call_ms > 0 else 0.0,
              "peak_gbs": hbm, "frac": (mv_bytes / (mv_call_ms / 1e3) / 1e9) / hbm if mv_call_ms > 0 else 0.0,
              "kernel_ms_sum": mv_ms,
              "kernel_sum_frac": (mv_bytes / (mv_ms / 1e3) / 1e9) / hbm if mv_ms > 0 else 0.0,
              "note": "Z v on the c-config product Z, device time of one whole call (nearfield stream "
                      "concurrent with the transform chain); bytes = matrix entries + vector reads"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_n = args.cpu_sample_n or CPU_SAMPLE_N[args.config]
        wall, tm = cpu_oracle_run(args.config, cpu_n, 1)
        cpu = {"value": cpu_n / wall, "unit": "DOF/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
               "sample": f"{args.config} generator at reduced n={cpu_n}, full product incl. weights "
                         f"({wall:.1f} s), oracle/h2_oracle.py (NumPy restatement of h2mul), 1 BLAS thread",
               "stages_s": tm}

    if rank == 0:
        line = {
            "metric": "h2_product_dof_per_s", "value": value, "unit": "DOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded points per BASELINE generator; interpolation inputs recompressed on GPU)",
            "config": {"workload": f"{args.config} product X*Y -> Z (multiply + coarsen onto X's tree)",
                       "n": n, "geometry": spec["geometry"], "kernel_x": spec["kernel_x"],
                       "kernel_y": spec["kernel_y"], "leaf": spec["leaf"], "eta": spec["eta"],
                       "order": spec["order"], "eps": eps,
                       "parallelism": f"row-subtree partition x{world}" if shard else f"replicas x{world}",
                       "l2": f"inputs larger than L2 (X packed {dx.packed_bytes() / 1e6:.0f} MB)"},
            "e2e": {"value": units / e2e_s, "unit": "DOF/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "seconds": e2e_s},
            "gpu_launches": cnt["launches"] // args.steps * args.steps,
            "host_syncs_per_step": cnt["syncs"] / args.steps,
            "clocks": clk,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "stages_s": stages,
            "ranks": {"final_max": int(max(zr)), "final_mean": float(sum(zr) / len(zr)),
                      "induced_max": int(max(g_ranks[0])), "induced_mean": float(g_ranks[0].mean())},
            "memory": {"engine_used_high_gb": mem["used_high"] / 1e9,
                       "engine_reserved_high_gb": mem["reserved_high"] / 1e9,
                       "note": "high-water marks of the engine's cudaMallocAsync arenas over the timed steps"},
            "accuracy": {"eps2_power_iteration": eps2, "eps2_induced": eps2_induced, "steps": 20, "seed": 0,
                         "eps": eps,
                         "estimator": "reference bench.py:147-174 on GPU matvecs"},
            "matvec": matvec,
            "exchange": xchg,
            "setup_s": {"build_inputs": t_build, "upload_recompress": t_prep},
        }
        if args.profile_json:
            with open(args.profile_json, "w") as fh:
                json.dump({"kernel_stats": ks, "host_ms": hts, "stages_s": stages, "line": line}, fh, indent=1)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
