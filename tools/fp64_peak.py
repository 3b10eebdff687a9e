"""Measure the FP64 roofline denominators on the box: torch float64 GEMM 8192^3 (cuBLAS DGEMM)
and the DMMA/DFMA microbenchmarks in fp64_peak_probe.cu. Writes gpurun_out/fp64_peak.json."""
import json, os, subprocess, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(2): a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
tf = 2 * n**3 / best / 1e9
print(f"torch fp64 matmul 8192^3: {best:.1f} ms, {tf:.2f} TFLOP/s")
out = subprocess.run([os.path.join(os.path.dirname(__file__), "fp64_peak_probe")], capture_output=True, text=True).stdout
print(out)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"dgemm_8192_tflops": tf, "probe": out}, open("gpurun_out/fp64_peak.json", "w"), indent=1)
