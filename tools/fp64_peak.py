"""Measure FP64 peaks on the B200: cuBLAS DGEMM (burst, sustained) plus the DFMA/DMMA loops."""
import json, subprocess, time, torch, os
r = {}
out = subprocess.run([os.path.join(os.path.dirname(__file__), "fp64_peak")], capture_output=True, text=True)
r["micro"] = out.stdout.strip()
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3): c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
r["dgemm_burst_tflops"] = 2 * n**3 / best * 1e-9
t0 = time.time(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
while time.time() - t0 < 4:
    for _ in range(4): c = a @ b
    k += 4
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
r["dgemm_sustained_tflops"] = 2 * n**3 * k / e0.elapsed_time(e1) * 1e-9
print(json.dumps(r))
