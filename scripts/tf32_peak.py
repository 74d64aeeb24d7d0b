"""Measure dense TF32 matmul throughput with torch/cuBLAS (8192^3), same protocol as
MEASURED_PEAKS.json:how (best of 10 burst; back-to-back 4 s sustained).  Context for the
roofline denominator of the TF32 conv passes."""
import json, time, torch
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
for _ in range(3): a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); a @ b; e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
t0 = time.time(); k = 0
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True); e0.record()
while time.time() - t0 < 4: a @ b; k += 1
e1.record(); e1.synchronize()
sus = 2 * n**3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12
print(json.dumps({"tf32_tflops_burst": 2 * n**3 / best / 1e12, "tf32_tflops_sustained": sus}))
