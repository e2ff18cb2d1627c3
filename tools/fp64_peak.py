"""FP64 roofline denominator: cuBLAS DGEMM (torch.matmul float64) 8192^3,
best of 10 (burst) and back to back for 3 s (sustained), CUDA events."""
import json, sys, time
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
    best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 3.0:
    torch.matmul(a, b); cnt += 1
e1.record(); e1.synchronize()
sus = 2 * n ** 3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
out = {"dgemm_tflops_burst": best, "dgemm_tflops_sustained": sus, "n": n,
       "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM, DMMA), best of 10 / back to back 3 s, CUDA events",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
