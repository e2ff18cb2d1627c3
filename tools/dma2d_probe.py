"""H2D / D2H rate of strided 2D DMA (column chunks of a row-major block) vs 1D."""
import time
import numpy as np, torch
from cuda.bindings import runtime as rt
N, R = 4190209, 64
h = torch.empty((N, R), dtype=torch.float64).pin_memory()
d = torch.empty((N, 16), dtype=torch.float64, device="cuda")
d64 = torch.empty((N, R), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for w in (16, 32):
    dd = torch.empty((N, w), dtype=torch.float64, device="cuda")
    for rep in range(2):
        t = time.perf_counter()
        err, = rt.cudaMemcpy2D(dd.data_ptr(), w * 8, h.data_ptr(), R * 8, w * 8, N, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
        torch.cuda.synchronize()
        t1 = time.perf_counter() - t
        t = time.perf_counter()
        err, = rt.cudaMemcpy2D(h.data_ptr(), R * 8, dd.data_ptr(), w * 8, w * 8, N, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        torch.cuda.synchronize()
        t2 = time.perf_counter() - t
        gb = N * w * 8 / 1e9
        print(f"w={w}: 2D H2D {gb/t1:.1f} GB/s  2D D2H {gb/t2:.1f} GB/s", flush=True)
t = time.perf_counter(); d64.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter() - t
print(f"1D H2D {N*R*8/1e9/t1:.1f} GB/s")
