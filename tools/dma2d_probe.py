"""PCIe DMA rates for the pipelined host solve: strided 2D copies of column
chunks of a row-major N x 64 block (widths 8-32 columns), alone and with the
opposite direction running at the same time, against contiguous 1D copies."""
import time
import torch
from cuda.bindings import runtime as rt
N, R = 4190209, 64
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
hi = torch.empty((N, R), dtype=torch.float64).pin_memory()
ho = torch.empty((N, R), dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(w, both):
    da = torch.empty((N, R), dtype=torch.float64, device="cuda")
    db = torch.empty((N, R), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    for c in range(0, R, w):
        rt.cudaMemcpy2DAsync(da.data_ptr() + c * N * 8, w * 8, hi.data_ptr() + c * 8, R * 8, w * 8, N, H2D,
                             s1.cuda_stream)
        if both:
            rt.cudaMemcpy2DAsync(ho.data_ptr() + c * 8, R * 8, db.data_ptr() + c * N * 8, w * 8, w * 8, N, D2H,
                                 s2.cuda_stream)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3


def run_d2h(w):
    db = torch.empty((N, R), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    for c in range(0, R, w):
        rt.cudaMemcpy2DAsync(ho.data_ptr() + c * 8, R * 8, db.data_ptr() + c * N * 8, w * 8, w * 8, N, D2H,
                             s2.cuda_stream)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3


gb = N * R * 8 / 1e9
for rep in range(2):
    for w in (8, 16, 32, 64):
        a, b, c = run(w, False), run_d2h(w), run(w, True)
        print(f"w={w:2d}: H2D {gb / a * 1e3:5.1f} GB/s ({a:.1f} ms) | D2H {gb / b * 1e3:5.1f} GB/s ({b:.1f} ms) | "
              f"both at once {c:.1f} ms ({2 * gb / c * 1e3:5.1f} GB/s total)", flush=True)
