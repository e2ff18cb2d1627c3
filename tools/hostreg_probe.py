"""Cost of page-locking a fresh pageable output (cudaHostRegister) vs staged copies."""
import time
import numpy as np, torch
from cuda.bindings import runtime as rt
N, R = 4190209, 64
d = torch.empty((N, R), dtype=torch.float64, device="cuda"); torch.cuda.synchronize()
for rep in range(3):
    x = np.empty((N, R))
    t = time.perf_counter()
    err, = rt.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    err2, = rt.cudaMemcpy(x.ctypes.data, d.data_ptr(), x.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    t2 = time.perf_counter() - t
    t = time.perf_counter()
    err3, = rt.cudaHostUnregister(x.ctypes.data)
    t3 = time.perf_counter() - t
    print(f"register {1e3*t1:.1f} ms ({err}) D2H {1e3*t2:.1f} ms ({err2}) unregister {1e3*t3:.1f} ms", flush=True)
    y = np.empty((N, R)); y[::512] = 0  # prefault-ish (one write per 4 KB page)
    t = time.perf_counter(); err, = rt.cudaHostRegister(y.ctypes.data, y.nbytes, 0); t1 = time.perf_counter() - t
    rt.cudaHostUnregister(y.ctypes.data)
    print(f"  register after prefault {1e3*t1:.1f} ms", flush=True)
