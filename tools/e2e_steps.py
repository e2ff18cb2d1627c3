"""Per-step split of the end-to-end path (public API, page-locked host
buffers): factor and solve wall times of consecutive steps, to find outliers."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
stream = torch.cuda.Stream(device=dev)
r = bench.Runner(3, dev, 0, stream, None, 1, 0)
nogc = "nogc" in sys.argv[1:]
wait = "async" not in sys.argv[1:]  # async: factor_hifde(..., wait=False)
if nogc:
    gc.disable()
for i in range(int(os.environ.get("E2E_STEPS", "12"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fe = r.fac(r.a_pin, r.g, r.eps, stream=stream.cuda_stream, device=0, wait=wait, kernel_log=bool(os.environ.get("HIFDE_PROFILE")))
    t1 = time.perf_counter()
    x = fe.apply_inverse(r.b_pin.numpy())
    t2 = time.perf_counter()
    del x
    t3 = time.perf_counter()
    fe.close()
    t4 = time.perf_counter()
    print(f"step {i}: factor {1e3*(t1-t0):7.2f} solve {1e3*(t2-t1):7.2f} del {1e3*(t3-t2):6.2f} close {1e3*(t4-t3):6.2f} gc {gc.get_count()}", flush=True)
