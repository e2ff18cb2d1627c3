"""Device-input factor of a BASELINE config exactly as bench.py times it
(CSR already in HBM, library stream), repeated; per-level host/GPU profile of
the last repetition (HIFDE_PROFILE) and optional host sampling (HIFDE_SAMPLE)."""
import ctypes as C, os, sys, time
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")  # before torch / libgomp initialize (as bench.py)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1307_2895_b200 as H
from paper_1307_2895_b200 import _lib

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
ip = torch.from_numpy(a.indptr.astype(np.int64)).to(dev)
ix = torch.from_numpy(a.indices.astype(np.int32)).to(dev)
va = torch.from_numpy(a.data.astype(np.float64)).to(dev)
lib = _lib.load()
walls = []
for r in range(reps):
    if r == reps - 1:
        os.environ["HIFDE_PROFILE"] = "1"
    opt = _lib.Options()
    lib.hifde_default_options(C.byref(opt), _lib.VARIANT_HIFDE if variant == "hifde" else _lib.VARIANT_HIFDE3X)
    opt.eps = eps
    opt.input_on_device = 1
    opt.stream = stream.cuda_stream
    h = C.c_void_p()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    code = lib.hifde_factor(ip.data_ptr(), ix.data_ptr(), va.data_ptr(), g.ndof, g.dim, g.n, g.m, g.nlevels,
                            C.byref(opt), C.byref(h))
    walls.append(time.perf_counter() - t0)
    assert code == 0, lib.hifde_last_error()
    f = H.GeneralizedLDL(h.value, lib, True)
    gpu = sum(d["gpu_seconds"] for d in f.level_info)
    print(f"rep {r}: wall {walls[-1]*1e3:.2f} ms gpu-sum {gpu*1e3:.2f} ms", flush=True)
    f.close()
print(f"median wall (reps 1..) {np.median(walls[1:])*1e3:.2f} ms")
