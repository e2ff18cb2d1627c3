"""Device timeline (HIFDE_PROFILE) of one factorization with the CSR already
resident in HBM: the bench's timed path (bench.Runner.factor_device).

usage: python tools/factor_timeline_dev.py CFG   (prints to stderr)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
stream = torch.cuda.Stream(device=dev)
r = bench.Runner(cfg, dev, 0, stream, None, 1, 0)
for _ in range(3):
    f, _ = r.factor_device()
    r.solve_device(f)
    stream.synchronize()
    f.close()
torch.cuda.synchronize()
os.environ["HIFDE_PROFILE"] = "1"
f, _ = r.factor_device()
stream.synchronize()
f.close()
