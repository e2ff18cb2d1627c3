"""Host sampling profile (HIFDE_SAMPLE) of one device-resident factorization:
writes the main thread's sampled stacks (library offsets) to gpurun_out/;
symbolize here with tools/host_sample_report.py.

usage: python tools/host_sample.py CFG OUT"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
cfg = int(sys.argv[1])
out = sys.argv[2]
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
stream = torch.cuda.Stream(device=dev)
r = bench.Runner(cfg, dev, 0, stream, None, 1, 0)
for _ in range(2):
    f, _ = r.factor_device()
    stream.synchronize()
    f.close()
torch.cuda.synchronize()
if os.path.exists(out):
    os.remove(out)
os.environ["HIFDE_SAMPLE"] = out
for _ in range(3):
    f, _ = r.factor_device()
    stream.synchronize()
    f.close()
