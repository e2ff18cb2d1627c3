"""Solve latency right after a factorization (as in bench.py's step): host
time of the hifde_solve call and the event interval, vs a back-to-back solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1307_2895_b200 as H
g, a, eps, variant, nrhs = H.baseline_problem(2)
st = torch.cuda.Stream()
b = torch.randn(g.ndof, nrhs, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
for rep in range(int(os.environ.get("REPS", "5"))):
    f = H.factor_hifde(a, g, eps, stream=st.cuda_stream)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(st)
    t0 = time.perf_counter()
    f.apply_inverse_device(b.data_ptr(), x.data_ptr(), nrhs, st.cuda_stream)
    t1 = time.perf_counter()
    e[1].record(st)
    f.apply_inverse_device(b.data_ptr(), x.data_ptr(), nrhs, st.cuda_stream)
    e[2].record(st)
    st.synchronize()
    print(f"rep {rep}: host call {1e3*(t1-t0):.3f} ms | first solve {e[0].elapsed_time(e[1]):.3f} ms | "
          f"second {e[1].elapsed_time(e[2]):.3f} ms")
    f.close()
