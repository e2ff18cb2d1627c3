"""Device solve time of a BASELINE config's factor for several RHS counts
(event time of back-to-back solves on resident buffers), and the launch
breakdown of one 1-RHS solve by kernel (HIFDE launches counted)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
f = fac(a, g, eps)
st = torch.cuda.Stream()
for k in (1, 16, 32):
    b = torch.randn(g.ndof, k, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(2):
        f.apply_inverse_device(b.data_ptr(), x.data_ptr(), k, st.cuda_stream)
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        f.apply_inverse_device(b.data_ptr(), x.data_ptr(), k, st.cuda_stream)
    e1.record(st)
    st.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"cfg{cfg} N={g.ndof} nrhs {k:3d}: solve {ms:.3f} ms  ({g.ndof*k/ms/1e3:.1f} M unknown-rhs/s), "
          f"factor bytes {f.metrics['m_f_bytes']/1e9:.2f} GB -> {f.metrics['m_f_bytes']/1e9/(ms/1e3):.0f} GB/s", flush=True)
