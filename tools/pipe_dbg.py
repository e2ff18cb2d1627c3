import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2895_b200 as H
for cfg in (2, 4):
    g, a, eps, variant, nrhs = H.baseline_problem(cfg)
    fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
    f = fac(a, g, eps)
    B = np.random.default_rng(3).standard_normal((g.ndof, 64))
    for R in (8, 32, 40, 64):
        bs = torch.from_numpy(np.ascontiguousarray(B[:, :R])).cuda(); xs = torch.empty_like(bs)
        f.apply_inverse_device(bs.data_ptr(), xs.data_ptr(), R); torch.cuda.synchronize()
        x = xs.cpu().numpy()
        res = np.linalg.norm(a @ x - B[:, :R], axis=0) / np.linalg.norm(B[:, :R], axis=0)
        print(os.environ.get("HIFDE_NO_SOLVE_SMALL", "small"), cfg, R, "resid max", res.max(), flush=True)
    for li in f.level_info:
        pass
