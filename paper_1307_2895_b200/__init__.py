"""B200-native HIF-DE factor/solve (arXiv 1307.2895) behind the reference's API.

The hot path (level sweep of eliminations and ID skeletonizations, and the
apply_inverse sweep) runs in hand-written sm_100a CUDA kernels in
``libhifde_gpu.so``; this package is the thin Python face of its C ABI.
"""

import os as _os

_os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")  # before libgomp initializes

from .driver import (FactorizationError, GeneralizedLDL, IndefiniteBlockError,
                     SingularBlockError, apply_inverse, densify, device_count, factor_hifde,
                     factor_hifde3x, factor_mf, pinned_csr, pinned_empty)
from .problems import (CoeffField, GridConfig, assemble, baseline_problem, build_grid,
                       constant_field, gaussian_contrast_field, high_contrast_field)
from .gldl import export_factor, import_factor, load_factor, read_gldl, save_factor, write_gldl
from .solvers import EstimateResult, estimate_apply_error, estimate_solve_error, gmres, pcg, pcg_gpu

__version__ = "0.1.0"
