"""ctypes binding of ``include/hifde_gpu.h`` (the C ABI of libhifde_gpu.so).

There is no CPU fallback: if the library is missing or no B200 is visible the
factor entry points raise.
"""

from __future__ import annotations

import ctypes as C
import os

from ._build import LIB

HIFDE_OK, HIFDE_INDEFINITE, HIFDE_SINGULAR, HIFDE_BADARG, HIFDE_CUDA, HIFDE_INTERNAL = range(6)
VARIANT_MF, VARIANT_HIFDE, VARIANT_HIFDE3X = 0, 1, 2
ORDER = {"auto": 0, "snapshot": 1, "exact": 2}
SYMBOLIC = {"auto": 0, "device": 0, "host": 1}


class Options(C.Structure):
    _fields_ = [
        ("variant", C.c_int),
        ("skip_levels", C.c_int),
        ("spd", C.c_int),
        ("order_mode", C.c_int),
        ("exact_max_batches", C.c_int),
        ("device", C.c_int),
        ("input_on_device", C.c_int),
        ("verify", C.c_int),
        ("eps", C.c_double),
        ("stream", C.c_void_p),
        ("comm", C.c_void_p),
        ("kernel_log", C.c_int),
        ("symbolic", C.c_int),
        ("indptr_int32", C.c_int),
        ("async_factor", C.c_int),
    ]


class Info(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("dim", C.c_int32),
        ("nlevels", C.c_int32),
        ("s_top", C.c_int64),
        ("m_f_bytes", C.c_int64),
        ("device_bytes", C.c_int64),
        ("t_f_seconds", C.c_double),
        ("eps", C.c_double),
        ("spd", C.c_int32),
        ("variant", C.c_int32),
        ("fac_len", C.c_int64),
        ("idx_len", C.c_int64),
        ("nranks", C.c_int32),
        ("factor_whole", C.c_int32),
        ("xfer_bytes", C.c_int64),
        ("solve_xfer_bytes", C.c_int64),
    ]


class Record(C.Structure):  # hifde_record_t
    _fields_ = [
        ("kind", C.c_int32), ("nc", C.c_int32), ("nq", C.c_int32), ("nr", C.c_int32),
        ("cell_off", C.c_int64), ("idx_off", C.c_int64), ("P_off", C.c_int64),
        ("W_off", C.c_int64), ("T_off", C.c_int64),
    ]


class LevelInfo(C.Structure):
    _fields_ = [
        ("tag", C.c_double),
        ("kind", C.c_int32),
        ("nbatches", C.c_int32),
        ("ngroups", C.c_int64),
        ("nskel", C.c_int64),
        ("nredundant", C.c_int64),
        ("active_after", C.c_int64),
        ("max_front", C.c_int64),
        ("seconds", C.c_double),
        ("gflop", C.c_double),
        ("gbytes", C.c_double),
        ("gpu_seconds", C.c_double),
    ]


class KernelStat(C.Structure):  # hifde_kernel_stat_t
    _fields_ = [
        ("name", C.c_char * 40), ("tag", C.c_double), ("phase", C.c_int32), ("launches", C.c_int32),
        ("seconds", C.c_double), ("gbytes", C.c_double), ("gflop", C.c_double),
    ]


# every symbol the public header declares
EXPORTS = [
    "hifde_version", "hifde_device_count", "hifde_default_options", "hifde_factor",
    "hifde_solve", "hifde_host_alloc", "hifde_host_free", "hifde_apply", "hifde_pcg", "hifde_level_records", "hifde_copy_arenas", "hifde_import", "hifde_power_norm", "hifde_get_info", "hifde_get_level", "hifde_last_launch_count", "hifde_kernel_stats",
    "hifde_free", "hifde_wait", "hifde_last_error", "hifde_partition",
    "hifde_comm_unique_id", "hifde_comm_init", "hifde_comm_emulated", "hifde_comm_host", "hifde_comm_info",
    "hifde_comm_free",
    "hifde_comm_last_error", "hifde_shard_owner", "hifde_shard_plan",
]

_lib = None


def load(path: str | None = None):
    """Load (once) and type the library; raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("HIFDE_LIB_PATH") or LIB  # override: A/B builds (tools/)
    # the host symbolic phase uses OpenMP between GPU launches: idle workers
    # must sleep, not spin (spinning libgomp workers starve the host thread)
    os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
    if not os.path.exists(p):
        raise RuntimeError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(p)
    P = C.POINTER
    lib.hifde_version.restype = C.c_char_p
    lib.hifde_device_count.restype = C.c_int
    lib.hifde_default_options.argtypes = [P(Options), C.c_int]
    lib.hifde_default_options.restype = None
    lib.hifde_factor.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                 C.c_int, C.c_int, P(Options), P(C.c_void_p)]
    lib.hifde_factor.restype = C.c_int
    lib.hifde_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                C.c_void_p]
    lib.hifde_solve.restype = C.c_int
    lib.hifde_apply.argtypes = lib.hifde_solve.argtypes
    lib.hifde_apply.restype = C.c_int
    lib.hifde_pcg.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_int64, C.c_double, C.c_int, C.c_int, C.c_void_p,
                              C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int)]
    lib.hifde_pcg.restype = C.c_int
    lib.hifde_level_records.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    lib.hifde_level_records.restype = C.c_int
    lib.hifde_copy_arenas.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
    lib.hifde_copy_arenas.restype = C.c_int
    lib.hifde_import.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int,
                                 C.POINTER(C.c_void_p)]
    lib.hifde_import.restype = C.c_int
    lib.hifde_power_norm.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                     C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.hifde_power_norm.restype = C.c_int
    lib.hifde_get_info.argtypes = [C.c_void_p, P(Info)]
    lib.hifde_get_info.restype = C.c_int
    lib.hifde_get_level.argtypes = [C.c_void_p, C.c_int, P(LevelInfo)]
    lib.hifde_get_level.restype = C.c_int
    lib.hifde_last_launch_count.restype = C.c_int64
    lib.hifde_kernel_stats.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    lib.hifde_kernel_stats.restype = C.c_int
    lib.hifde_host_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p)]
    lib.hifde_host_alloc.restype = C.c_int
    lib.hifde_host_free.argtypes = [C.c_void_p]
    lib.hifde_host_free.restype = C.c_int
    lib.hifde_free.argtypes = [C.c_void_p]
    lib.hifde_free.restype = None
    lib.hifde_wait.argtypes = [C.c_void_p]
    lib.hifde_wait.restype = C.c_int
    lib.hifde_last_error.restype = C.c_char_p
    lib.hifde_partition.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
    lib.hifde_partition.restype = C.c_int64
    lib.hifde_comm_unique_id.argtypes = [C.c_void_p]
    lib.hifde_comm_unique_id.restype = C.c_int
    lib.hifde_comm_init.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    lib.hifde_comm_init.restype = C.c_int
    lib.hifde_comm_emulated.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    lib.hifde_comm_emulated.restype = C.c_int
    lib.hifde_comm_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.hifde_comm_info.restype = C.c_int
    lib.hifde_comm_free.argtypes = [C.c_void_p]
    lib.hifde_comm_free.restype = None
    lib.hifde_comm_last_error.restype = C.c_char_p
    lib.hifde_shard_owner.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
    lib.hifde_shard_owner.restype = C.c_int
    lib.hifde_shard_plan.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
    lib.hifde_shard_plan.restype = C.c_int64
    if path is None:
        _lib = lib
    return lib
