"""Sharded factorization over several GPUs (DESIGN.md (e)).

One process per GPU (``torchrun``), ``torch.distributed`` for the plumbing:
rank 0 creates an NCCL unique id, the process group broadcasts it, and every
rank builds the library's own NCCL communicator on its device.  Passing the
communicator to ``factor_hifde`` / ``factor_hifde3x`` / ``factor_mf``
(``comm=``) partitions the level sweep spatially: each group is factored by the
rank owning its subdomain box, the blocks a rank's groups consume from its
neighbours travel as grouped ``ncclSend/ncclRecv`` before the level, and the
coarse exact-order levels run on rank 0.  Each rank keeps the factor values
of its own records only, and ``apply_inverse`` (and ``pcg_gpu``) is the
partitioned solve: every rank runs its records level by level, and the vector
rows a rank is about to read while another holds their current value move by
grouped ``ncclSend/ncclRecv`` (neighbour-row reductions run on the rank that
reads the row next, so the result is bit-identical to the single sweep); every
rank returns the whole solution.  The communicator must outlive the factor's
solves.  ``apply``, the export and the power estimators sum the ranks' factor
arenas once, on first use (a collective: every rank calls them).
``rhs_columns`` splits a block of right-hand sides over the ranks when
independent solves are wanted instead.

The reference (``src/driver.py:183``) is single-threaded and has no
multi-process path; this module has no reference counterpart beyond the
factor API it plugs into.

``emulated_comm(P)`` runs P virtual ranks in one process on one GPU (each with
a private block arena whose unwritten blocks are NaN), which is how the
sharded path is tested on a single device.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _lib as L


class Comm:
    """Library communicator (``hifde_comm_t``)."""

    def __init__(self, handle: int, device: int):
        self._lib = L.load()
        self._h = C.c_void_p(handle)
        self.device = device
        n, r, e = C.c_int(), C.c_int(), C.c_int()
        self._lib.hifde_comm_info(self._h, C.byref(n), C.byref(r), C.byref(e))
        self.nranks, self.rank, self.emulated = int(n.value), int(r.value), bool(e.value)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self):
        if self._h is not None and self._h.value:
            self._lib.hifde_comm_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _comm_error(lib) -> str:
    return lib.hifde_comm_last_error().decode(errors="replace")


def _ensure_nccl() -> None:
    """The library resolves libnccl.so.2 at run time and prefers a copy already
    in the process: import torch first (it loads its bundled NCCL), and point
    the fallback at that same file, so the system NCCL never shadows torch's."""
    import torch  # noqa: F401

    if "HIFDE_NCCL_LIB" not in os.environ:
        try:
            import nvidia.nccl
            cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["HIFDE_NCCL_LIB"] = cand
        except ImportError:
            pass


def share_unique_id(group=None) -> bytes:
    """Rank 0's NCCL unique id, broadcast to every rank of the process group."""
    import torch.distributed as dist

    _ensure_nccl()
    lib = L.load()
    uid = C.create_string_buffer(128)
    if dist.get_rank(group) == 0:
        code = lib.hifde_comm_unique_id(uid)
        if code:
            raise RuntimeError(_comm_error(lib))
    obj = [uid.raw]
    if dist.get_world_size(group) > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_comm(group=None, device: Optional[int] = None) -> Comm:
    """Communicator over the ranks of an initialized ``torch.distributed``
    process group (NCCL backend on the GPU box; any backend can carry the id)."""
    import torch.distributed as dist

    lib = L.load()
    rank = dist.get_rank(group)
    size = dist.get_world_size(group)
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank))
    uid = share_unique_id(group) if size > 1 else bytes(128)
    h = C.c_void_p()
    code = lib.hifde_comm_init(uid, size, rank, int(device), C.byref(h))
    if code:
        raise RuntimeError(_comm_error(lib))
    return Comm(h.value, int(device))


_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int)
_SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                        C.POINTER(C.c_size_t), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                        C.POINTER(C.c_size_t))


def host_comm(group=None, device: Optional[int] = None) -> Comm:
    """Real-rank communicator whose collectives are staged through host memory
    and carried by ``torch.distributed`` (any backend, gloo included).  It runs
    the sharded path's real-rank code (exchange, merges, factor sum) without
    NCCL, e.g. two processes on one GPU; it is a test transport, not a fast one."""
    import torch
    import torch.distributed as dist

    lib = L.load()
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank))
    dtypes = {0: np.int32, 1: np.uint8, 2: np.float64}
    ops = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MAX, 2: dist.ReduceOp.MIN}

    def view(ptr, nbytes, dtype=np.uint8):
        raw = (C.c_char * nbytes).from_address(ptr)
        return torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).view(dtype))

    def allreduce(ctx, buf, count, dtype, op):
        try:
            dt = dtypes[dtype]
            dist.all_reduce(view(buf, count * np.dtype(dt).itemsize, dt), op=ops[op], group=group)
            return 0
        except Exception:
            return 1

    def sendrecv(ctx, nsend, speer, sbuf, sbytes, nrecv, rpeer, rbuf, rbytes):
        try:
            reqs = []
            for i in range(nsend):
                reqs.append(dist.isend(view(sbuf[i], sbytes[i]), int(speer[i]), group=group))
            for i in range(nrecv):
                reqs.append(dist.irecv(view(rbuf[i], rbytes[i]), int(rpeer[i]), group=group))
            for r in reqs:
                r.wait()
            return 0
        except Exception:
            return 1

    cb_a, cb_s = _ALLREDUCE(allreduce), _SENDRECV(sendrecv)
    lib.hifde_comm_host.argtypes = [C.c_int, C.c_int, C.c_int, _ALLREDUCE, _SENDRECV, C.c_void_p,
                                    C.POINTER(C.c_void_p)]
    lib.hifde_comm_host.restype = C.c_int
    h = C.c_void_p()
    if lib.hifde_comm_host(size, rank, int(device), cb_a, cb_s, None, C.byref(h)):
        raise ValueError("bad host communicator arguments")
    c = Comm(h.value, int(device))
    c._callbacks = (cb_a, cb_s)  # kept alive with the communicator
    return c


def emulated_comm(nranks: int, device: int = 0) -> Comm:
    """P virtual ranks inside this process on one device (testing)."""
    lib = L.load()
    h = C.c_void_p()
    code = lib.hifde_comm_emulated(int(nranks), int(device), C.byref(h))
    if code:
        raise ValueError("bad rank count")
    return Comm(h.value, int(device))


def rhs_columns(nrhs: int, nranks: int, rank: int) -> slice:
    """This rank's contiguous share of nrhs right-hand-side columns."""
    lo = nrhs * rank // nranks
    hi = nrhs * (rank + 1) // nranks
    return slice(lo, hi)


def shard_owner(nranks: int, dim: int, n: int, dofs) -> np.ndarray:
    """Subdomain rank of each DOF (host-only; the runtime's ownership rule)."""
    lib = L.load()
    d = np.ascontiguousarray(dofs, dtype=np.int32)
    out = np.empty(d.shape, dtype=np.int32)
    code = lib.hifde_shard_owner(int(nranks), int(dim), int(n), d.ctypes.data, d.size, out.ctypes.data)
    if code:
        raise ValueError("bad sharding arguments")
    return out


def shard_plan(nranks: int, producer, have, owner, list_ptr, lists):
    """Block transfers making every block a task lists resident on its owner
    (host-only; the runtime's planner).  Returns (xfers[k, 3] = (src, dst,
    block) sorted, updated have bits)."""
    lib = L.load()
    prod = np.ascontiguousarray(producer, dtype=np.int32)
    hv = np.ascontiguousarray(have, dtype=np.uint32).copy()
    own = np.ascontiguousarray(owner, dtype=np.int32)
    ptr = np.ascontiguousarray(list_ptr, dtype=np.int64)
    lst = np.ascontiguousarray(lists, dtype=np.int32)
    args = (int(nranks), prod.size, prod.ctypes.data, hv.ctypes.data, own.size, own.ctypes.data,
            ptr.ctypes.data, lst.ctypes.data)
    cnt = lib.hifde_shard_plan(*args, None, 0)
    if cnt < 0:
        raise ValueError("bad plan arguments")
    out = np.empty((max(cnt, 1), 3), dtype=np.int32)
    got = lib.hifde_shard_plan(*args, out.ctypes.data, cnt)
    if got != cnt:
        raise RuntimeError("shard plan size changed")
    return out[:cnt], hv
