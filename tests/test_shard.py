"""Sharded level sweep.

CPU: the ownership rule and the block-transfer planner (the C++ code the
runtime uses, through its C hooks), and a world-size-2 gloo run in which two
processes hold only the blocks their own groups produced, move blocks exactly
as the planner says (each side computes the plan alone; sends and receives
must match without negotiation), and check every consumed block arrives with
the producer's payload.

GPU: the sharded factorization with P virtual ranks on one device (each with
a private, NaN-initialised block arena, so a missing transfer corrupts the
factor) against the unsharded factor -- every record byte-identical in 2D,
ranks identical and solutions within rounding in 3D.
"""

import io
import os
import socket

import numpy as np
import pytest

from paper_1307_2895_b200 import distributed as D
from paper_1307_2895_b200._build import build


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


# ---------------------------------------------------------------------------
# ownership


@pytest.mark.parametrize("dim,n", [(2, 16), (2, 64), (3, 8), (3, 16)])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_owner_boxes_cover_and_balance(dim, n, P):
    N = (n - 1) ** dim
    own = D.shard_owner(P, dim, n, np.arange(N))
    assert own.min() >= 0 and own.max() < P
    counts = np.bincount(own, minlength=P)
    assert (counts > 0).all()
    # boxes split the axes into slabs of (nearly) equal width
    assert counts.max() - counts.min() <= 2 * (n - 1) ** (dim - 1) * (1 + (P % 2))
    if P & (P - 1):
        return  # odd rank counts split axis 0 evenly, not along cell boundaries
    # every DOF of a level-0 leaf cell (interior of an m-box) shares one owner
    m = 4
    x = np.indices([n - 1] * dim).reshape(dim, -1)[::-1] + 1  # first axis fastest
    key = sum((x[ax] // m) * (n // m) ** ax for ax in range(dim))
    inner = np.all(x % m != 0, axis=0)
    for k in np.unique(key[inner])[:50]:
        assert len(set(own[(key == k) & inner])) == 1


def test_owner_split_planes():
    # P = 2 splits axis 0 at the middle separator (x = n/2 belongs to rank 1)
    n = 16
    own = D.shard_owner(2, 2, n, np.arange((n - 1) ** 2)).reshape(n - 1, n - 1)
    assert (own[:, : n // 2 - 1] == 0).all() and (own[:, n // 2 - 1:] == 1).all()
    with pytest.raises(ValueError):
        D.shard_owner(2, 2, n, [(n - 1) ** 2])


# ---------------------------------------------------------------------------
# planner


def _random_levels(rng, P, nlev=5, ntask=40, nb0=60):
    """Block producers and per-level consumption lists (tasks own blocks)."""
    producer = list(rng.integers(0, P, nb0))
    levels = []
    for _ in range(nlev):
        nb = len(producer)
        owner = rng.integers(0, P, ntask)
        lists, ptr = [], [0]
        for t in range(ntask):
            k = int(rng.integers(0, 6))
            lists += list(rng.choice(nb, size=k, replace=False))
            ptr.append(len(lists))
        levels.append((owner, np.array(ptr), np.array(lists, dtype=np.int32)))
        producer += list(owner)  # every task produces one new block
    return producer, levels


@pytest.mark.parametrize("P", [2, 3, 8])
def test_plan_makes_consumed_blocks_resident_once(P):
    rng = np.random.default_rng(P)
    producer, levels = _random_levels(rng, P)
    have = np.zeros(len(producer), dtype=np.uint32)
    nb_known = 60
    have[:nb_known] = 1 << np.array(producer[:nb_known], dtype=np.uint32)
    for owner, ptr, lists in levels:
        prod = np.array(producer[: nb_known], dtype=np.int32)
        x, hv = D.shard_plan(P, prod, have[:nb_known], owner, ptr, lists)
        # sorted by (src, dst, block), sources are producers, no duplicates
        keys = [tuple(r) for r in x]
        assert keys == sorted(keys) and len(set(keys)) == len(keys)
        for s_, d_, b_ in x:
            assert prod[b_] == s_ and s_ != d_
        for t in range(len(owner)):
            for b_ in lists[ptr[t]:ptr[t + 1]]:
                assert hv[b_] >> owner[t] & 1
        # a second plan over the same lists moves nothing
        x2, _ = D.shard_plan(P, prod, hv, owner, ptr, lists)
        assert len(x2) == 0
        have[:nb_known] = hv
        nb_new = len(owner)
        have[nb_known:nb_known + nb_new] = 1 << owner.astype(np.uint32)
        nb_known += nb_new


def test_plan_rejects_bad_input():
    with pytest.raises(ValueError):
        D.shard_plan(2, [0, 5], [0, 0], [0], [0, 1], [0])
    with pytest.raises(ValueError):
        D.shard_plan(2, [0, 1], [0, 0], [2], [0, 1], [0])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, seed, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)  # same structure on every rank
        producer, levels = _random_levels(rng, world, nlev=6, ntask=50, nb0=80)
        size = {b: 3 + (b * 7) % 11 for b in range(len(producer))}

        def payload(b):
            return np.sin(np.arange(size[b]) + 13.0 * b)

        store = {b: payload(b) for b in range(80) if producer[b] == rank}
        have = np.zeros(len(producer), dtype=np.uint32)
        have[:80] = 1 << np.array(producer[:80], dtype=np.uint32)
        nb_known, moved = 80, 0
        for owner, ptr, lists in levels:
            x, hv = D.shard_plan(world, np.array(producer[:nb_known], dtype=np.int32), have[:nb_known],
                                 owner, ptr, lists)
            have[:nb_known] = hv
            # packed per (src, dst) pair in plan order, exactly like the runtime
            for peer in range(world):
                if peer == rank:
                    continue
                out = [b for s_, d_, b in x if s_ == rank and d_ == peer]
                inc = [b for s_, d_, b in x if s_ == peer and d_ == rank]
                sbuf = torch.from_numpy(np.concatenate([store[b] for b in out]) if out else np.zeros(0))
                rbuf = torch.zeros(sum(size[b] for b in inc), dtype=torch.float64)
                if rank < peer:
                    if sbuf.numel():
                        dist.send(sbuf, peer)
                    if rbuf.numel():
                        dist.recv(rbuf, peer)
                else:
                    if rbuf.numel():
                        dist.recv(rbuf, peer)
                    if sbuf.numel():
                        dist.send(sbuf, peer)
                o = 0
                for b in inc:
                    store[b] = rbuf[o:o + size[b]].numpy().copy()
                    o += size[b]
                moved += len(inc)
            # every block my tasks consume is here with the producer's values
            for t in range(len(owner)):
                if owner[t] != rank:
                    continue
                for b in lists[ptr[t]:ptr[t + 1]]:
                    assert np.array_equal(store[int(b)], payload(int(b))), (rank, b)
            # my tasks produce their blocks
            for t in range(len(owner)):
                b = nb_known + t
                if owner[t] == rank:
                    store[b] = payload(b)
            have[nb_known:nb_known + len(owner)] = 1 << owner.astype(np.uint32)
            nb_known += len(owner)
        q.put((rank, "ok", moved))
    except Exception as e:  # reported to the parent
        q.put((rank, repr(e), 0))
    finally:
        dist.destroy_process_group()


def test_block_exchange_two_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, 7, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
    assert sum(r[2] for r in res) > 0


def _id_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, D.share_unique_id()))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_unique_id_is_shared_over_the_process_group():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert isinstance(res[0], bytes) and len(res[0]) == 128, res
    assert res[0] == res[1] and any(res[0])


def test_rhs_columns_partition():
    for nrhs in (1, 16, 17, 64):
        for P in (1, 2, 3, 8):
            cols = [D.rhs_columns(nrhs, P, r) for r in range(P)]
            got = np.concatenate([np.arange(nrhs)[c] for c in cols])
            assert np.array_equal(got, np.arange(nrhs))


# ---------------------------------------------------------------------------
# GPU: emulated ranks against the unsharded factor


def _gldl_bytes(f):
    from paper_1307_2895_b200 import gldl

    buf = io.BytesIO()
    path = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"shard_{os.getpid()}_{id(f)}.gldl")
    gldl.save_factor(f, path)
    with open(path, "rb") as fh:
        buf.write(fh.read())
    os.remove(path)
    return buf.getvalue()


def _raw_clone(f):
    """An unsharded device factor holding exactly f's records (arenas copied
    through hifde_copy_arenas / hifde_level_records into hifde_import)."""
    import ctypes as C
    from paper_1307_2895_b200 import _lib as L
    from paper_1307_2895_b200.driver import GeneralizedLDL

    lib = f._lib
    info = L.Info()
    lib.hifde_get_info(f._h, C.byref(info))
    fac = np.empty(int(info.fac_len), dtype=np.float64)
    idx = np.empty(int(info.idx_len), dtype=np.int32)
    assert lib.hifde_copy_arenas(f._h, fac.ctypes.data, fac.size, idx.ctypes.data, idx.size) == 0
    recs, ptr, tags, kinds = [], [0], [], []
    nlev = int(info.nlevels) + 1
    for li in range(nlev):
        cnt = C.c_int64()
        lib.hifde_level_records(f._h, li, None, 0, C.byref(cnt))
        rr = (L.Record * max(cnt.value, 1))()
        lib.hifde_level_records(f._h, li, rr, cnt.value, C.byref(cnt))
        recs.extend(rr[:cnt.value])
        ptr.append(len(recs))
        tags.append(float(f.level_info[li]["tag"]))
        kinds.append(2 if li == nlev - 1 else int(f.level_info[li]["kind"]))
    arr = (L.Record * len(recs))(*recs)
    tg, kd, pt = (np.asarray(tags, np.float64), np.asarray(kinds, np.int32), np.asarray(ptr, np.int64))
    h = C.c_void_p()
    code = lib.hifde_import(f.n, int(info.dim), float(info.eps), len(tags), tg.ctypes.data, kd.ctypes.data,
                            pt.ctypes.data, arr, fac.ctypes.data, fac.size, idx.ctypes.data, idx.size, 0, C.byref(h))
    assert code == 0, lib.hifde_last_error()
    return GeneralizedLDL(h.value, lib, True)


def _problem(dim, n, m, contrast):
    import paper_1307_2895_b200 as H

    g = H.build_grid(dim, n, m)
    field = H.gaussian_contrast_field(g, seed=3) if contrast else H.constant_field(g, 1.0, 0.0)
    return g, H.assemble(g, field)


@pytest.mark.gpu
@pytest.mark.parametrize("variant,dim,n,m,eps,contrast,ranks", [
    ("hifde", 2, 64, 8, 1e-6, True, (2, 3, 4, 8)),
    ("hifde", 2, 128, 8, 1e-9, False, (2, 4)),
    ("mf", 2, 64, 8, 0.0, False, (2, 4)),
])
def test_sharded_2d_factor_is_byte_identical(variant, dim, n, m, eps, contrast, ranks):
    import paper_1307_2895_b200 as H

    g, a = _problem(dim, n, m, contrast)
    fac = {"hifde": lambda **k: H.factor_hifde(a, g, eps, **k),
           "mf": lambda **k: H.factor_mf(a, g, **k)}[variant]
    b = np.random.default_rng(0).standard_normal((g.ndof, 3))
    f0 = fac()
    ref, x0 = _gldl_bytes(f0), f0.apply_inverse(b)
    for P in ranks:
        c = D.emulated_comm(P)
        f = fac(comm=c)
        assert f.metrics["nranks"] == P
        assert f.metrics["xfer_bytes"] > 0
        assert f.metrics["skeleton_counts"] == f0.metrics["skeleton_counts"]
        assert _gldl_bytes(f) == ref, P
        assert np.array_equal(f.apply_inverse(b), x0)
        f.close()
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("variant,dim,n,m,eps,P", [
    ("hifde", 2, 64, 8, 1e-6, 4),
    ("hifde", 2, 128, 8, 1e-9, 8),
    ("hifde3x", 3, 16, 4, 1e-6, 8),
    ("hifde3x", 3, 32, 4, 1e-6, 2),
    ("hifde3x", 3, 32, 4, 1e-6, 8),
    ("mf", 2, 64, 8, 0.0, 4),
])
def test_partitioned_solve_matches_whole_sweep(variant, dim, n, m, eps, P):
    """The partitioned solve (each virtual rank runs only its own records on
    its own copy of the vector; rows and contribution rows move as the
    per-level plans say) against the single-sweep solve of the same factor
    (exported and re-imported unsharded): identical for every RHS width --
    the same records, the same kernels' arithmetic, reductions in record
    order.  PCG with the partitioned preconditioner converges as the
    unsharded one."""
    import paper_1307_2895_b200 as H
    from paper_1307_2895_b200 import solvers

    g, a = _problem(dim, n, m, True)
    fac = {"hifde": lambda **k: H.factor_hifde(a, g, eps, **k), "mf": lambda **k: H.factor_mf(a, g, **k),
           "hifde3x": lambda **k: H.factor_hifde3x(a, g, eps, **k)}[variant]
    c = D.emulated_comm(P)
    f = fac(comm=c)
    f1 = _raw_clone(f)
    rng = np.random.default_rng(7)
    assert f.shard_info()["solve_xfer_bytes"] == 0
    for nrhs in (1, 2, 3, 8, 16, 64):
        b = rng.standard_normal((g.ndof, nrhs)) if nrhs > 1 else rng.standard_normal(g.ndof)
        x, x1 = f.apply_inverse(b), f1.apply_inverse(b)
        assert np.array_equal(x, x1), (nrhs, np.abs(x - x1).max())
    assert f.shard_info()["solve_xfer_bytes"] > 0
    b = rng.standard_normal(g.ndof)
    r, r1 = solvers.pcg_gpu(f, a, b), solvers.pcg_gpu(f1, a, b)
    assert r.converged and r.n_i == r1.n_i
    assert np.array_equal(r.x, r1.x)
    f.close()
    f1.close()
    c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n,m,contrast,ranks", [(3, 16, 4, False, (2, 4, 8)), (3, 32, 4, True, (8,))])
def test_sharded_3d_factor_matches(dim, n, m, contrast, ranks):
    """3D: the large-group CPQR splits SMs over the groups a launch holds, so
    a rank's subset can round differently; ranks and solutions must agree."""
    import paper_1307_2895_b200 as H

    g, a = _problem(dim, n, m, contrast)
    b = np.random.default_rng(0).standard_normal((g.ndof, 2))
    f0 = H.factor_hifde3x(a, g, 1e-6)
    x0 = f0.apply_inverse(b)
    for P in ranks:
        c = D.emulated_comm(P)
        f = H.factor_hifde3x(a, g, 1e-6, comm=c)
        for (t0, k0), (t1, k1) in zip(f0.metrics["skeleton_counts"], f.metrics["skeleton_counts"]):
            assert t0 == t1 and abs(k0 - k1) <= max(1, 0.02 * k0)
        x = f.apply_inverse(b)
        assert np.linalg.norm(x - x0) <= 1e-8 * np.linalg.norm(x0)
        f.close()
        c.close()


@pytest.mark.gpu
def test_sharded_full_size_config2_byte_identical():
    import paper_1307_2895_b200 as H

    g, a, eps, variant, nrhs = H.baseline_problem(2)
    f0 = H.factor_hifde(a, g, eps)
    ref = _gldl_bytes(f0)
    f0.close()
    c = D.emulated_comm(4)
    f = H.factor_hifde(a, g, eps, comm=c)
    assert _gldl_bytes(f) == ref
    f.close()
    c.close()


@pytest.mark.gpu
def test_emulated_single_rank_is_the_plain_path():
    import paper_1307_2895_b200 as H

    g, a = _problem(2, 32, 4, True)
    c = D.emulated_comm(1)
    f = H.factor_hifde(a, g, 1e-6, comm=c)
    assert f.metrics["nranks"] == 1 and f.metrics["xfer_bytes"] == 0
    assert _gldl_bytes(f) == _gldl_bytes(H.factor_hifde(a, g, 1e-6))


# ---------------------------------------------------------------------------
# GPU: the real-rank path (not emulated) with two processes on one GPU, the
# collectives staged through the host and carried by gloo (hifde_comm_host)


def _real_rank_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import paper_1307_2895_b200 as H

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        comm = D.host_comm(device=0)
        out = {}
        for name, (dim, n, m, eps, contrast, var) in {
                "2d": (2, 64, 8, 1e-6, True, "hifde"), "3d": (3, 16, 4, 1e-6, False, "hifde3x"),
                "3d_large": (3, 32, 4, 1e-6, True, "hifde3x")}.items():
            g, a = _problem(dim, n, m, contrast)
            fac = H.factor_hifde if var == "hifde" else H.factor_hifde3x
            f = fac(a, g, eps, comm=comm, device=0)
            b = np.random.default_rng(0).standard_normal((g.ndof, 2))
            # the partitioned solve runs on each rank's own records: the
            # factor arenas are not summed until the export needs them
            x = f.apply_inverse(b)
            st = f.shard_info()
            assert not st["factor_whole"] and st["solve_xfer_bytes"] > 0, st
            out[name] = (_gldl_bytes(f), x, f.metrics["skeleton_counts"], f.metrics["nranks"],
                         f.metrics["xfer_bytes"])
            assert f.shard_info()["factor_whole"]
            assert np.array_equal(f.apply_inverse(b), x)
            if rank == 0:
                f0 = fac(a, g, eps, device=0)
                out[name + "_ref"] = (_gldl_bytes(f0), f0.apply_inverse(b), f0.metrics["skeleton_counts"])
        comm.close()
        q.put((rank, "ok", out))
    except Exception as e:
        import traceback
        q.put((rank, traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_real_ranks_over_host_transport_two_processes():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_real_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, status, out = q.get(timeout=600)
        res[r] = (status, out)
    for p in procs:
        p.join(timeout=60)
    assert all(v[0] == "ok" for v in res.values()), res
    o0, o1 = res[0][1], res[1][1]
    for name in ("2d", "3d", "3d_large"):  # 3d_large: large groups (Gram path) split over the ranks per batch
        b0, x0, k0, nr, xb = o0[name]
        b1, x1, k1, _, _ = o1[name]
        rb, rx, rk = o0[name + "_ref"]
        assert nr == 2 and xb > 0
        assert b0 == b1 and np.array_equal(x0, x1)  # both ranks hold the same whole factor
        for (t0, c0), (t1, c1) in zip(k0, rk):
            assert t0 == t1 and abs(c0 - c1) <= max(1, 0.02 * c1)
        if name == "2d":
            assert b0 == rb and np.array_equal(x0, rx)  # the single-GPU factor, byte for byte
        else:
            assert np.linalg.norm(x0 - rx) <= 1e-8 * np.linalg.norm(rx)
