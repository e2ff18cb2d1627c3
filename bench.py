"""HIF-DE factor & solve benchmark (BASELINE.json metric) on B200.

Workload: BASELINE.json configs[2] ("config 3"), the largest configuration
that fits one B200 and the one the metric is quoted on at 1/2/4/8 GPUs:
2D five-point Laplacian, n = 2047 interior points per side (N = 4,190,209),
a = 1, b = 0, leaf 8x8, eps = 1e-6, 64 right-hand sides ~ N(0,1).  Synthetic,
seeded inputs generated in-process (the reference's own problems are
synthetic PDEs generated in code).

One step = factor_hifde of the matrix + apply_inverse of the 64-RHS block.
  value = N / (t_factor + t_solve)  [unknowns/s], inputs resident in HBM,
          CUDA events on the library's stream, L2 flushed between steps;
  e2e   = the same through the public Python API with host buffers (CSR and
          RHS host->device, solution device->host inside the timed region).
The line also carries config 5 (3D high-contrast hifde3x, N = 2,048,383,
eps = 1e-3, 32 RHS), the other 1/2/4/8-GPU configuration, as extra keys.

Multi-GPU (torchrun, --gpus N > 1): ONE instance of the config is factored
sharded over the N ranks (spatial group owners, NCCL block exchange; DESIGN.md
(e)) and the right-hand-side columns are split over the ranks: strong scaling.

`--impl reference` times the CPU oracle port of the reference algorithm
(oracle/hifde_oracle.py; the reference is pure Python and does not travel to
the GPU box) on this host: each step one bounded sample of the workload on
every host core (an independent process per core, each a 255x255 instance of
the config-3 operator, same leaf, eps and 64 RHS).
"""

from __future__ import annotations

import argparse
import json
import os

os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")  # before torch / libgomp initialize
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = 3
METRIC = "HIF-DE factor & solve unknowns/sec"
WORKLOADS = {
    2: "cfg2: 2D 5-point high-contrast (Gaussian, 4h, thr 0) n=511 N=261121, leaf 8x8, eps=1e-9, hifde, 16 RHS",
    3: "cfg3: 2D 5-point Laplacian n=2047 N=4190209, leaf 8x8, eps=1e-6, hifde, 64 RHS",
    4: "cfg4: 3D 7-point Laplacian n=63 N=250047, leaf 4^3, eps=1e-6, hifde3x, 16 RHS",
    5: "cfg5: 3D 7-point high-contrast (Gaussian, 4h, thr 0) n=127 N=2048383, leaf 4^3, eps=1e-3, hifde3x, 32 RHS",
}
# CPU sample of the reference arm / cpu_baseline: config 3's operator on a
# 255 x 255 grid (1/64 of its unknowns), same leaf, eps and RHS count
SAMPLE = (2, 256, 8, 1e-6, 64)
SAMPLE_TEXT = ("per host core one oracle-port factor_hifde + 64-RHS apply_inverse of the config-3 operator "
               "(2D Laplacian, leaf 8x8, eps 1e-6) on a 255x255 grid (N=65025), cores running concurrently")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk, kind = json.load(fh), "measured (MEASURED_PEAKS.json)"
    except Exception:
        pk, kind = {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"
    # FP64 roof: cuBLAS DGEMM 8192^3 sustained on this pool's B200
    # (profiles/r01_fp64_peak.json, tools/fp64_peak.py); not in MEASURED_PEAKS.json
    fp64 = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as fh:
            fp64 = float(json.load(fh)["dgemm_tflops_sustained"])
    except Exception:
        pass
    pk = dict(pk)
    pk["fp64_tflops"] = fp64 or 35.5
    return pk, kind


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        util = [float(s[7]) for s in self.samples if len(s) > 7 and s[7].replace(".", "").isdigit()]
        loaded = [c for c, u in zip(sm, util) if u > 0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(cfg, world, nranks=None):
    return {"workload": WORKLOADS[cfg] + "; step = factor + RHS-block solve",
            "parallelism": f"shard x{nranks or world}" if (nranks or world) > 1 else "single GPU",
            "l2": "flushed between timed steps (256 MiB write)"}


# --------------------------------------------------------------------------
# CPU side: the oracle port of the reference algorithm (reference arm and
# cpu_baseline).  Each worker process factors and solves one sample.
# --------------------------------------------------------------------------
_SAMPLE_PROBLEM = None


def _pool_init():
    """Worker start-up: BLAS on one thread (the reference pins its level loop to
    one, src/driver.py:35-41) and the sample problem assembled once."""
    global _SAMPLE_PROBLEM
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ROOT)
    import paper_1307_2895_b200.problems as P
    dim, n, m, eps, nrhs = SAMPLE
    g = P.build_grid(dim, n, m)
    a = P.assemble(g, P.constant_field(g))
    b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
    _SAMPLE_PROBLEM = (g, a, b)


def _sample_worker(_):
    from oracle import hifde_oracle as O
    g, a, b = _SAMPLE_PROBLEM
    dim, n, m, eps, nrhs = SAMPLE
    t0 = time.perf_counter()
    f = O.factor(a, O.make_grid(dim, n, m), eps, "hifde")
    tf = time.perf_counter() - t0
    x = f.apply_inverse(b)
    t = time.perf_counter() - t0
    resid = float(np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0)))
    return g.ndof, t, tf, resid, os.getpid()


class CpuPool:
    """One worker process per host core; a step runs one sample on each.  The
    step time is the slowest worker's factor + solve time (the samples run
    concurrently), or the pool's wall time if a worker ran two samples."""

    def __init__(self, cores):
        import multiprocessing as mp
        self.cores = cores
        self.pool = mp.get_context("spawn").Pool(cores, initializer=_pool_init)

    def step(self):
        t0 = time.perf_counter()
        res = self.pool.map(_sample_worker, range(self.cores), chunksize=1)
        wall = time.perf_counter() - t0
        t = max(r[1] for r in res) if len({r[4] for r in res}) == len(res) else wall
        return sum(r[0] for r in res), t, res

    def close(self):
        self.pool.close()
        self.pool.join()


def host_cores():
    try:
        return max(1, min(len(os.sched_getaffinity(0)), 32))
    except Exception:
        return max(1, min(os.cpu_count() or 1, 32))


def cpu_reference(args, world, rank):
    """Reference arm: the oracle port on all host cores, rank 0 only."""
    if rank != 0:
        return
    cores = host_cores()
    pool = CpuPool(cores)
    pool.step()  # worker start-up and imports, untimed
    times, unknowns, tfs, resid = [], 0, [], 0.0
    for i in range(args.warmup + args.steps):
        n, wall, res = pool.step()
        if i >= args.warmup:
            times.append(wall)
            unknowns = n
            tfs.append(max(r[2] for r in res))
            resid = max(r[3] for r in res)
    pool.close()
    tt = float(np.mean(times))
    value = unknowns / tt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "unknowns/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tt * 1e3,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic (seeded BASELINE cfg{args.config}-shaped sample)",
        "config": config_dict(args.config, world),
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": cores, "kind": "port",
                         "sample": SAMPLE_TEXT + "; oracle port = CPU restatement of the reference "
                                                 "(pure-Python reference cannot travel to the GPU box)"},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "resid": resid,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline():
    cores = host_cores()
    pool = CpuPool(cores)
    pool.step()
    vals = []
    for _ in range(2):
        n, wall, _ = pool.step()
        vals.append(n / wall)
    pool.close()
    return {"value": float(np.mean(vals)), "unit": "unknowns/s", "cores": cores, "kind": "port",
            "sample": SAMPLE_TEXT + ", 2 rounds"}


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
class Runner:
    """One configuration on this rank: device-resident inputs, the timed
    step through the C ABI, and the e2e step through the Python API."""

    def __init__(self, cfg, dev, local, stream, comm, world, rank):
        import torch
        import paper_1307_2895_b200 as H
        from paper_1307_2895_b200 import distributed as D
        self.H, self.torch = H, torch
        self.cfg, self.local, self.stream, self.comm = cfg, local, stream, comm
        g, a, eps, variant, nrhs = H.baseline_problem(cfg)
        self.g, self.a, self.eps, self.variant, self.nrhs = g, a, eps, variant, nrhs
        self.N = g.ndof
        cols = D.rhs_columns(nrhs, world, rank) if world > 1 else slice(0, nrhs)
        self.nloc = cols.stop - cols.start
        b_full = np.random.default_rng(1).standard_normal((self.N, nrhs))
        self.b_host = np.ascontiguousarray(b_full[:, cols])
        self.b_pin = torch.from_numpy(self.b_host).pin_memory()  # e2e: inputs from pinned host memory
        self.a_pin = H.pinned_csr(a)  # the CSR's three arrays page-locked too (direct DMA in factor_hifde)
        self.indptr_d = torch.from_numpy(a.indptr.astype(np.int64)).to(dev)
        self.indices_d = torch.from_numpy(a.indices.astype(np.int32)).to(dev)
        self.data_d = torch.from_numpy(a.data.astype(np.float64)).to(dev)
        self.b_d = torch.from_numpy(self.b_host).to(dev)
        self.x_d = torch.empty_like(self.b_d)
        self.fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x

    def factor_device(self, kernel_log=True):
        import ctypes as C
        from paper_1307_2895_b200 import _lib
        lib = _lib.load()
        opt = _lib.Options()
        lib.hifde_default_options(C.byref(opt), _lib.VARIANT_HIFDE if self.variant == "hifde" else _lib.VARIANT_HIFDE3X)
        opt.eps = self.eps
        opt.device = self.local
        opt.input_on_device = 1
        opt.stream = self.stream.cuda_stream
        opt.comm = self.comm.handle if self.comm is not None else None
        opt.kernel_log = int(kernel_log)
        h = C.c_void_p()
        code = lib.hifde_factor(self.indptr_d.data_ptr(), self.indices_d.data_ptr(), self.data_d.data_ptr(),
                                self.N, self.g.dim, self.g.n, self.g.m, self.g.nlevels, C.byref(opt), C.byref(h))
        if code:
            raise RuntimeError(lib.hifde_last_error().decode())
        return self.H.GeneralizedLDL(h.value, lib, True), int(lib.hifde_last_launch_count())

    def solve_device(self, f):
        from paper_1307_2895_b200 import _lib
        if not self.nloc:
            return 0
        f.apply_inverse_device(self.b_d.data_ptr(), self.x_d.data_ptr(), self.nloc, self.stream.cuda_stream)
        return int(_lib.load().hifde_last_launch_count())

    def timed(self, steps, warmup, flush, clock=None):
        torch = self.torch
        s = self.stream
        for _ in range(warmup):
            f, _ = self.factor_device()
            self.solve_device(f)
            s.synchronize()
            f.close()
        torch.cuda.synchronize()
        times, tfs, launches = [], [], 0
        kstats = None
        for i in range(steps):
            flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            s.wait_stream(torch.cuda.current_stream())
            e0.record(s)
            f, nl = self.factor_device()
            e1.record(s)
            nl += self.solve_device(f)
            e2.record(s)
            e2.synchronize()
            launches += nl
            times.append(e0.elapsed_time(e2) / 1e3)
            tfs.append(e0.elapsed_time(e1) / 1e3)
            if kstats is None:
                kstats = []
            for ph in (0, 1):
                for k in f.kernel_stats(ph):
                    kstats.append(k)
            if i == steps - 1:
                self.level_info = f.level_info
                self.skel = f.metrics["skeleton_counts"]
                self.xfer = f.metrics["xfer_bytes"]
                x = self.x_d.cpu().numpy()
                self.resid = (float(np.max(np.linalg.norm(self.a @ x - self.b_host, axis=0)
                                           / np.linalg.norm(self.b_host, axis=0))) if self.nloc else 0.0)
            f.close()
        torch.cuda.synchronize()
        self.kstats = kstats
        return float(np.mean(times)), float(np.mean(tfs)), launches

    def e2e(self, steps, dist, wait=True):
        """factor + apply_inverse through the public API, host buffers.
        wait=False: factor_hifde returns while the factorization runs on the
        library's thread, so the apply_inverse that follows uploads its
        right-hand sides meanwhile (one GPU; same calls, same results)."""
        torch = self.torch
        ts = []
        kw = {} if wait else {"wait": False}
        for i in range(steps + 1):
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fe = self.fac(self.a_pin, self.g, self.eps, stream=self.stream.cuda_stream, device=self.local,
                          comm=self.comm, **kw)
            if self.nloc:
                x = fe.apply_inverse(self.b_pin.numpy())
            else:
                fe.wait()
            t = time.perf_counter() - t0
            if i == steps and self.nloc and self.comm is None:  # the result is the solution (not timed)
                xs = np.asarray(x[:, :2])
                bs = self.b_host[:, :2]
                self.e2e_resid = float(np.max(np.linalg.norm(self.a @ xs - bs, axis=0) / np.linalg.norm(bs, axis=0)))
            x = None
            fe.close()
            if i > 0:  # first call warms the host caches of the public path
                ts.append(t)
        steps_ms = [round(t * 1e3, 2) for t in ts]
        if wait:
            self.e2e_blocking_steps_ms = steps_ms
        else:
            self.e2e_steps_ms = steps_ms
        return float(np.mean(ts))


def roofline(kstats, steps, pk, pk_kind):
    """Dominant kernel of the step by CUDA-event time (the kernel log of the
    library: every main launch bracketed by events on the stream it runs on).
    achieved = its algorithmic bytes (or FLOPs) per launch over its average
    launch duration; bound = FP64 tensor pipe when the work's arithmetic
    intensity is above the ridge (measured DGEMM / measured copy), else HBM."""
    agg = {}
    for k in kstats:
        key = (k["name"], round(k["tag"], 4), k["phase"])
        a = agg.setdefault(key, {"name": k["name"], "tag": k["tag"], "phase": k["phase"],
                                 "launches": 0, "seconds": 0.0, "gbytes": 0.0, "gflop": 0.0})
        for f in ("launches", "seconds", "gbytes", "gflop"):
            a[f] += k[f]
    total = sum(a["seconds"] for a in agg.values())
    # the roofline's kernel: the one with the most time among those with
    # algorithmic work (the device symbolic pass is integer bookkeeping with
    # no bytes/FLOPs model, and its interval on the second stream spans the
    # elimination kernels it overlaps)
    dom = max((a for a in agg.values() if a["gbytes"] > 0 or a["gflop"] > 0), key=lambda a: a["seconds"])
    per_launch_s = dom["seconds"] / max(dom["launches"], 1)
    gb_l = dom["gbytes"] / max(dom["launches"], 1)
    gf_l = dom["gflop"] / max(dom["launches"], 1)
    ridge = pk["fp64_tflops"] * 1e3 / pk["hbm_gbs"]
    ai = gf_l / gb_l if gb_l > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_r02.json")) as fh:
            tr = json.load(fh)["dram_bytes_per_launch"]
            v = tr.get(f"{dom['name']}@{dom['tag']:.3f}")
            traffic = v / 1e9 if v else None
    except Exception:
        pass
    if ai > ridge:
        achieved, peak, unit, bound = gf_l / per_launch_s * 1e-3, pk["fp64_tflops"], "TFLOP/s", "tensor"
        peak_kind = "measured cuBLAS DGEMM 8192^3 (profiles/r01_fp64_peak.json; FP64 DMMA pipe)"
    else:
        achieved, peak, unit, bound = gb_l / per_launch_s, pk["hbm_gbs"], "GB/s", "hbm"
        peak_kind = pk_kind + " hbm_gbs"
    top = sorted(agg.values(), key=lambda a: -a["seconds"])[:8]
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "traffic_unit": "GB per launch (ncu dram__bytes_read+write)",
            "kernel": dom["name"], "level": dom["tag"], "phase": "solve" if dom["phase"] else "factor",
            "launches_per_step": dom["launches"] / steps, "launch_seconds": per_launch_s,
            "algorithmic_gbytes_per_launch": gb_l, "algorithmic_gflop_per_launch": gf_l,
            "share_of_logged_time": dom["seconds"] / total if total else None,
            "launch_seconds_note": ("CUDA events around the launch inside the timed step; the level-0 elimination's "
                                    "interval includes the level-0.5 symbolic analysis, which runs on a high-priority "
                                    "stream on the same SMs (the kernel alone under ncu: profiles/r02_ncu_final.txt)"
                                    if dom["name"] == "elim_small_kernel" and dom["tag"] == 0.0 else
                                    "CUDA events around the launch inside the timed step"),
            "peak_kind": peak_kind,
            "top_kernels": [{"kernel": a["name"], "level": a["tag"], "phase": a["phase"],
                             "ms_per_step": a["seconds"] / steps * 1e3,
                             "gb_s": a["gbytes"] / a["seconds"] if a["seconds"] else None,
                             "tflop_s": a["gflop"] / a["seconds"] * 1e-3 if a["seconds"] else None}
                            for a in top]}


def run_gpu(args, world, rank, local):
    import torch
    from paper_1307_2895_b200 import distributed as D

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_baseline()  # before CUDA initializes (spawned worker processes)
    dist = None
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        comm = D.init_comm(device=local)
    elif args.emulate > 1:
        comm = D.emulated_comm(args.emulate, local)
    nranks = comm.nranks if comm is not None else 1
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    R = Runner(args.config, dev, local, stream, comm, world, rank)
    with torch.cuda.stream(stream):
        if dist:
            dist.barrier()
        with ClockSampler(local) as clk:
            t_step, t_f, launches = R.timed(args.steps, args.warmup, flush)
        if dist:
            dist.barrier()
        # e2e: the public calls with wait=False on one GPU (upload of the
        # right-hand sides under the factorization); the blocking calls beside it
        t_e2e_block = R.e2e(max(1, min(args.steps, 10)), dist, wait=True)
        t_e2e = R.e2e(max(1, min(args.steps, 10)), dist, wait=False) if world == 1 else t_e2e_block
        if world > 1:
            R.e2e_steps_ms = R.e2e_blocking_steps_ms
        extra = None
        if world == 1 and args.config == 3 and not args.no_extra:
            R5 = Runner(5, dev, local, stream, None, 1, 0)
            t5, tf5, _ = R5.timed(2, 2, flush)
            extra = {"workload": WORKLOADS[5] + "; device-resident, 2 warm-up + 2 timed steps",
                     "ms_per_step": t5 * 1e3, "factor_ms": tf5 * 1e3, "solve_ms": (t5 - tf5) * 1e3,
                     "unknowns_per_s": R5.N / t5, "factor_unknowns_per_s": R5.N / tf5,
                     "solve_unknown_rhs_per_s": R5.N * R5.nrhs / (t5 - tf5), "resid": R5.resid,
                     "skeleton_counts": [c for _, c in R5.skel],
                     "roofline": roofline(R5.kstats, 2, *peaks())}
            del R5
    t_s = t_step - t_f
    if dist:
        tt = torch.tensor([t_step, t_e2e, t_f, t_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_e2e, t_f, t_s = [float(v) for v in tt.cpu()]
        t_e2e_block = t_e2e
    pk, pk_kind = peaks()
    a = R.a
    h2d = a.indptr.size * 8 + a.indices.size * 4 + a.data.size * 8 + R.b_host.nbytes
    N = R.N
    line = {
        "metric": METRIC, "value": N / t_step, "unit": "unknowns/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded BASELINE cfg{args.config} inputs)",
        "config": config_dict(args.config, world, nranks),
        "factor_ms": t_f * 1e3, "solve_ms": t_s * 1e3,
        "factor_unknowns_per_s": N / t_f, "solve_unknown_rhs_per_s": N * R.nrhs / t_s if t_s > 0 else None,
        "e2e": {"value": N / t_e2e, "unit": "unknowns/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(R.b_host.nbytes),
                "note": "public API: factor_hifde(a, grid, eps, wait=False) + apply_inverse(b) with the host CSR and "
                        "RHS in page-locked memory (pinned_csr / pin_memory, outside the timed region); wait=False "
                        "lets apply_inverse upload the right-hand sides while the factorization runs on the "
                        "library's thread (one GPU; results identical); blocking_value: the same two calls with "
                        f"the default wait=True; mean of {max(1, min(args.steps, 10))} steps after one warm-up",
                "steps_ms": R.e2e_steps_ms,
                "blocking_value": N / t_e2e_block, "blocking_steps_ms": R.e2e_blocking_steps_ms,
                "resid": getattr(R, "e2e_resid", None)},
        "gpu_launches": int(launches // max(args.steps, 1)),
        "gpu_launches_note": "kernel launches of this library per step (factor + solve)",
        "clocks": clk.summary(),
        "resid": R.resid, "skeleton_counts": [c for _, c in R.skel],
    }
    if world > 1:
        line["xfer_bytes_rank0"] = int(R.xfer)
    line["roofline"] = roofline(R.kstats, args.steps, pk, pk_kind)
    if extra:
        line["cfg5"] = extra
    if cpu_base:
        line["cpu_baseline"] = cpu_base
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG, choices=[2, 3, 4, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config-5 extra keys")
    ap.add_argument("--emulate", type=int, default=1, help="virtual ranks on one GPU (sharded code path, N=1)")
    ap.add_argument("--shard", action="store_true", help=argparse.SUPPRESS)  # sharded is the N>1 default
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        cpu_reference(args, world, rank)
        return
    run_gpu(args, world, rank, local)


if __name__ == "__main__":
    main()
