"""HIF-DE factor & solve benchmark (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1], the config the metric is quoted on and the
largest that is a single-GPU case): 2D five-point high-contrast operator,
n = 511 interior points per side (N = 261,121), Gaussian-noise field smoothed
with width 4h thresholded at zero to {1e-2, 1e2}, leaf 8x8, eps = 1e-9,
16 right-hand sides ~ N(0,1).  Synthetic, seeded inputs generated in-process.

One step = factor_hifde of the matrix + apply_inverse of the 16-RHS block.
  value = N / (t_factor + t_solve)  [unknowns/s], inputs resident in HBM,
          timed with CUDA events on the library's stream;
  e2e   = the same through the public API with host buffers (CSR and RHS
          host->device, solution device->host inside the timed region).
`--impl reference` times the CPU oracle port of the reference algorithm
(oracle/hifde_oracle.py) on this host on the same workload.

Multi-GPU (torchrun, --gpus N): by default every rank factors and solves its
own independently seeded instance of config 2 (replicas; weak scaling).
`--shard --config {2,3,4,5}` instead factors ONE instance of that BASELINE
config sharded over the N ranks (spatial group owners, NCCL block exchange,
exact-order coarse levels on rank 0; strong scaling) and splits the
right-hand sides over the ranks -- DESIGN.md (e).  `--emulate P` runs the
sharded code path with P virtual ranks on one GPU (a correctness check; its
timing is not a multi-GPU number).
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

CONFIG = 2
WORKLOAD = ("cfg2: 2D 5-point high-contrast (Gaussian, 4h, thr 0) n=511 N=261121, "
            "leaf 8x8, eps=1e-9, hifde, 16 RHS; step = factor + 16-RHS solve")
METRIC = "HIF-DE factor & solve unknowns/sec"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


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


def cpu_reference(args, world, rank):
    """Reference arm: the CPU oracle port of the reference algorithm."""
    if rank != 0:
        return
    import paper_1307_2895_b200.problems as P
    from oracle import hifde_oracle as O
    g, a, eps, variant, nrhs = P.baseline_problem(CONFIG)
    og = O.make_grid(g.dim, g.n, g.m)
    b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
    steps = max(1, min(args.steps, 4))
    warm = min(args.warmup, 1)
    times = []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        f = O.factor(a, og, eps, variant)
        tf = time.perf_counter() - t0
        x = f.apply_inverse(b)
        t = time.perf_counter() - t0
        if i >= warm:
            times.append((t, tf, t - tf))
    tt = float(np.mean([t[0] for t in times]))
    value = g.ndof / tt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "unknowns/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": tt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE cfg2 inputs)",
        "config": {"workload": WORKLOAD},
        "factor_unknowns_per_s": g.ndof / float(np.mean([t[1] for t in times])),
        "solve_unknown_rhs_per_s": g.ndof * nrhs / float(np.mean([t[2] for t in times])),
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": 1, "kind": "port",
                         "sample": f"full cfg2 factor+16-RHS solve x{steps} (oracle port, BLAS 1 thread in the cell sweep as the reference)"},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "resid": float(np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0))),
    }
    print(json.dumps(line), flush=True)


def run_gpu(args, world, rank, local):
    import torch
    import paper_1307_2895_b200 as H
    from paper_1307_2895_b200 import _lib

    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    g, a, eps, variant, nrhs = H.baseline_problem(CONFIG, seed=rank)
    N = g.ndof
    rng = np.random.default_rng(1 + rank)
    b_host = rng.standard_normal((N, nrhs))
    # device-resident inputs for `value`
    indptr_d = torch.from_numpy(a.indptr.astype(np.int64)).to(dev)
    indices_d = torch.from_numpy(a.indices.astype(np.int32)).to(dev)
    data_d = torch.from_numpy(a.data.astype(np.float64)).to(dev)
    b_d = torch.from_numpy(b_host).to(dev)
    x_d = torch.empty_like(b_d)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    lib = _lib.load()

    import ctypes as C

    def factor_device():
        opt = _lib.Options()
        lib.hifde_default_options(C.byref(opt), _lib.VARIANT_HIFDE)
        opt.eps = eps
        opt.device = local
        opt.input_on_device = 1
        opt.stream = stream.cuda_stream
        h = C.c_void_p()
        code = lib.hifde_factor(indptr_d.data_ptr(), indices_d.data_ptr(), data_d.data_ptr(), N,
                                g.dim, g.n, g.m, g.nlevels, C.byref(opt), C.byref(h))
        if code:
            raise RuntimeError(lib.hifde_last_error().decode())
        launches = lib.hifde_last_launch_count()
        return H.GeneralizedLDL(h.value, lib, True), launches

    def one_step():
        f, nl_f = factor_device()
        f.apply_inverse_device(b_d.data_ptr(), x_d.data_ptr(), nrhs, stream.cuda_stream)
        nl_s = lib.hifde_last_launch_count()
        return f, nl_f + nl_s

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            f, _ = one_step()
            stream.synchronize()
        # correctness guard on the warm factor (not timed)
        x = x_d.cpu().numpy()
        resid = float(np.max(np.linalg.norm(a @ x - b_host, axis=0) / np.linalg.norm(b_host, axis=0)))
        level_info = f.level_info
        skel = f.metrics["skeleton_counts"]
        del f
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        times, tfs, launches = [], [], 0
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e2 = torch.cuda.Event(enable_timing=True)
                stream.wait_stream(torch.cuda.current_stream())
                e0.record(stream)
                f, nl_f = factor_device()
                e1.record(stream)
                f.apply_inverse_device(b_d.data_ptr(), x_d.data_ptr(), nrhs, stream.cuda_stream)
                launches += nl_f + lib.hifde_last_launch_count()
                e2.record(stream)
                e2.synchronize()
                times.append(e0.elapsed_time(e2) / 1e3)
                tfs.append(e0.elapsed_time(e1) / 1e3)
                level_info = f.level_info
                f.close()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t_step = float(np.mean(times))
        t_f = float(np.mean(tfs))
        t_s = t_step - t_f
        # end-to-end through the public API with host buffers
        e2e_times = []
        for _ in range(max(1, min(args.steps, 5))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fe = H.factor_hifde(a, g, eps, stream=stream.cuda_stream, device=local)
            xe = fe.apply_inverse(b_host)
            e2e_times.append(time.perf_counter() - t0)
            fe.close()
        t_e2e = float(np.median(e2e_times))
    if dist:
        tt = torch.tensor([t_step, t_e2e, t_f, t_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_e2e, t_f, t_s = [float(v) for v in tt.cpu()]

    # roofline of the dominant kernel class from the per-level accounting
    pk, pk_kind = peaks()
    dominant = max(level_info[:-1], key=lambda d: d["seconds"])
    h2d = a.indptr.size * 8 + a.indices.size * 4 + a.data.size * 8 + b_host.nbytes
    d2h = b_host.nbytes
    line = {
        "metric": METRIC, "value": world * N / t_step, "unit": "unknowns/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE cfg2 inputs)",
        "config": {"workload": WORKLOAD, "parallelism": f"replicas x{world}",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "factor_ms": t_f * 1e3, "solve_ms": t_s * 1e3,
        "factor_unknowns_per_s": N / t_f, "solve_unknown_rhs_per_s": N * nrhs / t_s,
        "e2e": {"value": world * N / t_e2e, "unit": "unknowns/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "resid": resid, "skeleton_counts": [c for _, c in skel],
    }
    line["roofline"] = roofline(level_info, pk, pk_kind, args)
    line["roofline_by_class"] = roofline_classes(level_info, pk)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_sharded(args, world, rank, local):
    """One BASELINE config sharded over the ranks (strong scaling)."""
    import ctypes as C

    import torch
    import paper_1307_2895_b200 as H
    from paper_1307_2895_b200 import _lib
    from paper_1307_2895_b200 import distributed as D

    dist = None
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        comm = D.init_comm(device=local)
    else:
        comm = D.emulated_comm(args.emulate, local) if args.emulate > 1 else None
    nr = comm.nranks if comm is not None else 1
    stream = torch.cuda.Stream(device=dev)
    g, a, eps, variant, nrhs = H.baseline_problem(args.config)
    N = g.ndof
    cols = D.rhs_columns(nrhs, world, rank)
    nloc = cols.stop - cols.start
    b_host = np.random.default_rng(1).standard_normal((N, nrhs))
    b_loc = np.ascontiguousarray(b_host[:, cols])
    indptr_d = torch.from_numpy(a.indptr.astype(np.int64)).to(dev)
    indices_d = torch.from_numpy(a.indices.astype(np.int32)).to(dev)
    data_d = torch.from_numpy(a.data.astype(np.float64)).to(dev)
    b_d = torch.from_numpy(b_loc).to(dev)
    x_d = torch.empty_like(b_d)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    lib = _lib.load()
    vcode = _lib.VARIANT_HIFDE if variant == "hifde" else _lib.VARIANT_HIFDE3X

    def factor_device():
        opt = _lib.Options()
        lib.hifde_default_options(C.byref(opt), vcode)
        opt.eps = eps
        opt.device = local
        opt.input_on_device = 1
        opt.stream = stream.cuda_stream
        opt.comm = comm.handle if comm is not None else None
        h = C.c_void_p()
        code = lib.hifde_factor(indptr_d.data_ptr(), indices_d.data_ptr(), data_d.data_ptr(), N,
                                g.dim, g.n, g.m, g.nlevels, C.byref(opt), C.byref(h))
        if code:
            raise RuntimeError(lib.hifde_last_error().decode())
        return H.GeneralizedLDL(h.value, lib, True), lib.hifde_last_launch_count()

    fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            f, _ = factor_device()
            if nloc:
                f.apply_inverse_device(b_d.data_ptr(), x_d.data_ptr(), nloc, stream.cuda_stream)
            stream.synchronize()
        x = x_d.cpu().numpy()
        resid = float(np.max(np.linalg.norm(a @ x - b_loc, axis=0) / np.linalg.norm(b_loc, axis=0))) if nloc else 0.0
        skel = f.metrics["skeleton_counts"]
        xfer = f.metrics["xfer_bytes"]
        f.close()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        times, tfs, launches = [], [], 0
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e2 = torch.cuda.Event(enable_timing=True)
                stream.wait_stream(torch.cuda.current_stream())
                e0.record(stream)
                f, nl = factor_device()
                e1.record(stream)
                if nloc:
                    f.apply_inverse_device(b_d.data_ptr(), x_d.data_ptr(), nloc, stream.cuda_stream)
                    nl += lib.hifde_last_launch_count()
                launches += nl
                e2.record(stream)
                e2.synchronize()
                times.append(e0.elapsed_time(e2) / 1e3)
                tfs.append(e0.elapsed_time(e1) / 1e3)
                level_info = f.level_info
                f.close()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t_step, t_f = float(np.mean(times)), float(np.mean(tfs))
        e2e_times = []
        for _ in range(max(1, min(args.steps, 3))):
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fe = fac(a, g, eps, stream=stream.cuda_stream, device=local, comm=comm)
            if nloc:
                fe.apply_inverse(b_loc)
            e2e_times.append(time.perf_counter() - t0)
            fe.close()
        t_e2e = float(np.median(e2e_times))
    t_s = t_step - t_f
    if dist:
        tt = torch.tensor([t_step, t_e2e, t_f, t_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_e2e, t_f, t_s = [float(v) for v in tt.cpu()]
    pk, pk_kind = peaks()
    h2d = a.indptr.size * 8 + a.indices.size * 4 + a.data.size * 8 + b_loc.nbytes
    line = {
        "metric": METRIC, "value": N / t_step, "unit": "unknowns/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded BASELINE cfg{args.config} inputs)",
        "config": {"workload": f"cfg{args.config}: {variant}, N={N}, eps={eps}, {nrhs} RHS; one instance "
                               f"sharded over {nr} rank(s){' (emulated on one GPU)' if comm is not None and comm.emulated else ''}; "
                               "step = factor + this rank's RHS columns",
                   "parallelism": f"shard x{nr}", "l2": "flushed between timed steps (256 MiB write)"},
        "factor_ms": t_f * 1e3, "solve_ms": t_s * 1e3,
        "factor_unknowns_per_s": N / t_f,
        "e2e": {"value": N / t_e2e, "unit": "unknowns/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(b_loc.nbytes)},
        "gpu_launches": int(launches), "clocks": clk.summary(), "resid": resid,
        "skeleton_counts": [c for _, c in skel], "xfer_bytes_rank0": int(xfer),
    }
    line["roofline"] = roofline(level_info, pk, pk_kind, args)
    line["roofline_by_class"] = roofline_classes(level_info, pk)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()


def roofline_classes(level_info, pk, fp64_tflops=35.5):
    """Whole-class fractions: the algorithmic bytes / FLOPs of
    all elimination levels, all skeletonization levels and the terminal block,
    over their summed CUDA-event time, against the HBM copy roof and the
    measured DGEMM roof (profiles/r01_fp64_peak.json)."""
    out = {}
    for name, kinds in (("elimination", (0,)), ("skeletonization", (1,)), ("terminal", (2,))):
        lv = [d for d in level_info if d["kind"] in kinds]
        sec = sum(d["gpu_seconds"] for d in lv)
        gb = sum(d["gbytes"] for d in lv)
        gf = sum(d["gflop"] for d in lv)
        if sec <= 0:
            continue
        out[name] = {"gpu_ms": sec * 1e3, "gb_per_s": gb / sec, "tflops": gf / sec * 1e-3,
                     "hbm_frac": gb / sec / pk.get("hbm_gbs", 6556.0), "fp64_frac": gf / sec * 1e-3 / fp64_tflops}
    return out


def roofline(level_info, pk, pk_kind, args):
    """HBM roofline of the dominant kernel launch.

    In exact order every skeletonization level is ONE launch of
    skel_ordered_kernel, and every level's launches are timed by CUDA events
    on the library's stream; the dominant launch is the level with the
    largest event time.  achieved = that level's algorithmic bytes (SURVEY.md
    8(d): 8[nq nc + nc^2 + k r + r^2 + r + r k + 2k^2] per group, 8[(nc+nq)^2
    + nc^2 + nc + nc nq + 2 nq^2] per cell) / its event time.  traffic = the
    DRAM bytes ncu measured for the same launch (profiles/roofline_r01.json).
    The launch is bound by the reference-order dependency chain, not by HBM
    (profiles/r01_summary.md), hence the small fraction."""
    dom = max(level_info[:-1], key=lambda d: d["gpu_seconds"])
    sec, gb, gf = dom["gpu_seconds"], dom["gbytes"], dom["gflop"]
    achieved = gb / sec if sec > 0 else None
    peak = pk.get("hbm_gbs")
    traffic = None
    prof = os.path.join(ROOT, "profiles", "roofline_r01.json")
    if os.path.exists(prof):
        try:
            tb = json.load(open(prof))["skel_levels_dram_bytes"].get(f"{dom['tag']:.1f}")
            traffic = tb / 1e9 if tb else None
        except Exception:
            traffic = None
    name = "skel_ordered_kernel" if dom["kind"] == 1 else "elim_kernels"
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved and peak else None,
            "traffic": traffic, "traffic_unit": "GB per launch", "kernel": name, "level": dom["tag"],
            "launch_seconds": sec, "algorithmic_gbytes": gb, "algorithmic_gflop": gf,
            "achieved_gflops": gf / sec if sec > 0 else None,
            "limiter": "reference-order dependency chain (latency), see profiles/r01_summary.md",
            "peak_kind": pk_kind + " (MEASURED_PEAKS.json hbm_gbs)"}


def cpu_baseline():
    import paper_1307_2895_b200.problems as P
    from oracle import hifde_oracle as O
    g, a, eps, variant, nrhs = P.baseline_problem(CONFIG)
    b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
    t0 = time.perf_counter()
    f = O.factor(a, O.make_grid(g.dim, g.n, g.m), eps, variant)
    f.apply_inverse(b)
    t = time.perf_counter() - t0
    return {"value": g.ndof / t, "unit": "unknowns/s", "cores": 1, "kind": "port",
            "sample": "one full cfg2 factor + 16-RHS solve (oracle port, 1 BLAS thread)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true", help="one instance sharded over the ranks")
    ap.add_argument("--config", type=int, default=CONFIG, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--emulate", type=int, default=1, help="virtual ranks on one GPU (--shard, N=1)")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        cpu_reference(args, world, rank)
        return
    if args.shard:
        run_sharded(args, world, rank, local)
        return
    run_gpu(args, world, rank, local)


if __name__ == "__main__":
    main()
