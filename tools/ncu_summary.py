"""Key metrics of .ncu-rep files (one captured launch each), one row per file."""
import csv, subprocess, sys
W = [("gpu__time_duration.sum", "dur"), ("launch__grid_size", "grid"), ("launch__block_size", "blk"),
     ("launch__registers_per_thread", "regs"), ("launch__shared_mem_per_block_dynamic", "smem"),
     ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
     ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
     ("sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active", "fmah%"),
     ("smsp__inst_executed.sum", "inst"),
     ("smsp__thread_inst_executed_per_inst_executed.ratio", "thr/inst"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankc")]
for f in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        print(f, "no data")
        continue
    h, u, v = rows[0], rows[1], rows[2]
    d = {n: (v[i], u[i]) for i, n in enumerate(h)}
    print(f.split("/")[-1], d.get("Kernel Name", ("?",))[0][:60])
    print("   " + "  ".join(f"{s}={d[n][0]}{d[n][1] if d[n][1] not in ('', 'inst', 'register/thread') else ''}" for n, s in W if n in d))
    st = sorted(((float(d[n][0]), n) for n in d if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio") or n.startswith("smsp__average_warp_latency_issue_stalled") ), reverse=True)[:6]
    print("   stalls: " + ", ".join(f"{n.split('stalled_')[1].split('_per')[0].split('.')[0]}={x:.2f}" for x, n in st))
