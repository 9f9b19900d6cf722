"""Print the headline metrics of every kernel in an .ncu-rep (ncu --page raw --csv)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "smsp__inst_executed.sum"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        print(rep, d.get("Kernel Name"))
        for k in KEYS:
            if k in d:
                print(f"  {k:65s} {d[k]:>16s} {u[h.index(k)]}")
        stalls = sorted(((float(d[k] or 0), k) for k in h if k.startswith("smsp__average_warp") and "issue_stalled" in k
                         and k.endswith("_per_issue_active.ratio")), reverse=True)[:6]
        for val, k in stalls:
            print(f"  {k:65s} {val:16.2f}")
