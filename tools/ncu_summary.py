"""Key metrics + warp-stall breakdown per launch of an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size"]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d.get("Kernel Name", "?"))
        for k in KEYS:
            if k in d:
                print(f"    {k:70s} {d[k]:>22s} {units[hdr.index(k)]}")
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        t = d.get("gpu__time_duration.sum")
        if rd and wr and t:
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
            b = float(rd) * scale.get(units[hdr.index("dram__bytes_read.sum")], 1) + \
                float(wr) * scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
            tu = units[hdr.index("gpu__time_duration.sum")]
            sec = float(t) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}.get(tu, 1)
            print(f"    {'achieved DRAM GB/s (isolated launch)':70s} {b / sec / 1e9:>22.1f}")
        st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[h] or 0) for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:9]
        print("    stalls (pc samples): " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
