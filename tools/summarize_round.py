"""Turn a tools/profile_round.sh output directory (gpurun_out/<tag>) into the committed evidence under
profiles/: the bench line, the launch-list summary, ncu key-metric summaries and per-launch DRAM
traffic (traffic.json, read by bench.py for roofline.traffic).  Runs here (needs ncu, no GPU).

Usage: python tools/summarize_round.py <tag>
"""
import csv
import io
import json
import shutil
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1]
src = ROOT / "gpurun_out" / tag
dst = ROOT / "profiles"

# 1. bench lines (config 3 headline; configs 1, 2 and the config-4 streaming slices when present)
shutil.copy(src / "bench.json", dst / f"{tag}_bench.json")
for extra in ("bench_config2.json", "bench_config1.json", "config4_replay.json", "config4_pinned.json",
              "config4_stream.json"):
    if (src / extra).exists():
        shutil.copy(src / extra, dst / f"{tag}_{extra}")
if (src / "bench_reference.log").exists():
    ref = [l for l in (src / "bench_reference.log").read_text().splitlines() if l.startswith("{")]
    if ref:
        (dst / f"{tag}_bench_reference.json").write_text(json.dumps(json.loads(ref[-1]), indent=1))

for extra in ("pytest_gpu.log", "step_gap.log"):
    if (src / extra).exists():
        shutil.copy(src / extra, dst / f"{tag}_{extra}")

# 2. launch list -> per-kernel averages and the fusion-step shares
rows = list(csv.reader(open(src / "launches.csv")))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("rlk::", "")
    per.setdefault(name, []).append(float(r[vi].replace(",", "")))
unit = "ns" if max(max(v) for v in per.values()) > 1e5 else "us"
scale = 1e-6 if unit == "ns" else 1e-3
fusion = [k for k in per if any(s in k for s in ("k_merge", "k_sumsq", "k_mask_bitmap", "k_finalize"))]
fsum = sum(statistics.mean(per[k]) for k in fusion)
lines = [f"# ncu launch list of `python bench.py --steps 3 --warmup 3 --quick --no-e2e --no-cpu` (our kernels only)",
         "# ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:k_sumsq|k_merge|k_mask_bitmap|k_finalize|k_grpo|k_segment_sum'",
         "# cold-cache, serialised per-launch times; compare shares with bench.json kernels_ms, not absolutes", ""]
for k, v in sorted(per.items(), key=lambda kv: -statistics.mean(kv[1]) * len(kv[1])):
    avg = statistics.mean(v) * scale
    share = f"  fusion-step share {statistics.mean(v) / fsum:.3f}" if k in fusion else ""
    lines.append(f"{k:45s} {len(v):4d} launches  avg {avg:10.4f} ms{share}")
(dst / f"{tag}_launches_summary.txt").write_text("\n".join(lines) + "\n")

# 3. ncu --set full summaries + traffic
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]
traffic = {}
for rep, out in (("fusion_full", "ncu_fusion_summary"), ("grpo_full", "ncu_grpo_summary"),
                 ("config1_full", "ncu_config1_summary")):
    f = src / f"{rep}.ncu-rep"
    if (src / f"{rep}.raw.csv").exists():  # exported on the GPU box (profile_round.sh)
        raw = (src / f"{rep}.raw.csv").read_text()
    elif f.exists():
        raw = subprocess.run(["ncu", "-i", str(f), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        continue
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = rr[0], rr[1]
    txt = [f"# ncu --set full --clock-control none ({rep}.ncu-rep): key metrics per captured launch", ""]
    for row in rr[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        name = d["Kernel Name"]
        txt.append(name)
        for k in KEYS:
            if k in d:
                txt.append(f"    {k:60s} {d[k]:>18s} {u.get(k, '')}")
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if rd and wr:
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = float(rd.replace(",", "")) * mult.get(u["dram__bytes_read.sum"], 1) + \
                float(wr.replace(",", "")) * mult.get(u["dram__bytes_write.sum"], 1)
            key = "rlk_fusion_merge_fixup" if "k_merge_fixup" in name else "rlk_fusion_merge" if "k_merge" in name else "rlk_fusion_sumsq" if "k_sumsq" in name else \
                "rlk_fusion_mask_bitmap" if "k_mask" in name else name.split("(")[0]
            if rep == "fusion_full":  # traffic.json describes the config-3 launches only
                traffic.setdefault(key, []).append(b)
            txt.append(f"    {'dram bytes read + write':60s} {b:18.0f} byte")
            dur = float(d["gpu__time_duration.sum"].replace(",", ""))
            dur_s = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(
                u.get("gpu__time_duration.sum", "ms"), 1e-3)
            gbs = b / dur_s / 1e9
            txt.append(f"    {'achieved DRAM GB/s (ncu, isolated launch)':60s} {gbs:18.1f} GB/s "
                       f"= {gbs / 8000 * 100:.1f}% of the 8 TB/s spec, {gbs / 6546.6 * 100:.1f}% of the measured copy peak")
        txt.append("")
    (dst / f"{tag}_{out}.txt").write_text("\n".join(txt))
raw_t = {k: v for k, v in traffic.items()}
(dst / f"{tag}_ncu_traffic_raw.json").write_text(json.dumps(raw_t, indent=1))
tj = json.loads((dst / "traffic.json").read_text()) if (dst / "traffic.json").exists() else {}
tj["_source"] = (f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch (profiles/{tag}_ncu_traffic_raw.json), "
                 "tools/prof_fusion.py --layout llama8b: the bench.py config-3 tensors and FusionConfig(dropout_p=0.5, seed=42), N=1")
tj.setdefault("llama8b", {})["1"] = {k: int(statistics.mean(v)) for k, v in traffic.items()
                                     if k in ("rlk_fusion_merge", "rlk_fusion_sumsq", "rlk_fusion_mask_bitmap")}
(dst / "traffic.json").write_text(json.dumps(tj, indent=1))
print("\n".join(lines))
print(json.dumps(tj, indent=1))
