"""Markdown summary of an ncu --set full report (per kernel: time, DRAM traffic,
achieved bandwidth, occupancy, registers, top stall reasons)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
print("| kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM GB/s | achieved occ. | regs | top stalls (cycles/issue) |")
print("|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    v = dict(zip(h, r))
    name = v["Kernel Name"].split("(")[0].replace("rs::<unnamed>::", "").replace("void ", "")
    f = lambda k: float(v.get(k, "0").replace(",", "") or 0)
    t = f("gpu__time_duration.sum")  # us
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")  # MB (ncu default units)
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(k)
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    top = ", ".join(f"{k} {x:.1f}" for k, x in sorted(stalls.items(), key=lambda kv: -kv[1])[:3])
    occ = v.get("sm__warps_active.avg.pct_of_peak_sustained_active", "")
    regs = v.get("launch__registers_per_thread", "")
    bw = (rd + wr) / t * 1e3 if t else 0  # MB/us -> GB/s
    print(f"| {name} | {t:.2f} | {rd:.2f} | {wr:.2f} | {bw:.0f} | {occ} | {regs} | {top} |")
