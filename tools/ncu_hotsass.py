"""Top SASS instructions by warp-stall samples of one kernel in an ncu report:
python tools/ncu_hotsass.py REPORT KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
si, ss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[hdr + 1:] if len(r) == len(h) and r[ss].isdigit()]
tot = sum(int(r[ss] or 0) for r in body)
print(f"total samples {tot}, instructions {len(body)}")
idx = sorted(range(len(body)), key=lambda i: -int(body[i][ss] or 0))[:n]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {int(r[ss]) / tot * 100:5.1f}%  {r[si].strip()[:90]}")
