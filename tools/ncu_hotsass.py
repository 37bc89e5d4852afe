"""Top SASS instructions by warp-stall samples of ONE kernel in an ncu report:
python tools/ncu_hotsass.py REPORT KERNEL_REGEX [N] [launch index]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdrs = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[hdrs[0]]
si, ss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
end = hdrs[1] if len(hdrs) > 1 else len(rows)
body = [r for r in rows[hdrs[0] + 1:end] if len(r) == len(h) and r[ss].isdigit()]
tot = sum(int(r[ss]) for r in body)
print(f"total samples {tot}, instructions {len(body)}")
idx = sorted(range(len(body)), key=lambda i: -int(body[i][ss]))[:n]
for i in sorted(idx):
    r = body[i]
    prev = body[i - 1][si].strip()[:50] if i else ""
    print(f"{i:5d} {int(r[ss]) / tot * 100:5.1f}%  {r[si].strip()[:70]:70s} | prev: {prev}")
