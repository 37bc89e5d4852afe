"""Top stall lines of one kernel from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
si, src, ex = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
val = lambda r, i: int(r[i]) if len(r) > i and r[i].isdigit() else 0
tot = sum(val(r, si) for r in data)
print("samples", tot, "instructions", sum(val(r, ex) for r in data))
top = sorted(range(len(data)), key=lambda i: -val(data[i], si))[:n]
for i in sorted(top):
    print(f"{i:5d} {val(data[i], si):6d} {val(data[i], ex):8d}  {data[i][src][:90]}")
