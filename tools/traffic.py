"""DRAM traffic per fast-step phase from ncu --set full captures of
tools/exp_phases.py (eager launches): one capture with caches flushed before
every kernel (ncu's default) and one with --cache-control none (the step's own
L2 state).  usage: python tools/traffic.py FLUSHED.ncu-rep INCONTEXT.ncu-rep OUT.json"""
import csv
import json
import subprocess
import sys

PHASE = {"k_fa": "dedup_probe", "k_fclean": "csr_update", "k_fc": "csr_update", "k_fh": "hot_update",
         "k_fhf": "hot_update", "k_fcs": "checksum"}


def per_phase(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    units = rows[1]
    res, seen = {}, {}
    for r in rows[2:]:
        v = dict(zip(h, r))
        name = v["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1].strip()
        ph = PHASE.get(name)
        if not ph:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(v[m].replace(",", "")) * scale.get(units[h.index(m)], 1)
        res[ph] = res.get(ph, 0.0) + b
        seen.setdefault(ph, []).append(name)
    return res, seen


flushed, names = per_phase(sys.argv[1])
ctx, _ = per_phase(sys.argv[2])
# one launch of every kernel of a step was captured per report
doc = dict(flushed)
doc["in_context"] = ctx
doc["_kernels"] = names
doc["_source"] = f"{sys.argv[1]} (ncu --set full, caches flushed per kernel) and {sys.argv[2]} (--cache-control none)"
json.dump(doc, open(sys.argv[3], "w"), indent=1)
print(json.dumps(doc, indent=1))
