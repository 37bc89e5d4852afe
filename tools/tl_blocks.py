"""Per-kernel block statistics of a dumped sharded-step timeline
(bench.py with RS_TRACE=1 RS_TRACE_DUMP=prefix).  usage: python tools/tl_blocks.py prefix [rank]"""
import sys

import numpy as np

NAMES = ["dedup_probe", "csr_light", "hot_tiles", "hot_finish", "scratch_clean", "csr_heavy", "req_gather",
         "req_grad_flags", "own_wait_ids", "own_dedup", "own_table_respond", "req_wait_rows", "own_wait_grads",
         "own_update_done", "own_update"]
t = np.load(f"{sys.argv[1]}_rank{sys.argv[2] if len(sys.argv) > 2 else 0}.npy")
rows = []
for i, n in enumerate(NAMES):
    s, e = t[i, :, 0], t[i, :, 1]
    ok = (e > 0) & (s < 1e6)
    if not ok.any():
        continue
    d = e[ok] - s[ok]
    rows.append((s[ok].min(), n, ok.sum(), s[ok].max(), np.percentile(e[ok], 50), e[ok].max(), np.median(d), np.percentile(d, 90)))
for r in sorted(rows):
    print(f"{r[1]:18s} blocks {r[2]:5d} start {r[0]:6.1f}..{r[3]:6.1f} end med {r[4]:6.1f} max {r[5]:6.1f}  dur med {r[6]:5.1f} p90 {r[7]:5.1f}")
