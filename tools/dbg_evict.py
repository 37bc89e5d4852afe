"""Debug: bounded-table eviction, GPU vs oracle, per batch (stamp-log selection)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12663_b200 as P  # noqa: E402
from oracle.bind import Oracle, Table  # noqa: E402

oracle = Oracle("oracle")
rng = np.random.default_rng(21)
dim, bound = 16, 3000
g = P.EmbedTable(P.TableConfig(capacity=1 << 13, embedding_dim=dim, chunk_rows=64, optimizer="adagrad", max_keys=bound))
o = Table(oracle, 1 << 13, dim, chunk_rows=4096)
fresh = 10**6
for b in range(12):
    old = rng.integers(0, 4000, 700).astype(np.uint64)
    new = np.arange(fresh, fresh + 150, dtype=np.uint64)
    fresh += 150
    keys = np.unique(np.concatenate([old, new]))
    rng.shuffle(keys)
    tick = g.tick() + 1
    g.ensure(keys)
    oracle.table_ensure_batch(o.h, keys, len(keys), tick, bound, None)
    if os.environ.get("NOEXPORT"):
        occ0 = g.occupied()
        torch.cuda.synchronize()
        print(b, "gpu occ", occ0, g.occupied(), "oracle occ", oracle.table_occupied(o.h), flush=True)
        continue
    ga, ob = g.export(), o.export()
    sg, so = set(ga["keys"].tolist()), set(ob["keys"].tolist())
    print(b, "n", len(keys), "gpu occ", g.occupied(), "oracle occ", oracle.table_occupied(o.h), "tick", g.tick(), tick,
          "only_gpu", len(sg - so), "only_oracle", len(so - sg), flush=True)
    if sg != so:
        og = sorted(sg - so)[:5]
        oo = sorted(so - sg)[:5]
        tg = dict(zip(ga["keys"].tolist(), ga["ts"].tolist()))
        to = dict(zip(ob["keys"].tolist(), ob["ts"].tolist()))
        print("  only gpu", [(k, tg[k]) for k in og], "only oracle", [(k, to[k]) for k in oo])
        break
