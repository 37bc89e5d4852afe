"""Experiment: config-1 rs_step device time under three L2 states between
timed steps: dirty-cold (512 MiB write, bench.py's flush), clean-cold (the
same write followed by a 256 MiB read, so the write-back happens outside the
bracket) and warm (no flush).  Prints one JSON line."""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_12663_b200 as P  # noqa: E402
from paper_2505_12663_b200 import workload as W  # noqa: E402

TAG1 = 1 << 62


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    torch.cuda.set_device(0)
    dim, vocab = 64, 1 << 20
    table = P.EmbedTable(P.TableConfig(capacity=1 << 22, embedding_dim=dim, optimizer="adagrad",
                                       chunk_rows=1 << 16, initial_rows=vocab + (1 << 20)))
    raw = torch.arange(0, vocab, dtype=torch.int64, device="cuda")
    table.insert(raw + TAG1, W.pseudo_grads(raw, 0, dim))
    nb = 6
    batches = [W.generate(1 + b, 1024, 128.0, 4096, 1.0, 1.1, [vocab]) for b in range(nb)]
    step = P.SparseStep(table, max(len(i) for _, i in batches), P.AdagradParams(lr=0.01, eps=1e-8))
    dev = []
    for b, (lengths, ids) in enumerate(batches):
        dev.append((P.as_keys(ids), W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), b,
                                                   dim), torch.empty((len(ids), dim), device="cuda")))
    wbuf = torch.empty(512 << 18, dtype=torch.float32, device="cuda")
    rbuf = torch.ones(256 << 18, dtype=torch.float32, device="cuda")
    sink = torch.empty(1, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    for k in range(2 * nb):
        step.step(*dev[k % nb])
    torch.cuda.synchronize()
    res = {}
    for mode in ("dirty", "clean", "warm", "dirty", "clean"):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            if mode in ("dirty", "clean"):
                wbuf.zero_()
            if mode == "clean":
                torch.sum(rbuf, dim=0, out=sink)
            evs[k][0].record(stream)
            step.step(*dev[k % nb])
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in evs]
        res.setdefault(mode, []).append({"median_ms": statistics.median(ms), "mean_ms": sum(ms) / len(ms),
                                         "min_ms": min(ms)})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
