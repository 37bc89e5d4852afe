"""Per-kernel-group device times of the config-1 rs_step (eager, serial, CUDA
events between the groups, L2 flushed before each step)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_12663_b200 as P  # noqa: E402
from paper_2505_12663_b200 import workload as W  # noqa: E402


def main():
    torch.cuda.set_device(0)
    dim, vocab = 64, 1 << 20
    table = P.EmbedTable(P.TableConfig(capacity=1 << 22, embedding_dim=dim, optimizer="adagrad",
                                       chunk_rows=1 << 16, initial_rows=vocab + (1 << 20)))
    raw = torch.arange(0, vocab, dtype=torch.int64, device="cuda")
    table.insert(raw + (1 << 62), W.pseudo_grads(raw, 0, dim))
    batches = [W.generate(1 + b, 1024, 128.0, 4096, 1.0, 1.1, [vocab]) for b in range(4)]
    step = P.SparseStep(table, max(len(i) for _, i in batches), P.AdagradParams(lr=0.01, eps=1e-8))
    dev = [(P.as_keys(ids), W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(l).view(np.int64)), b, dim),
            torch.empty((len(ids), dim), device="cuda")) for b, (l, ids) in enumerate(batches)]
    flush = torch.empty(512 << 18, dtype=torch.float32, device="cuda")
    lib = P.lib()
    for k in range(4):
        step.step(*dev[k % 4])
    P._lib.check(lib.rs_workspace_set_profiling(step.ws.handle, 1), "prof")
    for k in range(20):
        flush.zero_()
        step.step(*dev[k % 4])
    ms = (ctypes.c_double * 8)()
    cnt = ctypes.c_uint64()
    P._lib.check(lib.rs_workspace_phase_ms(step.ws.handle, ms, 8, ctypes.byref(cnt)), "phase")
    print(json.dumps({"phase_ms": [ms[i] for i in range(4)], "count": cnt.value}))


if __name__ == "__main__":
    main()
