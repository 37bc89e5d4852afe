"""Device-side timeline of one config-1 fast step inside its CUDA graph
(RS_TRACE=1, %globaltimer per block): per kernel the start / end relative to
the dedup kernel's first block, and block-duration percentiles."""
import ctypes
import json
import os
import sys

os.environ["RS_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_12663_b200 as P  # noqa: E402
from paper_2505_12663_b200 import workload as W  # noqa: E402

NAMES = ["dedup_probe", "csr_light", "hot_tiles", "hot_finish", "clean", "csr_heavy"]


def main():
    torch.cuda.set_device(0)
    dim, vocab = 64, 1 << 20
    table = P.EmbedTable(P.TableConfig(capacity=1 << 22, embedding_dim=dim, optimizer="adagrad",
                                       chunk_rows=1 << 16, initial_rows=vocab + (1 << 20)))
    raw = torch.arange(0, vocab, dtype=torch.int64, device="cuda")
    table.insert(raw + (1 << 62), W.pseudo_grads(raw, 0, dim))
    batches = [W.generate(1 + b, 1024, 128.0, 4096, 1.0, 1.1, [vocab]) for b in range(2)]
    step = P.SparseStep(table, max(len(i) for _, i in batches), P.AdagradParams(lr=0.01, eps=1e-8))
    dev = [(P.as_keys(ids), W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(l).view(np.int64)), b, dim),
            torch.empty((len(ids), dim), device="cuda")) for b, (l, ids) in enumerate(batches)]
    flush = torch.empty(512 << 18, dtype=torch.float32, device="cuda")
    lib = P.lib()
    n = ctypes.c_uint64()
    res = []
    for k in range(8):
        flush.zero_()
        torch.cuda.synchronize()
        buf = np.zeros(16 * 4096 * 2, np.uint64)
        P._lib.check(lib.rs_workspace_trace(step.ws.handle, buf.ctypes.data, buf.size, ctypes.byref(n)), "trace")
        step.step(*dev[k % 2])
        torch.cuda.synchronize()
        P._lib.check(lib.rs_workspace_trace(step.ws.handle, buf.ctypes.data, buf.size, ctypes.byref(n)), "trace")
        if k < 4:
            continue
        t = buf.reshape(16, 4096, 2).astype(np.float64)
        t0 = t[0, :, 0][t[0, :, 1] > 0].min()
        row = {}
        for i, name in enumerate(NAMES):
            ok = t[i, :, 1] > 0
            if not ok.any():
                continue
            st, en = (t[i, ok, 0] - t0) / 1e3, (t[i, ok, 1] - t0) / 1e3
            dur = en - st
            row[name] = {"blocks": int(ok.sum()), "start": round(st.min(), 2), "end": round(en.max(), 2),
                         "end_p50": round(float(np.percentile(en, 50)), 2), "end_p90": round(float(np.percentile(en, 90)), 2),
                         "dur_p50": round(float(np.percentile(dur, 50)), 2), "dur_max": round(dur.max(), 2)}
        res.append(row)
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
