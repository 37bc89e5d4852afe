"""Small cases of every kernel family for compute-sanitizer (one tool per
run: tools/sanitize.sh): table insert / ensure (duplicates) / find / lookup /
remove / expand / evict on a bounded table, exact dedup, the fast step (graph
and eager), the split-kernel step, the bounded-table step with device
eviction, the sharded step of a local 2-rank group.  Exits 0 and prints
SANITIZE_CASE_OK when every result is consistent."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_12663_b200 as P  # noqa: E402
from paper_2505_12663_b200 import workload as W  # noqa: E402
from paper_2505_12663_b200.dist import LocalShardGroup  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(1)
    dim = 16
    # table ops
    t = P.EmbedTable(P.TableConfig(capacity=64, embedding_dim=dim, chunk_rows=32, optimizer="adam"))
    keys = rng.integers(0, 200, 300).astype(np.uint64)
    t.insert(keys, torch.from_numpy(rng.standard_normal((300, dim)).astype(np.float32)))
    t.ensure(rng.integers(0, 400, 500).astype(np.uint64))
    t.find(keys[:50])
    t.lookup_batch(keys[:50])
    t.remove(keys[:40])
    t.expand()
    b = P.EmbedTable(P.TableConfig(capacity=1 << 10, embedding_dim=dim, chunk_rows=64, optimizer="adagrad",
                                   max_keys=300))
    for k in range(4):
        b.ensure(np.arange(k * 150, k * 150 + 200, dtype=np.uint64))
    b.evict(20)
    # exact dedup
    P.stage1_dedup((rng.zipf(1.2, 5000) % 700).astype(np.uint64))
    # steps: fast (graph + eager), split kernels, bounded
    lengths, ids = W.generate(3, 24, 32.0, 256, 1.0, 1.1, [3000])
    g = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), 0, dim)
    d_ids = P.as_keys(ids)
    out = torch.empty((len(ids), dim), device="cuda")
    for opt, params in (("adagrad", P.AdagradParams()), ("adam", P.AdamParams())):
        tab = P.EmbedTable(P.TableConfig(capacity=1 << 12, embedding_dim=dim, chunk_rows=256, optimizer=opt))
        st = P.SparseStep(tab, len(ids), params)
        for _ in range(3):
            st.step(d_ids, g, out)
        cs = torch.zeros(1, dtype=torch.float64, device="cuda")
        st.step_checksum(d_ids, g, out, cs)
    os.environ["RS_NO_GRAPH"] = "1"
    st = P.SparseStep(P.EmbedTable(P.TableConfig(capacity=1 << 12, embedding_dim=dim, optimizer="adagrad")),
                      len(ids), P.AdagradParams())
    st.step(d_ids, g, out)
    os.environ["RS_FAST_STEP"] = "0"
    st = P.SparseStep(P.EmbedTable(P.TableConfig(capacity=1 << 12, embedding_dim=dim, optimizer="adagrad")),
                      len(ids), P.AdagradParams())
    st.step(d_ids, g, out)
    del os.environ["RS_FAST_STEP"], os.environ["RS_NO_GRAPH"]
    bt = P.EmbedTable(P.TableConfig(capacity=1 << 12, embedding_dim=dim, optimizer="adagrad", max_keys=600))
    st = P.SparseStep(bt, len(ids), P.AdagradParams())
    for _ in range(2):
        st.step(d_ids, g, out)
    # sharded step of a local 2-rank group
    grp = LocalShardGroup(P.TableConfig(capacity=1 << 12, embedding_dim=dim, chunk_rows=256, optimizer="adagrad"),
                          2, 2048)
    grp.insert_all(np.arange(500, dtype=np.uint64), torch.ones((500, dim)))
    reqs = [torch.from_numpy((rng.zipf(1.2, n) % 900).astype(np.int64)).cuda() for n in (700, 300)]
    grads = [torch.randn((r.numel(), dim), device="cuda") for r in reqs]
    grp.step(reqs, grads, P.AdagradParams())
    grp.forward(reqs)
    grp.backward(grads, P.AdagradParams())
    grp.close()
    torch.cuda.synchronize()
    print("SANITIZE_CASE_OK", flush=True)


if __name__ == "__main__":
    main()
