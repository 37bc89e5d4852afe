"""The benchmarked path itself: rs_step at BASELINE config 1 (one table, D=64,
2^20 pre-populated keys, 1024 sequences mean 128, Zipf 1.1, Adagrad) through
the CUDA-graph path bench.py times (forked hot-id branch, split gather pass,
token ranks from the dedup kernel), against the UNMODIFIED reference compiled
from its sources (oracle/_ref: ref_c1_step = distributed_lookup W=1 two-stage
+ GradAccumulator accumulate + apply, workload.cpp:506-581; Adagrad rows by the
frozen restatement).

Three steps over batches A, B, A (the third replays A's captured graph on the
same scratch set):
* forward outputs: bit-exact (step 1 all tokens; later steps every token whose
  id has not yet been through the hot-id path -- a hot id's row after step 1 is
  within tolerance, not bit-identical);
* ids with <= 64 occurrences in every step so far: emb, Adagrad state and step
  counter bit-exact (sequential token-order sums);
* hot ids: the aggregated gradient through Adagrad's v' = v + g^2 under
  SURVEY §8(c)'s |dg| <= 1e-5 * sum|g_i|, accumulated over the steps;
* every row no batch touched: unchanged.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2505_12663_b200 as P
from paper_2505_12663_b200 import workload as W
from oracle.bind import Table

pytestmark = pytest.mark.gpu

TAG1 = 1 << 62
DIM, VOCAB, LR, EPS = 64, 1 << 20, 0.01, 1e-8
CSR_MAX = 64  # ids with more occurrences take the hot-id (tile partial) path


def test_config1_rs_step_vs_reference(cuda, ref):
    o = ref
    keys = np.arange(VOCAB, dtype=np.uint64) + np.uint64(TAG1)
    # GPU table exactly as bench.py builds it
    g = P.EmbedTable(P.TableConfig(capacity=1 << 22, embedding_dim=DIM, optimizer="adagrad",
                                   chunk_rows=1 << 16, initial_rows=VOCAB + (1 << 20)))
    raw = torch.arange(0, VOCAB, dtype=torch.int64, device="cuda")
    rows0 = W.pseudo_grads(raw, 0, DIM)
    g.insert(raw + TAG1, rows0)
    rows0 = rows0.cpu().numpy()
    # the reference's table: SimCluster(1) shard with the same rows (bench_main.cpp:105-108)
    h = C.c_void_p()
    assert o.cluster_create(1, 1 << 21, DIM, 1, 0.75, 1 << 16, 3, C.byref(h)) == 0
    shard = Table(o, 0, DIM, handle=o.cluster_shard(h, 0))
    shard.owned = False
    row = np.zeros(DIM, np.float32)
    o.pseudo_sparse_grad(5, 0, row, DIM)
    np.testing.assert_array_equal(row, rows0[5])  # device pseudo grads == the reference's
    for r in range(VOCAB):
        shard.insert(int(keys[r]), rows0[r])
    try:
        batches = [W.generate(1 + b, 1024, 128.0, 4096, 1.0, 1.1, [VOCAB]) for b in range(2)]
        plan = [0, 1, 0]
        max_t = max(len(i) for _, i in batches)
        step = P.SparseStep(g, max_t, P.AdagradParams(lr=LR, eps=EPS))
        dev = []
        for b, (lengths, ids) in enumerate(batches):
            grads = o.token_grads(lengths, b, DIM)  # the reference's pseudo_sparse_grad per token
            d_g = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), b, DIM)
            np.testing.assert_array_equal(d_g.cpu().numpy(), grads)
            dev.append((P.as_keys(ids), d_g, torch.empty((len(ids), DIM), device="cuda"), ids, grads))
        tainted = np.zeros(0, np.uint64)  # ids that went through the hot path
        vbound = {}                       # id -> accumulated |dv| bound (per element)
        touched = np.zeros(0, np.uint64)
        for k, b in enumerate(plan):
            d_ids, d_g, out, ids, grads = dev[b]
            step.step(d_ids, d_g, out)
            torch.cuda.synchronize()
            want = np.zeros((len(ids), DIM), np.float32)
            o.c1_step(h.value, ids, grads.reshape(-1), len(ids), 1, LR, EPS, want.ctypes.data)
            got = out.cpu().numpy()
            exact_tok = ~np.isin(ids, tainted)
            np.testing.assert_array_equal(got[exact_tok], want[exact_tok], err_msg=f"step {k}: gathered rows")
            assert np.abs(got - want).max() <= 1e-3, "hot rows drifted beyond the tolerance"
            u, cnt = np.unique(ids, return_counts=True)
            hot = u[cnt > CSR_MAX]
            assert 50 < len(hot) < 1000 and 20000 < len(u) < 40000, (len(hot), len(u))  # config-1 shape
            inv = np.searchsorted(u, ids)
            mass = np.zeros((len(u), DIM))
            np.add.at(mass, inv, np.abs(grads.astype(np.float64)))
            gsum = np.zeros((len(u), DIM))
            np.add.at(gsum, inv, grads.astype(np.float64))
            for i in np.nonzero(cnt > CSR_MAX)[0]:
                d = 1e-5 * mass[i]
                vbound[int(u[i])] = vbound.get(int(u[i]), 0.0) + (2 * np.abs(gsum[i]) + d) * d
            tainted = np.union1d(tainted, hot)
            touched = np.union1d(touched, u)
            a = g.export()
            bt = shard.export()
            np.testing.assert_array_equal(a["keys"], bt["keys"])
            np.testing.assert_array_equal(a["step"], bt["step"].astype(a["step"].dtype), err_msg="step counters")
            clean = ~np.isin(a["keys"], tainted)
            for f in ("emb", "v"):
                np.testing.assert_array_equal(a[f][clean], bt[f][clean], err_msg=f"step {k}: {f} of <=64-occurrence ids")
            sel = np.searchsorted(a["keys"], tainted)
            bound = np.stack([vbound[int(x)] for x in tainted]) + (k + 1) * 4 * np.spacing(np.abs(bt["v"][sel]))
            assert (np.abs(a["v"][sel].astype(np.float64) - bt["v"][sel]) <= bound).all(), "hot-id Adagrad state"
            assert np.abs(a["emb"][sel] - bt["emb"][sel]).max() <= 2 * LR * (k + 1)
            untouched = ~np.isin(a["keys"], touched)
            np.testing.assert_array_equal(a["emb"][untouched], rows0[(a["keys"][untouched] - np.uint64(TAG1)).astype(np.int64)])
    finally:
        o.cluster_destroy(h.value)
