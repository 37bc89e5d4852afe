"""One rank of the sharded-step parity check (launched by tests/test_dist.py
under torchrun, one process per GPU).

Every rank builds the same seeded inputs, runs its own slice through
``ShardedTable`` (NVLink peer-store exchanges), and rank 0 replays the whole
step on the oracle's SimCluster restatement (oracle.c or_distributed_lookup,
exchange_sim.cpp:117-233; the backward as run_workload, workload.cpp:519-581:
grads grouped per owner in (worker, token) order -> accumulate -> apply):

* outputs of every rank: bit-exact with distributed_lookup's outputs[rank];
* ExchangeTrace (ids_sent, embs_sent, lookups, ids_requested, ids_received):
  equal;
* shard contents after the optimizer (keys, emb, m/v, step): bit-exact --
  gradients are dyadic (k/64) so every f32 sum is exact in any order.

Usage: torchrun --nproc-per-node W tests/dist_worker.py [adam|adagrad] [dim]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_12663_b200 as P  # noqa: E402
from paper_2505_12663_b200.dist import ShardedTable  # noqa: E402


def main():
    opt = sys.argv[1] if len(sys.argv) > 1 else "adam"
    dim = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, W = dist.get_rank(), dist.get_world_size()
    cap, V, max_tokens = 1 << 14, 6000, 4096
    rng = np.random.default_rng(4242)  # identical stream on every rank
    keys = np.unique(rng.integers(0, 1 << 40, V).astype(np.uint64))
    emb0 = rng.standard_normal((len(keys), dim)).astype(np.float32)
    fresh = np.unique(rng.integers(1 << 41, 1 << 42, 800).astype(np.uint64))  # vivified by ensure
    params = P.AdamParams() if opt == "adam" else P.AdagradParams(lr=0.05)
    kind = 0 if opt == "adam" else 1

    st = ShardedTable(P.TableConfig(capacity=cap, embedding_dim=dim, chunk_rows=256, optimizer=opt),
                      max_tokens=max_tokens)
    st.insert_owned(keys, torch.from_numpy(emb0).cuda())

    o = cl = None
    if rank == 0:
        from oracle.bind import Oracle, Table
        o = Oracle("oracle")
        h = C.c_void_p()
        assert o.cluster_create(W, cap, dim, 1, 0.75, 256, 3, C.byref(h)) == 0
        cl = h.value
        for k, e in zip(keys, emb0):
            s = int(o.shard_of(int(k), W))
            o.table_insert(o.cluster_shard(cl, s), int(k), np.ascontiguousarray(e))

    pool = np.concatenate([keys, fresh])
    for step in range(6):
        counts = [int(rng.integers(1, max_tokens)) for _ in range(W)]
        if step == 2:
            counts[W - 1] = 0  # an idle rank still takes part in the exchange
        if step == 3:
            counts = [max_tokens] * W
        # zipf-like skew over the pool: many repeats + a tail of singletons
        reqs = [pool[np.minimum(rng.zipf(1.2, n) - 1, len(pool) - 1)] if n else np.zeros(0, np.uint64)
                for n in counts]
        grads = [(rng.integers(-64, 64, (n, dim)) / 64.0).astype(np.float32) for n in counts]
        ids_t = torch.from_numpy(reqs[rank].astype(np.uint64).view(np.int64)).cuda()
        g_t = torch.from_numpy(grads[rank]).cuda()
        if step % 2 == 0:  # the split API (distributed_lookup, then accumulate/apply) ...
            out = st.forward(ids_t)
            st.backward(g_t, params)
        elif step == 3:  # ... the fused step with the gather's checksum ...
            cs = torch.full((1,), -1.0, dtype=torch.float64, device="cuda")
            out = st.step(ids_t, g_t, params, checksum=cs)
            assert float(cs[0]) == float(out.double().sum()) or \
                abs(float(cs[0]) - float(out.double().sum())) <= 1e-9 * max(1.0, float(out.double().abs().sum())), \
                (float(cs[0]), float(out.double().sum()))
        else:  # ... and the fused step must give identical results
            out = st.step(ids_t, g_t, params)
        tr = st.trace()
        outs = [None] * W
        dist.all_gather_object(outs, out.cpu().numpy())
        if rank == 0:
            cnt = np.array(counts, np.uint64)
            flat = np.ascontiguousarray(np.concatenate(reqs).astype(np.uint64))
            ref_out = np.zeros((max(int(cnt.sum()), 1), dim), np.float32)
            ids_sent = np.zeros(W * W, np.uint64)
            embs_sent = np.zeros(W * W, np.uint64)
            lookups = np.zeros(W, np.uint64)
            totals = np.zeros(2, np.uint64)
            rc = o.distributed_lookup(cl, flat if len(flat) else np.zeros(1, np.uint64), cnt,
                                      ref_out.reshape(-1), ids_sent, embs_sent, lookups, totals)
            assert rc == 0
            off = 0
            for r in range(W):
                np.testing.assert_array_equal(outs[r], ref_out[off:off + counts[r]],
                                              err_msg=f"step {step} outputs of rank {r}")
                off += counts[r]
            np.testing.assert_array_equal(tr["ids_sent"], ids_sent.reshape(W, W), err_msg="ids_sent")
            np.testing.assert_array_equal(tr["embs_sent"], embs_sent.reshape(W, W), err_msg="embs_sent")
            np.testing.assert_array_equal(tr["lookups"], lookups, err_msg="lookups")
            assert tr["ids_requested"] == totals[0] and tr["ids_received"] == totals[1], (tr, totals)
            # backward: grads grouped per owner in (worker, token) order (workload.cpp:519-526)
            for s in range(W):
                gi, gg = [], []
                for w in range(W):
                    if counts[w] == 0:
                        continue
                    own = np.array([o.shard_of(int(k), W) for k in reqs[w]])
                    sel = np.nonzero(own == s)[0]
                    gi.append(reqs[w][sel])
                    gg.append(grads[w][sel])
                ids_s = np.concatenate(gi).astype(np.uint64) if gi else np.zeros(0, np.uint64)
                if len(ids_s) == 0:
                    continue
                i2, s2 = o.accumulate_np(ids_s, np.concatenate(gg), dim)
                o.apply(o.cluster_shard(cl, s), i2, s2.reshape(-1), len(i2), kind, params.lr,
                        getattr(params, "beta1", 0.9), getattr(params, "beta2", 0.999), params.eps)
    ex = st.shard.export()
    exs = [None] * W
    dist.all_gather_object(exs, ex)
    if rank == 0:
        from oracle.bind import Table
        fields = ("keys", "emb", "v", "step") + (("m",) if opt == "adam" else ())
        for s in range(W):
            ot = Table(o, cap, dim, handle=o.cluster_shard(cl, s))
            ot.owned = False
            b = ot.export()
            for f in fields:
                np.testing.assert_array_equal(exs[s][f], b[f].astype(exs[s][f].dtype),
                                              err_msg=f"shard {s} {f}")
        o.cluster_destroy(cl)
        print(f"DIST OK world={W} opt={opt} dim={dim}", flush=True)
    st.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
