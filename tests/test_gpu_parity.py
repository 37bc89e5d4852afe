"""GPU parity: the sm_100a kernels (through the C-ABI) against the CPU oracle.

Bars: bit-exact for hash/shard, dedup unique + inverse, table
contents after insert/ensure/remove/expand/evict, forward gathered rows, and
the optimizer given identical aggregated gradients; aggregated gradients
within |Δ| <= 1e-5 * Σ|g_i| of the reference's sequential f32 sums.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2505_12663_b200 as P
from paper_2505_12663_b200 import workload as W
from oracle.bind import Table

pytestmark = pytest.mark.gpu

TAG1 = 1 << 62  # catalog tag of a single-table workload (k = 1, ordinal 1)
GRAD_TOL = 1e-5


def dev(a):
    return P.as_keys(a)


def np_u64(t):
    return P.keys_to_numpy(t)


# ---------------------------------------------------------------- primitives
def test_hash64_and_shard_of(cuda, oracle, kat):
    rng = np.random.default_rng(1)
    keys = np.concatenate([np.array([c[0] for c in kat["hash64"]["cases"]], np.uint64),
                           rng.integers(0, 2**63, 5000, dtype=np.uint64) * 2 + 1,
                           np.array([0, 2**64 - 1, 2**64 - 2], np.uint64)])
    got = np_u64(P.hash64_batch(keys))
    want = np.array([oracle.hash64(int(k)) for k in keys], np.uint64)
    np.testing.assert_array_equal(got, want)
    for w in (1, 2, 3, 4, 7, 8):
        s = P.shard_of_batch(keys, w).cpu().numpy()
        np.testing.assert_array_equal(s, (want % np.uint64(w)).astype(np.int32))


# --------------------------------------------------------------------- dedup
def _dedup_cases():
    rng = np.random.default_rng(7)
    yield np.zeros(0, np.uint64)
    yield np.array([5, 3, 5, 9, 3], np.uint64)  # test_exchange_sim.cpp:77-82
    yield np.array([4, 8, 15, 16, 23, 42], np.uint64)
    yield np.full(3000, 77, np.uint64)
    yield np.arange(2049, dtype=np.uint64)[::-1].copy()
    yield np.array([2**64 - 1, 0, 2**64 - 2, 2**64 - 1, 0, 1], np.uint64)  # sentinel bit patterns
    for n in (1, 511, 512, 513, 1025, 40000):
        yield (rng.zipf(1.1, n) % 100000).astype(np.uint64) + np.uint64(TAG1)
    _, ids = W.generate(1, 1024, 128.0, 4096, 1.0, 1.1, [1 << 20])  # config 1 batch
    yield ids


def test_dedup_bit_exact(cuda, oracle):
    ws = P.Workspace(200000)
    for ids in _dedup_cases():
        u, inv = P.stage1_dedup(ids, ws)
        wu, winv = oracle.stage1(ids)
        np.testing.assert_array_equal(np_u64(u), wu)
        np.testing.assert_array_equal(inv.cpu().numpy().astype(np.int64), winv)


def test_stage2_is_dedup_over_concatenation(cuda, oracle):
    rng = np.random.default_rng(11)
    lists = [rng.integers(0, 300, int(rng.integers(0, 200))).astype(np.uint64) for _ in range(8)]
    wu, off, src, pos = oracle.stage2(lists)
    u, inv = P.stage1_dedup(np.concatenate(lists))
    np.testing.assert_array_equal(np_u64(u), wu)
    # the inverse gives every origin; grouped by unique in (source, position) order
    inv = inv.cpu().numpy()
    base = np.cumsum([0] + [len(x) for x in lists])
    for k in range(len(wu)):
        js = np.nonzero(inv == k)[0]
        s = np.searchsorted(base, js, side="right") - 1
        np.testing.assert_array_equal(s, src[off[k]:off[k + 1]])
        np.testing.assert_array_equal(js - base[s], pos[off[k]:off[k + 1]])


# --------------------------------------------------------------------- table
def _gpu_table(capacity, dim, opt="adam", **kw):
    return P.EmbedTable(P.TableConfig(capacity=capacity, embedding_dim=dim, chunk_rows=64, optimizer=opt, **kw))


def _compare_contents(gpu, ora, fields=("keys", "emb", "m", "v", "step")):
    a = gpu.export()
    b = ora.export()
    for f in fields:
        np.testing.assert_array_equal(a[f], b[f].astype(a[f].dtype), err_msg=f)


def test_insert_and_import_duplicate_keys_last_wins(cuda, oracle):
    # the reference inserts one key at a time (embed_table.cpp:193-227): within
    # one batch the LAST occurrence of a key determines its row
    rng = np.random.default_rng(17)
    dim = 8
    g = _gpu_table(64, dim)
    o = Table(oracle, 64, dim, chunk_rows=64)
    for it in range(6):
        keys = rng.integers(0, 40, 300).astype(np.uint64)  # many duplicates per batch
        keys[:3] = np.array([2**64 - 1, 2**64 - 2, 2**64 - 1], np.uint64)  # sentinel bit patterns, duplicated
        emb = rng.standard_normal((len(keys), dim)).astype(np.float32)
        g.insert(keys, torch.from_numpy(emb))
        for k, e in zip(keys, emb):
            o.insert(int(k), e)
        _compare_contents(g, o, ("keys", "emb", "step"))
    # import (host arrays): the same rule
    h = _gpu_table(64, dim)
    keys = rng.integers(0, 30, 200).astype(np.uint64)
    emb = rng.standard_normal((len(keys), dim)).astype(np.float32)
    h.import_entries(keys, emb, step=np.arange(len(keys), dtype=np.uint64))
    got = h.export()
    last = {int(k): i for i, k in enumerate(keys)}
    assert sorted(last) == [int(k) for k in got["keys"]]
    for j, k in enumerate(got["keys"]):
        np.testing.assert_array_equal(got["emb"][j], emb[last[int(k)]])
        assert int(got["step"][j]) == last[int(k)]
    with pytest.raises(P.ConfigError):  # 32-bit device step counters
        h.import_entries(np.array([5], np.uint64), emb[:1], step=np.array([1 << 33], np.uint64))


def test_table_model_vs_oracle(cuda, oracle):
    rng = np.random.default_rng(99)
    dim = 4
    g = _gpu_table(16, dim)
    o = Table(oracle, 16, dim, chunk_rows=64)
    for it in range(120):
        op = int(rng.integers(0, 5))
        keys = np.unique(rng.integers(0, 600, int(rng.integers(1, 40))).astype(np.uint64))
        rng.shuffle(keys)
        if op <= 1:
            emb = rng.standard_normal((len(keys), dim)).astype(np.float32)
            g.insert(keys, torch.from_numpy(emb))
            for k, e in zip(keys, emb):
                o.insert(int(k), e)
        elif op == 2:
            rows = g.ensure(keys).cpu().numpy()
            assert (rows >= 0).all()
            for k in keys:
                oracle.table_ensure(o.h, int(k))
        elif op == 3:
            rem = g.remove(keys).cpu().numpy()
            want = [oracle.table_remove(o.h, int(k)) for k in keys]
            np.testing.assert_array_equal(rem, np.array(want, bool))
        else:
            out = g.lookup_batch(np.concatenate([keys, keys])).cpu().numpy()
            want = np.zeros_like(out)
            for j, k in enumerate(np.concatenate([keys, keys])):
                r = oracle.table_find(o.h, int(k))
                if r >= 0:
                    want[j] = np.ctypeslib.as_array(oracle.table_emb(o.h, r), (dim,))
            np.testing.assert_array_equal(out, want)
        if it in (40, 80):
            g.expand()
        assert g.occupied() == oracle.table_occupied(o.h)
    _compare_contents(g, o)
    assert g.load_factor() <= 0.75


def test_table_expand_keeps_rows(cuda):
    g = _gpu_table(16, 4)
    keys = np.arange(5, dtype=np.uint64)
    g.insert(keys, torch.arange(20, dtype=torch.float32).reshape(5, 4))
    rows_before = g.find(keys).cpu().numpy()
    g.remove(np.array([4], np.uint64))
    assert g.tombstones() == 1
    assert g.expand() == 32
    assert g.tombstones() == 0
    np.testing.assert_array_equal(g.find(keys[:4]).cpu().numpy(), rows_before[:4])  # rows never move
    assert g.find(np.array([4], np.uint64)).item() == -1


def test_sentinel_keys(cuda):
    g = _gpu_table(64, 4)
    keys = np.array([2**64 - 1, 2**64 - 2, 0, 7], np.uint64)
    g.insert(keys, torch.arange(16, dtype=torch.float32).reshape(4, 4))
    out = g.lookup_batch(keys).cpu().numpy()
    np.testing.assert_array_equal(out, np.arange(16, dtype=np.float32).reshape(4, 4))
    assert g.occupied() == 4
    assert g.remove(keys[:1]).all()
    assert g.find(keys[:1]).item() == -1 and g.occupied() == 3
    e = g.export()
    np.testing.assert_array_equal(e["keys"], np.sort(keys[1:]))


def test_lookup_batch_ticks(cuda, oracle):
    g = _gpu_table(256, 4, opt="none")
    keys = np.arange(150, dtype=np.uint64)
    g.insert(keys, torch.zeros(150, 4))
    t0 = g.tick()
    q = np.random.default_rng(5).integers(0, 200, 500).astype(np.uint64)
    out = g.lookup_batch(q).cpu().numpy()
    assert g.tick() == t0 + 1
    e = g.export()
    hit = np.isin(e["keys"], q)
    assert (e["ts"][hit] == t0 + 1).all() and (e["ts"][~hit] == t0).all()
    assert (out[q >= 150] == 0).all()


# ------------------------------------------------------------- the C1 step
def _c1_like(seed, num_seq, vocab, dim, opt="adagrad", mean=128.0):
    lengths, ids = W.generate(seed, num_seq, mean, 4096, 1.0, 1.1, [vocab])
    keys = np.arange(vocab, dtype=np.uint64) + np.uint64(TAG1)
    rows = np.zeros((vocab, dim), np.float32)
    from oracle.bind import Oracle
    o = Oracle("oracle")
    for r in range(vocab):
        o.pseudo_sparse_grad(r, 0, rows[r], dim)
    g = _gpu_table(1 << max(4, int(np.ceil(np.log2(vocab * 2)))), dim, opt=opt)
    g.insert(keys, torch.from_numpy(rows))
    ot = Table(o, 1 << max(4, int(np.ceil(np.log2(vocab * 2)))), dim, chunk_rows=4096)
    for r in range(vocab):
        ot.insert(int(keys[r]), rows[r])
    return lengths, ids, g, ot


@pytest.mark.parametrize("dim,opt", [(64, "adagrad"), (64, "adam"), (128, "adagrad"), (32, "adam"), (20, "adagrad")])
def test_step_vs_oracle(cuda, oracle, dim, opt):
    vocab = 20000
    lengths, ids, g, ot = _c1_like(3, 256, vocab, dim, opt)
    params = P.AdagradParams() if opt == "adagrad" else P.AdamParams()
    step = P.SparseStep(g, len(ids), params)
    tok_sample = W.sample_of_tokens(lengths)
    for s in range(3):
        # new ids appear too (vivified as zero rows)
        batch = ids.copy()
        batch[::97] = np.uint64(TAG1) + np.uint64(vocab + s * 100000) + np.arange(len(batch[::97]), dtype=np.uint64)
        grads = W.pseudo_grads(torch.from_numpy(tok_sample.view(np.int64)), s, dim)
        out = step.forward(P.as_keys(batch))
        sums = step.accumulate(grads)
        step.backward(grads)
        torch.cuda.synchronize()
        # forward: bit-exact with distributed_lookup at W = 1 (vivified rows are zeros)
        want_out = np.zeros((len(batch), dim), np.float32)
        oracle.table_lookup_batch(ot.h, batch, len(batch), want_out.reshape(-1))
        np.testing.assert_array_equal(out.cpu().numpy(), want_out)
        # aggregated grads (rows indexed like step.last_unique()): tolerance
        # against the sequential f32 sums of the reference
        u, inv = oracle.stage1(batch)
        nu = len(u)
        gpu_ids = P.keys_to_numpy(step.last_unique())
        assert len(gpu_ids) == nu and np.array_equal(np.sort(gpu_ids), np.sort(u))
        g_np = grads.cpu().numpy()
        ids_acc, sums_ref = oracle.accumulate_np(batch, g_np, dim)
        order = np.argsort(gpu_ids)
        sums_gpu = sums[:nu].cpu().numpy()[order]
        np.testing.assert_array_equal(ids_acc, gpu_ids[order])
        absmass = np.zeros((nu, dim), np.float64)
        np.add.at(absmass, inv, np.abs(g_np).astype(np.float64))
        mass_sorted = absmass[np.argsort(u)]
        err = np.abs(sums_gpu.astype(np.float64) - sums_ref)
        assert (err <= GRAD_TOL * mass_sorted + 1e-30).all(), err.max()
        # ids with <= 64 occurrences are summed in the reference's token order:
        # bit-exact; hot ids within the tolerance above
        counts = np.bincount(inv, minlength=nu)[np.argsort(u)]
        exact = counts <= 64
        assert exact.mean() > 0.9
        np.testing.assert_array_equal(sums_gpu[exact], sums_ref[exact])
        # optimizer bit-exact given the GPU's aggregated grads (oracle apply)
        oracle.apply(ot.h, ids_acc, np.ascontiguousarray(sums_gpu).reshape(-1), nu,
                     1 if opt == "adagrad" else 0, params.lr, getattr(params, "beta1", 0.9),
                     getattr(params, "beta2", 0.999), params.eps)
        _compare_contents(g, ot, ("keys", "emb", "v", "step") + (("m",) if opt == "adam" else ()))


@pytest.mark.parametrize("opt", ["adagrad", "adam"])
def test_step_edge_batches(cuda, oracle, opt):
    """Ragged edge cases through the fused step (rs_step): an empty batch is a
    no-op, single-token and duplicate-only batches update exactly like the
    reference's accumulate + apply (sparse_update.cpp:45-83), and an id with
    65 occurrences (past the sequential-sum limit) stays within the tolerance."""
    dim, vocab = 16, 300
    _, _, g, ot = _c1_like(5, 4, vocab, dim, opt)
    params = P.AdagradParams() if opt == "adagrad" else P.AdamParams()
    st = P.SparseStep(g, 4096, params)
    batches = [np.zeros(0, np.uint64),
               np.array([7], np.uint64) + np.uint64(TAG1),
               np.array([9, 9, 9, 4, 9], np.uint64) + np.uint64(TAG1),
               np.array([vocab + 5], np.uint64) + np.uint64(TAG1),  # new id: vivified zero row
               np.concatenate([np.full(65, 11, np.uint64), np.arange(20, dtype=np.uint64)]) + np.uint64(TAG1)]
    for s, batch in enumerate(batches):
        n = len(batch)
        rng = np.random.default_rng(s)
        grads = torch.from_numpy(rng.uniform(-0.05, 0.05, (max(n, 1), dim)).astype(np.float32)).cuda()[:n]
        out = torch.empty((max(n, 1), dim), device="cuda")[:n]
        want_out = np.zeros((n, dim), np.float32)
        if n:
            oracle.table_lookup_batch(ot.h, batch, n, want_out.reshape(-1))
        st.step(P.as_keys(batch), grads.contiguous(), out)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), want_out)
        if n:
            ids_acc, sums_ref = oracle.accumulate_np(batch, grads.cpu().numpy(), dim)
            oracle.apply(ot.h, ids_acc, np.ascontiguousarray(sums_ref.astype(np.float32)).reshape(-1),
                         len(ids_acc), 1 if opt == "adagrad" else 0, params.lr, getattr(params, "beta1", 0.9),
                         getattr(params, "beta2", 0.999), params.eps)
        a, b = g.export(), ot.export()
        np.testing.assert_array_equal(a["keys"], b["keys"].astype(a["keys"].dtype))
        np.testing.assert_array_equal(a["step"], b["step"].astype(a["step"].dtype))
        if s < 4:  # every id summed in token order: bit-exact
            np.testing.assert_array_equal(a["emb"], b["emb"])
        else:  # the 65-occurrence id: tolerance on its updated row
            np.testing.assert_allclose(a["emb"], b["emb"], rtol=1e-5, atol=1e-6)
    # empty batch through the checksum variant: checksum 0, table untouched
    before = g.export()
    cs = torch.full((1,), 123.0, dtype=torch.float64, device="cuda")
    empty = torch.empty((1, dim), device="cuda")[:0]
    st.step_checksum(P.as_keys(np.zeros(0, np.uint64)), empty, empty, cs)
    torch.cuda.synchronize()
    assert float(cs[0]) == 0.0
    after = g.export()
    for f in ("keys", "emb", "v", "step"):
        np.testing.assert_array_equal(before[f], after[f], err_msg=f)


def test_step_deterministic(cuda):
    dim = 64
    lengths, ids = W.generate(4, 128, 128.0, 4096, 1.0, 1.1, [50000])
    res = []
    for _ in range(2):
        g = _gpu_table(1 << 17, dim, opt="adagrad")
        st = P.SparseStep(g, len(ids), P.AdagradParams())
        grads = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), 0, dim)
        out = torch.empty((len(ids), dim), device="cuda")
        for _ in range(3):
            st.step(P.as_keys(ids), grads, out)
        res.append(g.export())
    for f in ("keys", "emb", "v", "step"):
        np.testing.assert_array_equal(res[0][f], res[1][f])


@pytest.mark.parametrize("opt", ["adam", "adagrad"])
def test_apply_aggregated_bit_exact(cuda, oracle, opt):
    rng = np.random.default_rng(61)
    dim = 64
    g = _gpu_table(1024, dim, opt=opt)
    o = Table(oracle, 1024, dim, chunk_rows=64)
    keys = np.arange(300, dtype=np.uint64) * np.uint64(977)
    init = rng.standard_normal((300, dim)).astype(np.float32)
    g.insert(keys, torch.from_numpy(init))
    for k, e in zip(keys, init):
        o.insert(int(k), e)
    params = P.AdamParams(lr=0.003) if opt == "adam" else P.AdagradParams(lr=0.02)
    for step in range(25):
        sel = np.sort(rng.choice(np.concatenate([keys, keys[:20] + np.uint64(1)]), 120, replace=False))
        sums = (rng.standard_normal((120, dim)) * 0.1).astype(np.float32)
        P.apply_aggregated(g, sel, torch.from_numpy(sums), params)
        oracle.apply(o.h, sel, sums.reshape(-1), 120, 0 if opt == "adam" else 1, params.lr,
                     getattr(params, "beta1", 0.9), getattr(params, "beta2", 0.999), params.eps)
    _compare_contents(g, o, ("keys", "emb", "v", "step") + (("m",) if opt == "adam" else ()))


def test_sparse_update_matches_accumulate_apply(cuda, oracle):
    # GradAccumulator::accumulate + apply over one window, vivifying absent ids
    rng = np.random.default_rng(67)
    dim = 32
    g = _gpu_table(256, dim, opt="adam")
    o = Table(oracle, 256, dim, chunk_rows=64)
    ws = P.Workspace(1000)
    for _ in range(5):
        ids = rng.integers(0, 40, 700).astype(np.uint64)
        grads = (rng.integers(-64, 64, (700, dim)) / 64.0).astype(np.float32)  # dyadic: f32 sums exact in any order
        P.sparse_update(g, ws, ids, torch.from_numpy(grads).cuda(), P.AdamParams())
        i2, s2 = oracle.accumulate_np(ids, grads, dim)
        oracle.apply(o.h, i2, s2.reshape(-1), len(i2), 0, 0.01, 0.9, 0.999, 1e-8)
    _compare_contents(g, o, ("keys", "emb", "m", "v", "step"))


# ------------------------------------------------------- bounded + eviction
def test_bounded_table_eviction_vs_oracle(cuda, oracle):
    rng = np.random.default_rng(21)
    dim, bound = 16, 3000
    g = _gpu_table(1 << 13, dim, opt="adagrad", max_keys=bound)
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
        assert g.occupied() == oracle.table_occupied(o.h) <= bound
        assert g.tick() == tick
    _compare_contents(g, o, ("keys", "ts", "emb", "v", "step"))
    # explicit eviction of the k oldest (ts, key)
    g.evict(100)
    oracle.table_evict_oldest(o.h, 100)
    _compare_contents(g, o, ("keys", "ts"))


def test_evict_log_stream_vs_oracle(cuda, oracle):
    # the stamp-log victim selection (evict.cu k_lg_*) over a config-3-like
    # stream: a big fill (rebuilt into the (tick, key)-sorted region), then
    # batches of resident + never-seen ids evicting the oldest, a remove, an
    # explicit evict, the sentinel keys; no host sync between the batches
    rng = np.random.default_rng(77)
    dim, bound = 8, 6000
    g = _gpu_table(1 << 14, dim, opt="adagrad", max_keys=bound)
    o = Table(oracle, 1 << 14, dim, chunk_rows=4096)
    fill = rng.choice(1 << 40, bound - 2, replace=False).astype(np.uint64)
    fill = np.concatenate([fill, np.array([~np.uint64(0), ~np.uint64(0) - np.uint64(1)], np.uint64)])
    tick = g.tick() + 1
    g.ensure(fill)
    oracle.table_ensure_batch(o.h, fill, len(fill), tick, bound, None)
    fresh = np.uint64(1 << 50)
    resident = fill.copy()
    for b in range(40):
        old = rng.choice(resident, 400)
        new = fresh + np.arange(250, dtype=np.uint64)
        fresh += np.uint64(250)
        keys = np.unique(np.concatenate([old, new]))
        rng.shuffle(keys)
        tick = g.tick() + 1
        g.ensure(keys)
        oracle.table_ensure_batch(o.h, keys, len(keys), tick, bound, None)
        resident = np.concatenate([resident, new])[-bound:]
        if b == 12:
            rm = rng.choice(keys, 30, replace=False)
            g.remove(rm)
            for k in rm:
                oracle.table_remove(o.h, int(k))
        if b == 20:
            g.evict(500)
            oracle.table_evict_oldest(o.h, 500)
    assert g.occupied() == oracle.table_occupied(o.h)
    _compare_contents(g, o, ("keys", "ts", "emb", "v", "step"))


def test_step_graphs_survive_row_pool_growth(cuda):
    # the captured fast-step graphs bake the row pool's pointers in: a growth
    # of the pool between replays (new keys of another batch) must re-capture
    # them (buf_gen).  Same step sequence on a table that grows and on one
    # sized up front: bit-identical contents and outputs.
    rng = np.random.default_rng(91)
    dim, vocab = 64, 4000
    params = P.AdagradParams(lr=0.01, eps=1e-8)
    tabs = [P.EmbedTable(P.TableConfig(capacity=1 << 16, embedding_dim=dim, optimizer="adagrad", chunk_rows=64,
                                       initial_rows=r)) for r in (vocab + 64, 1 << 20)]
    keys0 = np.arange(vocab, dtype=np.uint64)
    for t in tabs:
        t.insert(keys0, torch.zeros(vocab, dim))
    batches = []
    for b, nb in enumerate((800, 2000, 5000)):  # growing batches: the pool grows at each new size
        ids = rng.integers(0, vocab, nb).astype(np.uint64)
        ids[::5] = np.uint64(10**6 * (b + 1)) + np.arange(len(ids[::5]), dtype=np.uint64)  # new keys
        ids[1::7] = np.uint64(7)  # a hot id: the hot-tile kernel reads the rows through the baked pointer
        batches.append((P.as_keys(ids), W.pseudo_grads(torch.arange(len(ids)), b, dim)))
    steps = [P.SparseStep(t, 5000, params) for t in tabs]
    outs = [[], []]
    for k, bi in enumerate((0, 0, 1, 0, 2, 1, 0, 2, 0)):  # replays of graphs captured before a growth
        ids, g = batches[bi]
        for j in range(2):
            out = torch.empty((ids.numel(), dim), device="cuda")
            steps[j].step(ids, g, out)
            outs[j].append(out.clone())
    torch.cuda.synchronize()
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    ea, eb = tabs[0].export(), tabs[1].export()
    oa, ob = np.argsort(ea["keys"]), np.argsort(eb["keys"])
    for f in ("keys", "emb", "v", "step"):
        np.testing.assert_array_equal(ea[f][oa], eb[f][ob], err_msg=f)


def test_ensure_duplicate_keys_in_one_batch(cuda, oracle):
    # ensure (embed_table.cpp:243-248) with every key repeated inside one batch:
    # one row per key, no row leaked, same contents as sequential ensures
    rng = np.random.default_rng(8)
    dim = 8
    g = _gpu_table(1 << 10, dim, opt="adam")
    o = Table(oracle, 1 << 10, dim, chunk_rows=64)
    for _ in range(6):
        keys = rng.integers(0, 300, 4000).astype(np.uint64)  # ~13 copies per key
        rows = g.ensure(keys).cpu().numpy()
        for k in keys:
            oracle.table_ensure(o.h, int(k))
        first = {}
        for k, r in zip(keys, rows):
            assert first.setdefault(int(k), r) == r
        i = g.info()
        assert i.occupied == o.o.table_occupied(o.h)
        assert i.rows_allocated - i.rows_free == i.occupied  # nothing leaked
    _compare_contents(g, o, ("keys", "emb", "m", "v", "step"))


@pytest.mark.parametrize("spread", [1, 5000])
def test_device_eviction_vs_oracle(cuda, oracle, spread):
    # bounded ensure with the device victim selection: ties in tick broken by
    # key (one initial tick for every key), ticks spread over many batches
    # (spread > 4096 exercises the narrowing tick windows), sentinel keys
    rng = np.random.default_rng(31 + spread)
    dim, bound = 8, 2000
    g = _gpu_table(1 << 12, dim, opt="adagrad", max_keys=bound)
    o = Table(oracle, 1 << 12, dim, chunk_rows=4096)
    init = rng.choice(1 << 40, bound - 2, replace=False).astype(np.uint64)
    init = np.concatenate([init, np.array([~np.uint64(0), ~np.uint64(0) - np.uint64(1)], np.uint64)])
    for lo in range(0, bound, 500):  # several initial ticks
        keys = init[lo:lo + 500]
        tick = g.tick() + 1
        g.ensure(keys)
        oracle.table_ensure_batch(o.h, keys, len(keys), tick, bound, None)
    if spread > 1:
        # spread the ticks of touched keys over > 4096 batch ops: lookups of an
        # absent key advance the tick and stamp nothing
        for _ in range(3):
            for _ in range(1500):
                g.lookup_batch(np.array([1], np.uint64))
            sel = rng.choice(init, 50, replace=False)
            tick = g.tick() + 1
            g.ensure(sel)
            oracle.table_ensure_batch(o.h, sel, len(sel), tick, bound, None)
    fresh = np.uint64(1 << 50)
    for b in range(10):
        old = rng.choice(init, 300)
        new = fresh + np.arange(120, dtype=np.uint64)
        fresh += np.uint64(120)
        keys = np.unique(np.concatenate([old, new]))
        tick = g.tick() + 1
        g.ensure(keys)
        oracle.table_ensure_batch(o.h, keys, len(keys), tick, bound, None)
        assert g.occupied() == oracle.table_occupied(o.h) == bound
    _compare_contents(g, o, ("keys", "ts", "emb", "v", "step"))
    for k in (1, 77, 600):
        g.evict(k)
        oracle.table_evict_oldest(o.h, k)
        _compare_contents(g, o, ("keys", "ts"))


def test_bounded_step_graph_equals_eager_and_oracle_keys(cuda, oracle):
    # the fused step on a bounded table replays from a CUDA graph (device
    # eviction, no host round trip); it must equal the eager forward/backward
    # path bit for bit, and its key set / ticks must follow the oracle's
    # ensure_batch eviction semantics
    rng = np.random.default_rng(41)
    dim, bound = 32, 1500
    tabs = [_gpu_table(1 << 12, dim, opt="adagrad", max_keys=bound) for _ in range(2)]
    o = Table(oracle, 1 << 12, dim, chunk_rows=4096)
    init = np.arange(bound, dtype=np.uint64) * np.uint64(7919)
    for t in tabs:
        t.ensure(init)
    tick0 = tabs[0].tick()
    oracle.table_ensure_batch(o.h, init, len(init), tick0, bound, None)
    steps = [P.SparseStep(t, 6000, P.AdagradParams(lr=0.05)) for t in tabs]
    fresh = np.uint64(1 << 45)
    buf_ids = torch.empty(6000, dtype=torch.int64, device="cuda")
    buf_g = torch.empty((6000, dim), device="cuda")
    outs = [torch.empty((6000, dim), device="cuda") for _ in tabs]
    for b in range(8):
        base = init[rng.integers(0, 900, 3000)]  # a batch must fit the bound
        new = fresh + rng.integers(0, 400, 1000).astype(np.uint64)
        fresh += np.uint64(400)
        ids = np.concatenate([base, new])
        rng.shuffle(ids)
        n = len(ids)
        buf_ids[:n] = P.as_keys(ids)
        buf_g[:n] = torch.from_numpy((rng.integers(-64, 64, (n, dim)) / 64.0).astype(np.float32)).cuda()
        tick = tabs[0].tick() + 1
        steps[0].step(buf_ids[:n], buf_g[:n], outs[0][:n])        # graph path
        steps[1].forward(buf_ids[:n], outs[1][:n])                # eager path
        steps[1].backward(buf_g[:n])
        torch.testing.assert_close(outs[0][:n], outs[1][:n], rtol=0, atol=0)
        u = np.unique(ids)
        oracle.table_ensure_batch(o.h, u, len(u), tick, bound, None)
        assert tabs[0].occupied() == tabs[1].occupied() == bound
    a, b2 = tabs[0].export(), tabs[1].export()
    for f in ("keys", "emb", "v", "step", "ts"):
        np.testing.assert_array_equal(a[f], b2[f], err_msg=f)
    oo = o.export()
    np.testing.assert_array_equal(a["keys"], oo["keys"])
    np.testing.assert_array_equal(a["ts"], oo["ts"].astype(a["ts"].dtype))


def test_pseudo_grads_jagged_equals_per_token(cuda, oracle):
    # pseudo_sparse_grad (workload.cpp:348-355) broadcast per sample == per token, == the oracle
    lengths = np.array([1, 5, 300, 2, 4096, 17], np.uint64)
    n = int(lengths.sum())
    a = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), 7, 64)
    b = W.pseudo_grads_jagged(torch.from_numpy(lengths.view(np.int64)), 7, 64, n)
    torch.testing.assert_close(a, b, rtol=0, atol=0)
    want = oracle.token_grads(lengths, 7, 64)
    np.testing.assert_array_equal(b.cpu().numpy(), want)
    offs = torch.from_numpy(np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)).cuda()
    c = torch.empty_like(b)
    P._lib.check(P.lib().rs_pseudo_grads_offsets(offs.data_ptr(), len(lengths), 1, 7, 64, c.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream), "offsets")
    torch.testing.assert_close(c, b, rtol=0, atol=0)


@pytest.mark.parametrize("dim,bound", [(64, 0), (6, 0), (64, 2000)])
def test_step_checksum_fused(cuda, dim, bound):
    # rs_step_checksum == rs_step (bit-exact outputs and table), its checksum ==
    # the f64 sum of the outputs, and it does not depend on timing (repeatable);
    # bound > 0: a bounded table (device eviction inside the step)
    kw = {"max_keys": bound} if bound else {}
    tabs = [_gpu_table(1 << 12, dim, opt="adagrad", **kw) for _ in range(2)]
    steps = [P.SparseStep(t, 40000, P.AdagradParams(lr=0.05)) for t in tabs]
    rng = np.random.default_rng(5)
    cs = torch.zeros(1, dtype=torch.float64, device="cuda")
    for k in range(5):
        n = int(rng.integers(1, 40000))
        raw = rng.zipf(1.2, n).astype(np.uint64)
        # bounded: <= 1500 distinct per batch, a sliding window -> evictions
        ids = P.as_keys(raw % 1500 + np.uint64(700 * k) if bound else raw % 3000)
        g = torch.randn((n, dim), device="cuda")
        o1, o2 = torch.empty((n, dim), device="cuda"), torch.empty((n, dim), device="cuda")
        steps[0].step_checksum(ids, g, o1, cs)
        steps[1].step(ids, g, o2)
        torch.testing.assert_close(o1, o2, rtol=0, atol=0)
        want = float(o2.double().sum())
        assert float(cs[0]) == pytest.approx(want, rel=1e-12, abs=1e-9)
    a, b = tabs[0].export(), tabs[1].export()
    for fld in ("keys", "emb", "v", "step"):
        np.testing.assert_array_equal(a[fld], b[fld], err_msg=fld)
    # same inputs, same table state -> bit-identical checksum
    t3 = [_gpu_table(1 << 12, dim, opt="adagrad", **kw) for _ in range(2)]
    s3 = [P.SparseStep(t, 40000, P.AdagradParams(lr=0.05)) for t in t3]
    ids = P.as_keys(rng.zipf(1.2, 30000).astype(np.uint64) % 1500)
    g = torch.randn((30000, dim), device="cuda")
    res = []
    for st in s3:
        o = torch.empty((30000, dim), device="cuda")
        c = torch.zeros(1, dtype=torch.float64, device="cuda")
        st.step_checksum(ids, g, o, c)
        res.append(float(c[0]))
    assert res[0] == res[1]


def test_feeder_step_matches_device_step(cuda):
    # rs_feeder_step (host ids + lengths -> device grads -> rs_step -> checksum)
    # equals the same step driven from device buffers, checksum included
    from paper_2505_12663_b200.feed import Feeder
    dim = 32
    tabs = [_gpu_table(1 << 12, dim, opt="adagrad") for _ in range(2)]
    steps = [P.SparseStep(t, 5000, P.AdagradParams(lr=0.05)) for t in tabs]
    f = Feeder(5000, 64, dim)
    rng = np.random.default_rng(12)
    for k in range(5):
        lengths = rng.integers(1, 120, 40).astype(np.uint64)
        if k == 2:  # ragged: empty sequences inside the batch
            lengths[::3] = 0
        if k == 3:  # every sequence empty: a no-op step, checksum 0
            lengths[:] = 0
        ids = rng.integers(0, 900, int(lengths.sum())).astype(np.uint64)
        h_ids = torch.from_numpy(ids.view(np.int64)).pin_memory()
        h_len = torch.from_numpy(lengths.view(np.int64)).pin_memory()
        f.step(steps[0], h_ids, h_len, k)
        got = f.checksum()
        g = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), k, dim)
        out = torch.empty((len(ids), dim), device="cuda")
        steps[1].step(P.as_keys(ids), g, out)
        assert got == pytest.approx(float(out.double().sum()), rel=1e-9, abs=1e-9)
    a, b = tabs[0].export(), tabs[1].export()
    for fld in ("keys", "emb", "v", "step"):
        np.testing.assert_array_equal(a[fld], b[fld], err_msg=fld)
