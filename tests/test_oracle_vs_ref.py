"""Pins the C restatement (oracle/oracle.c) to the reference itself, compiled
from /root/reference/proj sources into oracle/_ref/librsref.so, on seeded
random inputs (the reference's own test shapes: model test
test_embed_table.cpp:342-395, oracle equality test_exchange_sim.cpp:187-218,
optimizer trajectories acceptance_test.cpp:517-596)."""
import ctypes as C

import numpy as np
import pytest

from oracle.bind import Table


def digest(o, t):
    return (o.table_capacity(t.h), o.table_occupied(t.h), o.table_tombstones(t.h), o.table_tick(t.h))


@pytest.mark.parametrize("groups", [1, 2, 4])
def test_table_model_matches_reference(oracle, ref, groups):
    rng = np.random.default_rng(groups * 7 + 1)
    a = Table(oracle, 16, 2, groups=groups, chunk_rows=32)
    b = Table(ref, 16, 2, groups=groups, chunk_rows=32)
    for i in range(6000):
        k = int(rng.integers(0, 600))
        op = int(rng.integers(0, 100))
        if op < 50:
            e = np.array([op, -op], np.float32)
            assert a.insert(k, e) == b.insert(k, e)
        elif op < 70:
            assert oracle.table_lookup(a.h, k) == ref.table_lookup(b.h, k)
        elif op < 80:
            assert oracle.table_ensure(a.h, k) == ref.table_ensure(b.h, k)
        else:
            assert oracle.table_remove(a.h, k) == ref.table_remove(b.h, k)
        if i in (2000, 4000):  # forced expansions (test_embed_table.cpp:373-375)
            assert oracle.table_expand(a.h) == ref.table_expand(b.h)
        if i % 500 == 0:
            assert digest(oracle, a) == digest(ref, b)
    ea, eb = a.export(), b.export()
    for key in ea:
        np.testing.assert_array_equal(ea[key], eb[key])


def test_lookup_batch_matches_reference(oracle, ref):
    a = Table(oracle, 256, 4, chunk_rows=64)
    b = Table(ref, 256, 4, chunk_rows=64)
    for k in range(150):
        v = np.arange(4, dtype=np.float32) + k
        a.insert(k, v)
        b.insert(k, v)
    keys = np.random.default_rng(5).integers(0, 200, 500).astype(np.uint64)
    oa = np.zeros(500 * 4, np.float32)
    ob = np.zeros(500 * 4, np.float32)
    oracle.table_lookup_batch(a.h, keys, 500, oa)
    ref.table_lookup_batch(b.h, keys, 500, ob, 1)
    np.testing.assert_array_equal(oa, ob)
    for key in ("keys", "ts", "emb"):
        np.testing.assert_array_equal(a.export()[key], b.export()[key])


def test_dedup_matches_reference(oracle, ref):
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 1000, 50000):
        ids = (rng.zipf(1.2, n) % 5000).astype(np.uint64) if n else np.zeros(0, np.uint64)
        ua, ia = oracle.stage1(ids)
        ub, ib = ref.stage1(ids)
        np.testing.assert_array_equal(ua, ub)
        np.testing.assert_array_equal(ia, ib)
    lists = [rng.integers(0, 50, int(rng.integers(0, 40))).astype(np.uint64) for _ in range(5)]
    for x, y in zip(oracle.stage2(lists), ref.stage2(lists)):
        np.testing.assert_array_equal(x, y)


def _requests(rng, world, space):
    out = []
    for _ in range(world):
        n = int(rng.integers(0, 60))
        out.append(np.array([rng.integers(0, space // 4 + 1) for _ in range(n)], np.uint64) * 7919 % space)
    return out


def _dist(o, world, mode, populated, reqs, dim=4):
    h = C.c_void_p()
    assert o.cluster_create(world, 128, dim, 1, 0.75, 128, mode, C.byref(h)) == 0
    for idx in populated:
        s = o.shard_of(idx, world)
        sh = Table(o, 0, dim, handle=o.cluster_shard(h, s))
        sh.insert(idx, (np.arange(dim, dtype=np.float32) + idx) * 1e-3)
    counts = np.array([len(r) for r in reqs], np.uint64)
    flat = np.concatenate(reqs).astype(np.uint64) if counts.sum() else np.zeros(1, np.uint64)
    out = np.zeros(max(int(counts.sum()), 1) * dim, np.float32)
    ids_sent = np.zeros(world * world, np.uint64)
    embs_sent = np.zeros(world * world, np.uint64)
    lookups = np.zeros(world, np.uint64)
    totals = np.zeros(2, np.uint64)
    st = o.distributed_lookup(h, flat, counts, out, ids_sent, embs_sent, lookups, totals)
    o.cluster_destroy(h)
    assert st == 0
    return out, ids_sent, embs_sent, lookups, totals


def test_distributed_lookup_matches_reference(oracle, ref):
    rng = np.random.default_rng(17)
    for trial in range(12):
        world = int(rng.integers(1, 9))
        populated = sorted(set(int(x) for x in rng.integers(0, 500, 40)))
        reqs = _requests(rng, world, 500)
        for mode in range(4):
            a = _dist(oracle, world, mode, populated, reqs)
            b = _dist(ref, world, mode, populated, reqs)
            for x, y in zip(a, b):
                np.testing.assert_array_equal(x, y)


def test_accumulate_apply_adam_matches_reference(oracle, ref):
    rng = np.random.default_rng(67)
    dim = 4
    a = Table(oracle, 128, dim, chunk_rows=64)
    b = Table(ref, 128, dim, chunk_rows=64)
    for k in range(30):
        w = np.array([k, 0, -1, 1], np.float32)
        a.insert(k, w)
        b.insert(k, w)
    for step in range(20):
        ids = rng.integers(0, 40, 100).astype(np.uint64)
        grads = (rng.integers(0, 100, 400) / 50.0 - 1.0).astype(np.float32)
        ia, sa = oracle.accumulate_np(ids, grads, dim)
        ib, sb = ref.accumulate_np(ids, grads, dim)
        np.testing.assert_array_equal(ia, ib)
        np.testing.assert_array_equal(sa, sb)
        oracle.apply(a.h, ia, sa.reshape(-1), len(ia), 0, 0.01, 0.9, 0.999, 1e-8)
        ref.accumulate_apply_adam(b.h, ids, grads, len(ids), 0.01, 0.9, 0.999, 1e-8, 1)
    ea, eb = a.export(), b.export()
    for key in ("keys", "emb", "m", "v", "step"):
        np.testing.assert_array_equal(ea[key], eb[key])


def test_encode_decode_match_reference(oracle, ref):
    rng = np.random.default_rng(41)
    oa, ob = C.c_uint64(), C.c_uint64()
    for _ in range(2000):
        k = int(rng.integers(1, 5))
        lim = (1 << k) - 1
        idx = int(rng.integers(0, lim + 2))
        raw = int(rng.integers(0, 1 << 62)) >> int(rng.integers(0, 4))
        assert oracle.encode_tagged_id(k, idx, lim, raw, C.byref(oa)) == \
            ref.encode_tagged_id(k, idx, lim, raw, C.byref(ob))
        assert oa.value == ob.value


def test_batcher_matches_reference(oracle, ref):
    rng = np.random.default_rng(9)
    for trial in range(30):
        n = int(rng.integers(1, 400))
        lengths = rng.integers(1, 300, n).astype(np.uint64)
        target = int(rng.integers(1, 2000))
        chunk = int(rng.integers(1, 64))
        ba = np.zeros(n + 1, np.uint64)
        bb = np.zeros(n + 1, np.uint64)
        na = oracle.sequence_batches(lengths, n, target, chunk, ba)
        nb = ref.sequence_batches(lengths, n, target, chunk, bb)
        assert na == nb
        np.testing.assert_array_equal(ba[:na], bb[:nb])


@pytest.mark.parametrize("tables,vocab", [(1, [1 << 20]), (3, [1000, 50, 7])])
def test_generator_matches_reference(oracle, ref, tables, vocab):
    la, ia = oracle.generate(5, 300, 64.0, 1000, 1.2, 1.1, vocab)
    lb, ib = ref.generate(5, 300, 64.0, 1000, 1.2, 1.1, vocab)
    np.testing.assert_array_equal(la, lb)
    np.testing.assert_array_equal(ia, ib)
    for sid in (1, 77, 300):
        np.testing.assert_array_equal(oracle.grads(sid, 3, 64), ref.grads(sid, 3, 64))
