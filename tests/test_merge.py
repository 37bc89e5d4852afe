"""Table merging, pooling and per-token routing.

CPU: the oracle restatement (oracle/merge.py) against the compiled
reference (plan_merge incl. its ConfigErrors; HashTableCollection::lookup
outputs and table contents).  GPU: librsgpu's plan / collection lookup /
routing against the oracle, bit-exact.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import merge as M

F = M.Feature

CONFIGS = [
    [F("user", 32, ["user_table"]), F("item", 32, ["item_table"]), F("ctx", 64, ["ctx_table"])],
    # C2-like: 8 logical tables -> 2 groups (dims 64 / 128), shared tables, pooled features
    [F("f0", 64, ["t0"]), F("f1", 64, ["t1"]), F("f2", 128, ["t4"]), F("f3", 64, ["t2", "t3"], M.SUM),
     F("f4", 128, ["t5", "t6"], M.MEAN), F("f5", 128, ["t7", "t4"], M.SUM), F("f6", 64, ["t0", "t1", "t3"], M.MEAN)],
    [F("a", 8, ["x"]), F("b", 8, ["x", "y"], M.SUM), F("c", 16, ["z"]), F("d", 8, ["y"])],
]
BAD = [
    ([F("", 8, ["x"])], "empty name"),
    ([F("a", 8, ["x"]), F("a", 8, ["y"])], "duplicate feature"),
    ([F("a", 0, ["x"])], "embedding_dim"),
    ([F("a", 8, [])], "lookup_tables"),
    ([F("a", 8, ["x"]), F("b", 16, ["x"])], "conflicting"),
]


def _plan_tuple(groups):
    return [(g.dim, g.k_bits, list(g.members)) for g in groups]


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_plan_merge_oracle_vs_ref(ref, ci):
    groups, _ = M.plan_merge(CONFIGS[ci])
    assert _plan_tuple(groups) == [(d, k, m) for d, k, m in M.ref_plan(ref, CONFIGS[ci])]


@pytest.mark.parametrize("cfg,what", BAD)
def test_plan_merge_errors_oracle_vs_ref(ref, cfg, what):
    with pytest.raises(M.ConfigError, match=what.split()[0]):
        M.plan_merge(cfg)
    with pytest.raises(M.ConfigError):
        M.ref_plan(ref, cfg)


def _ref_collection(ref, features, cap, chunk):
    lib = ref.lib
    lib.ref_collection_create.restype = C.c_void_p
    lib.ref_collection_create.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_int)]
    lib.ref_collection_lookup.restype = C.c_int
    lib.ref_collection_lookup.argtypes = [C.c_void_p, C.c_char_p, np.ctypeslib.ndpointer(np.uint64), C.c_uint64,
                                          np.ctypeslib.ndpointer(np.float32)]
    lib.ref_collection_table.restype = C.c_void_p
    lib.ref_collection_table.argtypes = [C.c_void_p, C.c_uint64]
    lib.ref_collection_destroy.argtypes = [C.c_void_p]
    st = C.c_int()
    h = lib.ref_collection_create(M.spec_string(features).encode(), cap, chunk, C.byref(st))
    assert st.value == 0
    return h


def test_collection_lookup_oracle_vs_ref(ref, oracle):
    from oracle.bind import Table
    features = CONFIGS[1]
    groups, gof = M.plan_merge(features)
    cap, chunk = 1 << 12, 256
    rh = _ref_collection(ref, features, cap, chunk)
    otabs = [Table(oracle, cap, g.dim, chunk_rows=chunk) for g in groups]
    rng = np.random.default_rng(5)
    for rnd in range(4):
        for f in features:
            raw = rng.integers(0, 300, 97).astype(np.uint64)
            want = np.zeros((len(raw), f.dim), np.float32)
            assert ref.lib.ref_collection_lookup(rh, f.name.encode(), raw, len(raw), want.reshape(-1)) == 0
            got = M.collection_lookup(oracle, groups, gof, [t.h for t in otabs], f, raw)
            np.testing.assert_array_equal(got, want, err_msg=f"round {rnd} feature {f.name}")
    for gi, g in enumerate(groups):
        rt = Table(ref, cap, g.dim, handle=ref.lib.ref_collection_table(rh, gi))
        rt.owned = False
        a, b = otabs[gi].export(), rt.export()
        for k in ("keys", "emb", "m", "v", "step"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=f"group {gi} {k}")
    ref.lib.ref_collection_destroy(rh)


def test_collection_lookup_pooling_values(oracle):
    # non-zero rows: sum in lookup-table order, mean = sum * (1/n) (merge_registry.cpp:146-155)
    from oracle.bind import Table
    features = [F("s", 4, ["a", "b", "c"], M.SUM), F("m", 4, ["a", "b", "c"], M.MEAN), F("n", 4, ["b"])]
    groups, gof = M.plan_merge(features)
    t = Table(oracle, 64, 4, chunk_rows=16)
    rng = np.random.default_rng(1)
    vals = {}
    for name in ("a", "b", "c"):
        for raw in range(5):
            gid = M.encode(groups[0].k_bits, groups[0].index_of[name], 3, raw)
            v = rng.standard_normal(4).astype(np.float32)
            t.insert(gid, v)
            vals[(name, raw)] = v
    raw = np.array([0, 3, 4, 3], np.uint64)
    s = M.collection_lookup(oracle, groups, gof, [t.h], features[0], raw)
    m = M.collection_lookup(oracle, groups, gof, [t.h], features[1], raw)
    n = M.collection_lookup(oracle, groups, gof, [t.h], features[2], raw)
    for i, r in enumerate(raw):
        want = np.zeros(4, np.float32)
        for name in ("a", "b", "c"):
            want = want + vals[(name, int(r))]
        np.testing.assert_array_equal(s[i], want)
        np.testing.assert_array_equal(m[i], want * (np.float32(1) / np.float32(3)))
        np.testing.assert_array_equal(n[i], vals[("b", int(r))])


def test_route_tagged_restatement():
    # per token: decode the catalog tag, re-encode in the group's id space
    features = CONFIGS[1]
    names, ordinal_of, cat_k = M.catalog_from(features)
    assert cat_k == 4 and len(names) == 8
    rng = np.random.default_rng(2)
    ords = rng.integers(1, 9, 500)
    raws = rng.integers(0, 1 << 20, 500)
    tagged = np.array([M.encode(cat_k, int(o), 8, int(r)) for o, r in zip(ords, raws)], np.uint64)
    ids, pos = M.route_tagged(tagged, features)
    groups, gof = M.plan_merge(features)
    seen = np.zeros(500, bool)
    for g, (gi, gp) in enumerate(zip(ids, pos)):
        assert np.all(np.diff(gp) > 0)  # token order
        for x, p in zip(gi, gp):
            idx, raw = M.decode(groups[g].k_bits, len(groups[g].members), int(x))
            assert raw == raws[p] and groups[g].members[idx - 1] == names[ords[p] - 1]
            seen[p] = True
    assert seen.all()


# ------------------------------------------------------------------ librsgpu
def _pfeat(f):
    import paper_2505_12663_b200 as P
    return P.FeatureConfig(f.name, f.dim, list(f.tables), P.Pooling(f.pooling))


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_rs_plan_merge_vs_oracle(ci):
    # host planning in librsgpu (no device work): same groups / members / k
    import paper_2505_12663_b200 as P
    plan = P.plan_merge([_pfeat(f) for f in CONFIGS[ci]])
    groups, gof = M.plan_merge(CONFIGS[ci])
    assert [(g.embedding_dim, g.k_bits, g.member_tables) for g in plan.groups] == _plan_tuple(groups)
    for t, g in gof.items():
        assert plan.group_index_for(t) == g
        assert plan.group_for(t).table_index_of[t] == groups[g].index_of[t]


@pytest.mark.parametrize("cfg,what", BAD)
def test_rs_plan_merge_errors(cfg, what):
    import paper_2505_12663_b200 as P
    with pytest.raises(P.ConfigError, match=what.split()[0]):
        P.plan_merge([_pfeat(f) for f in cfg])


@pytest.mark.gpu
def test_collection_lookup_gpu_vs_oracle(cuda, oracle):
    import torch

    import paper_2505_12663_b200 as P
    from oracle.bind import Table
    features = CONFIGS[1] + [F("f7", 64, ["t2", "t0"], M.SUM)]
    pfs = [_pfeat(f) for f in features]
    plan = P.plan_merge(pfs)
    groups, gof = M.plan_merge(features)
    cap = 1 << 12
    coll = P.HashTableCollection(plan, P.TableConfig(capacity=cap, chunk_rows=256, optimizer="adam"))
    otabs = [Table(oracle, cap, g.dim, chunk_rows=256) for g in groups]
    rng = np.random.default_rng(11)
    # give some rows non-zero values in both so pooling sums real numbers
    for gi, g in enumerate(groups):
        keys = np.array([M.encode(g.k_bits, i, len(g.members), r) for i in range(1, len(g.members) + 1)
                         for r in range(0, 200, 3)], np.uint64)
        emb = rng.standard_normal((len(keys), g.dim)).astype(np.float32)
        coll.table(gi).insert(keys, torch.from_numpy(emb).cuda())
        for k, e in zip(keys, emb):
            otabs[gi].insert(int(k), e)
    for rnd in range(3):
        for f, pf in zip(features, pfs):
            raw = rng.integers(0, 260, 150).astype(np.uint64)  # hits, misses (vivified), duplicates
            got = coll.lookup(pf, raw).cpu().numpy()
            want = M.collection_lookup(oracle, groups, gof, [t.h for t in otabs], f, raw)
            np.testing.assert_array_equal(got, want, err_msg=f"round {rnd} feature {f.name}")
    for gi in range(len(groups)):
        a, b = coll.table(gi).export(), otabs[gi].export()
        for k in ("keys", "emb", "m", "v", "step"):
            np.testing.assert_array_equal(a[k], b[k].astype(a[k].dtype), err_msg=f"group {gi} {k}")
    # pooling=none needs exactly one table; a raw id beyond the payload fails before any ensure
    with pytest.raises(P.ConfigError):
        coll.lookup(P.FeatureConfig("bad", 64, ["t0", "t1"], P.Pooling.NONE), np.zeros(1, np.uint64))
    occ = coll.table(0).occupied()
    with pytest.raises(P.RangeError):
        coll.lookup(pfs[0], np.array([1, 1 << 62], np.uint64))
    assert coll.table(0).occupied() == occ


@pytest.mark.gpu
def test_route_tagged_gpu_vs_oracle(cuda):
    import paper_2505_12663_b200 as P
    features = CONFIGS[1]
    plan = P.plan_merge([_pfeat(f) for f in features])
    names, _, cat_k = M.catalog_from(features)
    router = P.Router(plan, names)
    rng = np.random.default_rng(3)
    for n in (0, 1, 1023, 1024, 1025, 70001, 1_300_001):  # > 1024 route blocks: chunked scan
        ords = rng.integers(0, 9, n).astype(np.uint64)  # ordinal 0 = untagged ids (identity of group 0)
        raws = rng.integers(0, 1 << 40, n).astype(np.uint64)
        tagged = (ords << np.uint64(63 - cat_k)) | raws
        gids, pos, counts = router.route(tagged)
        want_ids, want_pos = (M.route_tagged if n < 100_000 else M.route_tagged_np)(tagged, features)
        assert counts == [len(x) for x in want_ids]
        np.testing.assert_array_equal(P.keys_to_numpy(gids), np.concatenate(want_ids) if n else np.zeros(0, np.uint64))
        np.testing.assert_array_equal(pos.cpu().numpy(), np.concatenate(want_pos) if n else np.zeros(0))
    with pytest.raises(P.RangeError):
        router.route(np.array([1 << 63], np.uint64))
    with pytest.raises(P.RangeError):
        router.route(np.array([15 << (63 - cat_k)], np.uint64))
