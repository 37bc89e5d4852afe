"""Elastic checkpoint of device shards against the
compiled reference's save_cluster / load_cluster (checkpoint.cpp)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2505_12663_b200 as P
from paper_2505_12663_b200 import checkpoint as K


def _ref_fns(ref):
    lib = ref.lib
    lib.ref_ckpt_save_cluster.restype = C.c_int
    lib.ref_ckpt_save_cluster.argtypes = [C.c_void_p, C.c_char_p]
    lib.ref_ckpt_load_cluster.restype = C.c_void_p
    lib.ref_ckpt_load_cluster.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                          C.POINTER(C.c_int)]
    return lib


def _ref_cluster(ref, world, dim, keys, rng):
    # a reference SimCluster holding keys with non-trivial emb / Adam state / ticks
    from oracle.bind import Table
    h = C.c_void_p()
    assert ref.cluster_create(world, 1 << 12, dim, 1, 0.75, 256, 3, C.byref(h)) == 0
    for k in keys:
        s = int(ref.shard_of(int(k), world))
        tab = ref.cluster_shard(h.value, s)
        ref.table_insert(tab, int(k), rng.standard_normal(dim).astype(np.float32))
    # Adam steps on every shard so m / v / step are non-zero
    for s in range(world):
        tab = ref.cluster_shard(h.value, s)
        t = Table(ref, 1 << 12, dim, handle=tab)
        t.owned = False
        ks = t.export()["keys"]
        if len(ks):
            g = (rng.standard_normal((len(ks), dim)) * 0.1).astype(np.float32)
            ref.accumulate_apply_adam(tab, ks, g.reshape(-1), len(ks), 0.01, 0.9, 0.999, 1e-8, 1)
    return h.value


def _ref_export(ref, cluster, s, dim):
    from oracle.bind import Table
    t = Table(ref, 1 << 12, dim, handle=ref.cluster_shard(cluster, s))
    t.owned = False
    return t.export()


def _compare(a, b):
    for f in ("keys", "emb", "m", "v", "step", "ts"):
        np.testing.assert_array_equal(np.asarray(a[f]).astype(np.float64) if f in ("emb", "m", "v") else a[f].astype(np.uint64),
                                      np.asarray(b[f]).astype(np.float64) if f in ("emb", "m", "v") else b[f].astype(np.uint64),
                                      err_msg=f)


@pytest.mark.gpu
@pytest.mark.parametrize("saved,new", [(2, 2), (2, 4), (4, 2), (4, 1), (1, 4)])
def test_load_reference_checkpoint(cuda, ref, tmp_path, saved, new):
    lib = _ref_fns(ref)
    rng = np.random.default_rng(saved * 10 + new)
    dim = 16
    keys = np.unique(rng.integers(0, 1 << 40, 900).astype(np.uint64))
    cl = _ref_cluster(ref, saved, dim, keys, rng)
    assert lib.ref_ckpt_save_cluster(cl, str(tmp_path).encode()) == 0
    st = C.c_int()
    want = lib.ref_ckpt_load_cluster(str(tmp_path).encode(), saved, new, 1 << 12, dim, 256, C.byref(st))
    assert st.value == 0
    for r in range(new):
        t = P.EmbedTable(P.TableConfig(capacity=1 << 12, embedding_dim=dim, optimizer="adam"))
        K.load_shard(t, str(tmp_path), saved, new, r)
        _compare(t.export(), _ref_export(ref, want, r, dim))
        assert t.tick() >= int(_ref_export(ref, want, r, dim)["ts"].max(initial=0))
    ref.cluster_destroy(cl)
    ref.cluster_destroy(want)


@pytest.mark.gpu
def test_save_load_save_byte_identical_and_reference_reads_ours(cuda, ref, tmp_path):
    lib = _ref_fns(ref)
    rng = np.random.default_rng(3)
    dim, world = 8, 2
    keys = np.unique(rng.integers(0, 1 << 40, 700).astype(np.uint64))
    cl = _ref_cluster(ref, world, dim, keys, rng)
    assert lib.ref_ckpt_save_cluster(cl, str(tmp_path / "ref").encode()) == 0
    d1, d2 = tmp_path / "a", tmp_path / "b"
    os.makedirs(d1)
    os.makedirs(d2)
    tabs = []
    for r in range(world):
        t = P.EmbedTable(P.TableConfig(capacity=1 << 12, embedding_dim=dim, optimizer="adam"))
        K.load_shard(t, str(tmp_path / "ref"), world, world, r)
        K.save_shard(t, r, world, str(d1 / K.shard_file_name(r, world)))
        tabs.append(t)
    for r in range(world):  # reload our own files, save again: identical bytes
        t = P.EmbedTable(P.TableConfig(capacity=1 << 12, embedding_dim=dim, optimizer="adam"))
        K.load_shard(t, str(d1), world, world, r)
        K.save_shard(t, r, world, str(d2 / K.shard_file_name(r, world)))
        assert (d1 / K.shard_file_name(r, world)).read_bytes() == (d2 / K.shard_file_name(r, world)).read_bytes()
        h = K.read_header(str(d1 / K.shard_file_name(r, world)))
        assert (h.version, h.world_size, h.shard_rank, h.embedding_dim) == (1, world, r, dim)
    # the reference's elastic reload of OUR files (world 2 -> 4) equals its reload of its own
    st = C.c_int()
    a = lib.ref_ckpt_load_cluster(str(d1).encode(), world, 4, 1 << 12, dim, 256, C.byref(st))
    assert st.value == 0
    b = lib.ref_ckpt_load_cluster(str(tmp_path / "ref").encode(), world, 4, 1 << 12, dim, 256, C.byref(st))
    for r in range(4):
        _compare(_ref_export(ref, a, r, dim), _ref_export(ref, b, r, dim))
    for h in (cl, a, b):
        ref.cluster_destroy(h)


@pytest.mark.gpu
def test_checkpoint_errors(cuda, tmp_path):
    t = P.EmbedTable(P.TableConfig(capacity=1 << 10, embedding_dim=8, optimizer="adam"))
    with pytest.raises(P.ConfigError):
        K.load_shard(t, str(tmp_path), 3, 2, 0)  # worlds must divide
    with pytest.raises(P.IoError):
        K.load_shard(t, str(tmp_path), 2, 2, 0)  # missing file
    (tmp_path / K.shard_file_name(0, 2)).write_bytes(b"not a checkpoint at all")
    with pytest.raises(P.IoError):
        K.load_shard(t, str(tmp_path), 2, 2, 0)
    t2 = P.EmbedTable(P.TableConfig(capacity=1 << 10, embedding_dim=4, optimizer="adam"))
    K.save_shard(t2, 0, 1, str(tmp_path / K.shard_file_name(0, 1)))
    with pytest.raises(P.ConfigError):  # dim mismatch
        K.load_shard(t, str(tmp_path), 1, 1, 0)
